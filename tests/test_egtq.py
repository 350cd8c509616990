"""EGTQ files written by the reference's own serialize_compressed
(egtq_io.cpp:212-219, oracle/_ref) are read by the product's parser with the
reference's acceptance and FormatError messages (CPU); uploaded layers
dequantize bit-exactly to the oracle's unpack and multiply within tolerance
(GPU)."""
import numpy as np
import pytest

from oracle.oracle import OracleError, random_nm_mask
from tests.layers import close


def _layers(rng):
    w = lambda r, c: rng.uniform(-1, 1, (r, c)).astype(np.float32)  # noqa: E731
    return [
        dict(name="layers.0.wq", pattern=2, quant=True, w=w(32, 128), mask=random_nm_mask(rng, 32, 128, 2), group=32),
        dict(name="layers.0.wk", pattern=1, quant=True, w=w(48, 64), mask=random_nm_mask(rng, 48, 64, 1), group=64),
        dict(name="layers.0.wv", pattern=0, quant=True, w=w(16, 96), mask=None, group=32),
        dict(name="layers.0.wo", pattern=2, quant=False, w=w(32, 64), mask=random_nm_mask(rng, 32, 64, 2)),
        dict(name="layers.0.ff1", pattern=0, quant=False, w=w(8, 32), mask=None),
    ]


@pytest.fixture(scope="module")
def data(ref):
    return ref.ref_egtq_serialize(_layers(np.random.default_rng(3)))


def test_parse_reference_file(ref, data):
    from paper_2605_11582_b200.egtq import EgtqFile

    f = EgtqFile(data)
    assert ref.ref_egtq_parse(data) == len(f.layers) == 5
    assert [l.name for l in f.layers] == [l["name"] for l in _layers(np.random.default_rng(3))]
    assert [l.pattern for l in f.layers] == ["2:4", "1:4", "dense", "2:4", "dense"]
    assert [l.has_index for l in f.layers] == [True, True, False, False, False]


def _ref_error(ref, blob):
    try:
        ref.ref_egtq_parse(blob)
    except OracleError as e:
        return str(e).split(": ", 1)[1]
    return None


def test_malformed_files_match_reference(ref, data):
    """Every truncation and a set of single-byte corruptions: the product
    rejects exactly when the reference does, with the same message."""
    from paper_2605_11582_b200.egtq import EgtqFile
    from paper_2605_11582_b200.native import FormatError

    rng = np.random.default_rng(5)
    blobs = [data[:n] for n in range(0, len(data), 7)] + [data + b"\x00"]
    for _ in range(300):
        b = bytearray(data)
        i = int(rng.integers(0, len(b)))
        b[i] = int(rng.integers(0, 256))
        blobs.append(bytes(b))
    for blob in blobs:
        want = _ref_error(ref, blob)
        try:
            EgtqFile(blob)
            got = None
        except FormatError as e:
            got = str(e).split(": ", 1)[1]
        assert got == want, (len(blob), got, want)


@pytest.mark.gpu
def test_upload_dispatch_parity(ref, port, data):
    """Uploaded layers: bit-exact dequant vs the oracle's unpack of the same
    layer packed by the reference encoder; products within 1e-3 (1+|y|);
    dense fp is rejected as not on the path."""
    import torch

    from paper_2605_11582_b200.egtq import EgtqFile
    from paper_2605_11582_b200.native import InvalidArgument

    f = EgtqFile(data)
    rng = np.random.default_rng(3)
    specs = _layers(rng)
    for i, (info, spec) in enumerate(zip(f.layers, specs)):
        if info.pattern == "dense" and not info.has_quant:
            with pytest.raises(InvalidArgument, match="not on the SparseGemv path"):
                f.upload(i)
            continue
        w, mask = spec["w"], spec["mask"]
        if not info.has_quant and not np.array_equal(w.astype(np.float16).astype(np.float32), w):
            with pytest.raises(InvalidArgument, match="not representable in fp16"):
                f.upload(i)
        d = f.upload(i, round_fp16=not info.has_quant)
        rows, cols = w.shape
        if info.has_quant:
            gs = np.full(rows, spec["group"], np.uint32)
            q = port.quantize(w, gs, mask)
            if mask is None:
                want_w = port.dequantize(q)
            else:
                want_w, _ = port.unpack(port.pack_int4(mask, rows, cols, q, 2 if info.pattern == "2:4" else 1))
        else:  # sparse fp: f32 in the file, FP16 on the device when rounding is requested
            want_w, _ = port.unpack(port.pack_f32(mask, rows, cols, w, 2 if info.pattern == "2:4" else 1))
            raw_w = want_w.copy()
            want_w = want_w.astype(np.float16).astype(np.float32)
        got_w, _ = d.dequant()
        assert np.array_equal(got_w.cpu().numpy().view(np.uint32), want_w.astype(np.float32).view(np.uint32)), info.name
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        y = d.spmv(torch.from_numpy(x).cuda()).cpu().numpy()
        ok, err = close(y, want_w.astype(np.float64) @ x.astype(np.float64))
        assert ok, (info.name, err)
        if not info.has_quant:
            # against the reference's f32 spmv on the RAW f32 weights: the
            # rounding error of the opted-in fp16 storage, measured
            raw = port.pack_f32(mask, rows, cols, w, 2 if info.pattern == "2:4" else 1)
            ok, err = close(y, port.spmv(raw, x), tol=2e-3)
            assert ok, (info.name, "fp16 rounding vs raw f32", err)
