"""Generates tests/golden/ref_vectors.npz by running the UNMODIFIED reference
hot-path sources (oracle/_ref/libegt_ref.so, built by oracle/build_ref.sh from
/root/reference) on seeded inputs.  Run in the dev container, where the
reference tree exists:

    oracle/build_ref.sh && python tests/golden/make_golden.py

The fixtures let the CPU suite pin the C restatement (and the product's host
encoder) against the reference without the reference tree being present.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, random_nm_mask  # noqa: E402

# (rows, cols, n, group sizes spec, quant, dense-codes input)
CASES = [
    (1, 8, 2, [8], True, False),
    (4, 16, 2, [8], True, True),
    (7, 36, 1, [4], True, False),
    (5, 40, 2, [16], True, False),
    (16, 64, 2, [64], True, False),
    (16, 64, 1, [64], True, False),
    (32, 128, 2, [128], True, False),
    (32, 128, 1, [32], True, False),
    (24, 256, 2, "mixed64_128", True, False),
    (16, 96, 2, [48], True, False),
    (64, 512, 2, [128], True, False),
    (64, 512, 1, [128], True, False),
    (6, 20, 2, None, False, False),
    (9, 64, 1, None, False, False),
]


def main():
    R = Oracle("reference")
    rng = np.random.default_rng(20261017)
    out = {}
    for i, (rows, cols, n, gspec, quant, dense_codes) in enumerate(CASES):
        w = rng.uniform(-1, 1, (rows, cols)).astype(np.float32)
        x = rng.uniform(-1, 1, cols).astype(np.float32)
        mask = random_nm_mask(rng, rows, cols, n)
        key = f"c{i}_"
        out[key + "meta"] = np.array([rows, cols, n, int(quant), int(dense_codes)], np.int64)
        out[key + "w"] = w
        out[key + "x"] = x
        out[key + "mask"] = mask
        if quant:
            if gspec == "mixed64_128":
                gs = np.where(rng.random(rows) < 0.5, 64, 128).astype(np.uint32)
            else:
                gs = np.full(rows, gspec[0], np.uint32)
            q = R.quantize(w, gs) if dense_codes else R.quantize(w, gs, mask)
            p = R.pack_int4(mask, rows, cols, q, n)
            out[key + "group_sizes"] = gs
            out[key + "group_offsets"] = q.group_offsets
            out[key + "scales"] = q.scales
            out[key + "zero_points"] = q.zero_points
            out[key + "codes"] = q.codes
            out[key + "value_bytes"] = p.value_bytes
            out[key + "dequant"] = R.dequantize(q)
        else:
            p = R.pack_f32(mask, rows, cols, w, n)
            out[key + "values"] = p.values
        out[key + "index_words"] = p.index_words
        vals, bits = R.unpack(p)
        out[key + "unpack_values"] = vals
        out[key + "unpack_mask"] = bits
        out[key + "y"] = R.spmv(p, x)
        fp = R.footprint(p)
        out[key + "footprint"] = np.array([fp[k] for k in ("index_bytes", "value_bytes", "scale_bytes",
                                                             "packed_bytes", "baseline_bytes")], np.int64)
    # group-fit known answers run through the reference (test_compress.cpp:87-127)
    fits = []
    for vals in ([0.0, 1.0, 2.0, 3.0], [-1.0, 1.0], [0.0, 0.0, 0.0], [], [2.5, 2.5],
                 [-0.7, 0.3, 0.9], [1e-9, 2e-9], [-3.0, -1.0]):
        s, z = R.fit_group(vals)
        fits.append((s, z))
    out["fit_scale"] = np.array([f[0] for f in fits], np.float32)
    out["fit_zp"] = np.array([f[1] for f in fits], np.uint8)
    out["n_cases"] = np.array(len(CASES))
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ref_vectors.npz")
    np.savez_compressed(path, **out)
    print("wrote", path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
