"""The C++ drop-in boundary as a compiled consumer sees it: tests/cpp/
dropin_test.cpp includes egt_b200/packed.hpp, links -legt_b200 (the exported
egt_b200:: namespace) and checks quantize_matrix / pack / footprint (host)
and spmv / unpack (device, -m gpu) against the reference's golden vectors."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2605_11582_b200", "_lib")


def _golden_bin(path):
    z = np.load(os.path.join(ROOT, "tests", "golden", "ref_vectors.npz"))
    cases = []
    i = 0
    while f"c{i}_meta" in z:
        rows, cols, n, quant, dense_codes = (int(v) for v in z[f"c{i}_meta"])
        if quant and not dense_codes:
            cases.append(i)
        i += 1

    def put(f, a, dt):
        a = np.ascontiguousarray(a, dt).reshape(-1)
        f.write(np.uint64(a.size).tobytes())
        f.write(a.tobytes())

    with open(path, "wb") as f:
        put(f, [len(cases)], np.uint32)
        for i in cases:
            rows, cols, n = (int(v) for v in z[f"c{i}_meta"][:3])
            put(f, [rows, cols, n], np.uint32)
            put(f, z[f"c{i}_w"], np.float32)
            put(f, z[f"c{i}_x"], np.float32)
            put(f, z[f"c{i}_mask"], np.uint8)
            put(f, z[f"c{i}_group_sizes"], np.uint32)
            put(f, z[f"c{i}_scales"], np.float32)
            put(f, z[f"c{i}_zero_points"], np.uint8)
            put(f, z[f"c{i}_index_words"], np.uint16)
            put(f, z[f"c{i}_value_bytes"], np.uint8)
            fp = z[f"c{i}_footprint"]
            put(f, fp[:5], np.uint64)
            put(f, z[f"c{i}_y"], np.float32)
            put(f, z[f"c{i}_unpack_values"], np.float32)
    return len(cases)


@pytest.fixture(scope="module")
def dropin(tmp_path_factory):
    from paper_2605_11582_b200 import native

    if not os.path.exists(native.LIB_PATH):
        pytest.skip("libegt_b200.so not built")
    d = tmp_path_factory.mktemp("dropin")
    exe = str(d / "dropin_test")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I",
           os.path.join(ROOT, "paper_2605_11582_b200", "csrc", "host"), os.path.join(ROOT, "tests", "cpp",
                                                                                    "dropin_test.cpp"),
           "-L", LIBDIR, "-l:libegt_b200.so", f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    gold = str(d / "golden.bin")
    n = _golden_bin(gold)
    assert n >= 5
    return exe, gold


def test_cpp_dropin_host(dropin):
    exe, gold = dropin
    r = subprocess.run([exe, gold], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and r.stdout.count("PASS") >= 25


@pytest.mark.gpu
def test_cpp_dropin_device(dropin):
    exe, gold = dropin
    r = subprocess.run([exe, gold, "--gpu"], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout and "device spmv" in r.stdout
