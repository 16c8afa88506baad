"""The C-ABI from plain C (examples/rsa_c_example.c, gcc, no Python in the
process) and concurrent use from two streams with different keys."""
import json
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


def test_c_program(tmp_path):
    _cuda()
    lib_dir = os.path.join(ROOT, "paper_1407_1465_b200")
    # the library is named librsa_b200.so; link it by path
    exe = str(tmp_path / "rsa_c_example")
    subprocess.check_call(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
                           os.path.join(ROOT, "examples", "rsa_c_example.c"), os.path.join(lib_dir, "librsa_b200.so"),
                           "-L/usr/local/cuda/lib64", "-lcudart", f"-Wl,-rpath,{lib_dir}",
                           "-Wl,-rpath,/usr/local/cuda/lib64", "-o", exe])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    dv = json.load(open(os.path.join(GOLD, "survey_derived.json")))
    assert "decoded: parallelencryption" in r.stdout
    assert "cipher: " + " ".join(str(c) for c in dv["toy_ciphertexts"]) in r.stdout
    assert "paper's d=137: INVALID (d*e mod phi = 267)" in r.stdout


def test_concurrent_streams_different_keys():
    torch = _cuda()
    import oracle
    import paper_1407_1465_b200 as R
    import workload
    k1, k2 = workload.key("rsa2048"), workload.key("rsa1024")
    m1 = workload.packets(40000, 2048, n=k1["n"], config_id=41)
    m2 = workload.packets(60000, 1024, n=k2["n"], config_id=42)
    t1 = torch.from_numpy(m1.view(np.int32)).cuda()
    t2 = torch.from_numpy(m2.view(np.int32)).cuda()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    with torch.cuda.stream(s1):
        o1 = R.rsa_modexp_batch(t1, k1["d"], k1["n"], 2048, stream=s1)
    with torch.cuda.stream(s2):
        o2 = R.rsa_modexp_batch(t2, k2["e"], k2["n"], 1024, stream=s2)
        o3 = R.rsa_modexp_batch(o2, k2["d"], k2["n"], 1024, stream=s2)
    torch.cuda.synchronize()
    idx = np.arange(0, 40000, 997)
    assert np.array_equal(o1.cpu().numpy().view(np.uint32)[idx], oracle.modexp_batch(m1[idx], k1["d"], k1["n"]))
    assert np.array_equal(o3.cpu().numpy().view(np.uint32), m2)
