"""The C-ABI library loads and exports every symbol include/rsa_b200.h declares
(no GPU needed); host-only calls (keygen check, codec) work and agree with the
oracle / the paper."""
import json
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "rsa_b200.h")
GOLD = os.path.join(ROOT, "tests", "golden")


def declared():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(rsa_\w+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_calls():
    names = declared()
    for fn in ["rsa_keygen_check", "rsa_modexp_batch", "rsa_encode", "rsa_decode", "rsa_strerror"]:
        assert fn in names


def test_library_exports_every_declared_symbol():
    import paper_1407_1465_b200 as R
    out = subprocess.check_output(["nm", "-D", "--defined-only", R.LIB_PATH], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    for fn in declared():
        assert fn in exported, fn
        getattr(R._lib, fn)
    assert set(R.EXPORTS) <= exported


def test_library_is_sm100a():
    import paper_1407_1465_b200 as R
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", R.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_host_keygen_matches_oracle_and_paper():
    import oracle
    import paper_1407_1465_b200 as R
    import workload
    fig2 = json.load(open(os.path.join(GOLD, "fig2_key.json")))
    assert R.rsa_keygen_check(fig2["p"], fig2["q"], fig2["e"]) == (fig2["n"], fig2["phi"], fig2["d"])
    assert R.rsa_validate_key(131, 137, 131, 137) == (False, 267)
    assert R.rsa_validate_key(131, 14171, 131, 137) == (True, 1)
    for name in ["toy17947", "table2_513581", "rsa64", "rsa96", "rsa512", "rsa1024", "rsa2048"]:
        k = workload.key(name)
        assert R.rsa_keygen_check(k["p"], k["q"], k["e"]) == oracle.keygen_check(k["p"], k["q"], k["e"])


@pytest.mark.parametrize("args,code", [((13, 13, 3), -5), ((15, 17, 3), -4), ((17, 11, 2), -6),
                                       ((17, 11, 1), -2), ((17, 11, 160), -2), ((1005, 509, 131), -4),
                                       ((561, 11, 3), -4)])
def test_host_keygen_errors(args, code):
    import paper_1407_1465_b200 as R
    with pytest.raises(R.RsaError) as ei:
        R.rsa_keygen_check(*args)
    assert ei.value.code == code


def test_codec_matches_paper_and_oracle():
    import oracle
    import paper_1407_1465_b200 as R
    g = json.load(open(os.path.join(GOLD, "sec2_packets.json")))
    assert R.rsa_encode(g["text"]) == g["packets"] == oracle.encode(g["text"])
    assert R.rsa_decode(g["packets"]) == g["decoded"]
    for bad, code in [("a", R.RSA_EODD), ("aB", R.RSA_ECHAR)]:
        with pytest.raises(R.RsaError) as ei:
            R.rsa_encode(bad)
        assert ei.value.code == code
    with pytest.raises(R.RsaError) as ei:
        R.rsa_decode([2600])
    assert ei.value.code == R.RSA_EPACKET


def test_plan_montmul_counts():
    """Host plan: e=65537 costs 18 montmuls -- SURVEY.md sec. 8's 19 (16 S +
    1 M + 2 conversions) less one, because the final multiply by g takes the
    raw input and lands outside Montgomery form (RSA_OP_MULX, csrc/plan.h);
    an exponent whose scan ends in squarings keeps the explicit conversion;
    windowed plans never cost more than binary."""
    import paper_1407_1465_b200 as R
    import workload
    k = workload.key("rsa2048")
    p = R.rsa_plan_info(65537, k["n"], 2048)
    assert p["montmuls"] == 18 and p["squarings"] == 16 and p["width_class"] == 64
    for e, mm in [(1, 2), (2, 3), (3, 3), (6, 5), (7, 5)]:      # R2 [+ SQR/MUL ...] + ONE or MULX
        assert R.rsa_plan_info(e, k["n"], 2048)["montmuls"] == mm, e
    pd = R.rsa_plan_info(k["d"], k["n"], 2048)
    bits, pop = k["d"].bit_length(), bin(k["d"]).count("1")
    assert pd["montmuls"] < (bits - 1) + (pop - 1) + 2          # beats Fig 5 binary
    assert pd["squarings"] >= bits - 1 - pd["window"]


def test_kernel_path_knob():
    """rsa_set_kernel_path validates (class, path) pairs, resolves per class and
    changes the plan (executed products) without touching a device."""
    import paper_1407_1465_b200 as R
    import workload
    defaults = {2: R.RSA_PATH_INT_MULTI, 4: R.RSA_PATH_INT_MULTI, 8: R.RSA_PATH_INT, 16: R.RSA_PATH_INT,
                32: R.RSA_PATH_TC, 64: R.RSA_PATH_TC, 128: R.RSA_PATH_TC}
    for S, p in defaults.items():
        assert R.rsa_get_kernel_path(S) == p, S
    for S, p in [(8, R.RSA_PATH_FP64), (64, R.RSA_PATH_INT_PAIR), (128, R.RSA_PATH_INT_MULTI), (3, 0), (64, 9),
                 (16, R.RSA_PATH_TC), (8, R.RSA_PATH_TC)]:
        with pytest.raises(R.RsaError):
            R.rsa_set_kernel_path(S, p)
    with pytest.raises(R.RsaError):
        R.rsa_get_kernel_path(5)
    k = workload.key("rsa2048")
    fp = R.rsa_plan_info(k["d"], k["n"], 2048)
    with R.kernel_path(64, R.RSA_PATH_INT_GROUP):
        grp = R.rsa_plan_info(k["d"], k["n"], 2048)
        assert R.rsa_get_kernel_path(64) == R.RSA_PATH_INT_GROUP
    with R.kernel_path(128, R.RSA_PATH_INT):           # S = 128 integer = the lane pairs
        assert R.rsa_get_kernel_path(128) == R.RSA_PATH_INT_PAIR
    with R.kernel_path(64, R.RSA_PATH_FP64):
        f64 = R.rsa_plan_info(k["d"], k["n"], 2048)
    assert R.rsa_get_kernel_path(64) == R.RSA_PATH_TC
    assert fp["fp64_digits"] == 40 and fp["sqr_kernel"] == 1 and f64["fp64_digits"] == 40
    # the tensor-core path's CUDA-core digit products: the product T = A B only
    # (ND(ND+1)/2 per squaring, ND^2 per multiply); the FP64 kernel adds ND^2 of reduction
    nsq, nmul = fp["squarings"], fp["montmuls"] - fp["squarings"]
    assert fp["digit_products"] == nsq * 820 + nmul * 1600
    assert f64["digit_products"] == nsq * (820 + 1600) + nmul * 3200
    assert grp["fp64_digits"] == 0 and grp["sqr_kernel"] == 0
    assert grp["products"] > fp["products"]          # no dedicated squaring on the group kernel
    assert R.rsa_plan_info(k["d"], k["n"], 2048) == fp


def test_binding_rejects_bad_shapes():
    """The binding checks [count, s] / element size / residency before the C side
    trusts count*s (host arrays checked without a GPU)."""
    import numpy as np
    import paper_1407_1465_b200 as R
    import workload
    k = workload.key("rsa2048")
    # (numpy inputs are converted with ascontiguousarray(uint32): values, not layouts, are accepted)
    for bad in [np.zeros(64 * 3, np.uint32), np.zeros((3, 63), np.uint32), np.zeros((3, 64, 1), np.uint32)]:
        with pytest.raises(ValueError):
            R.rsa_modexp_batch_host(bad, 3, k["n"], 2048)
    with pytest.raises(ValueError):
        R.rsa_modexp_batch_host(np.zeros((3, 64), np.uint32), 3, k["n"], 2048, out=np.zeros((2, 64), np.uint32))
