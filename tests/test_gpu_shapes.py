"""The alternative kernel shapes kept for measurement ('chosen by
measurement'): the 1024/2048-bit classes on the integer pipe or the FP64 pipe
(RSA_B200_F64=0/1), the 4096-bit integer lane-pair kernel (RSA_B200_F64_4096=0),
2048-bit as a 2-lane group (RSA_B200_SHAPE64=group2) and
4096-bit as a 4-lane group (RSA_B200_TPI128=4), and the thread-per-packet
kernel for the small widths (RSA_B200_SMALL=0, instead of the multi-packet
one) stay bit-exact vs the oracle.
Run in subprocesses (the switch is read once per process)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import oracle, workload, paper_1407_1465_b200 as R
k = workload.key(sys.argv[1]); nb = k["nbits"]; s = workload.limbs_needed(nb)
m = workload.packets(int(sys.argv[2]), nb, n=k["n"], config_id=21)
R_ = 1 << (32 * s)                      # inputs at and above n as well (the call is total)
edge = [v for v in (k["n"], k["n"] + 1, 2 * k["n"] - 1, R_ - 1, R_ - 2) if v < R_]
m = np.concatenate([m, workload.ints_to_rows(edge, s)])
t = torch.from_numpy(m.view(np.int32)).cuda()
for e in (k["e"], k["d"], 3):
    got = R.rsa_modexp_batch(t, e, k["n"], nb).cpu().numpy().view(np.uint32)
    assert np.array_equal(got, oracle.modexp_batch(m, e, k["n"])[:, :s]), e
print("shape ok")
''' % ROOT


@pytest.mark.parametrize("env,key,count", [("RSA_B200_F64=0", "rsa2048", 300),
                                           ("RSA_B200_F64=0", "rsa1536", 300),
                                           ("RSA_B200_F64=1", "rsa2048", 300),
                                           ("RSA_B200_F64=1", "rsa1536", 300),
                                           ("RSA_B200_SHAPE64=group2", "rsa2048", 300),
                                           ("RSA_B200_SHAPE64=group2", "rsa1536", 300),
                                           ("RSA_B200_F64_4096=0", "rsa4096", 60),
                                           ("RSA_B200_F64_4096=0", "rsa3072", 60),
                                           ("RSA_B200_F64_4096=0,RSA_B200_TPI128=4", "rsa4096", 60),
                                           ("RSA_B200_F64_4096=0,RSA_B200_TPI128=4", "rsa3072", 60),
                                           ("RSA_B200_SMALL=0", "rsa64", 3001),
                                           ("RSA_B200_SMALL=0", "rsa128", 3001),
                                           ("RSA_B200_SMALL=0", "toy17947", 3001)])
def test_alternative_shapes(env, key, count):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    kv = dict(x.split("=") for x in env.split(","))
    r = subprocess.run([sys.executable, "-c", SCRIPT, key, str(count)], capture_output=True, text=True,
                       timeout=900, env=dict(os.environ, **kv))
    assert r.returncode == 0 and "shape ok" in r.stdout, (r.stdout + r.stderr)[-2000:]
