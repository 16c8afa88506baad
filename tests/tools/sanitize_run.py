#!/usr/bin/env python3
"""Exercise every kernel of librsa_b200.so on tiny inputs, checking results
against the oracle -- meant to run under compute-sanitizer (memcheck,
racecheck, initcheck, synccheck); see tests/test_gpu_sanitizer.py."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402  (checker)
import paper_1407_1465_b200 as R  # noqa: E402
import workload  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint32).view(np.int32)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy().view(np.uint32)


def main():
    count = int(os.environ.get("SAN_COUNT", "300"))
    # every width class and kernel shape, with short exponents (full-length
    # exponents are covered by the parity tests; under racecheck every smem
    # access is instrumented): d is used only for the small keys
    for name in ["toy17947", "rsa64", "rsa128", "rsa256", "rsa512", "rsa1024", "rsa2048", "rsa4096"]:
        k = workload.key(name)
        nb = k["n"].bit_length()
        m = workload.packets(count, nb, n=k["n"], config_id=1)
        c = R.rsa_modexp_batch(dev(m), k["e"], k["n"], nb)
        assert np.array_equal(host(c), oracle.modexp_batch(m, k["e"], k["n"])[:, :m.shape[1]]), name
        x = 0xF00D1 if nb > 256 else k["d"]                       # windowed path (w > 1)
        y = R.rsa_modexp_batch(c, x, k["n"], nb)
        assert np.array_equal(host(y), oracle.modexp_batch(host(c), x, k["n"])[:, :m.shape[1]]), name
        if name in ("rsa256", "rsa512"):
            z = R.rsa_decrypt_crt_batch(c, k["p"], k["q"], k["d"], nb)
            assert np.array_equal(host(z), m), name
    # host e2e entry
    k = workload.key("rsa256")
    m = workload.packets(count, 256, n=k["n"], config_id=2)
    assert np.array_equal(R.rsa_modexp_batch_host(m, k["e"], k["n"], 256), oracle.modexp_batch(m, k["e"], k["n"]))
    # paper kernel
    pp = workload.paper_packets(count)
    got = host(R.rsa_modexp_batch_paper(dev(pp.ravel()), 131, 17947))
    assert np.array_equal(got, oracle.modexp_batch(pp, 131, 17947).ravel())
    for sched in (R.RSA_SCHED_NAIVE, R.RSA_SCHED_R2L, R.RSA_SCHED_L2R):   # the paper's other schedules
        got = host(R.rsa_modexp_batch_schedule(dev(pp.ravel()), 131, 17947, sched))
        assert np.array_equal(got, oracle.modexp_batch(pp, 131, 17947).ravel()), sched
    # multi-key + MR + prime search helpers
    rng = np.random.default_rng(0)
    mods = rng.integers(0, 2**32, (count, 8), dtype=np.uint64).astype(np.uint32)
    mods[:, 0] |= 1
    mods[:, 7] |= np.uint32(1 << 31)
    base = rng.integers(0, 2**32, (count, 8), dtype=np.uint64).astype(np.uint32)
    exps = rng.integers(0, 2**32, (count, 8), dtype=np.uint64).astype(np.uint32)
    got = host(R.rsa_modexp_batch_multi(dev(base), dev(exps), dev(mods), 256))
    assert np.array_equal(got, oracle.modexp_multi(base, exps, mods))
    cand = R.rsa_prime_candidates(128, 3, 0, count)
    R.rsa_prime_sieve(cand, 128)
    R.rsa_miller_rabin_batch(cand, 128, 2)
    torch.cuda.synchronize()
    primes, _ = R.rsa_prime_search(64, 9, 2, rounds=4)
    assert all(oracle.is_prime(p) for p in primes)
    print("sanitize_run ok")


if __name__ == "__main__":
    main()
