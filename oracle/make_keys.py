"""Write workload/keys.json -- the committed key fixture.

Calls only ``oracle/`` (primality, key-generation check) plus the seeded
candidate generator of ``workload/`` (random bits only).  Run:
    python -m oracle.make_keys
Every stored n, phi, d is produced by ``oracle.keygen_check`` (Fig 1,
PAPER.md:53); the paper's own keys carry their citation.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import workload  # noqa: E402

SIZES = [64, 96, 128, 192, 256, 384, 512, 768, 1000, 1024, 1536, 2048, 3072, 4096]
E_PUBLIC = 65537


def find_prime(bits: int, rng) -> int:
    x = workload.prime_candidate(bits, rng)
    while not oracle.is_prime(x):
        x += 2
        if x.bit_length() > bits:
            x = workload.prime_candidate(bits, rng)
    return x


def make_key(nbits: int, e: int = E_PUBLIC) -> dict:
    rng = np.random.Generator(np.random.PCG64(workload.MASTER_SEED + 1000 + nbits))
    h1 = nbits // 2
    h2 = nbits - h1
    while True:
        p = find_prime(h1, rng)
        q = find_prime(h2, rng)
        if p == q:
            continue
        try:
            n, phi, d = oracle.keygen_check(p, q, e)
        except oracle.OracleError as ex:
            if ex.code == oracle.ENOTCOPRIME:
                continue
            raise
        assert n.bit_length() == nbits
        return dict(nbits=nbits, p=hex(p), q=hex(q), e=hex(e), n=hex(n), phi=hex(phi), d=hex(d),
                    d_bits=d.bit_length(), d_popcount=bin(d).count("1"),
                    note="seeded: PCG64(14071465 + 1000 + nbits), top two bits set, oracle MR")


def paper_key(p: int, q: int, e: int, cite: str, **extra) -> dict:
    n, phi, d = oracle.keygen_check(p, q, e)
    k = dict(nbits=n.bit_length(), p=hex(p), q=hex(q), e=hex(e), n=hex(n), phi=hex(phi), d=hex(d),
             d_bits=d.bit_length(), d_popcount=bin(d).count("1"), cite=cite)
    k.update(extra)
    return k


def main():
    keys = {}
    keys["toy17947"] = paper_key(131, 137, 131, "PAPER.md:37 sec. 2 (e=131, n=17947=131*137); "
                                 "the printed d=137 is invalid (reading Z1) -- d is e^-1 mod phi",
                                 paper_d=hex(137))
    keys["fig2_187"] = paper_key(17, 11, 7, "PAPER.md:73-79 Fig 2 (p=17, q=11, e=7, d=23)")
    keys["table2_513581"] = paper_key(1009, 509, 131, "PAPER.md:469 sec. 10.2.1 n=1009*509 "
                                      "(reading Z7: caption 1005 is composite; e=131 assumed)")
    for nb in SIZES:
        keys["rsa%d" % nb] = make_key(nb)
        print("rsa%d" % nb, "d bits", keys["rsa%d" % nb]["d_bits"], flush=True)
    out = dict(generator="oracle/make_keys.py", master_seed=workload.MASTER_SEED, keys=keys)
    with open(workload.KEYS_PATH, "w") as f:
        json.dump(out, f, indent=1)
        f.write("\n")


if __name__ == "__main__":
    main()
