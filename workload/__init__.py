"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no modular multiply, no
exponentiation, no primality test).  It only draws random limbs and reads the
committed key fixture ``workload/keys.json`` (written by
``oracle/make_keys.py``, which calls only ``oracle/``).

Recipe:
  * master seed 14071465;
  * packets: ``numpy.random.Generator(PCG64(seed + config_id))``,
    ``integers(0, 2**32, (count, s), uint32)`` with the top limb masked to
    nbits-1 bits, so every packet is uniform in [0, 2^(nbits-1)) < n;
  * rows 0..15 are overwritten with edge packets (0, 1, 2, 3, n-1, n-2,
    (n-1)/2, 2^(32k)-1, 2^(nbits-2), an all-ones pattern, ...);
  * keys: p, q random (nbits/2)-bit with the top two bits set (so n has exactly
    nbits bits), e = 65537, d = e^-1 mod phi (Fig 1).
The paper's own workloads ("values of message between 0 and
800"; sec. 2 packets <= 2525) are produced by ``paper_packets``.
"""
from __future__ import annotations

import json
import os

import numpy as np

MASTER_SEED = 14071465
_HERE = os.path.dirname(os.path.abspath(__file__))
KEYS_PATH = os.path.join(_HERE, "keys.json")

# BASELINE.json "configs", in order.  exp: "e" = public exponent, "d" = full
# private exponent, "both" = encrypt then decrypt (round trip).
CONFIGS = {
    "toy": dict(config_id=0, key="toy17947", count=9, exp="both",
                desc="paper toy key n=17947 (e=131): the 9 packets of 'parallel encryption'"),
    "u64": dict(config_id=1, key="rsa64", count=16 * 1024 * 1024, exp="both",
                desc="64-bit modulus, 16M random packets"),
    "rsa2048-enc": dict(config_id=2, key="rsa2048", count=1024 * 1024, exp="e",
                        desc="RSA-2048 encrypt e=65537, 1M packets"),
    "rsa2048-dec": dict(config_id=3, key="rsa2048", count=1024 * 1024, exp="d",
                        desc="RSA-2048 decrypt full d, 1M packets"),
    "rsa4096-dec": dict(config_id=4, key="rsa4096", count=256 * 1024, exp="d",
                        desc="RSA-4096 decrypt full d, 256K packets"),
}


def limbs_needed(nbits: int) -> int:
    return (nbits + 31) // 32


def to_limbs(x: int, n: int) -> np.ndarray:
    """Python int -> n little-endian uint32 limbs (representation only)."""
    out = np.zeros(n, dtype=np.uint32)
    for i in range(n):
        out[i] = x & 0xFFFFFFFF
        x >>= 32
    if x:
        raise ValueError("value does not fit")
    return out


def from_limbs(a) -> int:
    v = 0
    for w in reversed([int(t) for t in np.asarray(a, dtype=np.uint32).ravel()]):
        v = (v << 32) | w
    return v


def rows_to_ints(arr: np.ndarray):
    """[count, s] uint32 -> list of Python ints (vectorised via bytes)."""
    arr = np.ascontiguousarray(arr, dtype="<u4")
    nbytes = arr.shape[1] * 4
    raw = arr.tobytes()
    return [int.from_bytes(raw[i * nbytes:(i + 1) * nbytes], "little") for i in range(arr.shape[0])]


def ints_to_rows(vals, s: int) -> np.ndarray:
    buf = b"".join(int(v).to_bytes(4 * s, "little") for v in vals)
    return np.frombuffer(buf, dtype="<u4").reshape(len(vals), s).astype(np.uint32)


# ------------------------------------------------------------------ keys

def prime_candidate(bits: int, rng: np.random.Generator) -> int:
    """Random odd integer of exactly `bits` bits with the top two bits set."""
    nlimbs = limbs_needed(bits)
    x = from_limbs(rng.integers(0, 2**32, nlimbs, dtype=np.uint64).astype(np.uint32))
    x &= (1 << bits) - 1
    x |= (3 << (bits - 2)) | 1
    return x


def load_keys() -> dict:
    with open(KEYS_PATH) as f:
        raw = json.load(f)
    keys = {}
    for name, k in raw["keys"].items():
        keys[name] = {f: (int(v, 16) if isinstance(v, str) and f not in ("cite", "note") else v)
                      for f, v in k.items()}
    return keys


def key(name: str) -> dict:
    return load_keys()[name]


# ------------------------------------------------------------------ packets

def edge_ints(n: int, nbits: int):
    """Edge packets for modulus n (all < n except where noted by callers)."""
    s = limbs_needed(nbits)
    cand = [0, 1, 2, 3, n - 1, n - 2, (n - 1) // 2, (n + 1) // 2, 1 << (nbits - 2),
            (1 << (nbits - 1)) - 1]
    for k in range(1, s + 1):
        v = (1 << (32 * k)) - 1
        if v < n:
            cand.append(v)
    pat = int("5" * ((nbits + 3) // 4), 16) & ((1 << (nbits - 1)) - 1)
    cand.append(pat)
    out = []
    for v in cand:
        if 0 <= v < n and v not in out:
            out.append(v)
    return out[:16]


def packets(count: int, nbits: int, n: int | None = None, config_id: int = 0,
            seed: int = MASTER_SEED, s: int | None = None, edges: bool = True) -> np.ndarray:
    """Uniform packets in [0, 2^(nbits-1)) as uint32 [count, s], LE limbs.

    If ``n`` is given and ``edges`` is true, the first rows are the edge
    packets of ``edge_ints(n, nbits)``.
    """
    if s is None:
        s = limbs_needed(nbits)
    rng = np.random.Generator(np.random.PCG64(seed + config_id))
    out = rng.integers(0, 2**32, (count, s), dtype=np.uint64).astype(np.uint32)
    sn = limbs_needed(nbits)
    top_bits = (nbits - 1) - 32 * (sn - 1)      # in [0, 31]: bits kept in limb sn-1
    out[:, sn - 1] &= np.uint32((1 << top_bits) - 1)
    out[:, sn:] = 0
    if n is not None and edges and count > 0:
        e = edge_ints(n, nbits)[:count]
        out[: len(e)] = ints_to_rows(e, s)
    return out


def paper_packets(count: int, seed: int = MASTER_SEED, config_id: int = 0, high: int = 800) -> np.ndarray:
    """The paper's test inputs: values in [0, high], s = 1."""
    rng = np.random.Generator(np.random.PCG64(seed + config_id))
    return rng.integers(0, high + 1, (count, 1), dtype=np.uint64).astype(np.uint32)


# sec. 2 of the paper: the worked message
PAPER_TEXT = "parallel encryption"


# ------------------------------------------------------------------ prime-search candidates

_M64 = (1 << 64) - 1


def _splitmix_mix(x: int) -> int:
    x &= _M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & _M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & _M64
    return x ^ (x >> 31)


def prime_candidates(nbits: int, seed: int, first: int, count: int) -> np.ndarray:
    """The counter-based candidate generator of the GPU prime search
    (modexp_multi.cu), re-implemented independently: candidate i, limb pair j
    = splitmix64 finaliser of seed + (i * 2^16 + j + 1) * 0x9E3779B97F4A7C15;
    masked to nbits, bits nbits-1, nbits-2 and 0 set.  uint32 [count, s]."""
    s = limbs_needed(nbits)
    vals = []
    for i in range(first, first + count):
        x = 0
        for j in range((s + 1) // 2):
            z = _splitmix_mix(seed + ((i << 16) + j + 1) * 0x9E3779B97F4A7C15)
            x |= z << (64 * j)
        x &= (1 << nbits) - 1
        x |= (3 << (nbits - 2)) | 1
        vals.append(x)
    return ints_to_rows(vals, s)
