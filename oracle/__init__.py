"""CPU oracle for batched RSA modular exponentiation (arXiv 1407.1465).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product package ``paper_1407_1465_b200`` never imports it, and
this package never imports the product.

The arithmetic lives in plain C (``oracle/bn_oracle.c``: schoolbook multiply,
Knuth Algorithm D long division, Fig 5 left-to-right square-and-multiply,
PAPER.md:139-152).  This module only marshals Python ints <-> little-endian
uint32 limb arrays and calls it through ctypes.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

# status codes
OK, EINVAL, ERANGE, EEVEN, ENOTPRIME, EEQUAL, ENOTCOPRIME = 0, -1, -2, -3, -4, -5, -6
ECHAR, EODD, ENOSPC, EPACKET, EBADKEY = -7, -8, -9, -10, -11


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        super().__init__(f"oracle status {code} {what}".strip())
        self.code = code


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-O2", "-std=c99", "-fPIC", "-shared", "-pthread", "-Wall",
             "-o", _LIB, _SRC])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        u32p = ctypes.POINTER(ctypes.c_uint32)
        u64p = ctypes.POINTER(ctypes.c_uint64)
        L.oracle_modexp.argtypes = [u32p, ctypes.c_int, u32p, ctypes.c_int, u32p, ctypes.c_int, u32p]
        L.oracle_modexp_variant.argtypes = [ctypes.c_int, ctypes.c_int, u32p, ctypes.c_int, u32p,
                                            ctypes.c_int, u32p, ctypes.c_int, u32p]
        L.oracle_naive_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64, u64p, u64p]
        L.oracle_halving_u64.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_uint64,
                                         ctypes.c_int, u64p]
        L.oracle_is_prime.argtypes = [u32p, ctypes.c_int]
        L.oracle_keygen_check.argtypes = [u32p, u32p, ctypes.c_int, u32p, ctypes.c_int, u32p, u32p, u32p]
        L.oracle_validate_key.argtypes = [u32p, u32p, u32p, u32p, ctypes.c_int, u32p]
        L.oracle_modexp_batch.argtypes = [u32p, ctypes.c_size_t, ctypes.c_int, u32p, ctypes.c_int,
                                          u32p, ctypes.c_int, u32p, ctypes.c_int]
        L.oracle_modexp_multi.argtypes = [u32p, u32p, u32p, ctypes.c_size_t, ctypes.c_int, u32p, ctypes.c_int]
        L.oracle_mr_round.argtypes = [u32p, ctypes.c_int, ctypes.c_uint32]
        L.oracle_encode.argtypes = [ctypes.c_char_p, u32p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
        L.oracle_decode.argtypes = [u32p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
        _lib = L
    return _lib


# ---------------------------------------------------------------- marshalling

def limbs_of(x: int, n: int | None = None) -> np.ndarray:
    """Python int -> little-endian uint32 limbs (n limbs, zero padded)."""
    if x < 0:
        raise ValueError("negative")
    if n is None:
        n = max(1, (x.bit_length() + 31) // 32)
    out = np.zeros(n, dtype=np.uint32)
    for i in range(n):
        out[i] = x & 0xFFFFFFFF
        x >>= 32
    if x:
        raise ValueError("value does not fit in %d limbs" % n)
    return out


def int_of(limbs) -> int:
    v = 0
    for w in reversed([int(t) for t in np.asarray(limbs, dtype=np.uint32).ravel()]):
        v = (v << 32) | w
    return v


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_uint32))


def _nl(x: int) -> int:
    return max(1, (x.bit_length() + 31) // 32)


# ---------------------------------------------------------------- modexp

def modexp(g: int, e: int, m: int) -> int:
    """g^e mod m by Fig 5 left-to-right binary."""
    G, E, M = limbs_of(g), limbs_of(e), limbs_of(m)
    out = np.zeros(len(M), dtype=np.uint32)
    rc = lib().oracle_modexp(_p(G), len(G), _p(E), len(E), _p(M), len(M), _p(out))
    if rc:
        raise OracleError(rc, "modexp")
    return int_of(out)


_VARIANTS = {"l2r": 0, "r2l": 1, "kary": 2, "sliding": 3}


def modexp_variant(variant: str, g: int, e: int, m: int, k: int = 1) -> int:
    """Alternate schedules: 'r2l' (Fig 5a), 'kary' (Fig 6), 'sliding' (Fig 7)."""
    G, E, M = limbs_of(g), limbs_of(e), limbs_of(m)
    out = np.zeros(len(M), dtype=np.uint32)
    rc = lib().oracle_modexp_variant(_VARIANTS[variant], k, _p(G), len(G), _p(E), len(E),
                                     _p(M), len(M), _p(out))
    if rc:
        raise OracleError(rc, variant)
    return int_of(out)


def naive(g: int, e: int, m: int, trace: bool = False):
    """Fig 4 naive repeated multiplication (single-word), optional trace."""
    out = ctypes.c_uint64(0)
    tr = np.zeros(max(e, 1), dtype=np.uint64) if trace else None
    trp = tr.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)) if trace else None
    rc = lib().oracle_naive_u64(g, e, m, ctypes.byref(out), trp)
    if rc:
        raise OracleError(rc, "naive")
    if trace:
        return out.value, [int(t) for t in tr[:e]]
    return out.value


def halving(g: int, e: int, m: int, faithful: bool) -> int:
    """The paper's Fig 12 device loop, exact integers."""
    out = ctypes.c_uint64(0)
    rc = lib().oracle_halving_u64(g, e, m, 1 if faithful else 0, ctypes.byref(out))
    if rc:
        raise OracleError(rc, "halving")
    return out.value


def modexp_batch(base: np.ndarray, e: int, m: int, nthreads: int | None = None) -> np.ndarray:
    """out[i] = base[i]^e mod m; base is uint32 [count, s]; out [count, s_m]."""
    base = np.ascontiguousarray(base, dtype=np.uint32)
    count, s = base.shape
    E, M = limbs_of(e), limbs_of(m)
    out = np.zeros((count, len(M)), dtype=np.uint32)
    if nthreads is None:
        nthreads = os.cpu_count() or 1
    rc = lib().oracle_modexp_batch(_p(base), count, s, _p(E), len(E), _p(M), len(M), _p(out), nthreads)
    if rc:
        raise OracleError(rc, "modexp_batch")
    return out


def modexp_multi(base: np.ndarray, exps: np.ndarray, mods: np.ndarray, nthreads: int | None = None) -> np.ndarray:
    """out[i] = base[i]^exps[i] mod mods[i] (all uint32 [count, s])."""
    base = np.ascontiguousarray(base, dtype=np.uint32)
    exps = np.ascontiguousarray(exps, dtype=np.uint32)
    mods = np.ascontiguousarray(mods, dtype=np.uint32)
    count, s = base.shape
    assert exps.shape == mods.shape == base.shape
    out = np.zeros((count, s), dtype=np.uint32)
    rc = lib().oracle_modexp_multi(_p(base), _p(exps), _p(mods), count, s, _p(out), nthreads or os.cpu_count() or 1)
    if rc:
        raise OracleError(rc, "modexp_multi")
    return out


def mr_round(n: int, a: int) -> bool:
    """One Miller-Rabin round to base a (strong probable prime test)."""
    N = limbs_of(n)
    rc = lib().oracle_mr_round(_p(N), len(N), a)
    if rc < 0:
        raise OracleError(rc, "mr_round")
    return rc == 1


# ---------------------------------------------------------------- keys

def is_prime(x: int) -> bool:
    X = limbs_of(x)
    return lib().oracle_is_prime(_p(X), len(X)) == 1


def keygen_check(p: int, q: int, e: int):
    """Fig 1.  Returns (n, phi, d) or raises OracleError."""
    pl = max(_nl(p), _nl(q))
    P, Q, E = limbs_of(p, pl), limbs_of(q, pl), limbs_of(e)
    n = np.zeros(2 * pl, dtype=np.uint32)
    phi = np.zeros(2 * pl, dtype=np.uint32)
    d = np.zeros(2 * pl, dtype=np.uint32)
    rc = lib().oracle_keygen_check(_p(P), _p(Q), pl, _p(E), len(E), _p(n), _p(phi), _p(d))
    if rc:
        raise OracleError(rc, "keygen_check")
    return int_of(n), int_of(phi), int_of(d)


def validate_key(e: int, d: int, p: int, q: int):
    """Returns (ok, (d*e) mod phi)."""
    L = max(_nl(e), _nl(d), _nl(p), _nl(q))
    E, D, P, Q = (limbs_of(v, L) for v in (e, d, p, q))
    r = np.zeros(2 * L, dtype=np.uint32)
    rc = lib().oracle_validate_key(_p(E), _p(D), _p(P), _p(Q), L, _p(r))
    if rc not in (OK, EBADKEY):
        raise OracleError(rc, "validate_key")
    return rc == OK, int_of(r)


# ---------------------------------------------------------------- codec

def encode(text: str):
    cap = len(text) + 1
    pk = np.zeros(cap, dtype=np.uint32)
    cnt = ctypes.c_size_t(0)
    rc = lib().oracle_encode(text.encode("ascii"), _p(pk), cap, ctypes.byref(cnt))
    if rc:
        raise OracleError(rc, "encode")
    return [int(v) for v in pk[: cnt.value]]


def decode(packets) -> str:
    pk = np.asarray(packets, dtype=np.uint32)
    buf = ctypes.create_string_buffer(2 * len(pk) + 1)
    rc = lib().oracle_decode(_p(pk), len(pk), buf, len(buf))
    if rc:
        raise OracleError(rc, "decode")
    return buf.value.decode("ascii")
