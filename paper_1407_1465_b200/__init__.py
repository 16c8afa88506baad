"""B200-native batched RSA modular exponentiation (arXiv 1407.1465 hot path).

Thin Python binding over the C-ABI of ``librsa_b200.so`` (``include/rsa_b200.h``).
Argument marshalling only: every step of the hot path runs in the library's
CUDA kernels.  There is no CPU fallback -- importing this package without the
built library raises ``ImportError``.

Calls (same names as the C-ABI):
  rsa_modexp_batch(base, exp, n, nbits, out=None, stream=None)   device tensors
  rsa_modexp_batch_host(base, exp, n, nbits)                     host arrays (e2e)
  rsa_keygen_check(p, q, e) -> (n, phi, d)                       Fig 1
  rsa_validate_key(e, d, p, q) -> (ok, residue)
  rsa_encode(text) / rsa_decode(packets)                         sec. 2 codec
  rsa_plan_info(exp, n, nbits) -> dict
"""
from __future__ import annotations

import contextlib
import ctypes
import functools
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# RSA_B200_LIB: an alternate in-tree build of the same library (kernel A/B
# measurements only, e.g. paper_1407_1465_b200/librsa_b200_<variant>.so)
LIB_PATH = os.environ.get("RSA_B200_LIB") or os.path.join(_HERE, "librsa_b200.so")

RSA_OK, RSA_EINVAL, RSA_ERANGE, RSA_EEVEN = 0, -1, -2, -3
RSA_ENOTPRIME, RSA_EEQUAL, RSA_ENOTCOPRIME = -4, -5, -6
RSA_ECHAR, RSA_EODD, RSA_ENOSPC, RSA_EPACKET, RSA_EBADKEY, RSA_ECUDA = -7, -8, -9, -10, -11, -12
RSA_MAX_NBITS = 4096

EXPORTS = ["rsa_strerror", "rsa_keygen_check", "rsa_validate_key", "rsa_modexp_batch",
           "rsa_modexp_batch_host", "rsa_plan_info", "rsa_set_window", "rsa_encode", "rsa_decode",
           "rsa_kernel_launches", "rsa_modexp_batch_paper", "rsa_modexp_batch_multi", "rsa_miller_rabin_batch",
           "rsa_prime_candidates", "rsa_prime_sieve", "rsa_prime_search", "rsa_keygen", "rsa_multi_plan_info",
           "rsa_decrypt_crt_batch", "rsa_encrypt_text", "rsa_decrypt_text", "rsa_set_kernel_path",
           "rsa_get_kernel_path", "rsa_modexp_batch_schedule"]
# kernel paths per width class (rsa_set_kernel_path; include/rsa_b200.h)
# the paper's single-word schedules (rsa_modexp_batch_schedule)
RSA_SCHED_NAIVE, RSA_SCHED_R2L, RSA_SCHED_L2R, RSA_SCHED_HALVING, RSA_SCHED_HALVING_FAITHFUL = 1, 2, 3, 4, 5
RSA_PATH_DEFAULT, RSA_PATH_FP64, RSA_PATH_INT, RSA_PATH_INT_GROUP, RSA_PATH_INT_PAIR, RSA_PATH_INT_MULTI, RSA_PATH_TC = range(7)

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is not built: run `python paper_1407_1465_b200/build.py` "
                      "(no CPU fallback exists)")

_lib = ctypes.CDLL(LIB_PATH)
_u32p = ctypes.POINTER(ctypes.c_uint32)


class RsaPlanInfo(ctypes.Structure):
    _fields_ = [("width_class", ctypes.c_int), ("s_io", ctypes.c_int), ("window", ctypes.c_int),
                ("table_entries", ctypes.c_int), ("nops", ctypes.c_int), ("montmuls", ctypes.c_longlong),
                ("squarings", ctypes.c_longlong), ("exp_bits", ctypes.c_int), ("grid", ctypes.c_int),
                ("block", ctypes.c_int), ("sqr_kernel", ctypes.c_int), ("products", ctypes.c_longlong),
                ("fp64_digits", ctypes.c_int), ("digit_products", ctypes.c_longlong)]


_lib.rsa_strerror.restype = ctypes.c_char_p
_lib.rsa_strerror.argtypes = [ctypes.c_int]
_lib.rsa_keygen_check.argtypes = [_u32p, _u32p, ctypes.c_int, _u32p, ctypes.c_int, _u32p, _u32p, _u32p]
_lib.rsa_validate_key.argtypes = [_u32p, _u32p, _u32p, _u32p, ctypes.c_int, _u32p]
_lib.rsa_modexp_batch.argtypes = [ctypes.c_void_p, _u32p, _u32p, ctypes.c_int, ctypes.c_size_t,
                                  ctypes.c_void_p, ctypes.c_void_p]
_lib.rsa_modexp_batch_host.argtypes = [ctypes.c_void_p, _u32p, _u32p, ctypes.c_int, ctypes.c_size_t,
                                       ctypes.c_void_p]
_lib.rsa_plan_info.argtypes = [_u32p, _u32p, ctypes.c_int, ctypes.POINTER(RsaPlanInfo)]
_lib.rsa_set_window.argtypes = [ctypes.c_int]
_lib.rsa_modexp_batch_schedule.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t,
                                           ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]
_lib.rsa_set_kernel_path.argtypes = [ctypes.c_int, ctypes.c_int]
_lib.rsa_get_kernel_path.argtypes = [ctypes.c_int]
_lib.rsa_encode.argtypes = [ctypes.c_char_p, _u32p, ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
_lib.rsa_decode.argtypes = [_u32p, ctypes.c_size_t, ctypes.c_char_p, ctypes.c_size_t]
_lib.rsa_kernel_launches.restype = ctypes.c_ulonglong
_vp = ctypes.c_void_p
_lib.rsa_modexp_batch_multi.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_int, ctypes.c_size_t, _vp, _vp, _vp]
_lib.rsa_miller_rabin_batch.argtypes = [_vp, ctypes.c_int, ctypes.c_size_t, ctypes.c_uint32, _vp, _vp]
_lib.rsa_prime_candidates.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_ulonglong, ctypes.c_size_t, _vp, _vp]
_lib.rsa_prime_sieve.argtypes = [_vp, ctypes.c_int, ctypes.c_size_t, _vp, _vp]
_lib.rsa_prime_search.argtypes = [ctypes.c_int, ctypes.c_uint64, ctypes.c_int, ctypes.c_int, _u32p,
                                  ctypes.POINTER(ctypes.c_ulonglong)]
_lib.rsa_keygen.argtypes = [ctypes.c_int, _u32p, ctypes.c_int, ctypes.c_uint64, _u32p, _u32p, _u32p, _u32p, _u32p]
_lib.rsa_multi_plan_info.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(RsaPlanInfo)]
_lib.rsa_decrypt_crt_batch.argtypes = [_vp, _u32p, _u32p, ctypes.c_int, _u32p, ctypes.c_int, ctypes.c_size_t, _vp, _vp]
_lib.rsa_encrypt_text.argtypes = [_vp, ctypes.c_size_t, _u32p, _u32p, ctypes.c_int, _vp, _vp, _vp]
_lib.rsa_decrypt_text.argtypes = [_vp, ctypes.c_size_t, _u32p, _u32p, ctypes.c_int, _vp, _vp, _vp]
_lib.rsa_modexp_batch_paper.argtypes = [ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_size_t,
                                        ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p]


class RsaError(RuntimeError):
    def __init__(self, code: int, where: str = ""):
        msg = _lib.rsa_strerror(code).decode()
        super().__init__(f"{where}: {msg} ({code})" if where else f"{msg} ({code})")
        self.code = code


def _check(rc: int, where: str):
    if rc != RSA_OK:
        raise RsaError(rc, where)


def limbs(x: int, n: int) -> np.ndarray:
    """Python int -> n little-endian uint32 limbs."""
    if x < 0 or x >> (32 * n):
        raise ValueError("value does not fit in %d limbs" % n)
    return np.frombuffer(int(x).to_bytes(4 * n, "little"), dtype="<u4").astype(np.uint32)


@functools.lru_cache(maxsize=256)
def _climbs(x: int, n: int) -> np.ndarray:
    """limbs() for the per-call key arguments (exp, n, ...), cached read-only:
    the same key is converted once, not on every batch."""
    a = limbs(x, n)
    a.flags.writeable = False
    return a


def _on(device):
    """Make `device` current for the call unless it already is (entering
    torch.cuda.device costs two device switches per call)."""
    import torch
    if device.index is None or device.index == torch.cuda.current_device():
        return contextlib.nullcontext()
    return torch.cuda.device(device)


def _rows(t, s: int, name: str, cuda: bool = True, like=None):
    """Check a packet array at the boundary: 2-D [count, s], 4-byte elements,
    C-contiguous, on a CUDA device (cuda=True) or in host memory (cuda=False),
    and shaped like `like` if given.  The C side trusts count*s, so a wrong
    shape here would be an out-of-bounds access there."""
    import torch
    if isinstance(t, np.ndarray):
        ok = (not cuda and t.ndim == 2 and t.shape[1] == s and t.itemsize == 4 and t.flags.c_contiguous)
    elif isinstance(t, torch.Tensor):
        ok = (t.dim() == 2 and t.shape[1] == s and t.element_size() == 4 and t.is_contiguous()
              and t.is_cuda == cuda and not (t.dtype.is_floating_point or t.dtype.is_complex))
    else:
        ok = False
    if ok and like is not None:
        ok = tuple(t.shape) == tuple(like.shape) and (not cuda or t.device == like.device)
    if not ok:
        where = "CUDA" if cuda else "host (numpy or CPU tensor)"
        shape = f"[{like.shape[0]}, {s}]" if like is not None else f"[count, {s}]"
        raise ValueError(f"{name} must be a contiguous {where} {shape} array of 32-bit integers")
    return t


def _vec(t, n: int, name: str, itemsize: int, cuda: bool = True):
    """A contiguous 1-D CUDA tensor of n elements of `itemsize` bytes."""
    if t.dim() != 1 or t.numel() != n or t.element_size() != itemsize or not t.is_contiguous() or t.is_cuda != cuda:
        raise ValueError(f"{name} must be a contiguous 1-D CUDA tensor of {n} {8 * itemsize}-bit elements")
    return t


def to_int(a) -> int:
    return int.from_bytes(np.ascontiguousarray(a, dtype="<u4").tobytes(), "little")


def _p(a: np.ndarray):
    return a.ctypes.data_as(_u32p)


def nlimbs(nbits: int) -> int:
    return (nbits + 31) // 32


# ------------------------------------------------------------------ hot path

def rsa_modexp_batch(base, exp: int, n: int, nbits: int, out=None, stream=None):
    """out[i] = base[i]^exp mod n on the GPU (asynchronous on `stream`).

    base: CUDA tensor [count, s] of int32/uint32 limbs (s = ceil(nbits/32)).
    out:  CUDA tensor of the same shape (allocated if None; may be `base`).
    stream: a torch.cuda.Stream, a raw cudaStream_t int, or None for the
            current torch stream.
    """
    import torch
    s = nlimbs(nbits)
    base = _rows(base.contiguous() if isinstance(base, torch.Tensor) else base, s, "base")
    if out is None:
        out = torch.empty_like(base)
    _rows(out, s, "out", like=base)
    if stream is None:
        stream = torch.cuda.current_stream(base.device).cuda_stream
    elif hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    E, N = _climbs(exp, s), _climbs(n, s)
    with _on(base.device):
        rc = _lib.rsa_modexp_batch(ctypes.c_void_p(base.data_ptr()), _p(E), _p(N), nbits, base.shape[0],
                                   ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(stream))
    _check(rc, "rsa_modexp_batch")
    return out


def rsa_decrypt_crt_batch(c, p: int, q: int, d: int, nbits: int, out=None, stream=None):
    """M = c^d mod pq by the CRT (two half-width exponentiations + Garner)."""
    import torch
    s = nlimbs(nbits)
    c = _rows(c.contiguous(), s, "c")
    if out is None:
        out = torch.empty_like(c)
    _rows(out, s, "out", like=c)
    pl = nlimbs(max(p.bit_length(), q.bit_length(), 1))
    with _on(c.device):
        rc = _lib.rsa_decrypt_crt_batch(_vp(c.data_ptr()), _p(limbs(p, pl)), _p(limbs(q, pl)), pl, _p(limbs(d, s)),
                                        nbits, c.shape[0], _vp(out.data_ptr()), _vp(_stream_of(c, stream)))
    _check(rc, "rsa_decrypt_crt_batch")
    return out


def rsa_encrypt_text(text, e: int, n: int, nbits: int, status=None, out=None, stream=None):
    """Fused sec. 2 codec + encryption.  text: CUDA uint8 tensor of lowercase
    letters (spaces stripped, even length) or a str; returns [count, s]."""
    import torch
    if isinstance(text, str):
        text = torch.tensor(list(text.replace(" ", "").encode("ascii")), dtype=torch.uint8, device="cuda")
    s = nlimbs(nbits)
    if text.dim() != 1 or text.element_size() != 1 or not text.is_cuda or not text.is_contiguous():
        raise ValueError("text must be a contiguous 1-D CUDA uint8 tensor")
    if out is None:
        out = torch.empty((text.numel() // 2, s), dtype=torch.int32, device=text.device)
    _rows(out, s, "out")
    if out.shape[0] != text.numel() // 2 or out.device != text.device:
        raise ValueError(f"out must be [{text.numel() // 2}, {s}] on {text.device}")
    if status is not None:
        _vec(status, text.numel() // 2, "status", 4)
    with _on(text.device):
        rc = _lib.rsa_encrypt_text(_vp(text.data_ptr()), text.numel(), _p(limbs(e, s)), _p(limbs(n, s)), nbits,
                                   _vp(out.data_ptr()), _vp(status.data_ptr() if status is not None else 0),
                                   _vp(_stream_of(text, stream)))
    _check(rc, "rsa_encrypt_text")
    return out


def rsa_decrypt_text(cipher, d: int, n: int, nbits: int, status=None, out=None, stream=None):
    """Fused decryption + sec. 2 decoding; returns a CUDA uint8 tensor of letters."""
    import torch
    s = nlimbs(nbits)
    cipher = _rows(cipher.contiguous(), s, "cipher")
    if out is None:
        out = torch.empty(2 * cipher.shape[0], dtype=torch.uint8, device=cipher.device)
    _vec(out, 2 * cipher.shape[0], "out", 1)
    if status is not None:
        _vec(status, cipher.shape[0], "status", 4)
    with _on(cipher.device):
        rc = _lib.rsa_decrypt_text(_vp(cipher.data_ptr()), cipher.shape[0], _p(limbs(d, s)), _p(limbs(n, s)), nbits,
                                   _vp(out.data_ptr()), _vp(status.data_ptr() if status is not None else 0),
                                   _vp(_stream_of(cipher, stream)))
    _check(rc, "rsa_decrypt_text")
    return out


def rsa_modexp_batch_host(base: np.ndarray, exp: int, n: int, nbits: int, out: np.ndarray | None = None):
    """End-to-end from host memory (H2D, kernel, D2H pipelined); synchronous."""
    s = nlimbs(nbits)
    base = np.ascontiguousarray(base, dtype=np.uint32) if isinstance(base, np.ndarray) else base
    _rows(base, s, "base", cuda=False)
    if out is None:
        out = np.empty_like(base)
    _rows(out, s, "out", cuda=False, like=base)
    E, N = limbs(exp, s), limbs(n, s)
    bp = base.ctypes.data if isinstance(base, np.ndarray) else base.data_ptr()
    op = out.ctypes.data if isinstance(out, np.ndarray) else out.data_ptr()
    rc = _lib.rsa_modexp_batch_host(ctypes.c_void_p(bp), _p(E), _p(N), nbits, base.shape[0], ctypes.c_void_p(op))
    _check(rc, "rsa_modexp_batch_host")
    return out


def rsa_modexp_batch_paper(num, key: int, den: int, faithful: bool = True, out=None, stream=None):
    """The paper's Fig 12 kernel on the GPU (prior art): num is a CUDA
    int32/uint32 tensor of single-word packets; returns result tensor."""
    import torch
    if not num.is_cuda or num.element_size() != 4:
        raise ValueError("num must be a CUDA tensor of 32-bit packets")
    num = num.contiguous().view(-1)
    if out is None:
        out = torch.empty_like(num)
    _vec(out, num.numel(), "out", 4)
    if stream is None:
        stream = torch.cuda.current_stream(num.device).cuda_stream
    elif hasattr(stream, "cuda_stream"):
        stream = stream.cuda_stream
    with _on(num.device):
        rc = _lib.rsa_modexp_batch_paper(ctypes.c_void_p(num.data_ptr()), key, den, num.numel(),
                                         ctypes.c_void_p(out.data_ptr()), 1 if faithful else 0, ctypes.c_void_p(stream))
    _check(rc, "rsa_modexp_batch_paper")
    return out


def rsa_modexp_batch_schedule(num, exp: int, den: int, schedule: int, out=None, stream=None):
    """num^exp mod den by one of the paper's schedules (Fig 4 naive, Fig 5a
    right-to-left, Fig 5b left-to-right, Fig 12 halving) on the GPU: num is a
    CUDA tensor of 32-bit single-word packets; returns the result tensor."""
    import torch
    if not num.is_cuda or num.element_size() != 4:
        raise ValueError("num must be a CUDA tensor of 32-bit packets")
    num = num.contiguous().view(-1)
    if out is None:
        out = torch.empty_like(num)
    _vec(out, num.numel(), "out", 4)
    with _on(num.device):
        rc = _lib.rsa_modexp_batch_schedule(ctypes.c_void_p(num.data_ptr()), exp, den, num.numel(),
                                            ctypes.c_void_p(out.data_ptr()), schedule,
                                            ctypes.c_void_p(_stream_of(num, stream)))
    _check(rc, "rsa_modexp_batch_schedule")
    return out


def _stream_of(t, stream):
    import torch
    if stream is None:
        return torch.cuda.current_stream(t.device).cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else stream


def rsa_modexp_batch_multi(base, exps, mods, nbits: int, exp_bits: int | None = None, out=None, status=None,
                           stream=None):
    """out[i] = base[i]^exps[i] mod mods[i] (CUDA [count, s] 32-bit tensors)."""
    import torch
    s = nlimbs(nbits)
    base, exps, mods = base.contiguous(), exps.contiguous(), mods.contiguous()
    _rows(base, s, "base")
    _rows(exps, s, "exps", like=base)
    _rows(mods, s, "mods", like=base)
    if out is None:
        out = torch.empty_like(base)
    _rows(out, s, "out", like=base)
    if status is not None:
        _vec(status, base.shape[0], "status", 4)
    exp_bits = 32 * s if exp_bits is None else exp_bits
    with _on(base.device):
        rc = _lib.rsa_modexp_batch_multi(_vp(base.data_ptr()), _vp(exps.data_ptr()), _vp(mods.data_ptr()), nbits,
                                         exp_bits, base.shape[0], _vp(out.data_ptr()),
                                         _vp(status.data_ptr() if status is not None else 0),
                                         _vp(_stream_of(base, stream)))
    _check(rc, "rsa_modexp_batch_multi")
    return out


def rsa_miller_rabin_batch(cand, nbits: int, base: int, out=None, stream=None):
    import torch
    cand = _rows(cand.contiguous(), nlimbs(nbits), "cand")
    if out is None:
        out = torch.empty(cand.shape[0], dtype=torch.int32, device=cand.device)
    _vec(out, cand.shape[0], "out", 4)
    with _on(cand.device):
        rc = _lib.rsa_miller_rabin_batch(_vp(cand.data_ptr()), nbits, cand.shape[0], base, _vp(out.data_ptr()),
                                         _vp(_stream_of(cand, stream)))
    _check(rc, "rsa_miller_rabin_batch")
    return out


def rsa_prime_candidates(nbits: int, seed: int, first: int, count: int, device="cuda", stream=None):
    import torch
    out = torch.empty((count, nlimbs(nbits)), dtype=torch.int32, device=device)
    with _on(out.device):
        rc = _lib.rsa_prime_candidates(nbits, seed, first, count, _vp(out.data_ptr()), _vp(_stream_of(out, stream)))
    _check(rc, "rsa_prime_candidates")
    return out


def rsa_prime_sieve(cand, nbits: int, stream=None):
    import torch
    cand = _rows(cand.contiguous(), nlimbs(nbits), "cand")
    out = torch.empty(cand.shape[0], dtype=torch.int32, device=cand.device)
    with _on(cand.device):
        rc = _lib.rsa_prime_sieve(_vp(cand.data_ptr()), nbits, cand.shape[0], _vp(out.data_ptr()),
                                  _vp(_stream_of(cand, stream)))
    _check(rc, "rsa_prime_sieve")
    return out


def rsa_prime_search(nbits: int, seed: int, want: int, rounds: int = 8):
    """Returns (primes as Python ints, candidates tried)."""
    s = nlimbs(nbits)
    buf = np.zeros(max(want, 1) * s, np.uint32)
    tried = ctypes.c_ulonglong(0)
    _check(_lib.rsa_prime_search(nbits, seed, want, rounds, _p(buf), ctypes.byref(tried)), "rsa_prime_search")
    return [to_int(buf[i * s:(i + 1) * s]) for i in range(want)], tried.value


def rsa_keygen(nbits: int, e: int = 65537, seed: int = 1):
    """Fig 1 key generation with the GPU prime search -> dict(p, q, n, phi, d, e)."""
    h = nlimbs(nbits - nbits // 2)
    el = nlimbs(max(e.bit_length(), 1))
    P, Q = np.zeros(h, np.uint32), np.zeros(h, np.uint32)
    N, PHI, D = (np.zeros(2 * h, np.uint32) for _ in range(3))
    _check(_lib.rsa_keygen(nbits, _p(limbs(e, el)), el, seed, _p(P), _p(Q), _p(N), _p(PHI), _p(D)), "rsa_keygen")
    return dict(p=to_int(P), q=to_int(Q), n=to_int(N), phi=to_int(PHI), d=to_int(D), e=e)


def rsa_plan_info(exp: int, n: int, nbits: int) -> dict:
    s = nlimbs(nbits)
    info = RsaPlanInfo()
    _check(_lib.rsa_plan_info(_p(limbs(exp, s)), _p(limbs(n, s)), nbits, ctypes.byref(info)), "rsa_plan_info")
    return {f: getattr(info, f) for f, _ in RsaPlanInfo._fields_}


def rsa_multi_plan_info(nbits: int, exp_bits: int, mr: bool = False) -> dict:
    info = RsaPlanInfo()
    _check(_lib.rsa_multi_plan_info(nbits, exp_bits, 1 if mr else 0, ctypes.byref(info)), "rsa_multi_plan_info")
    return {f: getattr(info, f) for f, _ in RsaPlanInfo._fields_}


def rsa_set_window(w: int) -> None:
    _check(_lib.rsa_set_window(w), "rsa_set_window")


def rsa_set_kernel_path(width_class: int, path: int) -> None:
    """Select the kernel of a width class (A/B measurement; include/rsa_b200.h)."""
    _check(_lib.rsa_set_kernel_path(width_class, path), "rsa_set_kernel_path")


def rsa_get_kernel_path(width_class: int) -> int:
    rc = _lib.rsa_get_kernel_path(width_class)
    if rc < 0:
        _check(rc, "rsa_get_kernel_path")
    return rc


@contextlib.contextmanager
def kernel_path(width_class: int, path: int):
    """with kernel_path(64, RSA_PATH_INT): ... -- restores the default after."""
    rsa_set_kernel_path(width_class, path)
    try:
        yield
    finally:
        rsa_set_kernel_path(width_class, RSA_PATH_DEFAULT)


def rsa_kernel_launches() -> int:
    return int(_lib.rsa_kernel_launches())


# ------------------------------------------------------------------ keys

def rsa_keygen_check(p: int, q: int, e: int):
    pl = max(nlimbs(max(p.bit_length(), q.bit_length(), 1)), 1)
    el = nlimbs(max(e.bit_length(), 1))
    n = np.zeros(2 * pl, np.uint32)
    phi = np.zeros(2 * pl, np.uint32)
    d = np.zeros(2 * pl, np.uint32)
    rc = _lib.rsa_keygen_check(_p(limbs(p, pl)), _p(limbs(q, pl)), pl, _p(limbs(e, el)), el, _p(n), _p(phi), _p(d))
    _check(rc, "rsa_keygen_check")
    return to_int(n), to_int(phi), to_int(d)


def rsa_validate_key(e: int, d: int, p: int, q: int):
    L = max(nlimbs(max(v.bit_length(), 1)) for v in (e, d, p, q))
    r = np.zeros(2 * L, np.uint32)
    rc = _lib.rsa_validate_key(*(_p(limbs(v, L)) for v in (e, d, p, q)), L, _p(r))
    if rc not in (RSA_OK, RSA_EBADKEY):
        _check(rc, "rsa_validate_key")
    return rc == RSA_OK, to_int(r)


# ------------------------------------------------------------------ codec

def rsa_encode(text: str):
    cap = len(text) // 2 + 1
    pk = np.zeros(cap, np.uint32)
    cnt = ctypes.c_size_t(0)
    _check(_lib.rsa_encode(text.encode("ascii"), _p(pk), cap, ctypes.byref(cnt)), "rsa_encode")
    return [int(v) for v in pk[: cnt.value]]


def rsa_decode(packets) -> str:
    pk = np.ascontiguousarray(packets, dtype=np.uint32)
    buf = ctypes.create_string_buffer(2 * len(pk) + 1)
    _check(_lib.rsa_decode(_p(pk), len(pk), buf, len(buf)), "rsa_decode")
    return buf.value.decode("ascii")
