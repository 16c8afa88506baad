"""Multi-GPU batch sharding (sec. 8(a) row a9).

Packets are independent (sec. 9: the plaintext is divided "into
packets of same length and then apply encryption or decryption transformation
on each packet"), and the paper's flow is one batch in, one result array out
(sec. 6).  So one batch of `count` packets shards into
contiguous slices, one per rank (one process per GPU); every rank derives the
same key; the only collective is the reassembly of the result slices (one
NCCL all-gather over NVLink/NVSwitch), which is step a9 of the hot path.

    shard_bounds(count, world) -> ([(lo, hi)] per rank, per)
    shard_range(count, rank, world) -> (lo, hi)
    modexp_sharded(local, exp, n, nbits, count, ...)        device slice in, whole result out
    modexp_sharded_host(local_host, exp, n, nbits, count, ...)  end to end from host memory

Layout: rank r owns rows [r*per, min(count, (r+1)*per)) with per = ceil(count /
world).  Every slice except the last is exactly `per` rows, so when each rank
writes its result straight into its own chunk of a [per*world, s] gather
buffer, the in-place all-gather (send buffer = the rank's chunk of the receive
buffer) leaves the whole result in rows [0, count) with no re-assembly copy.
"""
from __future__ import annotations


def shard_bounds(count: int, world: int):
    """Contiguous slices: rank r gets [r*ceil(N/k), min(N, (r+1)*ceil(N/k)))."""
    if world < 1 or count < 0:
        raise ValueError("bad count/world")
    per = -(-count // world) if count else 0
    return [(min(count, r * per), min(count, (r + 1) * per)) for r in range(world)], per


def shard_range(count: int, rank: int, world: int):
    b, _ = shard_bounds(count, world)
    return b[rank]


def _world(group):
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(group), dist.get_rank(group)
    return 1, 0


def _exps(exp):
    return [int(e) for e in exp] if isinstance(exp, (list, tuple)) else [int(exp)]


def gather_slices(full, per: int, group=None):
    """In-place all-gather: this rank's result is already in its chunk
    full[rank*per:(rank+1)*per]; afterwards every chunk is filled.  NCCL gathers
    device memory directly (over NVLink); a gloo group (CPU tests, or several
    ranks sharing one GPU) stages device tensors through host memory."""
    import torch
    import torch.distributed as dist
    world, rank = _world(group)
    if world == 1 or per == 0:
        return full
    chunk = full[rank * per:(rank + 1) * per]
    if full.is_cuda and dist.get_backend(group) != "nccl":
        hf = torch.empty(full.shape, dtype=full.dtype)
        dist.all_gather_into_tensor(hf, chunk.cpu(), group=group)
        full.copy_(hf)
    else:
        dist.all_gather_into_tensor(full, chunk, group=group)
    return full


def modexp_sharded(local, exp, n: int, nbits: int, count: int, group=None, gather: bool = True, out=None,
                   stream=None, compute=None):
    """Exponentiate this rank's slice and reassemble the batch.

    local:   this rank's rows [lo, hi) of a global batch of `count` packets,
             a [hi - lo, s] tensor on this rank's device (s = ceil(nbits/32));
    exp:     an exponent, or a sequence applied in order (e.g. (e, d): the
             encrypt-then-decrypt round trip);
    gather:  if True return the whole [count, s] result on every rank (one
             all-gather); else this rank's [hi - lo, s] result;
    out:     optional gather buffer, [per * world, s] (gather) or [hi - lo, s];
    compute: compute(x, e, out) -> out, defaults to the CUDA path
             (paper_1407_1465_b200.rsa_modexp_batch; out may alias x); it is
             injectable so the reassembly logic runs on CPU with gloo.
    """
    import torch
    world, rank = _world(group)
    bounds, per = shard_bounds(count, world)
    lo, hi = bounds[rank]
    if local.dim() != 2 or local.shape[0] != hi - lo:
        raise ValueError(f"rank {rank} of {world} owns rows [{lo}, {hi}) of {count}: "
                         f"local must be [{hi - lo}, s], got {tuple(local.shape)}")
    s = local.shape[1]
    if compute is None:
        from . import rsa_modexp_batch

        def compute(x, e, o):
            return rsa_modexp_batch(x, e, n, nbits, out=o, stream=stream)
    gathering = gather and world > 1
    rows = per * world if gathering else hi - lo
    if out is None:
        out = torch.empty((rows, s), dtype=local.dtype, device=local.device)
    elif tuple(out.shape) != (rows, s) or out.device != local.device:
        raise ValueError(f"out must be [{rows}, {s}] on {local.device}")
    mine = out[rank * per:rank * per + (hi - lo)] if gathering else out
    if hi > lo:
        exps = _exps(exp)
        if not exps:
            mine.copy_(local)
        src = local
        for e in exps:
            r = compute(src, e, mine)
            if r is not None and r.data_ptr() != mine.data_ptr():
                mine.copy_(r)
            src = mine
    if not gathering:
        return out
    gather_slices(out, per, group)
    return out[:count]


def modexp_sharded_host(local_host, exp, n: int, nbits: int, count: int, group=None, root: int = 0, out=None,
                        device=None):
    """End to end from host memory, one process per GPU: every rank copies its
    host slice to its device, exponentiates it (exp or a sequence of
    exponents), the slices are all-gathered on the devices, and rank `root`
    copies the whole [count, s] result back to host memory (`out`, pinned if
    given) and returns it; other ranks return None.  At world size 1 this is
    the C-ABI host entry (rsa_modexp_batch_host: H2D, kernel and D2H pipelined
    in chunks) once per exponent."""
    import numpy as np
    import torch
    world, rank = _world(group)
    exps = _exps(exp)
    if world == 1:
        from . import rsa_modexp_batch_host
        cur = local_host
        if out is None:
            out = torch.empty(tuple(local_host.shape), dtype=torch.int32).pin_memory() \
                if isinstance(local_host, torch.Tensor) else np.empty_like(local_host)
        for e in exps:
            rsa_modexp_batch_host(cur, e, n, nbits, out=out)
            cur = out
        return out
    dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
    x = torch.as_tensor(local_host).to(dev, non_blocking=True)
    full = modexp_sharded(x, exps, n, nbits, count, group=group)
    if rank != root:
        torch.cuda.current_stream(dev).synchronize()
        return None
    if out is None:
        out = torch.empty(tuple(full.shape), dtype=full.dtype).pin_memory()
    out.copy_(full, non_blocking=True)
    torch.cuda.current_stream(dev).synchronize()
    return out
