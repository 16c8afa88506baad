"""Multi-GPU batch sharding.

Packets are independent ("divides the plaintext ... into packets
of same length and then apply encryption or decryption transformation on each
packet"), so a batch shards into contiguous slices, one per rank; the key is
shared.  The only collective is the optional reassembly of the result slices
(NCCL all-gather over NVLink); it is not part of the hot path.

    shard_range(count, rank, world) -> (lo, hi)
    modexp_sharded(local_or_full, exp, n, nbits, group=None, gather=True)
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


def modexp_sharded(full, exp: int, n: int, nbits: int, group=None, gather: bool = True, compute=None):
    """Exponentiate this rank's slice of `full` ([count, s] tensor, on this
    rank's device) and, if `gather`, reassemble the whole result on every rank
    with one all-gather (slices padded to equal length).

    `compute(slice) -> slice` defaults to the CUDA path
    (paper_1407_1465_b200.rsa_modexp_batch); it is injectable so the
    reassembly logic can be tested on CPU with the gloo backend.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    count = full.shape[0]
    bounds, per = shard_bounds(count, world)
    lo, hi = bounds[rank]
    if compute is None:
        from . import rsa_modexp_batch

        def compute(x):
            return rsa_modexp_batch(x, exp, n, nbits)
    mine = compute(full[lo:hi].contiguous()) if hi > lo else full[lo:hi].clone()
    if not gather or world == 1:
        return mine
    padded = torch.zeros((per, full.shape[1]), dtype=full.dtype, device=full.device)
    padded[: hi - lo] = mine
    out = torch.empty((per * world, full.shape[1]), dtype=full.dtype, device=full.device)
    dist.all_gather_into_tensor(out, padded, group=group)
    # drop per-rank padding
    pieces = [out[r * per: r * per + (bounds[r][1] - bounds[r][0])] for r in range(world)]
    return torch.cat(pieces, 0)
