"""Multi-process (world_size 2..4, gloo, CPU) tests of the batch sharder:
each rank holds only its contiguous slice; in-place all-gather into the padded
buffer; round-trip pipelines; empty slices (count < world) and an empty batch.
The per-slice compute is the oracle here (test infrastructure); on the GPU
(tests/test_gpu_shard.py) it is the CUDA path."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1407_1465_b200.shard import shard_bounds, shard_range


@pytest.mark.parametrize("world", [1, 2, 3, 4, 7, 8])
@pytest.mark.parametrize("count", [0, 1, 5, 8, 9, 1000, 1 << 20])
def test_shard_bounds_partition(world, count):
    b, per = shard_bounds(count, world)
    covered = []
    for lo, hi in b:
        assert 0 <= lo <= hi <= count and hi - lo <= per
        covered.extend(range(lo, hi)) if count < 5000 else None
    if count < 5000:
        assert covered == list(range(count))
    assert b[0][0] == 0 and b[-1][1] == count
    assert sum(hi - lo for lo, hi in b) == count


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, count, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        import workload
        from paper_1407_1465_b200.shard import modexp_sharded, modexp_sharded_host
        k = workload.key("rsa256")
        base = workload.packets(count, 256, n=k["n"], config_id=9)
        lo, hi = shard_range(count, rank, world)
        local = torch.from_numpy(base[lo:hi].view(np.int32))      # this rank's slice only

        def compute(x, e, o):
            o.copy_(torch.from_numpy(oracle.modexp_batch(x.numpy().view(np.uint32), e, k["n"]).view(np.int32)))
            return o

        out = modexp_sharded(local, k["e"], k["n"], 256, count, compute=compute)
        mine = modexp_sharded(local, k["e"], k["n"], 256, count, compute=compute, gather=False)
        both = modexp_sharded(local, (k["e"], k["d"]), k["n"], 256, count, compute=compute)
        want = oracle.modexp_batch(base, k["e"], k["n"])
        ok = out.shape[0] == count and np.array_equal(out.numpy().view(np.uint32), want) and \
            np.array_equal(mine.numpy().view(np.uint32), want[lo:hi]) and \
            np.array_equal(both.numpy().view(np.uint32), base)
        # a wrong slice is rejected before any compute
        try:
            modexp_sharded(torch.zeros((hi - lo + 1, 8), dtype=torch.int32), 3, k["n"], 256, count, compute=compute)
            ok = False
        except ValueError:
            pass
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 1001), (3, 10), (2, 1), (4, 3), (3, 0)])
def test_gloo_all_gather_reassembly(world, count):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
