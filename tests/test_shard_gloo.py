"""Multi-process (world_size 2 and 3, gloo, CPU) tests of the batch sharder:
contiguous slices, padding, all-gather reassembly.  The per-slice compute is
the oracle here (test infrastructure); on GPUs it is the CUDA path."""
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
        from paper_1407_1465_b200.shard import modexp_sharded
        k = workload.key("rsa256")
        base = workload.packets(count, 256, n=k["n"], config_id=9)
        full = torch.from_numpy(base.view(np.int32))

        def compute(x):
            return torch.from_numpy(oracle.modexp_batch(x.numpy().view(np.uint32), k["e"], k["n"]).view(np.int32))

        out = modexp_sharded(full, k["e"], k["n"], 256, compute=compute)
        lo, hi = shard_range(count, rank, world)
        mine = modexp_sharded(full, k["e"], k["n"], 256, compute=compute, gather=False)
        want = oracle.modexp_batch(base, k["e"], k["n"])
        ok = np.array_equal(out.numpy().view(np.uint32), want) and \
            np.array_equal(mine.numpy().view(np.uint32), want[lo:hi])
        q.put((rank, ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,count", [(2, 1001), (3, 10), (2, 1)])
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
