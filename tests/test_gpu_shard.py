"""The sharded multi-GPU path with the
CUDA compute, bit-exact against the oracle element by element:
  * world size 1 (no process group): modexp_sharded and modexp_sharded_host;
  * 2 ranks with the gloo backend sharing the visible GPU (the gather is staged
    through host memory; on an 8-GPU box the same code all-gathers with NCCL):
    each rank holds only its slice, the result is reassembled on every rank,
    the host entry returns it on rank 0;
  * several devices in one process (the per-device launch caches), when the
    box has more than one GPU;
  * several host threads calling the C-ABI at once on their own streams."""
import os
import socket

import numpy as np
import pytest

import oracle
import workload

pytestmark = pytest.mark.gpu


def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return torch


@pytest.mark.parametrize("key,count", [("rsa2048", 777), ("rsa4096", 131), ("rsa1024", 1000), ("rsa64", 5000)])
def test_sharded_world1(key, count):
    torch = _cuda()
    from paper_1407_1465_b200.shard import modexp_sharded, modexp_sharded_host
    k = workload.key(key)
    nb = k["nbits"]
    base = workload.packets(count, nb, n=k["n"], config_id=31)
    x = torch.from_numpy(base.view(np.int32)).cuda()
    enc = modexp_sharded(x, k["e"], k["n"], nb, count).cpu().numpy().view(np.uint32)
    assert np.array_equal(enc, oracle.modexp_batch(base, k["e"], k["n"]))
    rt = modexp_sharded(x, (k["e"], k["d"]), k["n"], nb, count).cpu().numpy().view(np.uint32)
    assert np.array_equal(rt, base)
    host = torch.from_numpy(base.view(np.int32)).pin_memory()
    rth = modexp_sharded_host(host, (k["e"], k["d"]), k["n"], nb, count)
    assert np.array_equal(np.asarray(rth).view(np.uint32), base)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, key, count, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1407_1465_b200.shard import modexp_sharded, modexp_sharded_host, shard_range
        torch.cuda.set_device(rank % torch.cuda.device_count())
        k = workload.key(key)
        nb = k["nbits"]
        base = workload.packets(count, nb, n=k["n"], config_id=32)
        lo, hi = shard_range(count, rank, world)
        local = torch.from_numpy(base[lo:hi].view(np.int32)).cuda()
        enc = modexp_sharded(local, k["e"], k["n"], nb, count)
        want = oracle.modexp_batch(base, k["e"], k["n"])
        ok = enc.is_cuda and np.array_equal(enc.cpu().numpy().view(np.uint32), want)
        mine = modexp_sharded(local, k["e"], k["n"], nb, count, gather=False)
        ok = ok and np.array_equal(mine.cpu().numpy().view(np.uint32), want[lo:hi])
        # the round trip through the host entry: H2D slice, kernels, gather, D2H on rank 0
        host = torch.from_numpy(base[lo:hi].view(np.int32)).pin_memory()
        got = modexp_sharded_host(host, (k["e"], k["d"]), k["n"], nb, count)
        if rank == 0:
            ok = ok and got is not None and np.array_equal(got.numpy().view(np.uint32), base)
        else:
            ok = ok and got is None
        q.put((rank, bool(ok)))
    except Exception as ex:       # report, do not hang the parent
        q.put((rank, repr(ex)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("key,count", [("rsa2048", 1001), ("rsa4096", 67), ("rsa256", 3)])
def test_sharded_two_ranks_gloo(key, count):
    _cuda()
    import torch.multiprocessing as mp
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, key, count, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert all(ok is True for _, ok in res), res


def test_device_switch_in_one_process():
    """Every launcher's shared-memory opt-in and occupancy are cached per
    device: alternate devices in one process, each launch bit-exact."""
    torch = _cuda()
    if torch.cuda.device_count() < 2:
        pytest.skip("one visible GPU")
    import paper_1407_1465_b200 as R
    k = workload.key("rsa2048")
    base = workload.packets(300, 2048, n=k["n"], config_id=33)
    want = oracle.modexp_batch(base, k["d"], k["n"])
    for dev in [0, 1, 0, 1]:
        x = torch.from_numpy(base.view(np.int32)).to(f"cuda:{dev}")
        got = R.rsa_modexp_batch(x, k["d"], k["n"], 2048).cpu().numpy().view(np.uint32)
        assert np.array_equal(got, want), dev


def test_concurrent_calls_from_threads():
    """Several host threads, each on its own CUDA stream with its own key and
    width class, call the C-ABI at once: the plan cache, the per-device launch
    caches and the stream-ordered workspaces are shared; every result stays
    bit-exact."""
    torch = _cuda()
    import threading
    import paper_1407_1465_b200 as R
    jobs = [("rsa2048", 300), ("rsa1024", 500), ("rsa4096", 80), ("rsa64", 3000), ("rsa512", 700),
            ("rsa2048", 301), ("toy17947", 999), ("rsa3072", 90)]
    want, errors = {}, []
    for idx, (key, count) in enumerate(jobs):
        k = workload.key(key)
        m = workload.packets(count, k["nbits"], n=k["n"], config_id=40 + idx)
        want[idx] = (m, oracle.modexp_batch(m, k["d"], k["n"])[:, :m.shape[1]])
    start = threading.Barrier(len(jobs))

    def run(idx):
        try:
            key, _ = jobs[idx]
            k = workload.key(key)
            m, w = want[idx]
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                x = torch.from_numpy(m.view(np.int32)).cuda()
                start.wait()
                for _ in range(3):
                    y = R.rsa_modexp_batch(x, k["d"], k["n"], k["nbits"], stream=st)
                st.synchronize()
            if not np.array_equal(y.cpu().numpy().view(np.uint32), w):
                errors.append(idx)
        except Exception as ex:            # surfaced below
            errors.append((idx, repr(ex)))
    ths = [threading.Thread(target=run, args=(i,)) for i in range(len(jobs))]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert not errors, errors
