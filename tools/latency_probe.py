#!/usr/bin/env python3
"""Call latency of small batches (the paper's toy workload: 9 packets, and
the Table 1 sizes) through rsa_modexp_batch, vs the paper's Fig 12 kernel.

Per call, medians over 50 calls:
  wall_us     host wall time of one Python-level call + synchronize
  capi_us     host wall time of the bare C-ABI call (ctypes, arguments prebuilt)
  device_us   CUDA events around one call (includes host gaps if the GPU idles)
  queued_us   CUDA events around one call enqueued behind a GPU spin, so the host
              is ahead of the GPU: pure device time of what the call launches
"""
import ctypes
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_1465_b200 as R  # noqa: E402
import workload  # noqa: E402


def med(xs):
    return statistics.median(xs)


def probe(fn, capi=None, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()
    wall, dev, queued, capi_t = [], [], [], []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        wall.append(time.perf_counter() - w0)
        dev.append(a.elapsed_time(b))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(2_000_000)          # ~1 ms of GPU spin: the host gets ahead
        a.record(s)
        fn()
        b.record(s)
        torch.cuda.synchronize()
        queued.append(a.elapsed_time(b))
        if capi is not None:
            torch.cuda._sleep(2_000_000)
            c0 = time.perf_counter()
            capi()
            capi_t.append(time.perf_counter() - c0)
            torch.cuda.synchronize()
    out = {"wall_us": 1e6 * med(wall), "device_us": 1e3 * med(dev), "queued_us": 1e3 * med(queued)}
    if capi_t:
        out["capi_us"] = 1e6 * med(capi_t)
    return out


def main():
    k = workload.key("toy17947")
    lib = R._lib
    rows = []
    for count in (9, 256, 4096, 32784):
        pk = workload.paper_packets(count)
        t = torch.from_numpy(pk.view(np.int32)).cuda()
        o = torch.empty_like(t)
        t1 = t.view(-1)
        o1 = torch.empty_like(t1)
        E, N = R.limbs(k["e"], 1), R.limbs(k["n"], 1)
        stream = torch.cuda.current_stream().cuda_stream
        args = (ctypes.c_void_p(t.data_ptr()), R._p(E), R._p(N), 15, count, ctypes.c_void_p(o.data_ptr()),
                ctypes.c_void_p(stream))
        res = {
            "montgomery": probe(lambda: R.rsa_modexp_batch(t, k["e"], k["n"], 15, out=o),
                                capi=lambda: lib.rsa_modexp_batch(*args)),
            "paper_fig12": probe(lambda: R.rsa_modexp_batch_paper(t1, k["e"], k["n"], out=o1)),
        }
        rows.append({"packets": count, **res})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"key": "toy17947 (n=17947, e=131)", "rows": rows}, indent=1))


if __name__ == "__main__":
    main()
