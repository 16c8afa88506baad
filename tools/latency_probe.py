#!/usr/bin/env python3
"""Call latency of small batches (the paper's toy workload: 9 packets, and
the Table 1 sizes) through rsa_modexp_batch, device time by CUDA events and
host wall time per call, vs the paper's Fig 12 kernel."""
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

k = workload.key("toy17947")
rows = []
for count in (9, 256, 4096, 32784):
    pk = workload.paper_packets(count)
    t = torch.from_numpy(pk.view(np.int32)).cuda()
    o = torch.empty_like(t)
    t1 = t.view(-1)
    o1 = torch.empty_like(t1)
    res = {}
    for label, fn in (("montgomery", lambda: R.rsa_modexp_batch(t, k["e"], k["n"], 15, out=o)),
                      ("paper_fig12", lambda: R.rsa_modexp_batch_paper(t1, k["e"], k["n"], out=o1))):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        dev, wall = [], []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            wall.append(time.perf_counter() - w0)
            dev.append(a.elapsed_time(b))
        res[label] = {"device_us": 1e3 * statistics.median(dev), "wall_us": 1e6 * statistics.median(wall)}
    rows.append({"packets": count, **res})
print(json.dumps({"key": "toy17947 (n=17947, e=131)", "rows": rows}, indent=1))
