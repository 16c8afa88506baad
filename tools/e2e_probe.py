#!/usr/bin/env python3
"""Where does the end-to-end (host buffers) time go?  Times each leg through
rsa_modexp_batch_host against the device-only call on the same data."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_1465_b200 as R  # noqa: E402
import workload  # noqa: E402

k = workload.key("rsa2048")
m = workload.packets(1 << 20, 2048, n=k["n"], config_id=2)
host_in = torch.from_numpy(m.view(np.int32)).pin_memory()
host_out = torch.empty_like(host_in).pin_memory()
dev_in = host_in.cuda()
dev_out = torch.empty_like(dev_in)
for label, e in (("enc", k["e"]), ("dec", k["d"])):
    R.rsa_modexp_batch_host(host_in, e, k["n"], 2048, out=host_out)
    t0 = time.perf_counter()
    R.rsa_modexp_batch_host(host_in, e, k["n"], 2048, out=host_out)
    th = time.perf_counter() - t0
    R.rsa_modexp_batch(dev_in, e, k["n"], 2048, out=dev_out)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    R.rsa_modexp_batch(dev_in, e, k["n"], 2048, out=dev_out)
    torch.cuda.synchronize()
    td = time.perf_counter() - t0
    t0 = time.perf_counter()
    x = host_in.cuda(non_blocking=True)
    torch.cuda.synchronize()
    h2d = time.perf_counter() - t0
    print(f"{label}: host-path {th*1e3:.1f} ms, device-only {td*1e3:.1f} ms, plain H2D 256 MiB {h2d*1e3:.1f} ms")
