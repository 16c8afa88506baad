#!/usr/bin/env python3
"""Full-d decrypt throughput and % of the IMAD peak for every width class
(one seeded key per modulus size, workload/keys.json), through
rsa_modexp_batch with device-resident inputs; device time by CUDA events
on the launching stream.  Products per packet come from rsa_plan_info (the
kernel that actually runs the class).  No correctness check here -- the
parity tests cover every class; this only measures."""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1407_1465_b200 as R  # noqa: E402
import workload  # noqa: E402

PEAK = 32 * 148 * 1965e6        # products/s (profiles/r01_imad_peak.jsonl, MEASURED_PEAKS sm_max_mhz)
KEYS = ["rsa64", "rsa128", "rsa256", "rsa512", "rsa1024", "rsa2048", "rsa4096"]


def main():
    only = sys.argv[1:] or KEYS
    props = torch.cuda.get_device_properties(0)
    rows = []
    for name in only:
        k = workload.key(name)
        nb = k["nbits"]
        info = R.rsa_plan_info(k["d"], k["n"], nb)
        # about 0.3 s of work per launch at the expected rate, at least 4 waves of the grid
        per_pkt = info["products"] / (0.8 * PEAK)
        count = int(max(4 * info["grid"] * info["block"], min(1 << 24, 0.3 / per_pkt)))
        m = workload.packets(count, nb, n=k["n"], config_id=3)
        t = torch.from_numpy(m.view(np.int32)).cuda()
        o = torch.empty_like(t)
        s = torch.cuda.current_stream()
        for _ in range(2):
            R.rsa_modexp_batch(t, k["d"], k["n"], nb, out=o)
        torch.cuda.synchronize()
        ms = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            R.rsa_modexp_batch(t, k["d"], k["n"], nb, out=o)
            b.record(s)
            torch.cuda.synchronize()
            ms.append(a.elapsed_time(b))
        t_ms = statistics.median(ms)
        rate = count / (t_ms / 1e3)
        rows.append({"key": name, "nbits": nb, "S": info["width_class"], "window": info["window"],
                     "packets": count, "ms": round(t_ms, 3), "modexp_per_s": rate,
                     "products_per_packet": info["products"], "sqr_kernel": info["sqr_kernel"],
                     "grid": info["grid"], "block": info["block"],
                     "frac": info["products"] * rate / PEAK})
        print(json.dumps(rows[-1]), flush=True)
    print(json.dumps({"device": props.name, "sms": props.multi_processor_count, "peak_products_per_s": PEAK,
                      "rows": rows}))


if __name__ == "__main__":
    main()
