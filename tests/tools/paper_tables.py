#!/usr/bin/env python3
"""Replay the paper's Table 1 / Table 2 shapes on B200 (SURVEY.md sec. 8(f)
row f2): the paper's own Fig 12 kernel (rsa_modexp_batch_paper, 64 threads
per block, O(e) loop), its other schedules as GPU kernels (Fig 4 naive, Fig 5a
right-to-left, Fig 5b left-to-right: rsa_modexp_batch_schedule) beside the
Montgomery path (rsa_modexp_batch), same
inputs (values 0..800), device time by CUDA events (median of
20 runs, the paper averaged 20).  Context only: the paper's
seconds were GT 630M wall clock including transfers.

    python tests/tools/paper_tables.py > profiles/r02_paper_tables.json
"""
import json
import os
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import oracle  # noqa: E402  (checker only)
import paper_1407_1465_b200 as R  # noqa: E402
import workload  # noqa: E402

SIZES = [256, 512, 1024, 2048, 4096, 8192, 16392, 32784, 1 << 20, 16 << 20]
TABLES = {"table1": (17947, 131, 15, "PAPER.md:431-441, n=131*137, e=131"),
          "table2": (513581, 131, 19, "PAPER.md:455-465, n=1009*509 (reading Z7), e=131 assumed")}


def timed(fn, reps=20):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    for a, b in ev:
        a.record()
        fn()
        b.record()
    torch.cuda.synchronize()
    return statistics.median(a.elapsed_time(b) for a, b in ev)


def main():
    out = {"device": torch.cuda.get_device_name(0), "rows": []}
    for name, (n, e, nbits, cite) in TABLES.items():
        for size in SIZES:
            pp = workload.paper_packets(size, config_id=size)
            t1 = torch.from_numpy(pp.ravel().view(np.int32)).cuda()
            t2 = torch.from_numpy(pp.view(np.int32)).cuda()
            o1 = torch.empty_like(t1)
            o2 = torch.empty_like(t2)
            ms_paper = timed(lambda: R.rsa_modexp_batch_paper(t1, e, n, out=o1))
            ms_mont = timed(lambda: R.rsa_modexp_batch(t2, e, n, nbits, out=o2))
            k = min(size, 4096)
            want = oracle.modexp_batch(pp[:k], e, n).ravel()
            ok = bool(np.array_equal(o1.cpu().numpy().view(np.uint32)[:k], want) and
                      np.array_equal(o2.cpu().numpy().view(np.uint32).ravel()[:k], want))
            row = {"table": name, "cite": cite, "size": size, "paper_fig12_ms": ms_paper,
                   "montgomery_ms": ms_mont, "paper_fig12_modexp_per_s": size / ms_paper * 1e3,
                   "montgomery_modexp_per_s": size / ms_mont * 1e3}
            for label, sched in (("naive_fig4", R.RSA_SCHED_NAIVE), ("r2l_fig5a", R.RSA_SCHED_R2L),
                                 ("l2r_fig5b", R.RSA_SCHED_L2R)):
                o3 = torch.empty_like(t1)
                row[label + "_ms"] = timed(lambda: R.rsa_modexp_batch_schedule(t1, e, n, sched, out=o3))
                row[label + "_modexp_per_s"] = size / row[label + "_ms"] * 1e3
                ok = ok and bool(np.array_equal(o3.cpu().numpy().view(np.uint32)[:k], want))
            row["oracle_checked"] = ok
            out["rows"].append(row)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
