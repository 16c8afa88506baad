#!/usr/bin/env python3
"""Benchmark of the batched RSA hot path (arXiv 1407.1465) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl ours|reference]

Default workload (BASELINE.json metric "RSA-2048 modexps/sec (e=65537 and full
d)"): one step = encrypt a 1M-packet batch with e = 65537, then decrypt the
ciphertexts with the full private exponent d (configs[2] then configs[3]), all
packets resident in HBM.  value = modexps per second (2 x packets per step),
whole job.  Under torchrun (N > 1) the SAME batch is sharded (strong scaling,
SURVEY.md sec. 8(e)): rank r holds only its contiguous slice
(paper_1407_1465_b200.shard), runs the legs on it, and the step ends with the
all-gather of the result slices into the whole result on every rank (row a9);
time = max over ranks.

Prints ONE JSON line on rank 0.  See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workload  # noqa: E402

METRIC = "RSA-2048 modexps/sec (e=65537 and full d) at 1/2/4/8 B200; % of IMAD peak"
R_PRODUCTS_PER_CLK_PER_SM = 32      # measured: profiles/r01_imad_peak.jsonl (IMAD.WIDE half rate)
DFMA_PER_CLK_PER_SM = 64            # nominal FP64 pipe (ncu); fma.rn.f64 microbenchmark sustains 53.6
LANE_OPS_PER_CLK_PER_SM = 64        # 16-lane pipes (FP64, INT32 ALU, IMAD) share issue: 4 SMSPs x 16 lanes
                                    # per clock (profiles/r02_dfma_mix.jsonl: each such instruction costs
                                    # 2 SMSP cycles whichever of them it is; only FP32 co-issues)


def tc_macs_per_op(S: int) -> int:
    """u8 MACs per packet per Montgomery op on the tensor core (mont_tc.cuh, KB = 4S
    bytes): GEMM1 = N = 128 blocks b with 4b + 4 K-blocks of 32, GEMM2 = KB x KB."""
    kb = 4 * S
    return sum((4 * b + 4) * 32 * 128 for b in range(kb // 128)) + kb * kb   # 114688 at S = 64


def tc_words_per_op(S: int) -> int:
    """32-bit words assembled from the two GEMMs' byte columns per op (2 x S)."""
    return 2 * S


WORKLOADS = {
    # name: (key, count, legs)   legs: list of (label, exponent field, input)
    "rsa2048-roundtrip": ("rsa2048", 1 << 20, [("enc_e65537", "e"), ("dec_full_d", "d")]),
    "rsa2048-enc": ("rsa2048", 1 << 20, [("enc_e65537", "e")]),
    "rsa2048-dec": ("rsa2048", 1 << 20, [("dec_full_d", "d")]),
    "rsa4096-dec": ("rsa4096", 256 << 10, [("dec_full_d", "d")]),
    "rsa4096-roundtrip": ("rsa4096", 256 << 10, [("enc_e65537", "e"), ("dec_full_d", "d")]),
    "u64-roundtrip": ("rsa64", 16 << 20, [("enc_e65537", "e"), ("dec_full_d", "d")]),
    # every packet with its own (random odd, 2048-bit) modulus, e = 65537
    "multikey2048-enc": ("rsa2048", 1 << 20, [("multi_enc_e65537", "multi:65537")]),
    # f3: CRT decryption of 1M RSA-2048 ciphertexts (same result as full d)
    "rsa2048-dec-crt": ("rsa2048", 1 << 20, [("dec_crt", "crt:d")]),
    "rsa4096-dec-crt": ("rsa4096", 256 << 10, [("dec_crt", "crt:d")]),
    # f4: sec. 2 text -> packets -> C -> M -> text, fused, toy key, 16M letters
    "toy-text-roundtrip": ("toy17947", 8 << 20, [("enc_text_e131", "text:e"), ("dec_text_d14171", "text:d")]),
    # f1: one Miller-Rabin round (base 2) on 1M 1024-bit prime-search candidates
    "mr1024": ("rsa2048", 1 << 20, [("mr_base2_1024", "mr:1024")]),
    "toy-roundtrip": ("toy17947", 9, [("enc_e131", "e"), ("dec_d14171", "d")]),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="rsa2048-roundtrip", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--count", type=int, default=0, help="override packets per rank (profiling only)")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: test the multi-rank path on fewer GPUs)")
    ap.add_argument("--kernel-path", action="append", default=[], metavar="S=PATH",
                    help="A/B only: run width class S on another kernel (rsa_set_kernel_path), PATH one of "
                         "tc, fp64, int, int_group, int_pair, int_multi; e.g. --kernel-path 64=fp64")
    ap.add_argument("--window", type=int, default=0,
                    help="A/B only: force the sliding-window width (rsa_set_window; 0 = the plan's cost model)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="CPU-seconds budget of the oracle sample")
    return ap.parse_args()


# ------------------------------------------------------------------ clocks

class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.sw_power_cap",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "power.draw"]

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"rsa_bench_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "200"], stdout=self.f, stderr=subprocess.DEVNULL)
        except (OSError, FileNotFoundError):
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.f.close()
        sm, smax, reasons, power = [], [], set(), []
        names = ["sw_power_cap", "hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"]
        with open(self.path) as f:
            for line in f:
                parts = [p.strip() for p in line.split(",")]
                if len(parts) < len(self.FIELDS):
                    continue
                try:
                    sm.append(float(parts[0]))
                    smax.append(float(parts[1]))
                    power.append(float(parts[6]))
                except ValueError:
                    continue
                for nm, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
        os.unlink(self.path)
        note = None
        if not sm:
            # timed region shorter than nvidia-smi's start-up: one direct query
            try:
                q = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                                    "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=20)
                parts = [p.strip() for p in q.stdout.strip().split(",")]
                sm, smax, power = [float(parts[0])], [float(parts[1])], [float(parts[6])]
                for nm, v in zip(names, parts[2:6]):
                    if v.lower().startswith("active"):
                        reasons.add(nm)
                note = "single sample after the timed region (shorter than nvidia-smi start-up)"
            except (OSError, ValueError, IndexError, subprocess.TimeoutExpired):
                pass
        loaded = [c for c in sm if smax and c > 0.5 * max(smax)] or sm
        out = {"sm_mhz": statistics.median(loaded) if loaded else None,
               "sm_max_mhz": max(smax) if smax else None,
               "reasons": sorted(reasons), "samples": len(sm),
               "power_w_max": max(power) if power else None}
        if note:
            out["note"] = note
        return out


# ------------------------------------------------------------------ oracle baseline

def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def cpu_baseline(key: dict, base: np.ndarray, legs, cpu_seconds: float):
    """The oracle (oracle/, plain C, as it stands) on the host cores, on a
    bounded sample of the same workload, every leg (SURVEY.md sec. 8(d)
    "Oracle timing"): a fixed 4096-packet subsample (the first 4096 packets of
    the batch, edge packets included) for the expensive full-d legs, more
    packets for cheap legs (about cpu_seconds of single-core work); all cores
    (one thread each); plus the single-core rate on a smaller share; the CPU
    model is named (the paper names its CPU)."""
    import oracle
    cores = os.cpu_count() or 1
    # calibrate on 2 random (non-edge) packets of the most expensive leg
    t0 = time.perf_counter()
    oracle.modexp_batch(base[16:18], key[legs[-1][1]], key["n"], nthreads=1)
    per = max(time.perf_counter() - t0, 1e-6) / 2 * len(legs)
    k = min(len(base), 4096 if per > 1e-3 else max(4096, int(cpu_seconds / per)))
    t0 = time.perf_counter()
    cur = base[:k]
    for _, field in legs:
        cur = oracle.modexp_batch(cur, key[field], key["n"], nthreads=cores)
    wall = time.perf_counter() - t0
    k1 = min(k, max(16, k // (2 * cores)))
    t0 = time.perf_counter()
    cur = base[:k1]
    for _, field in legs:
        cur = oracle.modexp_batch(cur, key[field], key["n"], nthreads=1)
    wall1 = time.perf_counter() - t0
    return {"value": k * len(legs) / wall, "unit": "modexp/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(),
            "single_core": {"value": k1 * len(legs) / wall1, "unit": "modexp/s",
                            "sample": f"first {k1} packets, {len(legs)} leg(s), 1 thread, {wall1:.1f} s"},
            "sample": f"first {k} packets of the batch, {len(legs)} leg(s) each "
                      f"({', '.join(l for l, _ in legs)}); {wall:.1f} s wall on {cores} threads"}


def measured_chain_rate():
    """Best products/clk/SM of the IMAD.WIDE.U32.X chain form in the committed
    microbenchmark (profiles/r01_imad_peak.jsonl), or None."""
    best = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_imad_peak.jsonl")) as f:
            for line in f:
                if line.startswith("{"):
                    rec = json.loads(line)
                    if "IMAD.WIDE.U32.X" in rec.get("form", ""):
                        v = rec.get("products_per_clk_per_sm")
                        best = v if best is None or v > best else best
    except (OSError, ValueError):
        return None
    return best


def measured_dfma_rate():
    """Best fma.rn.f64 results/clk/SM in the committed microbenchmark
    (profiles/r01_imad_peak.jsonl), or None."""
    best = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_imad_peak.jsonl")) as f:
            for line in f:
                if line.startswith("{"):
                    rec = json.loads(line)
                    v = rec.get("dfma_per_clk_per_sm")
                    if v is not None:
                        best = v if best is None or v > best else best
    except (OSError, ValueError):
        return None
    return best


def measured_digit_mix_rate():
    """Best FP64 ops/clk/SM of the kernel's digit-product instruction mix
    (DFMA.RZ, DADD, DFMA.RZ + the 64-bit column add: the rows with mix
    'dfma+dadd+dfma+iadd3x2' only, not the add-free or IMAD.X variants) in
    profiles/r01_dfma_latency.jsonl, or None."""
    best = None
    try:
        with open(os.path.join(ROOT, "profiles", "r01_dfma_latency.jsonl")) as f:
            for line in f:
                if line.startswith("{"):
                    rec = json.loads(line)
                    if rec.get("mix") != "dfma+dadd+dfma+iadd3x2":
                        continue
                    v = rec.get("fp64_ops_per_clk_per_sm")
                    if v is not None:
                        best = v if best is None or v > best else best
    except (OSError, ValueError):
        return None
    return best


def measured_i8_tops():
    """Best int8 tcgen05.mma rate (T int8-op/s, whole GPU) measured by
    csrc/microbench/tc_i8_peak.cu (profiles/r02_tc_i8_peak.jsonl), or None."""
    best = None
    try:
        with open(os.path.join(ROOT, "profiles", "r02_tc_i8_peak.jsonl")) as f:
            for line in f:
                if line.startswith("{"):
                    v = json.loads(line).get("int8_tops")
                    best = v if best is None or (v and v > best) else best
    except (OSError, ValueError):
        return None
    return best


def batch_kernel_name(R, S: int) -> str:
    """The kernel modexp.cu launches for width class S (its resolved path)."""
    path = R.rsa_get_kernel_path(S)
    if path == R.RSA_PATH_FP64:
        return f"modexp_f64_kernel<{S}>"
    if path == R.RSA_PATH_TC:
        return "modexp_tc_kernel"
    if path == R.RSA_PATH_INT_MULTI:
        return f"modexp_small_kernel<{S}>"
    if path == R.RSA_PATH_INT_GROUP:
        return f"modexp_group_kernel<{S}, {2 if S == 64 else 4}>"
    if path == R.RSA_PATH_INT_PAIR:
        return f"modexp_pair_kernel<{S}>"
    return f"modexp_kernel<{S}>"


def ncu_traffic(key_name: str, leg: str, count: int, kernel_tag: str = ""):
    """DRAM bytes (read + write) per launch of the dominant kernel, from the
    committed ncu --set full capture (profiles/ncu_traffic.json, bytes per
    packet; entry `leg + kernel_tag` when the kernel has its own capture)
    scaled to this launch's packets; None if not captured."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            recs = json.load(f).get(key_name, {})
            rec = recs.get(leg + kernel_tag)     # a kernel without its own capture: None
    except (OSError, ValueError):
        return None
    return None if not rec else rec["bytes_per_packet"] * count


# ------------------------------------------------------------------ arms

def run_reference(args, rank, world):
    """--impl reference: the oracle as it stands, on host cores, rank 0 only."""
    if rank != 0:
        return
    key_name, count, legs = WORKLOADS[args.config]
    key = workload.key(key_name)
    nb = key["nbits"]
    base = workload.packets(count, nb, n=key["n"], config_id=2)
    import oracle
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    oracle.modexp_batch(base[16:18], key[legs[-1][1]], key["n"], nthreads=1)
    per = max(time.perf_counter() - t0, 1e-6) / 2 * len(legs)
    budget = 120.0 / max(1, args.steps + args.warmup)          # whole run within a few minutes
    k = int(min(count, max(cores, budget * cores / per)))
    times = []
    for it in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cur = base[:k]
        for _, field in legs:
            cur = oracle.modexp_batch(cur, key[field], key["n"], nthreads=cores)
        if it >= args.warmup:
            times.append(time.perf_counter() - t0)
    ms = 1e3 * statistics.mean(times)
    value = k * len(legs) / (ms / 1e3)
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": "modexp/s", "n_gpus": 1,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": args.config, "packets_per_step": k, "key": key_name,
                       "note": "oracle (plain C bignum, Fig 5 L2R) on host cores; bounded sample per step"},
            "cpu_baseline": {"value": value, "unit": "modexp/s", "cores": cores, "kind": "oracle",
                             "cpu_model": cpu_model(),
                             "sample": f"first {k} packets of the batch x {len(legs)} legs per step"},
            "e2e": {"value": value, "unit": "modexp/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1407_1465_b200 as R
    from paper_1407_1465_b200.shard import gather_slices, modexp_sharded_host, shard_bounds

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    for kp in args.kernel_path:
        cls, path = kp.split("=")
        R.rsa_set_kernel_path(int(cls), getattr(R, "RSA_PATH_" + path.upper()))
    if args.window:
        R.rsa_set_window(args.window)
    key_name, total, legs = WORKLOADS[args.config]
    if args.count:
        total = args.count
    key = workload.key(key_name)
    nb, n = key["nbits"], key["n"]
    s = workload.limbs_needed(nb)
    # strong scaling: ONE batch of `total` packets (the same on every rank), rank
    # r holds only rows [lo, hi) on its device
    bounds, per = shard_bounds(total, world)
    lo, hi = bounds[rank]
    count = hi - lo
    kind = legs[0][1].split(":")[0] if ":" in legs[0][1] else "batch"
    stream = torch.cuda.current_stream(dev)
    base_np = None
    if kind == "text":
        rng = np.random.default_rng(workload.MASTER_SEED)
        text_np = (rng.integers(0, 26, 2 * total) + ord("a")).astype(np.uint8)
        letters = torch.from_numpy(text_np[2 * lo:2 * hi].copy()).to(dev)
        base = letters
    elif kind == "mr":
        nb = int(legs[0][1].split(":")[1])
        s = workload.limbs_needed(nb)
        # counter-based generator: this rank's candidates are indices [lo, hi)
        base = R.rsa_prime_candidates(nb, workload.MASTER_SEED, lo, count, device=dev)
    else:
        full_np = workload.packets(total, nb, n=n, config_id=2)
        base_np = full_np[lo:hi]
        base = torch.from_numpy(np.ascontiguousarray(base_np).view(np.int32)).to(dev)
    # the result rows go straight into this rank's chunk of the gather buffer
    # (shard.py layout): rows [rank*per, rank*per + count) of [per*world, s]
    gathered = kind in ("batch", "crt", "multi")
    full = torch.empty((per * world if world > 1 else count, s), dtype=torch.int32, device=dev) if gathered else None
    mine = full[rank * per:rank * per + count] if (gathered and world > 1) else full
    bufs = [base] + [torch.empty_like(base) for _ in legs[:-1]] + [mine if gathered else torch.empty_like(base)]
    if kind == "text":
        bufs = [letters, torch.empty((count, s), dtype=torch.int32, device=dev), torch.empty_like(letters)]
        exps = [key["e"], key["d"]]
        plans = [R.rsa_plan_info(e, n, nb) for e in exps]
    elif kind == "batch":
        exps = [key[f] for _, f in legs]
        plans = [R.rsa_plan_info(e, n, nb) for e in exps]
    elif kind == "multi":
        ev = int(legs[0][1].split(":")[1])
        rng = np.random.Generator(np.random.PCG64(workload.MASTER_SEED + 500))
        mods_np = rng.integers(0, 2**32, (total, s), dtype=np.uint64).astype(np.uint32)[lo:hi]
        mods_np[:, 0] |= 1
        mods_np[:, s - 1] |= np.uint32(1 << 31)
        mods = torch.from_numpy(np.ascontiguousarray(mods_np).view(np.int32)).to(dev)
        expt = torch.from_numpy(workload.ints_to_rows([ev] * 1, s).view(np.int32)).to(dev).expand(count, s).contiguous()
        exps = [ev]
        pm = R.rsa_multi_plan_info(nb, ev.bit_length())
        # the kernel skips a window's multiply when every digit in the CTA is 0
        # (modexp_multi.cu RSA_MULTI_SKIP0); this batch has one exponent, so the
        # executed multiplies are the nonzero digits below the top window
        w_, nwin_ = pm["window"], (ev.bit_length() + pm["window"] - 1) // pm["window"]
        zero_ = sum(1 for wi in range(nwin_ - 1) if (ev >> (wi * w_)) & ((1 << w_) - 1) == 0)
        S_ = pm["width_class"]
        plans = [dict(pm, montmuls=pm["montmuls"] - zero_, products=pm["products"] - zero_ * (2 * S_ * S_ + S_),
                      skipped_zero_windows=zero_)]
    elif kind == "crt":
        exps = [key["d"]]
        p_, q_ = max(key["p"], key["q"]), min(key["p"], key["q"])
        hb = 32 * workload.limbs_needed(p_.bit_length())
        hp = R.rsa_plan_info(key["d"] % (p_ - 1), p_, hb)
        hq = R.rsa_plan_info(key["d"] % (q_ - 1), q_, hb)
        plans = [dict(hp, montmuls=hp["montmuls"] + hq["montmuls"], squarings=hp["squarings"] + hq["squarings"],
                      products=hp["products"] + hq["products"], window=hp["window"], exp_bits=hp["exp_bits"],
                      digit_products=hp["digit_products"] + hq["digit_products"])]
    else:
        exps = [0]
        plans = [R.rsa_multi_plan_info(nb, 0, mr=True)]
        mr_out = torch.empty(count, dtype=torch.int32, device=dev)

    def step(evs=None, gev=None):
        for j, e in enumerate(exps):
            if evs is not None:
                evs[j][0].record(stream)
            if count == 0:
                pass
            elif kind == "batch":
                R.rsa_modexp_batch(bufs[j], e, n, nb, out=bufs[j + 1], stream=stream)
            elif kind == "multi":
                R.rsa_modexp_batch_multi(bufs[j], expt, mods, nb, exp_bits=e.bit_length(), out=bufs[j + 1],
                                         stream=stream)
            elif kind == "text" and j == 0:
                R.rsa_encrypt_text(bufs[0], e, n, nb, out=bufs[1], stream=stream)
            elif kind == "text":
                R.rsa_decrypt_text(bufs[1], e, n, nb, out=bufs[2], stream=stream)
            elif kind == "crt":
                R.rsa_decrypt_crt_batch(bufs[j], key["p"], key["q"], key["d"], nb, out=bufs[j + 1], stream=stream)
            else:
                R.rsa_miller_rabin_batch(bufs[j], nb, 2, out=mr_out, stream=stream)
            if evs is not None:
                evs[j][1].record(stream)
        if gathered and world > 1:
            # step a9: reassemble the whole result on every rank (in-place all-gather)
            gather_slices(full, per)
            if gev is not None:
                gev.record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # correctness of the last warm-up round trip: the whole reassembled batch
    # equals the input batch (compared on the host: each rank holds only its
    # input slice on the device)
    verified = None
    if len(legs) == 2 and kind == "batch":
        verified = bool(np.array_equal(full[:total].cpu().numpy().view(np.uint32), full_np))
    elif len(legs) == 2:
        verified = bool(torch.equal(bufs[-1], bufs[0]))

    clocks = ClockSampler(local_rank if "CUDA_VISIBLE_DEVICES" not in os.environ else 0)
    if rank == 0:
        clocks.start()
        time.sleep(0.3)
    leg_events = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)] for _ in legs]
                  for _ in range(args.steps)]
    gather_events = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = R.rsa_kernel_launches()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    t_start.record(stream)
    for k in range(args.steps):
        step(leg_events[k], gather_events[k])
    t_end.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    launches = R.rsa_kernel_launches() - launches0
    clk = clocks.stop() if rank == 0 else None
    elapsed_ms = t_start.elapsed_time(t_end)
    leg_ms = [statistics.mean(leg_events[k][j][0].elapsed_time(leg_events[k][j][1]) for k in range(args.steps))
              for j in range(len(legs))]
    gather_ms = (statistics.mean(leg_events[k][-1][1].elapsed_time(gather_events[k]) for k in range(args.steps))
                 if gathered and world > 1 else 0.0)
    if world > 1:
        on_dev = dist.get_backend() == "nccl"
        t = torch.tensor([elapsed_ms, gather_ms] + leg_ms, device=dev if on_dev else "cpu", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms, gather_ms, leg_ms = float(t[0]), float(t[1]), [float(v) for v in t[2:]]
        lt = torch.tensor([launches], device=dev if on_dev else "cpu", dtype=torch.int64)
        dist.all_reduce(lt, op=dist.ReduceOp.SUM)
        launches = int(lt[0])

    # ---- end to end through the public API (pinned host buffers): every rank
    # copies its slice host -> device, runs the legs, the slices are
    # all-gathered, rank 0 copies the whole result device -> host
    e2e = None
    if not args.no_e2e and kind == "batch":
        host_in = torch.from_numpy(np.ascontiguousarray(base_np).view(np.int32)).pin_memory()
        host_out = torch.empty((total, s), dtype=torch.int32).pin_memory() if rank == 0 else None
        modexp_sharded_host(host_in, exps[:1], n, nb, total, out=host_out)      # warm
        ts = []
        for _ in range(max(1, min(args.steps, 3))):
            if world > 1:
                dist.barrier()
            t0 = time.perf_counter()
            modexp_sharded_host(host_in, exps, n, nb, total, out=host_out)
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                tt = torch.tensor([dt], dtype=torch.float64,
                                  device=dev if dist.get_backend() == "nccl" else "cpu")
                dist.all_reduce(tt, op=dist.ReduceOp.MAX)
                dt = float(tt[0])
            ts.append(dt)
        e2e_s = statistics.median(ts)
        row = s * 4
        if world == 1:
            nh2d = nd2h = total * row * len(legs)
            path = "rsa_modexp_batch_host per leg: pinned host -> device -> kernel -> host, chunk-pipelined"
        else:
            nh2d, nd2h = total * row, total * row
            path = ("shard.modexp_sharded_host: each rank pinned slice -> its device, legs, NCCL all-gather of the "
                    "result slices, rank 0 whole result -> pinned host")
        e2e = {"value": total * len(legs) / e2e_s, "unit": "modexp/s", "h2d_bytes_per_step": nh2d,
               "d2h_bytes_per_step": nd2h, "ms_per_step": 1e3 * e2e_s, "path": path}
        if len(legs) == 2 and rank == 0:
            e2e["verified"] = bool(np.array_equal(host_out.numpy().view(np.uint32), full_np))

    if rank != 0:
        return
    ms_per_step = elapsed_ms / args.steps
    value = total * len(legs) / (ms_per_step / 1e3)
    # ---- roofline of the dominant kernel
    props = torch.cuda.get_device_properties(dev)
    sms = props.multi_processor_count
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except (OSError, ValueError):
        pass
    f_max = float(peaks.get("sm_max_mhz", 1965.0))
    dom = max(range(len(legs)), key=lambda j: leg_ms[j])
    S = plans[dom]["width_class"]
    products = count * plans[dom]["products"]
    achieved = products / (leg_ms[dom] / 1e3) / 1e12
    peak = R_PRODUCTS_PER_CLK_PER_SM * sms * f_max * 1e6 / 1e12
    fp64 = kind in ("batch", "crt") and plans[dom].get("fp64_digits", 0) > 0 and \
        batch_kernel_name(R, S) != "modexp_tc_kernel"
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tprod/s", "frac": achieved / peak,
                "traffic": ncu_traffic(key_name, legs[dom][0], count,
                                       "_tc" if kind in ("batch", "crt") and batch_kernel_name(R, S) == "modexp_tc_kernel"
                                       else ""),
                "traffic_unit": "bytes per launch", "algorithmic_bytes": count * s * 4 * 2,
                "kernel": ({"multi": f"modexp_multi_kernel<{S}>", "mr": f"modexp_multi_kernel<{S}> (MR mode)",
                            "crt": f"2 x {batch_kernel_name(R, S)} + crt_split/combine (half-width CRT legs; "
                                   f"products of both)"}.get(
                    kind, batch_kernel_name(R, S))) + f" ({legs[dom][0]})",
                "algorithmic": f"{plans[dom]['products']} 32x32->64 limb products/packet "
                               f"({plans[dom]['squarings']} squarings x "
                               f"{'1.5S^2+1.5S' if plans[dom]['sqr_kernel'] else '2S^2+S'} + "
                               f"{plans[dom]['montmuls'] - plans[dom]['squarings']} other montmuls x 2S^2+S, S={S})"
                               f" x {count} packets per launch",
                "peak_basis": f"{R_PRODUCTS_PER_CLK_PER_SM} products/clk/SM (IMAD.WIDE half rate, "
                              f"profiles/r01_imad_peak.jsonl) x {sms} SMs x {f_max:.0f} MHz "
                              f"(MEASURED_PEAKS sm_max_mhz)",
                "peak_source": "nominal: MEASURED_PEAKS.json has no INT32 entry; frac is 'of nominal'"}
    if fp64:
        # The dominant kernel runs on the FP64 pipe (mont_f64.cuh): its own
        # roofline is FP64 ops against the measured DFMA issue rate.  The
        # metric's "% of IMAD peak" (the same limb-product count against the
        # integer pipe's peak) is kept beside it: above 1 means the path beats
        # the integer-pipe ceiling.
        nd = plans[dom]["fp64_digits"]
        dfma = measured_dfma_rate()
        ops = 3 * count * plans[dom]["digit_products"]
        f_ach = ops / (leg_ms[dom] / 1e3) / 1e12
        f_peak = DFMA_PER_CLK_PER_SM * sms * f_max * 1e6 / 1e12
        roofline.update({
            "achieved": f_ach, "peak": f_peak, "unit": "T fp64-op/s", "frac": f_ach / f_peak,
            "algorithmic": f"{plans[dom]['digit_products']} 52x52-bit digit products/packet x 3 FP64 ops "
                           f"(DFMA.RZ hi, DADD, DFMA.RZ lo; {plans[dom]['squarings']} squarings x ND(ND+1)/2+ND^2 + "
                           f"{plans[dom]['montmuls'] - plans[dom]['squarings']} other montmuls x 2ND^2, ND={nd}) "
                           f"x {count} packets per launch",
            "peak_basis": f"{DFMA_PER_CLK_PER_SM} FP64 ops/clk/SM (16 FP64 lanes per SM sub-partition: the "
                          f"peak of ncu's sm__inst_executed_pipe_fp64) x {sms} SMs x {f_max:.0f} MHz "
                          f"(MEASURED_PEAKS sm_max_mhz)",
            "peak_source": "nominal: MEASURED_PEAKS.json has no FP64 entry (hbm_gbs and bf16 only); frac is "
                           "'of nominal'. peak_measured_* below are this repo's microbenchmarks",
            **({"peak_measured_dfma": dfma * sms * f_max * 1e6 / 1e12,
                "frac_of_measured_dfma": f_ach / (dfma * sms * f_max * 1e6 / 1e12)} if dfma else {}),
            **({"peak_measured_digit_mix": mix * sms * f_max * 1e6 / 1e12,
                "frac_of_measured_digit_mix": f_ach / (mix * sms * f_max * 1e6 / 1e12)}
               if (mix := measured_digit_mix_rate()) else {}),
            "imad_equiv": {"achieved": achieved, "peak": peak, "unit": "Tprod/s", "frac": achieved / peak,
                           "peak_source": "nominal (half-rate IMAD.WIDE, profiles/r01_imad_peak.jsonl)",
                           "basis": "the path's 32x32->64 limb-product count (the metric's '% of IMAD peak') "
                                    "against 32 products/clk/SM on the integer pipe"}})
    tc = kind in ("batch", "crt") and batch_kernel_name(R, S) == "modexp_tc_kernel"
    if tc:
        # Tensor-core reduction kernel (modexp_tc.cu): the CUDA cores' 16-lane
        # issue (FP64 + INT32 share it) is the bound.  Algorithmic lane-ops per
        # packet: 5 per 52x52 digit product of T = A B (3 FP64 for the exact
        # split + the 64-bit column add, the representation's floor:
        # r02_dfma_mix) and 4 per word assembled from the GEMMs' byte columns
        # (3 IMAD.WIDE + 1 add-with-carry).  The tensor core's own share is
        # reported beside it against the int8 peak.
        pd = plans[dom]
        lane_ops = 5 * pd["digit_products"] + 4 * tc_words_per_op(S) * pd["montmuls"]
        l_ach = count * lane_ops / (leg_ms[dom] / 1e3) / 1e12
        l_peak = LANE_OPS_PER_CLK_PER_SM * sms * f_max * 1e6 / 1e12
        i8_meas = measured_i8_tops()
        i8_peak = i8_meas or 2 * float(peaks.get("bf16_tflops_sustained", 1378.2))   # int8 = 2 x bf16
        i8_ach = count * 2 * tc_macs_per_op(S) * pd["montmuls"] / (leg_ms[dom] / 1e3) / 1e12
        roofline.update({
            "bound": "alu", "achieved": l_ach, "peak": l_peak, "unit": "T lane-op/s", "frac": l_ach / l_peak,
            "algorithmic": f"{lane_ops} CUDA-core lane-ops/packet: {pd['digit_products']} 52x52 digit products "
                           f"x 5 (T = A B; {pd['squarings']} squarings x ND(ND+1)/2 + "
                           f"{pd['montmuls'] - pd['squarings']} multiplies x ND^2, ND={pd['fp64_digits']}) + "
                           f"{pd['montmuls']} ops x {tc_words_per_op(S)} GEMM output words x 4, x {count} packets"
                           + (" (both CRT halves)" if kind == "crt" else ""),
            "peak_basis": f"{LANE_OPS_PER_CLK_PER_SM} lane-ops/clk/SM (4 SMSPs x 16 lanes of the FP64 / INT32 "
                          f"pipes, one shared issue) x {sms} SMs x {f_max:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "peak_source": "nominal: MEASURED_PEAKS.json has no FP64/INT32 entry; frac is 'of nominal'",
            "tensor": {"achieved": i8_ach, "peak": i8_peak, "unit": "T int8-op/s", "frac": i8_ach / i8_peak,
                       "algorithmic": f"{tc_macs_per_op(S)} u8 MACs x 2 per packet per Montgomery op "
                                      f"(m = T n' mod R, columns of m n) x {pd['montmuls']} ops",
                       "peak_source": ("measured: best u8 tcgen05.mma rate of profiles/r02_tc_i8_peak.jsonl "
                                       "(csrc/microbench/tc_i8_peak.cu, back-to-back M=128 N=256 K=32)")
                                      if i8_meas else
                                      "2 x MEASURED_PEAKS bf16_tflops_sustained (guide: int8/fp8 = 2 x bf16 dense)"},
            "imad_equiv": {"achieved": achieved, "peak": peak, "unit": "Tprod/s", "frac": achieved / peak,
                           "peak_source": "nominal (half-rate IMAD.WIDE, profiles/r01_imad_peak.jsonl)",
                           "basis": "the metric's '% of IMAD peak': the textbook 32x32->64 limb-product count "
                                    "of the same Montgomery ops against 32 products/clk/SM on the integer pipe"}})
    if kind == "batch":
        # the window table is algorithmic state too: every entry written once,
        # read by each window multiply (+ the A loads); per resident thread it is
        # ntab x S limbs, larger than L2 at S = 64 / w = 7, so it streams to DRAM
        pd = plans[dom]
        touches = pd["table_entries"] + (pd["montmuls"] - pd["squarings"] - 2) + 2
        entry = 8 * pd["fp64_digits"] if (fp64 or tc) else S * 4   # 52-bit digits as doubles, or limbs
        roofline["algorithmic_table_bytes"] = count * entry * touches
        roofline["traffic_note"] = ("DRAM traffic = packet I/O + the per-thread sliding-window table "
                                    f"({pd['table_entries']} entries x {entry} B, {touches} entry reads/writes per "
                                    "packet); compare traffic with algorithmic_bytes + algorithmic_table_bytes")
    chain = measured_chain_rate()
    if chain and not fp64:
        # context, not the contract's peak: the best rate the IMAD microbenchmark
        # sustained for dependent IMAD.WIDE.U32.X chains (any occupancy)
        roofline["peak_measured_chain"] = chain * sms * f_max * 1e6 / 1e12
        roofline["frac_of_measured_chain"] = achieved / roofline["peak_measured_chain"]
    if clk and clk.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = roofline["frac"] * f_max / clk["sm_mhz"]
    legs_out = {}
    for j, (label, field) in enumerate(legs):
        legs_out[label] = {"ms": leg_ms[j], "modexp_per_s": total / (leg_ms[j] / 1e3),
                           "montmuls_per_packet": plans[j]["montmuls"], "squarings_per_packet": plans[j]["squarings"],
                           "products_per_packet": plans[j]["products"], "window": plans[j]["window"],
                           "exp_bits": plans[j]["exp_bits"]}
    cpu = None
    if not args.no_cpu_baseline and world == 1 and kind == "batch":
        cpu = cpu_baseline(key, base_np, legs, args.cpu_seconds)
    line = {"metric": METRIC, "value": value, "unit": "modexp/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64+u8" if tc else ("f64" if fp64 else "u32"), "data": "synthetic",
            "config": {"workload": args.config, "packets_total": total, "packets_per_rank": per,
                       **({"kernel_path": args.kernel_path} if args.kernel_path else {}),
                       **({"window_forced": args.window} if args.window else {}),
                       "key": key_name + " (seeded, "
                       "workload/keys.json)", "legs": [l for l, _ in legs], "modulus_bits": nb,
                       "l2": f"inputs {count * s * 4 / 2**20:.0f} MiB per leg vs 126 MB L2"
                             + (" (larger than L2)" if count * s * 4 > 126e6 else " (fits L2)"),
                       "parallelism": (f"dp{world}: contiguous slices of one {total}-packet batch, one per rank; "
                                       f"the step ends with the all-gather of the result slices (row a9)"
                                       if world > 1 else "dp1 (one GPU, the whole batch)")},
            "legs": legs_out, **({"gather_ms": gather_ms} if world > 1 and gathered else {}), "verified_roundtrip": verified, "roofline": roofline, "cpu_baseline": cpu,
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            torch.cuda.set_device(local_rank)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            # ranks share the visible devices round-robin (testing the N > 1 path)
            local_rank = local_rank % max(1, torch.cuda.device_count())
            torch.cuda.set_device(local_rank)
            dist.init_process_group("gloo")
    try:
        run_ours(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
