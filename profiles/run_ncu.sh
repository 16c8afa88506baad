#!/bin/bash
# ncu evidence for the bench's kernels (run on the GPU box via gpurun, 1 GPU).
# 1) launch list of the exact bench command (cold-cache, serialised: compare shares)
# 2) --set full capture of the dominant kernel (decrypt) and of the encrypt kernel
set -x
OUT=${1:-gpurun_out}
mkdir -p $OUT
python paper_1407_1465_b200/build.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --no-cpu-baseline > $OUT/bench_under_ncu.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_kernel -s 1 -c 1 -o $OUT/prof_dec -f \
    python bench.py --config rsa2048-dec --count 75776 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_kernel -s 1 -c 1 -o $OUT/prof_enc -f \
    python bench.py --config rsa2048-enc --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT
