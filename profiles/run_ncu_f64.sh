#!/bin/bash
# ncu evidence for the FP64-pipe kernel (gpurun, 1 GPU):
# 1) launch list of the default bench command (cold-cache, serialised: compare shares)
# 2) --set full capture of the decrypt kernel (one persistent wave) and of the encrypt kernel
OUT=${1:-gpurun_out}
mkdir -p $OUT
python paper_1407_1465_b200/build.py > /dev/null
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_f64.csv \
    python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > $OUT/bench_under_ncu_f64.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_f64 -s 1 -c 1 -o $OUT/prof_f64_dec -f \
    python bench.py --config rsa2048-dec --count 37888 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_f64 -s 1 -c 1 -o $OUT/prof_f64_enc -f \
    python bench.py --config rsa2048-enc --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la $OUT | grep -E "f64"
