#!/bin/bash
# ncu --set full capture of the 4096-bit tensor-core kernel (one persistent wave: 148 x 128 packets),
# raw page exported for profiles/ and the per-source-line stall summary (tools/ncu_regions.py).
OUT=gpurun_out
mkdir -p $OUT
timeout 900 ncu --set full --clock-control none --import-source on -k regex:modexp_tc -c 1 -o $OUT/tc4096 \
    python bench.py --config rsa4096-dec --count 18944 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
    > $OUT/tc4096_ncu.log 2>&1
ncu -i $OUT/tc4096.ncu-rep --page raw --csv > $OUT/r02_ncu_raw_tc_4096_dec.csv 2>/dev/null
ncu -i $OUT/tc4096.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum 2>/dev/null | tail -2
