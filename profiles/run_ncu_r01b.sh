#!/bin/bash
# Round-1 final ncu captures (gpurun, 1 GPU): one --set full launch per kernel family.
OUT=${1:-gpurun_out}
mkdir -p $OUT
python paper_1407_1465_b200/build.py >/dev/null
cap() {  # name config extra-args
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s 1 -c 1 -o $OUT/prof_$1 -f \
      python bench.py --config $2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline $4 > /dev/null 2>&1
}
cap enc rsa2048-enc modexp_kernel
cap dec4096 rsa4096-dec modexp_pair_kernel "--count 37888"
cap multikey multikey2048-enc modexp_multi_kernel
cap mr1024 mr1024 modexp_multi_kernel
cap u64 u64-roundtrip modexp_kernel
ls -la $OUT/prof_*.ncu-rep
