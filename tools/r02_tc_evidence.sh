#!/bin/bash
# Round-2 evidence for the tensor-core kernels (one GPU; run from the repo root under gpurun).
# Bench lines of the configs the TC kernels serve, the launch list of the default command and
# one ncu --set full capture of each TC kernel (decrypt, one persistent wave).
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/r02_bench_default_tc.json 2> $OUT/r02_bench_default_tc.err
for c in rsa2048-dec rsa2048-enc rsa2048-dec-crt rsa4096-dec-crt; do
  timeout 600 python bench.py --config $c --steps 5 --warmup 3 > $OUT/r02_bench_${c}_tc.json 2> /dev/null
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_launches_tc.csv \
    python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > $OUT/bench_under_ncu_tc.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_tc -s 1 -c 1 -o $OUT/prof_tc_2048 -f \
    python bench.py --config rsa2048-dec --count 37888 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:modexp_tc -s 2 -c 1 -o $OUT/prof_tc_1024 -f \
    python bench.py --config rsa2048-dec-crt --count 75776 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
for c in default rsa2048-dec rsa2048-enc rsa2048-dec-crt rsa4096-dec-crt; do
  python -c "
import json
d = json.loads(open('$OUT/r02_bench_${c}_tc.json').read().strip().splitlines()[-1])
print('$c', round(d['value']), round(d['e2e']['value']) if d.get('e2e') else None, round(d['roofline']['frac'], 3),
      d['roofline'].get('tensor', {}).get('frac'), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
