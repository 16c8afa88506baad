#!/bin/bash
# Final round-2 evidence in one gpurun call (repo root): full GPU suite + smoke, the default
# bench line, one bench line per config, and the ncu launch list of the default command.
# (compute-sanitizer is closed on this GPU pool: its round-2 logs predate the TC kernels.)
OUT=gpurun_out
mkdir -p $OUT
timeout 1800 python -m pytest tests -m gpu -q > $OUT/r02_final_gpu_suite.log 2>&1; tail -2 $OUT/r02_final_gpu_suite.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/r02_final_smoke.log 2>&1; tail -1 $OUT/r02_final_smoke.log
timeout 900 python bench.py > $OUT/r02_final_bench_default.json 2> $OUT/r02_final_bench_default.err
for c in rsa2048-enc rsa2048-dec rsa4096-dec rsa4096-roundtrip rsa2048-dec-crt rsa4096-dec-crt u64-roundtrip \
         multikey2048-enc mr1024 toy-text-roundtrip toy-roundtrip; do
  timeout 900 python bench.py --config $c --cpu-seconds 5 > $OUT/r02_final_bench_$c.json 2> $OUT/r02_final_bench_$c.err
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/r02_final_launches_default.csv \
    python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > $OUT/r02_final_bench_under_ncu.json 2>&1
for c in default rsa2048-enc rsa2048-dec rsa4096-dec rsa4096-roundtrip rsa2048-dec-crt rsa4096-dec-crt u64-roundtrip \
         multikey2048-enc mr1024 toy-text-roundtrip toy-roundtrip; do
  python -c "
import json
d = json.loads(open('$OUT/r02_final_bench_$c.json').read().strip().splitlines()[-1])
e = d.get('e2e') or {}
print('$c', round(d['value']), round(e['value']) if e.get('value') else None, round(d['roofline']['frac'], 3),
      d['roofline']['kernel'][:34], d['clocks']['sm_mhz'], d['clocks']['reasons'])" || tail -2 $OUT/r02_final_bench_$c.err
done
