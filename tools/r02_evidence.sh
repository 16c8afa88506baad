#!/bin/bash
# Round-2 GPU evidence in one gpurun call (from the repo root): ncu launch list
# of the default bench command, compute-sanitizer logs, and a bench line per
# config.  Outputs land in gpurun_out/ (scratch); profiles/ keeps what is judged.
mkdir -p gpurun_out/sanitizer
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_default.csv \
    python bench.py --no-cpu-baseline --no-e2e --steps 2 --warmup 3 > gpurun_out/r02_bench_under_ncu.json 2>&1
for tool in memcheck racecheck initcheck synccheck; do
  SAN_COUNT=40 PYTORCH_NO_CUDA_MEMORY_CACHING=1 timeout 900 compute-sanitizer --tool $tool --error-exitcode 99 \
      --target-processes all python tests/tools/sanitize_run.py > gpurun_out/sanitizer/r02_$tool.log 2>&1
  echo "$tool rc=$? $(tail -1 gpurun_out/sanitizer/r02_$tool.log)"
done
for c in rsa2048-enc rsa2048-dec rsa4096-dec rsa4096-roundtrip rsa2048-dec-crt rsa4096-dec-crt u64-roundtrip \
         multikey2048-enc mr1024 toy-text-roundtrip toy-roundtrip; do
  timeout 900 python bench.py --config $c --cpu-seconds 5 > gpurun_out/r02_bench_$c.json 2> gpurun_out/r02_bench_$c.err
  python -c "import json; d=json.load(open('gpurun_out/r02_bench_$c.json')); print('$c', round(d['value']), d['roofline']['frac'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/r02_bench_$c.err
done
