#!/bin/bash
# One-call GPU validation (run via gpurun from the repo root):
#   smoke, the full GPU test suite, the default bench line, RSA-4096 lines.
# Outputs land in gpurun_out/ (scratch); copy what is judged into profiles/.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE OK')" > gpurun_out/final_smoke.log 2>&1; tail -1 gpurun_out/final_smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final_gpu_tests.log 2>&1; tail -2 gpurun_out/final_gpu_tests.log
timeout 600 python bench.py > gpurun_out/final_bench_default.json 2> gpurun_out/final_bench_default.err
python -c "import json; d=json.load(open('gpurun_out/final_bench_default.json')); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline'].get('imad_equiv',{}).get('frac'), d['clocks'])"
for c in rsa4096-dec rsa4096-dec-crt; do
  timeout 600 python bench.py --config $c --cpu-seconds 5 > gpurun_out/fb_$c.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/fb_$c.json')); print('$c', d['value'], d['roofline']['frac'], d['roofline'].get('imad_equiv',{}).get('frac'))"
done
