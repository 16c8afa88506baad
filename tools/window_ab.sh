#!/bin/bash
# A/B of the sliding-window width (bench.py --window; 0 = the plan's cost model) on a GPU box.
#   tools/window_ab.sh CONFIG [CONFIG...]
for cfg in "$@"; do
for w in 0 ${WINDOWS:-4 5 6 7}; do
  timeout 600 python bench.py --config $cfg --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --window $w \
      > gpurun_out/win_${cfg}_$w.json 2> gpurun_out/win_${cfg}_$w.err
  python -c "
import json
d=json.load(open('gpurun_out/win_${cfg}_$w.json'))
print('$cfg', 'w=$w', round(d['value']), {k: (round(v['modexp_per_s']), v['window']) for k, v in d['legs'].items()}, 'mhz', d['clocks']['sm_mhz'])
" || tail -3 gpurun_out/win_${cfg}_$w.err
done; done
