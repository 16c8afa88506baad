#!/bin/bash
# A/B of compile-time kernel variants (run from the repo root).
#   build here:  tools/ab_variants.sh build NAME "-DMACRO=V ..." [NAME "-D..."]...
#   run on GPU:  tools/ab_variants.sh run CONFIG NAME [NAME...]   (bench.py --config CONFIG, one line each)
# Variant libraries: paper_1407_1465_b200/librsa_b200_<NAME>.so (git-ignored),
# loaded through RSA_B200_LIB; DESIGN.md / profiles/ record the outcomes.
set -e
cmd=$1; shift
if [ "$cmd" = build ]; then
  pids=()
  while [ $# -ge 2 ]; do
    name=$1; flags=$2; shift 2
    RSA_B200_NVCC_EXTRA="$flags" python paper_1407_1465_b200/build.py --out=paper_1407_1465_b200/librsa_b200_$name.so > /dev/null &
    pids+=($!)
  done
  for p in "${pids[@]}"; do wait $p; done
  ls -la paper_1407_1465_b200/librsa_b200_*.so
elif [ "$cmd" = run ]; then
  config=$1; shift
  mkdir -p gpurun_out
  for name in "$@"; do
    lib=paper_1407_1465_b200/librsa_b200_$name.so
    [ "$name" = default ] && lib=paper_1407_1465_b200/librsa_b200.so
    RSA_B200_LIB=$PWD/$lib timeout 900 python bench.py --config $config --steps ${AB_STEPS:-3} --warmup 3 \
        --no-cpu-baseline --no-e2e ${AB_EXTRA} > gpurun_out/ab_${config}_$name.json 2> gpurun_out/ab_${config}_$name.err || true
    python -c "
import json,sys
try:
    d=json.load(open('gpurun_out/ab_${config}_$name.json'))
    print('$config', '$name', round(d['value']), {k: round(v['modexp_per_s']) for k,v in d['legs'].items()}, 'frac', round(d['roofline']['frac'],3), 'mhz', d['clocks']['sm_mhz'])
except Exception as e: print('$config', '$name', 'FAILED', e, open('gpurun_out/ab_${config}_$name.err').read()[-500:])
"
  done
fi
