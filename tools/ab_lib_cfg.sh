#!/bin/bash
# A/B builds of libparadiag.so on one config: tools/ab_lib_cfg.sh CONFIG libA.so libB.so ...
cfg=$1; shift
for lib in "$@"; do
  cp "$lib" paper_2304_14021_b200/lib/libparadiag.so
  touch paper_2304_14021_b200/lib/libparadiag.so
  echo "=== $cfg $lib"
  timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
