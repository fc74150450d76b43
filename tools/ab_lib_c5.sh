#!/bin/bash
# A/B two or more builds of libparadiag.so on the c5 bench: tools/ab_lib_c5.sh libA.so libB.so ...
for lib in "$@"; do
  cp "$lib" paper_2304_14021_b200/lib/libparadiag.so
  touch paper_2304_14021_b200/lib/libparadiag.so
  echo "=== $lib"
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],2)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.2f}\" for k,v in d['kernels'].items()))"
done
