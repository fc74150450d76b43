#!/bin/bash
# A/B two builds of libparadiag.so on the c6 bench: tools/ab_lib.sh libA.so libB.so
for lib in "$@"; do
  cp "$lib" paper_2304_14021_b200/lib/libparadiag.so
  touch paper_2304_14021_b200/lib/libparadiag.so
  timeout 600 python bench.py --config c6 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
