#!/bin/bash
# A/B builds of libparadiag.so on the c5 bench (per-kernel event times): tools/ab_c5.sh libA.so libB.so ...
cp paper_2304_14021_b200/lib/libparadiag.so /tmp/lib_orig.so
for rep in 1 2; do
for lib in "$@"; do
  cp "$lib" paper_2304_14021_b200/lib/libparadiag.so
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$lib', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
done
cp /tmp/lib_orig.so paper_2304_14021_b200/lib/libparadiag.so
