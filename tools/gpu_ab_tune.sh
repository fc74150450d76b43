#!/bin/bash
# A/B of PARADIAG_TUNE settings on one config's bench line: tools/gpu_ab_tune.sh CONFIG TUNE1 TUNE2 ...
cfg=$1; shift
for t in "$@"; do
  echo "=== tune $t"
  PARADIAG_TUNE=$t timeout 600 python bench.py --config $cfg --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
