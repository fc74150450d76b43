#!/bin/bash
# A/B environment settings on the c5 bench (per-kernel event times): tools/ab_env.sh "VAR=a" "VAR=b" ...
for rep in 1 2; do
for envs in "$@"; do
  env $envs timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline ${AB_ARGS} 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$envs', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
done
