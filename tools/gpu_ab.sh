#!/bin/bash
# A/B bench runs: each argument is an env assignment list, e.g. "PARADIAG_TUNE=1" "PARADIAG_TUNE=2"
mkdir -p gpurun_out
for cfg in "$@"; do
  echo "=== $cfg"
  env $cfg timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1 || { tail -5 gpurun_out/ab.log; continue; }
  python - <<'PY'
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ms/step', round(d['ms_per_step'],2))
        print('  ' + '  '.join(f"{k}={v['avg_ms']:.2f}" for k,v in d['kernels'].items()))
PY
done
