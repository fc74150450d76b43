#!/bin/bash
# A/B bench runs on one config: tools/gpu_ab_cfg.sh CONFIG "ENV=..." "ENV=..."
cfg=$1; shift
mkdir -p gpurun_out
for e in "$@"; do
  echo "=== $cfg $e"
  env $e timeout 600 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab.log 2>&1 || { tail -5 gpurun_out/ab.log; continue; }
  python - <<'PY'
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('ms/step', round(d['ms_per_step'],3))
        print('  ' + '  '.join(f"{k}={v['avg_ms']:.3f}" for k,v in d['kernels'].items()))
PY
done
