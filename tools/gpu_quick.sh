#!/bin/bash
# quick GPU loop: parity tests (+ full-size with 'full'), then the c5 bench; env passes through.
tag=${1:-q}; mode=${2:-parity}
mkdir -p gpurun_out
if [ "$mode" != "bench" ]; then
  T=tests/test_gpu_parity.py; [ "$mode" = "full" ] && T="tests/test_gpu_parity.py tests/test_gpu_fullsize.py"
  timeout 420 python -m pytest $T -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/${tag}_tests.log
  tail -4 gpurun_out/${tag}_tests.log
fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${tag}_bench.log 2>&1; echo "bench rc=$?"
python - <<'PY'
import json,glob,sys
for l in open(sorted(glob.glob('gpurun_out/*_bench.log'), key=lambda f: __import__('os').path.getmtime(f))[-1]):
    if l.startswith('{'):
        d=json.loads(l); print('ms/step', round(d['ms_per_step'],2), 'value', '%.3e'%d['value'])
        for k,v in d['kernels'].items(): print(f"  {k:14s} {v['avg_ms']:8.3f} ms  {v['gbs'] or 0:8.0f} GB/s")
PY
