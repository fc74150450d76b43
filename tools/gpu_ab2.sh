#!/bin/bash
# usage: tools/gpu_ab2.sh TAG "ENV=a" "ENV=b" ... — parity tests (test_gpu_parity.py), then the c5 bench
# per-kernel times for each environment setting (2 reps).  AB_CONFIG (default c5), AB_TESTS (pytest -k)
tag=$1; shift
mkdir -p gpurun_out
O=gpurun_out
if [ "${AB_NOTEST:-0}" != "1" ]; then
  timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x ${AB_TESTS:+-k "$AB_TESTS"} > $O/${tag}_tests.log 2>&1
  echo "tests rc=$?" >> $O/${tag}_tests.log; tail -4 $O/${tag}_tests.log
fi
for rep in 1 2; do
for envs in "$@"; do
  env $envs timeout 600 python bench.py --config ${AB_CONFIG:-c5} --steps 3 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$envs', round(d['ms_per_step'],3), 'precond', round(d['precond']['ms_per_step'],3) if d.get('precond') else None); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))" 2>&1 | tee -a $O/${tag}_ab.log
done
done
