#!/bin/bash
# slab path at N = 1 (NCCL world of one): block-addressed transposes vs pack/unpack copies
for f in 1 0; do
  PARADIAG_SLAB_FUSED=$f timeout 600 python bench.py --parallelism slab --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fused', $f, round(d['ms_per_step'],2)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.2f}\" for k,v in d['kernels'].items()))"
done
