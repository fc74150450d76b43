#!/bin/bash
# slab path at N = 1 (NCCL world of one): block-addressed transposes (1 and 4 slice ranges) vs
# pack/unpack copies
for cfg in "PARADIAG_SLAB_FUSED=1 PARADIAG_SLAB_CHUNKS=1" "PARADIAG_SLAB_FUSED=1 PARADIAG_SLAB_CHUNKS=4" "PARADIAG_SLAB_FUSED=0"; do
  env $cfg timeout 600 python bench.py --parallelism slab --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],2)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.2f}\" for k,v in d['kernels'].items()))"
done
