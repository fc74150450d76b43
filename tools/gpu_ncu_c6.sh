#!/bin/bash
# ncu --set full of the c6 (NEXT-3) kernels: k_x1d (x transforms) and the four-step time passes.
# usage: tools/gpu_ncu_c6.sh TAG [kernel-regex]
O=gpurun_out
tag=${1:-c6}
re=${2:-"k_x1d|k_tl_"}
BC="python bench.py --config c6 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 $BC > $O/${tag}_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$re" -c 8 -o $O/${tag}_full -f $BC > $O/${tag}_ncu.log 2>&1
echo "ncu rc=$?"
