#!/bin/bash
# ncu --set full of one launch of each c5 hot kernel (full sizes), inside a short bench run.
tag=${1:-r01b}
mkdir -p gpurun_out
BC="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $BC > gpurun_out/${tag}_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"${KRE:-k_time2d|k_cols|k_rows|k_residual|k_update}" -c ${KC:-6} -o gpurun_out/${tag}_c5full -f $BC \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -5 gpurun_out/${tag}_ncu.log
