#!/bin/bash
# usage: tools/gpu_ncu1.sh TAG KERNEL_REGEX [count] — one ncu --set full capture of the c5 bench's kernel
tag=$1; kre=$2; cnt=${3:-1}
mkdir -p gpurun_out
BC="python bench.py --config ${NCU_CONFIG:-c5} --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $BC > gpurun_out/${tag}_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$kre" -c $cnt -o gpurun_out/${tag} -f $BC \
  > gpurun_out/${tag}_ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/${tag}_ncu.log
