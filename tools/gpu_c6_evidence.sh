#!/bin/bash
# c6 (NEXT-3) evidence: bench line (with e2e and cpu_baseline), launch list, ncu --set full of the
# hot kernels.  usage: tools/gpu_c6_evidence.sh TAG
O=gpurun_out
tag=${1:-r01d_c6}
timeout 600 python bench.py --config c6 --steps 10 --warmup 3 > $O/${tag}_bench.log 2>&1; echo "bench rc=$?"
tail -1 $O/${tag}_bench.log | cut -c1-400
BC="python bench.py --config c6 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 $BC > $O/${tag}_launch_plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
echo "launches rc=$?"
BC1="python bench.py --config c6 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 300 $BC1 > $O/${tag}_full_plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_x1d|k_tl_" -c 8 \
    -o $O/${tag}_full -f $BC1 > $O/${tag}_full_ncu.log 2>&1
echo "ncu full rc=$?"
