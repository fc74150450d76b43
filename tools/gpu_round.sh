#!/bin/bash
# One gpurun call for the round's evidence: all GPU tests, the default bench line, the ncu launch
# list of the bench command, and an `ncu --set full` capture of one launch of every c5 hot kernel.
# usage: tools/gpu_round.sh TAG
tag=${1:-r01}
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi > $O/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $O/${tag}_tests.log
tail -3 $O/${tag}_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/${tag}_bench.log 2>&1; echo "bench rc=$?" >> $O/${tag}_bench.log
tail -c 1500 $O/${tag}_bench.log
BC="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $BC > $O/${tag}_launch_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
echo "launches rc=$?"
BC1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $BC1 > $O/${tag}_full_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_time2d|k_cols3|k_rows3|k_residual_tile|k_update" -c 5 -o $O/${tag}_full -f $BC1 \
  > $O/${tag}_full_ncu.log 2>&1
echo "ncu full rc=$?"
