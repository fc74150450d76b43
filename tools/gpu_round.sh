#!/bin/bash
# One gpurun call: parity + full-size tests, bench, ncu launch list of the bench command and one
# `ncu --set full` capture of the top kernels on a short c5-shaped driver.
# usage: tools/gpu_round.sh TAG [skip-tests] [skip-ncu]
tag=${1:-r01}; shift
mkdir -p gpurun_out
O=gpurun_out
nvidia-smi > $O/${tag}_smi.txt 2>&1
if [ "$1" != "skip-tests" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $O/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $O/${tag}_tests.log
  tail -3 $O/${tag}_tests.log
fi
timeout 600 python bench.py --steps 5 --warmup 3 > $O/${tag}_bench.log 2>&1; echo "bench rc=$?" >> $O/${tag}_bench.log
tail -c 2500 $O/${tag}_bench.log
if [ "$2" != "skip-ncu" ]; then
  BC="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
  timeout 600 $BC > $O/${tag}_launch_plain.log 2>&1 &&
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
      --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
  echo "launches rc=$?"
  PC="python tools/prof_driver.py 16 2"
  timeout 300 $PC > $O/${tag}_prof_plain.log 2>&1 &&
  timeout 1200 ncu --set full --clock-control none --import-source on -s 7 -c 7 \
      -o $O/${tag}_full -f $PC > $O/${tag}_full_ncu.log 2>&1
  echo "ncu full rc=$?"
fi
