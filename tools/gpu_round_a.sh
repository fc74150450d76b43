#!/bin/bash
# Round evidence, part 1: all GPU tests, the default bench line, the ncu launch list of the bench
# command.  usage: tools/gpu_round_a.sh TAG   (part 2, the --set full capture: tools/gpu_ncu_c5.sh)
tag=${1:-r01}
if [ -n "$(find paper_2304_14021_b200/csrc include -newer paper_2304_14021_b200/lib/libparadiag.so -type f)" ]; then
  echo "libparadiag.so is older than its sources: rebuild first"; exit 3
fi
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
