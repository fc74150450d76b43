#!/bin/bash
# Round-2 evidence: bench lines for every config, the CPU oracle baseline table, the ncu launch list
# and one `ncu --set full` capture of each c5 hot kernel.  usage: tools/gpu_evidence2.sh TAG
tag=${1:-r02}
O=gpurun_out
mkdir -p $O
nvidia-smi > $O/${tag}_smi.txt 2>&1
for c in c5 c3 c4 c2 c1 c6; do
  timeout 900 python bench.py --config $c --steps 5 --warmup 3 > $O/${tag}_bench_$c.log 2>&1; echo "bench $c rc=$?"
done
timeout 1200 python tools/cpu_baseline.py $O/${tag}_cpu_baseline.json > $O/${tag}_cpu_baseline.log 2>&1; echo "cpu rc=$?"
BC="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $BC > $O/${tag}_launch_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
echo "launches rc=$?"
BC1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $BC1 > $O/${tag}_full_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_time2d_v4|k_cols_cm|k_rows3|k_residual_tile|k_update" -c 6 -o $O/${tag}_full -f $BC1 \
  > $O/${tag}_full_ncu.log 2>&1
echo "ncu full rc=$?"
