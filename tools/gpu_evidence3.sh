#!/bin/bash
# Round-2 late evidence: GPU tests, smoke, bench lines (c5, c6n, c3), ncu launch list of the c5
# bench and one `ncu --set full` capture of each c5 hot kernel.  usage: tools/gpu_evidence3.sh TAG
tag=${1:-r02z}
O=gpurun_out
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/${tag}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${tag}_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${tag}_smoke.log 2>&1
for c in c5 c6n c3; do
  timeout 900 python bench.py --config $c > $O/${tag}_bench_$c.log 2>&1; echo "bench $c rc=$?"
done
BC="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
echo "launches rc=$?"
BC1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_time2d_v4|k_cols_cm|k_cols_tma_inv|k_rows3|k_residual_tile|k_update" -c 6 -o $O/${tag}_full -f $BC1 \
  > $O/${tag}_full_ncu.log 2>&1
echo "ncu full rc=$?"
