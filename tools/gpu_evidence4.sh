#!/bin/bash
# Round-2 final evidence: GPU tests, smoke, bench lines (c5, c6n, c3), ncu launch list of the c5
# bench and one `ncu --set full` capture of each c5 hot kernel.  usage: tools/gpu_evidence4.sh TAG
tag=${1:-r02zc}
O=gpurun_out
mkdir -p $O
if [ -n "$(find paper_2304_14021_b200/csrc include -newer paper_2304_14021_b200/lib/libparadiag.so -type f)" ]; then
  echo "libparadiag.so is older than its sources: rebuild first"; exit 3
fi
nvidia-smi > $O/${tag}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/${tag}_gpu_tests.log 2>&1; echo "rc=$?" >> $O/${tag}_gpu_tests.log
tail -3 $O/${tag}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${tag}_smoke.log 2>&1
tail -1 $O/${tag}_smoke.log
for c in c5 c6n c3; do
  timeout 900 python bench.py --config $c > $O/${tag}_bench_$c.log 2>&1; echo "bench $c rc=$?"
done
BC="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $BC > $O/${tag}_launch_plain.log 2>&1 &&
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file $O/${tag}_launches.csv $BC > $O/${tag}_launch_ncu.log 2>&1
echo "launches rc=$?"
BC1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 $BC1 > $O/${tag}_full_plain.log 2>&1 &&
timeout 1500 ncu --set full --clock-control none --import-source on \
  -k regex:"k_time2d_v4|k_cols_cm|k_cols_tma_inv|k_rows3|k_residual_tile|k_update" -c 7 -o $O/${tag}_full -f $BC1 \
  > $O/${tag}_full_ncu.log 2>&1
echo "ncu full rc=$?"
# gpurun brings back at most 64 MiB: export the raw page here and leave a large report on the box
ncu -i $O/${tag}_full.ncu-rep --page raw --csv > $O/${tag}_full_raw.csv 2>/dev/null
if [ $(stat -c %s $O/${tag}_full.ncu-rep) -gt 40000000 ]; then rm -f $O/${tag}_full.ncu-rep; fi
du -sh $O
