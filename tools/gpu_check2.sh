#!/bin/bash
# usage: tools/gpu_check2.sh TAG [pytest args...] — GPU tests (default: all -m gpu) + the default bench line
tag=${1:-r02}; shift
mkdir -p gpurun_out
O=gpurun_out
T=${@:-tests}
timeout 1500 python -m pytest $T -m gpu -q -x > $O/${tag}_tests.log 2>&1; echo "tests rc=$?" >> $O/${tag}_tests.log
tail -5 $O/${tag}_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > $O/${tag}_bench.log 2>&1; echo "bench rc=$?" >> $O/${tag}_bench.log
tail -c 3000 $O/${tag}_bench.log
