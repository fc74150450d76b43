#!/bin/bash
# Run on a GPU box via gpurun: parity tests, full-size tests (optional), bench.
# usage: tools/gpu_check.sh [quick|full] [bench args...]
mode=${1:-quick}; shift
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity.log 2>&1; echo "parity rc=$?" >> gpurun_out/parity.log
if [ "$mode" = "full" ]; then
  timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q > gpurun_out/full.log 2>&1; echo "full rc=$?" >> gpurun_out/full.log
fi
timeout 600 python bench.py "$@" > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
tail -3 gpurun_out/parity.log; tail -2 gpurun_out/full.log 2>/dev/null; tail -c 3000 gpurun_out/bench.log
