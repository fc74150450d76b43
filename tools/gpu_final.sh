#!/bin/bash
# Full GPU evidence: all GPU tests, smoke(), and the c6n bench line.  usage: tools/gpu_final.sh TAG
tag=${1:-r02}
O=gpurun_out
mkdir -p $O
timeout 2400 python -m pytest tests -m gpu -q > $O/${tag}_gpu_tests.log 2>&1; echo "tests rc=$?" >> $O/${tag}_gpu_tests.log
tail -3 $O/${tag}_gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/${tag}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${tag}_smoke.log
tail -2 $O/${tag}_smoke.log
timeout 900 python bench.py --config c6n --steps 5 --warmup 3 > $O/${tag}_bench_c6n.log 2>&1; echo "bench c6n rc=$?"
