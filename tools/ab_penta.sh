# c1 / c2 per-iteration time of the pentadiagonal solve; parity of the 1D cases incl. m = 8191
for c in c1 c2; do python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(d['config']['workload'][:30], round(d['ms_per_step'],4), {k:round(v['avg_ms'],4) for k,v in d['kernels'].items() if 'penta' in k})"; done
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "c1 or c2" 2>&1 | tail -2
PARADIAG_PENTA=0 python -m pytest tests/test_gpu_parity.py -q -x -k "c2_m8191 or c2_theta or c1_theta" 2>&1 | tail -2
