for f in 1 0; do PARADIAG_TLFUSE=$f python bench.py --config c6 --steps 10 --warmup 3 --no-e2e --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('fuse', $f, d['ms_per_step']); [print(k, round(v['avg_ms'],3), round(v['gbs'] or 0)) for k,v in d['kernels'].items()]"; done
