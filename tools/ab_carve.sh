for c in none 58 60 72 100 none; do
  echo "=== carve $c"
  if [ $c = none ]; then unset PARADIAG_CARVE; else export PARADIAG_CARVE=$c; fi
  timeout 600 python bench.py --config c5 --steps 3 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('ms/step', round(d['ms_per_step'],3)); print('  ' + '  '.join(f\"{k}={v['avg_ms']:.3f}\" for k,v in d['kernels'].items()))"
done
