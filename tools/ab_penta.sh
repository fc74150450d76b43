set -e
python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or c2" 2>&1 | tail -3
for f in 1 0; do echo "PARADIAG_PENTA=$f"; PARADIAG_PENTA=$f python tools/time_solve.py c1 c2 2>&1 | grep graph=1; done
