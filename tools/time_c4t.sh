#!/bin/bash
# c4t (NEXT-4) full-size solve, device-side Arnoldi graph vs the host loop
for g in 1 0; do
  echo "=== PARADIAG_KRYGRAPH=$g"
  C4T_PROFILE=0 PARADIAG_KRYGRAPH=$g timeout 900 python tools/run_c4t.py c4t 2>&1 | tail -2
done
