#!/bin/bash
# stress step timing with and without the solo passes (tools/fit_only.py), q = 2 metric shape
for it in 50 100 200; do
  echo "iters=$it solo:    $(python tools/fit_only.py $it)"
  echo "iters=$it no-solo: $(GMDS_NO_SOLO=1 python tools/fit_only.py $it)"
done
