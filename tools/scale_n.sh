#!/bin/bash
# Distance (nu = 2, gini_gmd2_kernel) and stress (Kruskal, q = 2, seeded init) rates over n on one B200:
# tools/dist_only.py and tools/fit_only.py (metric generator, packed fp32 D).
for n in 5000 10000 20000 40000 60000; do
  echo "n=$n distance: $(python tools/dist_only.py $n 2.0 2 | tail -1)"
  a=$(FIT_N=$n python tools/fit_only.py 50 | tail -1); b=$(FIT_N=$n python tools/fit_only.py 100 | tail -1)
  echo "n=$n fit50: $a"
  echo "n=$n fit100: $b"
done
