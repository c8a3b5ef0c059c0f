#!/bin/bash
# A/B of the stress step between the in-tree build and another build of libgmds (lib_prev/)
for rep in 1 2; do
for it in 50 100; do
  echo "cur  iters=$it: $(python tools/fit_only.py $it)"
  echo "prev iters=$it: $(GMDS_LIB_PATH=/root/repo/paper_2605_25124_b200/lib_prev/libgmds.so python tools/fit_only.py $it)"
done; done
