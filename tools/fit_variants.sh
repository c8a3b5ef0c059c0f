#!/bin/bash
# stress step timing across experimental builds of the stress passes (tools/build_variant.sh)
for v in "" _dgsplit _q2split _q2split3; do
  lib=/root/repo/paper_2605_25124_b200/lib$v/libgmds.so
  [ -f $lib ] || continue
  for it in 50 100; do
    echo "lib$v iters=$it: $(GMDS_LIB_PATH=$lib python tools/fit_only.py $it)"
  done
done
