#!/bin/bash
# stress step timing across experimental builds of the stress passes (tools/build_variant.sh <name> <flags>)
for v in "" "$@"; do
  lib=/root/repo/paper_2605_25124_b200/lib${v:+_$v}/libgmds.so
  [ -f $lib ] || continue
  for it in 50 100; do
    echo "lib${v:+_$v} iters=$it: $(GMDS_LIB_PATH=$lib python tools/fit_only.py $it)"
  done
done
