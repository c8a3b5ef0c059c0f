#!/bin/bash
# Stand-in for compute-sanitizer memcheck (closed on the GPU pool): rebuild the round-2b distance
# kernels with -DGMDS_BOUNDS_CHECK (every list / panel / bucket-table / scratch index they form is
# checked, and the bucket scan's result is checked to be the exact lower bound; a violation prints
# and traps) into lib_chk/, then run the distance parity tests against that library.
set -e
cd /root/repo
OUT=paper_2605_25124_b200/lib_chk
mkdir -p $OUT/obj
cp paper_2605_25124_b200/lib/obj/*.o $OUT/obj/
(cd paper_2605_25124_b200/csrc && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I/root/repo/include -I. --expt-relaxed-constexpr -DGMDS_BOUNDS_CHECK -dc -o ../lib_chk/obj/gini_gmd.o gini_gmd.cu)
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libgmds.so $OUT/obj/*.o -lcusolver -ldl
GMDS_LIB_PATH=/root/repo/$OUT/libgmds.so python -m pytest tests/test_gpu_metrics.py tests/test_gpu_large.py tests/test_gpu_sweep.py -m gpu -x -q
GMDS_LIB_PATH=/root/repo/$OUT/libgmds.so python tools/dist_only.py 20000 2.0 1
GMDS_LIB_PATH=/root/repo/$OUT/libgmds.so python tools/dist_only.py 20000 2.5 1
