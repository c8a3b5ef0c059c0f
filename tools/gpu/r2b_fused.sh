#!/bin/bash
# ncu --set full of the device loop's main pass (stress_tma_multi_kernel<2, 1>, fused body) at the
# metric shape, iterations ~75 of a 100-iteration fit (two consecutive multi launches: the empty
# difference slot and the fused pass)
ncu --set full --import-source on --clock-control none -k regex:stress_tma_multi_kernel -s 150 -c 2 -o /tmp/r2b_fused -f \
  python tools/fit_only.py 100 > gpurun_out/r2b_fused_ncu.log 2>&1
ncu -i /tmp/r2b_fused.ncu-rep --page details --csv > gpurun_out/r2b_fused_details.csv
ncu -i /tmp/r2b_fused.ncu-rep --page raw --csv > gpurun_out/r2b_fused_raw.csv
ls -la gpurun_out/
