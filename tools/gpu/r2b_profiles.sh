#!/bin/bash
# Round-2 (second half) evidence: launch list of the bench command, ncu --set full of the headline
# distance kernel (gini_gmd2_kernel) and of the device loop's main pass in the fused regime
# (stress_tma_multi_kernel<2, 1>) at the metric shape.  CSV exports only (reports stay on the box).
set -x
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2b_launches_bench.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:gini_gmd2 -c 1 -o /tmp/r2b_gmd2 -f \
  python tools/dist_only.py 20000 2.0 1 > gpurun_out/r2b_gmd2_ncu.log 2>&1
ncu -i /tmp/r2b_gmd2.ncu-rep --page details --csv > gpurun_out/r2b_gmd2_details.csv
ncu -i /tmp/r2b_gmd2.ncu-rep --page raw --csv > gpurun_out/r2b_gmd2_raw.csv
ncu --set full --import-source on --clock-control none -k regex:"stress_tma_multi_kernel<2, 1>" -s 75 -c 1 -o /tmp/r2b_fused -f \
  python tools/fit_only.py 100 > gpurun_out/r2b_fused_ncu.log 2>&1
ncu -i /tmp/r2b_fused.ncu-rep --page details --csv > gpurun_out/r2b_fused_details.csv
ncu -i /tmp/r2b_fused.ncu-rep --page raw --csv > gpurun_out/r2b_fused_raw.csv
ncu -i /tmp/r2b_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/r2b_fused_sass.csv 2>/dev/null
ls -la gpurun_out/
