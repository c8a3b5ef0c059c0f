python tools/dist_only.py 4000 2.0 1 > gpurun_out/r2_dist4000.log 2>&1 && \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none -k regex:"gini_gmd_kernel" -s 1 -c 1 -o /tmp/r2_prof_gmd2 python tools/dist_only.py 4000 2.0 1 > gpurun_out/r2_ncu_gmd.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_gmd2.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_prof_gmd_lines.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_gmd2.ncu-rep --page raw --csv > gpurun_out/r2_prof_gmd_raw.csv 2>&1
