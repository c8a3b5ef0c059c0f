python tools/fit_only.py 50 > gpurun_out/r2_fit_only.log 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stress|gd_step|reduce|finish|sum_parts|combine" --csv --log-file gpurun_out/r2_fit_launches.csv python tools/fit_only.py 50 > gpurun_out/r2_ncu_fit.log 2>&1
