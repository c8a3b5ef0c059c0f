timeout 900 python -m pytest tests/test_gpu_distributed.py tests/test_gpu_stress.py -q -x -k "partials or gradient_accuracy or small" 2>&1 | tail -4 > gpurun_out/r2_t21.log
python tools/fit_only.py 50 > gpurun_out/r2_fit_only.log 2>&1 && \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"stress_tma_kernel<.int.2, .int.7" --launch-skip 12 -c 1 -o /tmp/r2_prof_dg7b python tools/fit_only.py 50 > gpurun_out/r2_ncu_dg7.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_dg7b.ncu-rep --page details > gpurun_out/r2_prof_dg7_details.txt 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_dg7b.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_prof_dg7_source.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_dg7b.ncu-rep --page raw --csv > gpurun_out/r2_prof_dg7_raw.csv 2>&1
