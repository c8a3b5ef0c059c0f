timeout 1200 python -m pytest tests/test_gpu_stress.py tests/test_gpu_large.py tests/test_gpu_distributed.py -q -x -k "not metric" 2>&1 | tail -5 > gpurun_out/r2_t13.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench13.json 2> gpurun_out/r2_bench13.err
python tools/fit_only.py 50 > gpurun_out/r2_fit_only.log 2>&1 && \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"stress_tma_kernel<.int.2, .int.2," --launch-skip 40 -c 1 -o /tmp/r2_prof_fused python tools/fit_only.py 50 > gpurun_out/r2_ncu_fused.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_fused.ncu-rep --page details > gpurun_out/r2_prof_fused_details.txt 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_prof_fused_source.csv 2>&1
