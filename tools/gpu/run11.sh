timeout 1200 python -m pytest tests/test_gpu_stress.py tests/test_gpu_large.py tests/test_gpu_distributed.py -q -x -k "not metric" 2>&1 | tail -15 > gpurun_out/r2_tiny_tests.log
python tools/fit_only.py 50 > gpurun_out/r2_fit_only.log 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"stress|gd_step|reduce|finish|sum_parts|combine" --csv --log-file gpurun_out/r2_fit_launches2.csv python tools/fit_only.py 50 > gpurun_out/r2_ncu_fit.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_tiny.json 2> gpurun_out/r2_bench_tiny.err
