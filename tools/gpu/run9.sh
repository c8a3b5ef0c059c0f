timeout 1200 python -m pytest tests/test_gpu_stress.py tests/test_gpu_large.py tests/test_gpu_distributed.py -q -x -k "not metric" 2>&1 | tail -15 > gpurun_out/r2_tiny_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_tiny.json 2> gpurun_out/r2_bench_tiny.err
