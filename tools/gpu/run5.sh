timeout 900 python -m pytest tests/test_gpu_euclid.py -q -x 2>&1 | tail -25 > gpurun_out/r2_euclid_tests.log
timeout 600 python tools/bench_euclid.py > gpurun_out/r2_bench_euclid.json 2> gpurun_out/r2_bench_euclid.err
