timeout 1500 python -m pytest tests/ -q -m gpu -x 2>&1 | tail -8 > gpurun_out/r2_all_gpu.log
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench16.json 2> gpurun_out/r2_bench16.err
