set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests/test_gpu_large.py -x -q -k "img2600 or c2 or c4" 2>&1 | tail -30 > gpurun_out/r2_large1.log
timeout 1200 python -m pytest tests/ -q -m gpu -k "not large" 2>&1 | tail -30 > gpurun_out/r2_gpu_all.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err
tail -3 gpurun_out/r2_large1.log gpurun_out/r2_gpu_all.log
cat gpurun_out/r2_bench1.json
