timeout 1200 python -m pytest tests/test_gpu_large.py -q -k "c3" 2>&1 | tail -25 > gpurun_out/r2_c3.log
