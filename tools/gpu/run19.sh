python tools/dist_only.py 20000 2.0 3 > gpurun_out/r2_d19.log 2>&1
python tools/dist_only.py 20000 2.5 2 >> gpurun_out/r2_d19.log 2>&1
timeout 900 python -m pytest tests/test_gpu_metrics.py tests/test_gpu_large.py -q -x -k "metric or linear or gmd or c2 or c3_dist or c4 or pairwise" 2>&1 | tail -4 >> gpurun_out/r2_d19.log
