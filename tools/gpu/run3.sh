timeout 900 python -m pytest tests/test_gpu_large.py -q -x -k "topq" 2>&1 | tail -15 > gpurun_out/r2_topq.log
timeout 900 python -m pytest tests/test_gpu_stress.py -q -x -k "topq or subspace or weight or smacof" 2>&1 | tail -15 > gpurun_out/r2_topq2.log
python tools/prof_classical.py > gpurun_out/r2_prof_classical.log 2>&1
