# multi-GPU libgmds path + facade + large golden (available ones)
timeout 900 python -m pytest tests/test_gpu_distributed.py -x -q 2>&1 | tail -30 > gpurun_out/r2_dist.log
timeout 600 python -m pytest tests/test_cpp_facade.py tests/test_gpu_large.py -q -k "not c3 and not metric" 2>&1 | tail -30 > gpurun_out/r2_facade_large.log
timeout 900 python -m pytest tests/test_gpu_stress.py -q -x 2>&1 | tail -5 > gpurun_out/r2_stress.log
