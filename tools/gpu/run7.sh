timeout 900 python -m pytest tests/test_gpu_euclid.py -q -x 2>&1 | tail -5 > gpurun_out/r2_euclid_tests.log
python tools/bench_euclid.py > gpurun_out/r2_bench_euclid3.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_euclid_launches2.csv python tools/bench_euclid.py 8000 > gpurun_out/r2_ncu_euclid2.log 2>&1
