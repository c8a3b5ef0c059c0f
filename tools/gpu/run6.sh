python tools/bench_euclid.py > gpurun_out/r2_bench_euclid2.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_euclid_launches.csv python tools/bench_euclid.py 8000 > gpurun_out/r2_ncu_euclid.log 2>&1
