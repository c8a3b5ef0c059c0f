timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench20.json 2> gpurun_out/r2_bench20.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 >> gpurun_out/r2_bench20.json 2>> gpurun_out/r2_bench20.err
timeout 1200 python tools/bench_configs.py c1 c2 c3 c4 c5 > gpurun_out/r2_configs.jsonl 2> gpurun_out/r2_configs.err
python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_bench_plain.json 2>&1 && \
/usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_bench.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/r2_ncu_bench.log 2>&1
