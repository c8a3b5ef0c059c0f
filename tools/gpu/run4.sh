python tools/sanitize_small.py > gpurun_out/r2_sanitize_plain.log 2>&1 && \
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --racecheck-report all --print-limit 50 python tools/sanitize_small.py > gpurun_out/r2_racecheck.log 2>&1
echo "exit $?" >> gpurun_out/r2_racecheck.log
