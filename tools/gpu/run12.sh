python tools/fit_only.py 50 > gpurun_out/r2_fit_only.log 2>&1 && \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"stress_tma_kernel<.int.2, .int.7" --launch-skip 10 -c 1 -o /tmp/r2_prof_dg7 python tools/fit_only.py 50 > gpurun_out/r2_ncu_dg7.log 2>&1; \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"stress_tma_kernel<.int.2, .int.2," --launch-skip 40 -c 1 -o /tmp/r2_prof_fused python tools/fit_only.py 50 > gpurun_out/r2_ncu_fused.log 2>&1
for k in dg7 fused; do
  /usr/local/cuda/bin/ncu -i /tmp/r2_prof_$k.ncu-rep --page details > gpurun_out/r2_prof_${k}_details.txt 2>&1
  /usr/local/cuda/bin/ncu -i /tmp/r2_prof_$k.ncu-rep --page raw --csv > gpurun_out/r2_prof_${k}_raw.csv 2>&1
  /usr/local/cuda/bin/ncu -i /tmp/r2_prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_prof_${k}_source.csv 2>&1
done
ls -la gpurun_out/ | tail
