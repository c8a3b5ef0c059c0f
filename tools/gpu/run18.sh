python tools/dist_c4.py 20000 > gpurun_out/r2_c4.log 2>&1
python tools/dist_c4.py 4000 1 > gpurun_out/r2_c4s.log 2>&1 && \
/usr/local/cuda/bin/ncu -f --set full --import-source on --clock-control none -s 1 -c 1 -k regex:"gini_split" -o /tmp/r2_prof_split python tools/dist_c4.py 4000 1 > gpurun_out/r2_ncu_split.log 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_split.ncu-rep --page details > gpurun_out/r2_prof_split_details.txt 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_split.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/r2_prof_split_lines.csv 2>&1
/usr/local/cuda/bin/ncu -i /tmp/r2_prof_split.ncu-rep --page source --csv --print-source sass > gpurun_out/r2_prof_split_source.csv 2>&1
