for v in lib lib_p4s2m3 lib_p4s2m2 lib_p4s3m3; do
  echo "$v 50: $(GMDS_LIB_PATH=paper_2605_25124_b200/$v/libgmds.so python tools/fit_only.py 50 2>&1 | tail -1)  100: $(GMDS_LIB_PATH=paper_2605_25124_b200/$v/libgmds.so python tools/fit_only.py 100 2>&1 | tail -1)" >> gpurun_out/r2_variants.log
done
