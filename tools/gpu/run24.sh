for v in lib lib_g16u4 lib_g8u8 lib_g16u8 lib; do
  echo "$v 50: $(GMDS_LIB_PATH=paper_2605_25124_b200/$v/libgmds.so python tools/fit_only.py 50 2>&1 | tail -1)  100: $(GMDS_LIB_PATH=paper_2605_25124_b200/$v/libgmds.so python tools/fit_only.py 100 2>&1 | tail -1)" >> gpurun_out/r2_variants2.log
done
