set -e
V=$1; shift
OUT=/root/repo/paper_2605_25124_b200/lib_$V
mkdir -p $OUT/obj
cd /root/repo/paper_2605_25124_b200/csrc
for f in pool comm euclid_tc gini_gmd gini_merge capi_extra gini_k32 gini_split_k16 gini_split_k8 gini_k16 stress_pass_f32_grad stress_pass_f32_loss stress_pass_f32_fused stress_pass_f64_grad stress_pass_f64_loss stress_pass_f32x64_loss stress_pass_f32_diff stress_pass_f32_diffgrad stress_pass_f32_multi gini_k8 gini_k4 gini_k2 gini_k1 gini_kernels gini_plan capi_metrics stress_kernels dmat_kernels fit small_fit classical_topq tune; do
  case $f in stress_pass_f32_*|stress_kernels|fit|classical_topq) 
    echo "nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I/root/repo/include -I. --expt-relaxed-constexpr $* -dc -o $OUT/obj/$f.o $f.cu";;
  *) echo "cp /root/repo/paper_2605_25124_b200/lib/obj/$f.o $OUT/obj/$f.o";;
  esac
done | xargs -P 8 -I{} sh -c "{}"
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libgmds.so $OUT/obj/*.o -lcusolver -ldl
ls -la $OUT/libgmds.so
