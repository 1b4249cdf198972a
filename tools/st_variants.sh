# build variant libraries of the stencil kernel (diagnostics): name and extra nvcc flags
set -e
cd paper_2407_18352_b200/csrc
build_var() {
  name=$1; shift
  mkdir -p build_var/$name
  for f in plan kernels_simt exact_c1 exact_c5 exact_small exact_generic cnn_exact mlp_tc gemm_tc capi peak; do
    cp -f build/$f.o build_var/$name/$f.o
  done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr "$@" -c stencil_tc.cu -o build_var/$name/stencil_tc.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libsmlrt_var_$name.so build_var/$name/*.o -lcudart
}
build_var rb32 -DSM_RB_=32
build_var ns3 -DSM_NS_=3
build_var ns4 -DSM_NS_=4
