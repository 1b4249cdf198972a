# build variant libraries (diagnostics): each variant recompiles ONE source
# file with extra nvcc flags and links it with the main build's other objects.
#   build_var <name> <file.cu> [flags...]  ->  paper_2407_18352_b200/libsmlrt_var_<name>.so
set -e
cd paper_2407_18352_b200/csrc
build_var() {
  name=$1; src=$2; shift 2
  mkdir -p build_var/$name
  for o in build/*.o; do cp -f $o build_var/$name/; done
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC,-O3 --expt-relaxed-constexpr -Xptxas -v "$@" -c $src -o build_var/$name/${src%.cu}.o 2> build_var/$name/ptxas.txt || (cat build_var/$name/ptxas.txt; false)
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../libsmlrt_var_$name.so build_var/$name/*.o -lcudart
}
if [ $# -gt 0 ]; then "$@"; fi
