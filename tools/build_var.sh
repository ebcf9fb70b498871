# Build variant libraries into build/var/<name>.so with extra nvcc flags:
#   tools/build_var.sh name "-DHOS_K2_PAIRS=4" [name2 "flags2" ...]
set -e
cd "$(dirname "$0")/.."
mkdir -p build/var
C=paper_1805_11775_b200/csrc
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared \
    $flags -o build/var/$name.so $C/hos_capi.cu $C/hos_kernels.cu $C/hos_geometry.cpp \
    -L/usr/local/cuda/lib64 -lcufft -Xlinker -rpath=/usr/local/cuda/lib64 &
done
wait
ls build/var
