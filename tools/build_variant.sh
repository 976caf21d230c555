#!/bin/bash
# Build a variant of libvba with extra nvcc defines into build/var_<name>.so (tuning sweeps).
# usage: tools/build_variant.sh NAME "-DFOO=1 -DBAR=2"
set -e
name=$1; defs=$2
cd "$(dirname "$0")/../paper_2512_02293_b200/csrc"
mkdir -p build/var_$name
for f in vba_vision.cu vba_imu.cu vba_dense.cu vba_chol.cu vba_small.cu vba_preint.cu vba_host.cu vba_pgba.cu vba_init.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr $defs -c $f -o build/var_$name/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o ../../build/var_$name.so build/var_$name/*.o -lcudart
echo built build/var_$name.so
