#!/bin/bash
# Build a tuning variant of libvba with extra nvcc flags into $1 (e.g. /tmp/v1.so):
#   bash tools/build_variant.sh build/var_s4.so -DVBA_K1_STAGES=4 -DVBA_K1_MINB=2
# Select it at run time with VBA_LIB=<path>.  Not used by the product build.
out=$1; shift
d=$(mktemp -d)
cd "$(dirname "$0")/../paper_2512_02293_b200/csrc" || exit 1
for f in vba_vision.cu vba_imu.cu vba_dense.cu vba_chol.cu vba_host.cu; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -Xcompiler -fvisibility=hidden \
    --expt-relaxed-constexpr "$@" -c $f -o $d/${f%.cu}.o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o "$out" $d/*.o -lcudart && echo "built $out"
rm -rf $d
