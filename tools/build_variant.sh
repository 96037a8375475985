#!/bin/bash
# Build an A/B variant of the kernel library into lib/libmb_sm100_<name>.so (select it at run time
# with MB_KERNELS_LIB=libmb_sm100_<name>.so).  usage: tools/build_variant.sh <name> "<nvcc defines>"
set -e
name=$1; shift
defs="$*"
root=$(cd "$(dirname "$0")/.." && pwd)
src=$root/paper_2605_08639_b200/csrc/kernels
out=/tmp/mb_variant_$name
mkdir -p $out
objs=()
for f in $src/*.cu; do
  b=$(basename $f .cu)
  extra=""
  [ "$b" = anneal ] && extra="-fmad=false"
  nvcc -std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC --expt-relaxed-constexpr \
       -I$root/include $defs $extra -c $f -o $out/$b.o &
  objs+=($out/$b.o)
done
wait
nvcc -shared -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC "${objs[@]}" \
     -o $root/paper_2605_08639_b200/lib/libmb_sm100_$name.so
echo built lib/libmb_sm100_$name.so
