#!/bin/bash
# Build variants of the config-4 kernels (only sipg_h3.cu is recompiled; the other objects come from
# the default build) into paper_2504_03573_b200/build/var/NAME.so.
# usage: tools/h3c_variants.sh NAME "-DFLAG=.. -DFLAG2=.." [NAME2 "flags" ...]
cd "$(dirname "$0")/.."
P=paper_2504_03573_b200
mkdir -p $P/build/var
while [ $# -ge 2 ]; do
  name=$1; flags=$2; shift 2
  ( nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr \
      -I include $flags -c $P/csrc/sipg_h3.cu -o $P/build/var/$name.o &&
    nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/build/var/$name.so $P/build/var/$name.o \
      $P/build/sipg_capi.o $P/build/sipg_quad.o $P/build/sipg_tri.o $P/build/sipg_hex.o $P/build/sipg_krylov.o -lcudart &&
    echo "built $name ($flags)" ) &
done
wait
