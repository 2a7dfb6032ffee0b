#!/bin/bash
# Builds an experimental variant of the product library with extra nvcc
# defines: scripts/build_variant.sh NAME "-DFOO=1 ..." ->
# paper_2506_03887_b200/libpre3gmask_NAME.so (load it with PRE3_GMASK_LIB).
set -e
cd "$(dirname "$0")/.."
NAME=$1; shift
D=build/var_$NAME; mkdir -p $D
NV="/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -O3 -lineinfo -Xcompiler -fPIC -Iinclude -Ipaper_2506_03887_b200/csrc $*"
$NV -Xptxas -v -c ${KSRC:-paper_2506_03887_b200/csrc/kernels.cu} -o $D/kernels.o 2> $D/ptxas.txt &
$NV -c paper_2506_03887_b200/csrc/capi.cu -o $D/capi.o &
$NV -c paper_2506_03887_b200/csrc/workload_dev.cu -o $D/workload_dev.o &
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart static -Xcompiler -static-libstdc++ \
  -Xcompiler -static-libgcc -Xlinker --exclude-libs,ALL -o paper_2506_03887_b200/libpre3gmask_$NAME.so \
  $D/kernels.o $D/capi.o $D/workload_dev.o build/obj/automaton.o build/obj/workload.o build/obj/compiler.o build/obj/serialize.o
grep -A3 "FillKernelILi0ELi0" $D/ptxas.txt | grep -i "registers\|spill" | tr '\n' ' '; echo
