#!/bin/bash
# Build an experimental variant of libhwgpu.so with extra -D flags on the
# double-double TU (solver and fast-tier objects reused), for A/B runs with
# HWG_LIB:   tools/build_dd_variant.sh NAME -DHWG_DD_MINB=4 -DHWG_DD_SEQ
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_2010_04760_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off"
nvcc $F "$@" -Xptxas -v -c -o $P/_obj/dd_$name.o $P/csrc/hwg_stage_dd.cu 2> $P/_obj/dd_$name.ptxas
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libhwgpu_$name.so \
  $P/_obj/hwg_solver.cu.o $P/_obj/hwg_stage_fast.cu.o $P/_obj/dd_$name.o $P/_obj/hwg_peer_emu.cu.o $P/_obj/hwg_coef.cu.o
for k in "ILi0ELi1ELi2E" "ILi0ELi0ELi2E"; do
  grep -A2 "Compiling entry function '_ZN3hwg15stage_kernel_dd$k" $P/_obj/dd_$name.ptxas | grep -E "spill|Used" | sed "s/^/$name $k: /"
done
