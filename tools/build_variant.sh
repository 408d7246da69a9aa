#!/bin/bash
# Build an experimental variant of libhwgpu.so with extra -D flags on the
# fast-tier TU (solver and DD objects reused), for A/B runs with HWG_LIB:
#   tools/build_variant.sh NAME -DHWG_UNROLL=6 -DHWG_MINB=3
set -e
cd "$(dirname "$0")/.."
name=$1; shift
P=paper_2010_04760_b200
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false -Xcompiler -fPIC,-ffp-contract=off"
nvcc $F "$@" -Xptxas -v -c -o $P/_obj/fast_$name.o $P/csrc/hwg_stage_fast.cu 2> $P/_obj/fast_$name.ptxas
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $P/libhwgpu_$name.so \
  $P/_obj/hwg_solver.cu.o $P/_obj/fast_$name.o $P/_obj/hwg_stage_dd.cu.o $P/_obj/hwg_peer_emu.cu.o $P/_obj/hwg_coef.cu.o
grep -A1 "stage_kernelILi0ELi[01]ELi[123]" $P/_obj/fast_$name.ptxas | grep -E "spill|Used" | sed "s/^/$name: /"
