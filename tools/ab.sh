#!/bin/bash
# Interleaved A/B of library variants (HWG_LIB) at C5: R rounds of
# (mixed, f64) x variants, 50 RK3 steps each after 3 warm-up steps.
cd "$(dirname "$0")/.."
out=gpurun_out/ab.txt
: > $out
R=${R:-3}
for r in $(seq $R); do
  for L in libhwgpu.so "$@"; do
    for m in mixed f64; do
      echo -n "$L r$r " >> $out
      HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 300 python tools/prof_stage.py --mode $m --steps ${STEPS:-50} >> $out 2>&1 || echo "$L $m failed" >> $out
    done
  done
done
