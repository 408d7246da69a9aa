#!/bin/bash
# Interleaved A/B of double-double library variants (HWG_LIB) at C5 and C3:
#   tools/ab_dd.sh libhwgpu_x.so ...   -> gpurun_out/ab_dd.txt
cd "$(dirname "$0")/.."
out=${OUT:-gpurun_out/ab_dd.txt}
: > $out
R=${R:-2}
MODES=${MODES:-"dd-mixed dd-full"}
for r in $(seq $R); do
  for L in libhwgpu.so "$@"; do
    for m in $MODES; do
      echo -n "$L r$r " >> $out
      HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 300 python tools/prof_stage.py --mode $m ${SHAPE:-} --warmup ${WARM:-1} --steps ${STEPS:-3} >> $out 2>&1 || echo "$L $m failed" >> $out
    done
  done
done
