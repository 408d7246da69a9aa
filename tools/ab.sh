#!/bin/bash
# Interleaved A/B of library variants (HWG_LIB): R rounds of
# (modes) x variants at C5 (50 RK3 steps) and, with SMALL=1, at C2 4096x128
# (1000 steps), each after 3 warm-up steps.
cd "$(dirname "$0")/.."
out=gpurun_out/ab.txt
: > $out
R=${R:-3}
MODES=${MODES:-"mixed f64"}
for r in $(seq $R); do
  for L in libhwgpu.so "$@"; do
    for m in $MODES; do
      echo -n "$L r$r " >> $out
      HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 300 python tools/prof_stage.py --mode $m --steps ${STEPS:-50} >> $out 2>&1 || echo "$L $m failed" >> $out
      if [ -n "$SMALL" ]; then
        echo -n "$L r$r " >> $out
        HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 300 python tools/prof_stage.py --mode $m --nrho 4096 --ntheta 128 --steps 1000 >> $out 2>&1 || echo "$L $m small failed" >> $out
      fi
    done
  done
done
