#!/bin/bash
# A/B the experimental builds of the stage kernel (HWG_LIB override) at C5:
# wall-clock of 20 RK3 steps per mode after 3 warm-up steps, then parity.
cd "$(dirname "$0")/.."
out=gpurun_out/variants.txt
: > $out
for L in libhwgpu.so "$@"; do
  for m in mixed f64; do
    HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 300 python tools/prof_stage.py --mode $m --steps 20 >> $out 2>&1 || echo "$L $m failed" >> $out
    echo "  ^ $L" >> $out
  done
done
