cd $GRAFT_REPO_ROOT
for r in 1 2; do
for sp in 0 16 64; do for cp in 0 16 72; do
  echo -n "sp=$sp cp=$cp " >> gpurun_out/pad.txt
  HWG_STATE_PAD=$sp HWG_COEF_PAD=$cp python tools/prof_stage.py --mode mixed --steps 50 2>&1 | sed -E 's/launch.*//' >> gpurun_out/pad.txt
done; done; done
