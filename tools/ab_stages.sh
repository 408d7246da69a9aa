mkdir -p gpurun_out; : > gpurun_out/r01h_ab.txt
for r in 1 2; do for L in libhwgpu.so libhwgpu_m4u1.so libhwgpu_m4u2.so; do
  echo "== $L r$r" >> gpurun_out/r01h_ab.txt
  HWG_LIB=$PWD/paper_2010_04760_b200/$L timeout 600 python bench.py --no-cpu --no-dd --e2e-steps 2 --e2e-lanes 1 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); [print(m, round(v['value']/1e9,2), [round(x,4) for x in v['step_or_stage_ms_mean']]) for m,v in d['modes'].items()]; print('launch', d['launch'])" >> gpurun_out/r01h_ab.txt 2>&1
done; done
