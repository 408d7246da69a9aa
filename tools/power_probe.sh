#!/bin/bash
# Sample power / clocks / throttle reasons every 50 ms while the C5 stage
# kernels run (200 RK3 steps), to see what bounds sustained throughput.
cd "$(dirname "$0")/.."
nvidia-smi -q -d POWER > gpurun_out/power_limits.txt 2>&1
nvidia-smi --query-gpu=timestamp,power.draw,enforced.power.limit,clocks.sm,clocks.mem,temperature.gpu,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown --format=csv -lms 50 > gpurun_out/power_trace.csv &
P=$!
sleep 1
python tools/prof_stage.py --mode ${MODE:-mixed} --steps ${STEPS:-200} > gpurun_out/power_run.txt 2>&1
sleep 1
kill $P
