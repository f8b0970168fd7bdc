#!/bin/bash
# One GPU call: the bench line, its ncu launch list, and full captures of the two kernels at step 200.
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
python tools/profile_step.py --warm 198 --steps 4 --mode run > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:plan_tile -s 200 -c 1 -o gpurun_out/plan_full \
    python tools/profile_step.py --warm 198 --steps 4 --mode run > gpurun_out/ncu_plan.log 2>&1; echo "plan rc=$?"
ncu --set full --import-source on --clock-control none -k regex:move_rounds -s 200 -c 1 -o gpurun_out/move_full \
    python tools/profile_step.py --warm 198 --steps 4 --mode run > gpurun_out/ncu_move.log 2>&1; echo "move rc=$?"
python tools/profile_step.py --warm 4 --steps 2 --mode run > gpurun_out/prof_start.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:plan_tile -s 5 -c 1 -o gpurun_out/plan_start \
    python tools/profile_step.py --warm 4 --steps 2 --mode run > gpurun_out/ncu_plan_start.log 2>&1; echo "plan start rc=$?"
