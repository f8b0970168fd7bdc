#!/bin/bash
# One GPU call for profiles/: the launch list of a short bench run (every kernel, cold and
# serialised: shares, not absolute times), and full ncu captures of the plan kernel on the
# bench's start and end states and of the motion kernel at plaza step 200.
set -x
mkdir -p gpurun_out
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/short.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/ncu_launch.log 2>&1; echo "launches rc=$?"
ncu --set full --import-source on --clock-control none -k regex:plan_stream_kernel --launch-skip 1 --launch-count 1 \
    -o gpurun_out/plan_start python bench.py --plan-state start > gpurun_out/ncu_plan_start.log 2>&1; echo "plan start rc=$?"
ncu --set full --import-source on --clock-control none -k regex:plan_stream_kernel --launch-skip 397 --launch-count 1 \
    -o gpurun_out/plan_end python bench.py --plan-state end > gpurun_out/ncu_plan_end.log 2>&1; echo "plan end rc=$?"
ncu --set full --import-source on --clock-control none -k regex:move_rounds -s 200 -c 1 -o gpurun_out/move_full \
    python tools/profile_step.py --warm 198 --steps 4 --mode run > gpurun_out/ncu_move.log 2>&1; echo "move rc=$?"
