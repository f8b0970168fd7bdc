# ncu --set full captures of plan_stream_kernel on the bench's start and end states (plaza).
mkdir -p gpurun_out
CFG=${1:-plaza}
TAG=${2:-cur}
timeout 600 python tools/plan_timing.py $CFG 396 > gpurun_out/plan_timing_$TAG.txt 2>&1; echo "timing rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plan_stream_kernel --launch-skip 1 --launch-count 1 \
  -o gpurun_out/plan_start_$TAG python bench.py --config $CFG --plan-state start > gpurun_out/ncu_plan_start_$TAG.log 2>&1; echo "ncu start rc=$?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:plan_stream_kernel --launch-skip 397 --launch-count 1 \
  -o gpurun_out/plan_end_$TAG python bench.py --config $CFG --plan-state end > gpurun_out/ncu_plan_end_$TAG.log 2>&1; echo "ncu end rc=$?"
