# Quick A/B loop on the GPU box: plan-kernel timing on plaza (+ optional configs), then the GPU tests.
mkdir -p gpurun_out
TAG=${1:-cur}
shift
for cfg in plaza "$@"; do
  timeout 600 python tools/plan_timing.py $cfg 396 >> gpurun_out/plan_timing_$TAG.txt 2>&1; echo "timing $cfg rc=$?"
done
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
