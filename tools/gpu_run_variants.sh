# Whole-run timing (plaza, 396 steps) for the in-tree library and each exp/*.so variant.
mkdir -p gpurun_out
TAG=${1:-v}
CFG=${2:-plaza}
timeout 600 python tools/plan_timing.py $CFG 396 >> gpurun_out/runvar_$TAG.txt 2>&1
shopt -s nullglob
for so in exp/*.so; do
  echo "== $so" >> gpurun_out/runvar_$TAG.txt
  FASTPED_B200_LIB=$PWD/$so timeout 600 python tools/plan_timing.py $CFG 396 >> gpurun_out/runvar_$TAG.txt 2>&1
done
cat gpurun_out/runvar_$TAG.txt
