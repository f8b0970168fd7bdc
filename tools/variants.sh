# Times the plan kernel on the start state for each prebuilt variant in exp/*.so plus the
# in-tree library:  bash tools/variants.sh TAG [config]
mkdir -p gpurun_out
TAG=${1:-v}
CFG=${2:-plaza}
timeout 300 python tools/plan_start_time.py $CFG base >> gpurun_out/variants_$TAG.txt 2>&1
shopt -s nullglob
for so in exp/*.so; do
  FASTPED_B200_LIB=$PWD/$so timeout 300 python tools/plan_start_time.py $CFG $(basename $so) >> gpurun_out/variants_$TAG.txt 2>&1
done
cat gpurun_out/variants_$TAG.txt
