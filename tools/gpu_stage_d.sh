export FP_STAGE_BUCKET=1
for v in stageb o2 b4 o2b4; do
export FASTPED_B200_LIB=$PWD/exp/$v.so
echo $v
timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/stage_timing.py plaza 380 390
timeout 300 python tools/plan_timing.py plaza 396
done
