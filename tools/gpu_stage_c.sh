export FP_STAGE_BUCKET=1
for v in stageb; do
export FASTPED_B200_LIB=$PWD/exp/$v.so
echo $v
timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/stage_timing.py plaza 380 390
done
unset FASTPED_B200_LIB FP_STAGE_BUCKET; timeout 600 python tools/plan_timing.py plaza 396
