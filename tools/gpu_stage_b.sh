export FASTPED_B200_LIB=$PWD/exp/stageb.so FP_STAGE_BUCKET=1
timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/stage_timing.py plaza 380 390
