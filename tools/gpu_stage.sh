export FASTPED_B200_LIB=$PWD/exp/stage.so
timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/stage_timing.py plaza 195 205
timeout 300 python tools/stage_timing.py plaza 380 390
unset FASTPED_B200_LIB
timeout 600 python tools/plan_timing.py plaza 396
