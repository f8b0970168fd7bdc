bash tools/gpu_run_variants.sh w
FASTPED_B200_LIB=$PWD/exp/stageb.so FP_STAGE_BUCKET=1 timeout 300 python tools/stage_timing.py plaza 0 10
timeout 300 python tools/motion_phases.py plaza | head -3
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_w.log 2>&1; tail -2 gpurun_out/pytest_w.log
