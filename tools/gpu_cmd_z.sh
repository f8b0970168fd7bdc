bash tools/gpu_stage.sh exp/stage.so bucket
timeout 600 python tools/plan_timing.py plaza 396
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_z.log 2>&1; tail -2 gpurun_out/pytest_z.log
