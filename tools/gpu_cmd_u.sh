bash tools/gpu_stage_c.sh
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_u.log 2>&1; tail -2 gpurun_out/pytest_u.log
