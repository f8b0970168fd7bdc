bash tools/variants.sh r
timeout 600 python tools/plan_timing.py plaza 396 > gpurun_out/plan_timing_r.txt 2>&1; cat gpurun_out/plan_timing_r.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_r.log 2>&1; tail -2 gpurun_out/pytest_r.log
