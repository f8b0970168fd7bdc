bash tools/variants.sh v
timeout 600 python tools/plan_timing.py plaza 396 > gpurun_out/plan_timing_v.txt 2>&1; cat gpurun_out/plan_timing_v.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_v.log 2>&1; tail -2 gpurun_out/pytest_v.log
