bash tools/variants.sh m
timeout 600 python tools/plan_timing.py plaza 396 > gpurun_out/plan_timing_m.txt 2>&1; cat gpurun_out/plan_timing_m.txt
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_golden.py -x -q -m gpu > gpurun_out/pytest_m.log 2>&1; tail -2 gpurun_out/pytest_m.log
