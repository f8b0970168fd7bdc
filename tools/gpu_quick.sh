mkdir -p gpurun_out
: > gpurun_out/timing.log
timeout 300 python tools/plan_timing.py plaza 396 >> gpurun_out/timing.log 2>&1
timeout 600 python tools/plan_timing.py obstacles 20 >> gpurun_out/timing.log 2>&1
timeout 300 python -m pytest tests/test_fullsize_golden.py -m gpu -q -x -k "plaza or room_v4 or obstacles or ring" >> gpurun_out/timing.log 2>&1
