mkdir -p gpurun_out
timeout 600 python tools/plan_timing.py plaza 396 > gpurun_out/plan_timing_i.txt 2>&1; cat gpurun_out/plan_timing_i.txt
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_i.log 2>&1; tail -3 gpurun_out/pytest_i.log
bash tools/gpu_launches.sh i
python tools/launch_table.py gpurun_out/launch_i_w198.csv 30 | head -34
