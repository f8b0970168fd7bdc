set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 2000 python -m pytest tests -m gpu -q -rf --timeout 1800 > gpurun_out/pytest_gpu.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/dump_state.py plaza 396 gpurun_out/plaza_end.npz > gpurun_out/dump.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 3 > gpurun_out/bench20.json 2> gpurun_out/bench20.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref20.json 2> gpurun_out/ref20.err
ls -la gpurun_out
