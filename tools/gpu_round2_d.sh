mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_golden.py tests/test_golden.py -m gpu -q -rf -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench20.json 2> gpurun_out/bench20.err
