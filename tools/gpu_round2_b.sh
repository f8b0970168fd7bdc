mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_strips.py -m gpu -q -rf --timeout 900 -x > gpurun_out/pytest_strips.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_strips.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_fullsize_golden.py -m gpu -q -rf -x > gpurun_out/pytest_parity.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_parity.log
