mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_strips.py -m gpu -q -rf --timeout 900 > gpurun_out/pytest_strips.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_strips.log
