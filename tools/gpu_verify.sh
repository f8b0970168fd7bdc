# HEAD verification on a fresh box: GPU tests, smoke, the default bench line.
mkdir -p gpurun_out/verify
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/verify/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/verify/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/verify/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/verify/smoke.log
timeout 900 python bench.py > gpurun_out/verify/bench_plaza.json 2> gpurun_out/verify/bench_plaza.err; echo "bench rc=$?"
