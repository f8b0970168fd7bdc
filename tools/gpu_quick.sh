mkdir -p gpurun_out
: > gpurun_out/timing.log
for v in m_base m_li6 m_li12 m_b1 m_pb4; do
  echo "== $v" >> gpurun_out/timing.log
  FASTPED_B200_LIB=exp/lib_$v.so timeout 300 python tools/plan_timing.py plaza 396 >> gpurun_out/timing.log 2>&1
done
timeout 600 python -m pytest tests/test_acceptance_dropin.py -m gpu -q >> gpurun_out/timing.log 2>&1
timeout 1500 python bench.py --capacity --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_capacity.json 2> gpurun_out/bench_capacity.err
