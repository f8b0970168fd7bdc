# A/B of the unrolled run() graph (FASTPED_RUN_UNROLL steps per graph launch) against one graph
# launch per phase: whole-run step time per config, then the GPU tests at the default.
mkdir -p gpurun_out/unroll
O=gpurun_out/unroll/ab.txt
for rep in 1 2; do
  for cfg in plaza corridor room ring; do
    for u in 1 8 33; do
      echo "== rep $rep unroll $u" >> $O; FASTPED_RUN_UNROLL=$u timeout 300 python tools/plan_timing.py $cfg 396 >> $O 2>&1
    done
  done
done
cat $O
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/unroll/pytest.log 2>&1; echo "gpu tests rc=$?"; tail -1 gpurun_out/unroll/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
