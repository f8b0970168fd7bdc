# A/B of programmatic dependent launch: whole-run step time per config with the attribute off
# (FASTPED_PDL=0), on (in-tree library), and the FP_PDL_TRIGGER variant (exp/pdl_trigger.so);
# then the GPU tests under each PDL build.
mkdir -p gpurun_out/pdl
O=gpurun_out/pdl/ab.txt
for rep in 1 2; do
  for cfg in plaza corridor room ring; do
    echo "== rep $rep off" >> $O; FASTPED_PDL=0 timeout 300 python tools/plan_timing.py $cfg 396 >> $O 2>&1
    echo "== rep $rep on" >> $O; timeout 300 python tools/plan_timing.py $cfg 396 >> $O 2>&1
    echo "== rep $rep trigger" >> $O; FASTPED_B200_LIB=$PWD/exp/pdl_trigger.so timeout 300 python tools/plan_timing.py $cfg 396 >> $O 2>&1
  done
done
cat $O
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pdl/pytest_on.log 2>&1; echo "gpu tests (pdl on) rc=$?"; tail -1 gpurun_out/pdl/pytest_on.log
FASTPED_B200_LIB=$PWD/exp/pdl_trigger.so timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pdl/pytest_trigger.log 2>&1; echo "gpu tests (trigger) rc=$?"; tail -1 gpurun_out/pdl/pytest_trigger.log
