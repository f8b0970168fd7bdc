mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:"plan_exact_list" --launch-skip 5 --launch-count 1 \
  -o gpurun_out/exact5 python tools/profile_step.py --config plaza --warm 0 --steps 8 --mode run > gpurun_out/ncu_exact5.log 2>&1
echo "ncu rc=$?"
