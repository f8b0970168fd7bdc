# ncu --set full of the motion's prep and seed kernels at plaza step ~200 (one launch each).
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"seed_classify|bk_count|bk_sort_kernel|bk_final|p2_number|move_rounds" \
  --launch-skip 1194 --launch-count 6 -o gpurun_out/motion200 python tools/profile_step.py --config plaza --warm 198 --steps 2 --mode run > gpurun_out/ncu_motion200.log 2>&1
echo "ncu rc=$?"
