mkdir -p gpurun_out
: > gpurun_out/timing.log
for v in t512 t640 t768 t640n2k; do
  echo "== $v" >> gpurun_out/timing.log
  FASTPED_B200_LIB=exp/lib_$v.so timeout 300 python tools/plan_timing.py plaza 396 >> gpurun_out/timing.log 2>&1
done
