# Per-kernel durations of whole steps with warm caches (ncu --cache-control none): step 1-3 and 200-202.
mkdir -p gpurun_out
TAG=${1:-x}
for W in 0 198; do
timeout 900 ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv \
  --log-file gpurun_out/launch_${TAG}_w$W.csv python tools/profile_step.py --config plaza --warm $W --steps 3 --mode run \
  > gpurun_out/launch_${TAG}_w$W.log 2>&1; echo "ncu w$W rc=$?"
done
