# Closing bench refresh after the last plan-phase changes (plaza 396 / 20 steps, obstacles, ring),
# the plan kernel launch list and ncu summaries.
mkdir -p gpurun_out/final2
F=gpurun_out/final2
timeout 900 python bench.py > $F/bench_plaza.json 2> $F/bench_plaza.err; echo "plaza rc=$?"
timeout 900 python bench.py --steps 20 --warmup 3 > $F/bench_plaza20.json 2> $F/bench_plaza20.err; echo "plaza20 rc=$?"
timeout 1500 python bench.py --config obstacles --steps 20 --warmup 3 > $F/bench_obstacles.json 2> $F/bench_obstacles.err; echo "obstacles rc=$?"
timeout 600 python bench.py --config ring > $F/bench_ring.json 2> $F/bench_ring.err; echo "ring rc=$?"
for v in 1 4 5; do timeout 600 python bench.py --config room --v $v > $F/bench_room_v$v.json 2> $F/bench_room_v$v.err; done
timeout 600 python bench.py --config corridor > $F/bench_corridor.json 2> $F/bench_corridor.err; echo "corridor rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $F/ncu_launch.log 2>&1; echo "launches rc=$?"
ls -la $F
