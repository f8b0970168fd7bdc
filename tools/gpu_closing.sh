# Closing bench refresh: every BASELINE config through bench.py, the reference arm, and the
# launch list of a short plaza run (ncu, cold and serialised: shares, not absolute times).
F=gpurun_out/closing
mkdir -p $F
timeout 900 python bench.py > $F/bench_plaza.json 2> $F/bench_plaza.err; echo "plaza rc=$?"
timeout 900 python bench.py --steps 20 --warmup 3 > $F/bench_plaza20.json 2> $F/bench_plaza20.err; echo "plaza20 rc=$?"
for v in 1 2 3 4 5; do
  timeout 600 python bench.py --config room --v $v > $F/bench_room_v$v.json 2> $F/bench_room_v$v.err; echo "room v$v rc=$?"
done
timeout 600 python bench.py --config ring > $F/bench_ring.json 2> $F/bench_ring.err; echo "ring rc=$?"
timeout 600 python bench.py --config corridor > $F/bench_corridor.json 2> $F/bench_corridor.err; echo "corridor rc=$?"
timeout 1500 python bench.py --config obstacles --steps 20 --warmup 3 > $F/bench_obstacles.json 2> $F/bench_obstacles.err; echo "obstacles rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > $F/ref_plaza.json 2> $F/ref_plaza.err; echo "ref rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $F/launches.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 1 > $F/ncu_launch.log 2>&1; echo "launches rc=$?"
ls -la $F
