# Round-2 closing measurements: every BASELINE config through bench.py, the reference arm,
# the measured capacity, and ncu captures of the step's kernels at plaza step ~200.
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_plaza.json 2> gpurun_out/bench_plaza.err
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_plaza20.json 2> gpurun_out/bench_plaza20.err
for v in 1 2 3 4 5; do
  timeout 600 python bench.py --config room --v $v > gpurun_out/bench_room_v$v.json 2> gpurun_out/bench_room_v$v.err
done
timeout 600 python bench.py --config ring > gpurun_out/bench_ring.json 2> gpurun_out/bench_ring.err
timeout 600 python bench.py --config corridor > gpurun_out/bench_corridor.json 2> gpurun_out/bench_corridor.err
timeout 1500 python bench.py --config obstacles --steps 20 --warmup 3 > gpurun_out/bench_obstacles.json 2> gpurun_out/bench_obstacles.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_plaza.json 2> gpurun_out/ref_plaza.err
ncu --set full --import-source on --clock-control none -k regex:"seed_|bk_|p2_|move_rounds" --launch-skip 2376 --launch-count 12 \
    -o gpurun_out/move_step199 python tools/profile_step.py --warm 198 --steps 2 --mode run > gpurun_out/ncu_move199.log 2>&1
echo "ncu move rc=$?"
timeout 2400 python bench.py --capacity --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_capacity.json 2> gpurun_out/bench_capacity.err
ls -la gpurun_out | tail -30
