mkdir -p gpurun_out
python tools/traffic_capture.py plaza > gpurun_out/traffic.log 2>&1
cp profiles/plan_kernel_ncu.json gpurun_out/plan_kernel_ncu.json
timeout 900 python bench.py > gpurun_out/bench_plaza.json 2> gpurun_out/bench_plaza.err
timeout 900 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_plaza20.json 2> gpurun_out/bench_plaza20.err
for v in 1 2 3 4 5; do
  timeout 600 python bench.py --config room --v $v > gpurun_out/bench_room_v$v.json 2> gpurun_out/bench_room_v$v.err
done
timeout 600 python bench.py --config ring > gpurun_out/bench_ring.json 2> gpurun_out/bench_ring.err
timeout 600 python bench.py --config corridor > gpurun_out/bench_corridor.json 2> gpurun_out/bench_corridor.err
timeout 1500 python bench.py --config obstacles --steps 20 --warmup 3 > gpurun_out/bench_obstacles.json 2> gpurun_out/bench_obstacles.err
timeout 1500 python bench.py --capacity --no-cpu-baseline --steps 20 --warmup 3 > gpurun_out/bench_capacity.json 2> gpurun_out/bench_capacity.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/ref_plaza.json 2> gpurun_out/ref_plaza.err
ls -la gpurun_out
