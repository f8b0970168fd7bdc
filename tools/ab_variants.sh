for v in base s4h32 s4h36 base s4h32 s4h36; do
  cp exp/lib_$v.so paper_0911_2900_b200/libfastped_b200.so; touch paper_0911_2900_b200/libfastped_b200.so
  python bench.py --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', round(d['value']/1e6,1), round(d['e2e']['value']/1e6,1), d['phases_ms'], d['roofline']['plan_ms_start_end'], d['roofline']['frac'])"
done
cp exp/lib_base.so paper_0911_2900_b200/libfastped_b200.so
