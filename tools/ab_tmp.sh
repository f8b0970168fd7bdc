run() { python bench.py --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$1', 'value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), d['phases_ms'])"; for w in 20 200; do python tools/debug_rounds.py --warm $w | grep seed_ns; done; }
FP_SEED_STATIC=0 run dyn
FP_SEED_STATIC=1 run static
