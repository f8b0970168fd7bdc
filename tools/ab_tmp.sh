python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/debug_rounds.py --warm 300 | head -6
for w in 20 200 350; do python tools/profile_step.py --warm $w --steps 1 --mode run --each 2>&1 | tail -2 | head -1 | cut -c1-300; done
python bench.py --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), d['phases_ms'], 'rounds/step', d['motion_rounds_per_step'])"
