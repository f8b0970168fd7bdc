python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python tools/debug_rounds.py --warm 200 | head -8
python tools/profile_step.py --warm 200 --steps 2 --mode run --each 2>&1 | tail -3 | head -2
python tools/profile_step.py --warm 20 --steps 2 --mode run --each 2>&1 | tail -3 | head -2
python bench.py --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), d['phases_ms'], 'rounds/step', d['motion_rounds_per_step'])"
