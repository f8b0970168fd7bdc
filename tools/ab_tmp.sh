python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for w in 100 200 300; do python tools/debug_rounds.py --warm $w | grep -i "seed_ns\|round  \(0\|1\|5\|10\|20\|30\) "; done
python bench.py --no-cpu-baseline --e2e-steps 20 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('value %.4g ms/step %.3f' % (d['value'], d['ms_per_step']), d['phases_ms'], 'rounds/step', d['motion_rounds_per_step'])"
