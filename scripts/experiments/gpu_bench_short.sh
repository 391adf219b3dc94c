cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline "$@" > /tmp/bench.json 2>/tmp/bench.err
tail -3 /tmp/bench.err
python - <<'PY'
import json
d = json.loads(open('/tmp/bench.json').read().strip().splitlines()[-1])
print(d['config']['workload'], d['ms_per_step'], 'tok/s', d['value'], 'roof', d['roofline']['kernel'], d['roofline']['frac'], d['roofline']['achieved'], '|', ' '.join(f"{k}={v}" for k, v in d['profile_ms_per_step'].items()))
PY
