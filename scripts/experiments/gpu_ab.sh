cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
HSD_PDL=0 timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=0', d['ms_per_step'], d['profile_ms_per_step'])"
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('PDL=1', d['ms_per_step'], d['roofline'], d['profile_ms_per_step'])"
