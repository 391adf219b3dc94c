cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
nproc; free -g | head -2
(time timeout 600 python bench.py --impl reference --steps 1 --warmup 0 2>&1 | tail -2) 2>&1 | tail -6
timeout 900 python bench.py --config c3 --steps 3 --warmup 2 --no-cpu-baseline 2>&1 | tail -3
