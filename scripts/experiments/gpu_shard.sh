# vocab-sharded lm_head on one GPU (simulated shards) + the full GPU suite
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-e2e --no-planted --steps 20"
for extra in "--config c2" "--config c2 --vocab-shard" "--config c5 --batch 2" "--config c5 --batch 2 --vocab-shard"; do
  timeout 900 $B $extra 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$extra', d['ms_per_step'], d['config']['lm_head'], d['profile_ms_per_step'].get('head_verify'), d['profile_ms_per_step'].get('head_draft'), d['verify_latency_ms'])"
done
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
