# quick GPU check: selected tests (-k $1) + c3 / c2 bench lines (no cpu baseline / planted leg)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out; T=${TAG:-q}
timeout 1500 python -m pytest tests -m gpu -q -rf -x -k "${1:-tcgen05 or fullsize or attention}" 2>&1 | tail -15 > $O/${T}_tests.txt
for c in ${CONFIGS:-c3 c2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
tail -2 $O/${T}_tests.txt
