# full GPU check: the whole -m gpu suite, smoke(), c3 / c2 bench lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out; T=${TAG:-full}
timeout 2400 python -m pytest tests -m gpu -q -rf ${PYARGS} 2>&1 | tail -25 > $O/${T}_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${T}_smoke.txt 2>&1
for c in ${CONFIGS:-c3 c2}; do
  timeout 600 python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/${T}_bench_$c.json 2> $O/${T}_bench_$c.err
done
tail -3 $O/${T}_tests.txt; tail -1 $O/${T}_smoke.txt
