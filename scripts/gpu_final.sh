# end-of-round validation: full -m gpu suite, smoke(), default bench line (c3) + c2 / c4 / c5 lines,
# then the round-2 ncu evidence (scripts/gpu_profiles_r02.sh)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -rf 2>&1 | tail -6 > $O/final_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/final_smoke.txt 2>&1
timeout 900 python bench.py > $O/final_bench_c3.json 2> $O/final_bench_c3.err
timeout 600 python bench.py --config c2 --steps 20 --warmup 5 > $O/final_bench_c2.json 2> $O/final_bench_c2.err
timeout 900 python bench.py --config c4 --steps 5 --warmup 3 --no-cpu-baseline --no-planted > $O/final_bench_c4.json 2> $O/final_bench_c4.err
timeout 900 python bench.py --config c5 --batch-per-gpu 2 --steps 5 --warmup 3 --no-cpu-baseline --no-planted > $O/final_bench_c5.json 2> $O/final_bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/final_ref.json 2> $O/final_ref.err
bash scripts/gpu_profiles_r02.sh > /dev/null 2>&1
cat $O/final_tests.txt; tail -2 $O/final_smoke.txt
