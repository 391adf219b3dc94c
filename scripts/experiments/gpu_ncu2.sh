cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 1 --no-profile --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_tc -s 200 -c 3 -o gpurun_out/prof_attn python bench.py --steps 1 --warmup 1 --no-profile --no-cpu-baseline > gpurun_out/ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 2 -c 1 -o gpurun_out/prof_tree python bench.py --steps 1 --warmup 1 --no-profile --no-cpu-baseline > gpurun_out/ncu_tree.log 2>&1
tail -2 gpurun_out/*.log
