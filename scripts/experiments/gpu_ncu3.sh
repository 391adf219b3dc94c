cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_tc_kernel -s 60 -c 2 -o gpurun_out/prof_attn2 python bench.py --steps 1 --warmup 1 --no-profile --no-cpu-baseline > gpurun_out/ncu_attn2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 1 -c 1 -o gpurun_out/prof_tree2 python bench.py --steps 1 --warmup 1 --no-profile --no-cpu-baseline > gpurun_out/ncu_tree2.log 2>&1
ls gpurun_out
