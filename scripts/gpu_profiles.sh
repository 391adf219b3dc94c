# ncu evidence for profiles/ (one GPU; never a multi-rank command)
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 1 --no-profile --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv --log-file gpurun_out/r01_launches_c2.csv $B > gpurun_out/r01_ncu_launch.log 2>&1
B1="python bench.py --steps 1 --warmup 1 --no-profile --no-cpu-baseline"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 160 -c 4 -o gpurun_out/r01_gemm_c2 $B1 > gpurun_out/r01_ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attention_tc_kernel -s 39 -c 1 -o gpurun_out/r01_attn_c2 $B1 > gpurun_out/r01_ncu_attn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tree_kernel -s 0 -c 2 -o gpurun_out/r01_tree_c2 $B1 > gpurun_out/r01_ncu_tree.log 2>&1
ls -la gpurun_out | tail -8
