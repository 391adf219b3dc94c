cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m paper_2602_21224_b200.build >/dev/null
M="gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sectors_srcunit_tex.sum,l1tex__m_xbar2l1tex_read_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__block_size,launch__cluster_dim_x,launch__cluster_dim_y,smsp__cycles_active.avg,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__throughput.avg.pct_of_peak_sustained_elapsed"
ncu --metrics $M --clock-control none --csv python scripts/gemm_one.py 2080 6144 4096 > gpurun_out/ncu_gemm_qkv.csv 2>&1
ncu --metrics $M --clock-control none --csv python scripts/gemm_one.py 2080 4096 14336 > gpurun_out/ncu_gemm_down.csv 2>&1
