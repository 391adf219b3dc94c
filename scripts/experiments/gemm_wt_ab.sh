# A/B of the pair-GEMM super-tile width, alternating processes (box clocks drift)
cd $GRAFT_REPO_ROOT; python -m paper_2602_21224_b200.build >/dev/null
O=gpurun_out/gab.txt; : > $O
for rep in 1 2; do for wt in 1 2; do
  echo "WT=$wt rep $rep $(HSD_GEMM_WT=$wt python scripts/gemm_vs_cublas.py c3 | tail -1)" >> $O
done; done
for rep in 1 2; do for wt in 1 0; do
  HSD_GEMM_WT=$wt timeout 600 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > gpurun_out/gab_bench_${wt}_$rep.json 2>/dev/null
  echo "bench WT=$wt rep $rep $(python scripts/bench_summary.py gpurun_out/gab_bench_${wt}_$rep.json | head -1)" >> $O
done; done
