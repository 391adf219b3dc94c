cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
for cfg in "200 1" "100 2" "70 3" "150 1" "100 1"; do set -- $cfg; echo "RING_KB=$1 PER_SM=$2"; HSD_GEMM_RING_KB=$1 HSD_GEMM_CTAS_PER_SM=$2 python scripts/gemm_bench.py | tail -1; done
