# attention timing experiments on c3 (bench line per variant), single-CTA kernel
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out; T=${TAG:-x}
B="python bench.py --config c3 --steps 6 --warmup 3 --no-cpu-baseline --no-planted --no-e2e"
for e in 0 2 4 6; do HSD_ATTN_PAIR=0 HSD_ATTN_EXP=$e timeout 300 $B > $O/${T}_exp$e.json 2>&1; done
HSD_ATTN_PAIR=1 timeout 300 $B > $O/${T}_pair.json 2>&1
