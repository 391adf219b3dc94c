# A/B sweep of the L2 weight prefetch (HSD_L2PF_MB cap, HSD_L2PF_WHERE windows, HSD_L2PF_LATE) on c2.
cd $GRAFT_REPO_ROOT
python -m paper_2602_21224_b200.build > /dev/null
B="python bench.py --no-cpu-baseline --no-profile --no-e2e --no-planted --config c2 --steps 30 --warmup 5"
run() { r=$(env "$@" timeout 600 $B 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'])"); echo "$* ms/step=$r"; }
run HSD_L2PF_MB=0
for late in 0 1; do for w in 2 4 16 32; do run HSD_L2PF_MB=48 HSD_L2PF_WHERE=$w HSD_L2PF_LATE=$late; done; done
run HSD_L2PF_MB=8 HSD_L2PF_WHERE=2 HSD_L2PF_LATE=1
run HSD_L2PF_MB=0
