cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv --log-file $O/c21_prefill_c3.csv python scripts/profile_step.py c3 --stage prefill > $O/c21.log 2>&1
timeout 300 python scripts/prefill_time.py c3 > $O/c21_pt.txt 2>&1
tail -2 $O/c21.log; cat $O/c21_pt.txt
