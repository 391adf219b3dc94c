cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
export HSD_STAGE_GRAPHS=0
for tool in memcheck initcheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 0 python scripts/sanitize_run.py pair > $O/sanitize_${tool}_pair.log 2>&1
  echo "pair $tool: $(tail -1 $O/sanitize_${tool}_pair.log)"
done
unset HSD_STAGE_GRAPHS
/usr/bin/time -v timeout 900 python bench.py > $O/c23_default.json 2> $O/c23_default.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/c23_ref.json 2> $O/c23_ref.err
tail -c 600 $O/c23_default.json; echo; grep -E "Elapsed|Maximum resident" $O/c23_default.err; tail -c 400 $O/c23_ref.json
