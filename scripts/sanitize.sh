# compute-sanitizer over the library's kernels (one GPU): memcheck, racecheck,
# synccheck, initcheck on the c1 fp32-verify path and a small bf16 tcgen05 config.
# Logs -> gpurun_out/sanitize_<tool>_<mode>.log (summaries copied to profiles/ by hand).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
export HSD_STAGE_GRAPHS=0          # eager launches: every kernel visible to the tools
for mode in fp32 bf16; do
  for tool in memcheck racecheck synccheck initcheck; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 30 --error-exitcode 0 \
      python scripts/sanitize_run.py $mode > gpurun_out/sanitize_${tool}_${mode}.log 2>&1
    echo "$mode $tool: $(tail -1 gpurun_out/sanitize_${tool}_${mode}.log)"
  done
done
