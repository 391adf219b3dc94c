cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
HSD_ATTN_DUAL=1 timeout 300 python -m pytest tests/test_gpu_fullsize_logits.py -q -x -k "c3" > $O/c18_c3logits.txt 2>&1
tail -3 $O/c18_c3logits.txt
HSD_ATTN_DUAL=1 timeout 300 python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --no-planted > $O/c18_bench_c3_dual.json 2> $O/c18_bench_c3_dual.err
HSD_ATTN_DUAL=1 timeout 900 python -m pytest tests -m gpu -q -x -k "tcgen05 or fullsize_logits or bf16" > $O/c18_tests.txt 2>&1
tail -3 $O/c18_tests.txt
