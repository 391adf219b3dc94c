cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
python -m paper_2602_21224_b200.build > /dev/null
O=gpurun_out
for i in 1 2; do timeout 300 python bench.py --config c2 --steps 20 --warmup 5 --no-cpu-baseline --no-planted --no-profile > $O/c28_c2_$i.json 2>/dev/null; done
timeout 300 python bench.py --config c5 --batch-per-gpu 2 --steps 5 --warmup 3 --no-cpu-baseline --no-planted --no-profile > $O/c28_c5.json 2>/dev/null
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2 > $O/c28_tests.txt
cat $O/c28_tests.txt
python -c "
import json
for f in ['c28_c2_1','c28_c2_2','c28_c5']:
    d=json.loads(open('$O/'+f+'.json').read().strip().splitlines()[-1]); print(f, d['ms_per_step'], d['value'])
"
