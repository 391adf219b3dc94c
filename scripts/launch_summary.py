"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel
for one speculative step (between consecutive fresh tree_kernel launches)."""
import csv, collections, re, sys

def load(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if 'Kernel Name' in r][0]
    h = rows[hi]
    ki, vi = h.index('Kernel Name'), h.index('Metric Value')
    out = []
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        m = re.search(r'([A-Za-z_0-9]+_kernel|[A-Za-z_0-9]+kernel)', r[ki])
        out.append((m.group(1) if m else r[ki][:40], float(r[vi].replace(',', ''))))
    return out

def step_slice(names, which=1):
    tk = [i for i, (n, _) in enumerate(names) if n == 'tree_kernel']
    # tree_kernel launches come in (fresh, resample) pairs per step; a capture of
    # exactly one step (scripts/profile_step.py --stage step) is taken whole
    if len(tk) <= 2:
        return names
    return names[tk[2 * which]:tk[2 * which + 2]]

if __name__ == '__main__':
    names = load(sys.argv[1])
    which = int(sys.argv[2]) if len(sys.argv) > 2 else 1
    step = step_slice(names, which)
    agg = collections.defaultdict(lambda: [0, 0.0])
    for n, v in step:
        agg[n][0] += 1; agg[n][1] += v
    tot = sum(v for _, v in step)
    print(f"launches per step {len(step)}  total {tot/1e3:.1f} us (serialised, cold-cache)")
    for k, (c, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:40s} {c:5d} {v/1e3:10.1f} us {100*v/tot:5.1f}%  avg {v/c/1e3:8.2f} us")
