# Per-kernel device time of the fused attention at the bench shape (mbs 16):
# ncu launch list (gpu__time_duration, no clock control) of a few attn_bench calls.
G=${WP_BW_GROUP:-32}
WP_BW_GROUP=$G timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  python -c "import sys; sys.path.insert(0, 'tools'); import attn_bench; attn_bench.main(mbs=16, n=3, causal=int(__import__(\"os\").environ.get(\"CAUSAL\", \"1\")))" 2>/dev/null \
  | python -c "
import csv, sys, collections
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
h = rows[0]; k = h.index('Kernel Name'); v = h.index('Metric Value'); u = h.index('Metric Unit')
acc = collections.defaultdict(list)
for r in rows[1:]:
    t = float(r[v].replace(',', '')) * (1e-3 if r[u] in ('nsecond', 'ns') else 1.0)
    acc[r[k].split('(')[0].split('::')[-1][:60]].append(t)
for name, ts in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
    print(f'{name:60s} n={len(ts):3d} min={min(ts):8.1f} us  median={sorted(ts)[len(ts)//2]:8.1f} us')
"
