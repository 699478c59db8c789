"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list by kernel."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6}
for r in rows[1:]:
    name = r[ki].split("(")[0].replace("hpbj::<unnamed>::", "").replace("void ", "")[:70]
    agg[name][0] += 1
    agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
tot = sum(t for _, t in agg.values())
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1])[: int(sys.argv[2]) if len(sys.argv) > 2 else 20]:
    print(f"  {k:70s} {n:6d} {t:12.1f} us {t / n:10.2f} us/launch {100 * t / tot:5.1f}%")
print(f"  total {tot:.1f} us")
