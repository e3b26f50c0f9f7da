"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv):
per-kernel launch count, total and mean duration, share of the listed time."""
import collections, csv, sys

rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
K, V, M = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[M] != "gpu__time_duration.sum" or not r[V]:
        continue
    name = r[K].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")
    t = float(r[V].replace(",", ""))
    c, s = agg.get(name, (0, 0.0))
    agg[name] = (c + 1, s + t)
tot = sum(s for _, s in agg.values())
print(f"{'kernel':60s} {'launches':>8s} {'total_us':>10s} {'mean_us':>9s} {'share':>6s}")
for name, (c, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{name[:60]:60s} {c:8d} {s / 1e3:10.1f} {s / c / 1e3:9.2f} {s / tot:6.1%}")
print(f"total listed kernel time {tot / 1e3:.1f} us over {sum(c for c, _ in agg.values())} launches")
