"""Summarise an ncu --csv launch list: per-kernel count and total device time (us)."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h, rows = rows[0], rows[1:]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
agg = collections.defaultdict(lambda: collections.defaultdict(float))
cnt = collections.Counter()
for r in rows:
    name = r[ki].split("(")[0].replace("ucudnn::<unnamed>::", "").replace("void ", "")
    agg[name][r[mi]] += float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        cnt[name] += 1
tot = sum(v.get("gpu__time_duration.sum", 0) for v in agg.values())
for name, v in sorted(agg.items(), key=lambda x: -x[1].get("gpu__time_duration.sum", 0)):
    t = v.get("gpu__time_duration.sum", 0)
    extra = " ".join(f"{k.split('__')[1]}={v[k] / max(cnt[name], 1):.3g}" for k in v if k != "gpu__time_duration.sum")
    print(f"{name:34s} n={cnt[name]:5d} total={t / 1e3:10.1f} us  avg={t / 1e3 / max(cnt[name], 1):8.2f} us  {100 * t / tot:5.1f}%  {extra}")
