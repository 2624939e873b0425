"""Per-region warp-stall breakdown from an `ncu --page source --csv
--print-source sass` dump (debug helper: python scripts/stall_summary.py dump.csv [lo_addr hi_addr])."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h, data = rows[1], rows[2:]
ia = h.index("Address")
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
lo = int(sys.argv[2], 16) if len(sys.argv) > 3 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 64
tot = collections.Counter()
for r in data:
    a = int(r[ia], 16) & 0xFFFFF
    if lo <= a < hi:
        for c in cols:
            tot[c] += float(r[h.index(c)] or 0)
s = sum(tot.values())
for c, v in tot.most_common(10):
    print(f"{c:28s} {v:8.0f} {100 * v / max(s, 1):5.1f}%")
