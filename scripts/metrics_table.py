"""Per-kernel duration / DRAM bytes / GB/s / tensor-pipe % from ncu --metrics
CSV logs (scripts/r02_prof1.sh: one log per one_conv.py call with reps = 2;
the second call of each kernel is reported -- the first one also pays the
filter packing and first-touch costs).

  python scripts/metrics_table.py gpurun_out/r02_m_*.csv > profiles/r02_kernel_metrics.txt
"""
import csv
import io
import os
import sys

HBM = 6555.2  # GB/s, MEASURED_PEAKS.json hbm_gbs (copy bandwidth, read + write)


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(text[start:])))
    by = {}
    order = []
    for r in rows:
        key = (r["ID"], r["Kernel Name"])
        if key not in by:
            by[key] = {}
            order.append(key)
        try:
            v = float(r["Metric Value"].replace(",", ""))
        except ValueError:
            continue
        # ncu scales units per row: normalise to ns and bytes
        v *= {"ns": 1, "nsecond": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6, "byte": 1,
              "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "%": 1}.get(r.get("Metric Unit", ""), 1)
        by[key][r["Metric Name"]] = v
    return [(k[1], by[k]) for k in order]


def short(name):
    name = name.split("(")[0]
    for pre in ("ucudnn::", "(anonymous namespace)::", "<unnamed>::"):
        name = name.replace(pre, "")
    return name[:40]


def main():
    print(f"{'call (layer op algo batch)':30s} {'kernel':40s} {'us':>9s} {'DRAM MB':>9s} {'GB/s':>8s} "
          f"{'of HBM':>7s} {'tensor%':>8s}")
    for path in sys.argv[1:]:
        tag = os.path.basename(path)[len("r02_m_"):-4]
        ls = launches(path)
        # second occurrence of each kernel name (reps = 2)
        seen, picked = {}, []
        for name, m in ls:
            seen[name] = seen.get(name, 0) + 1
            if seen[name] == 2:
                picked.append((name, m))
        if not picked:
            picked = ls
        for name, m in picked:
            if name.startswith("void at::"):
                continue  # torch's input initialisation
            us = m.get("gpu__time_duration.sum", 0) / 1e3
            mb = (m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)) / 1e6
            gbs = mb / us * 1e3 if us else 0.0
            tp = m.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0)
            print(f"{tag:30s} {short(name):40s} {us:9.1f} {mb:9.1f} {gbs:8.0f} {gbs / HBM:7.2f} {tp:8.1f}")


if __name__ == "__main__":
    main()
