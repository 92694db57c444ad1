"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares: python scripts/launch_summary.py launches.csv"""
import csv
import re
import sys
from collections import defaultdict


def main(path):
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        short = re.sub(r"\(.*", "", name)
        short = re.sub(r"^void ", "", short)
        m = re.match(r"adaptra::gemm_tc_kernel<(.*?)>", short)
        if m:
            short = f"gemm_tc_kernel<{m.group(1)}>"
        val = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        scale = {"ns": 1.0, "usecond": 1e3, "us": 1e3, "msecond": 1e6, "ms": 1e6, "nsecond": 1.0}.get(unit, 1.0)
        rows.append((short, val * scale))
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for k, v in rows:
        tot[k] += v
        cnt[k] += 1
    total = sum(tot.values())
    print(f"launches {len(rows)}  total {total / 1e6:.3f} ms (cold-cache, serialised)")
    fam = defaultdict(float)
    for k, v in tot.items():
        fam["gemm_tc (all)" if k.startswith("gemm_tc") else k] += v
    print("\nby family:")
    for k, v in sorted(fam.items(), key=lambda x: -x[1]):
        print(f"  {v / total * 100:6.2f}%  {v / 1e3:10.1f} us  {k}")
    print("\nby kernel:")
    for k, v in sorted(tot.items(), key=lambda x: -x[1])[:25]:
        print(f"  {v / total * 100:6.2f}%  {v / 1e3:10.1f} us  n={cnt[k]:6d}  avg {v / cnt[k] / 1e3:8.2f} us  {k}")


if __name__ == "__main__":
    main(sys.argv[1])
