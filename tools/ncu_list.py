"""Compact per-launch table from an ncu --metrics ... --csv launch list."""
import collections
import csv
import re
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
k = collections.OrderedDict()
for r in csv.DictReader(lines):
    name = re.sub(r"\(.*", "", r["Kernel Name"]).replace("void ", "").split("::")[-1][:28]
    k.setdefault((r["ID"], name, r["Grid Size"]), {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
for (i, name, grid), v in k.items():
    t = v.get("gpu__time_duration.sum", 0) / 1e3
    rd = v.get("dram__bytes_read.sum", 0)
    wr = v.get("dram__bytes_write.sum", 0)
    print(f"{name:28s} {grid:14s} {t:8.1f}us rd={rd/1e6:8.1f}MB wr={wr/1e6:8.1f}MB "
          f"{(rd+wr)/max(t,1e-9)/1e3:7.1f}GB/s inst={v.get('sm__inst_executed.sum',0)/1e6:7.1f}M "
          f"issue={v.get('smsp__issue_active.avg.pct_of_peak_sustained_active',0):5.1f}% "
          f"l1={v.get('l1tex__throughput.avg.pct_of_peak_sustained_elapsed',0):5.1f}% "
          f"warps={v.get('sm__warps_active.avg.pct_of_peak_sustained_active',0):5.1f}%")
