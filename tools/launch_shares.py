"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) into
per-kernel launch counts and time shares."""
import csv
import re
import sys
from collections import defaultdict


def main(path, header=""):
    rows = []
    with open(path) as fh:
        lines = [ln for ln in fh if ln.startswith('"')]
    for r in csv.DictReader(lines):
        if r["Metric Name"] == "gpu__time_duration.sum":
            name = re.sub(r"\(.*", "", r["Kernel Name"]).split("::")[-1]
            name = re.sub(r"<.*", "", name).replace("void ", "")
            rows.append((name, float(r["Metric Value"])))
    tot = sum(t for _, t in rows)
    agg = defaultdict(lambda: [0, 0.0])
    for n, t in rows:
        agg[n][0] += 1
        agg[n][1] += t
    if header:
        print(header)
    print(f"{len(rows)} launches, {tot / 1e6:.3f} ms total")
    for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:32s} launches={c:5d} share={t / tot:.3f} mean_us={t / c / 1e3:9.2f}")


if __name__ == "__main__":
    main(sys.argv[1], " ".join(sys.argv[2:]))
