"""Per-kernel-family DRAM traffic of one steady-state c2 Uzawa iteration from
an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum, serialised cold-cache replay).  The last complete
iteration (first launch = the r1 residual kernel) is used.  Writes JSON with
bytes per launch and ms per launch for each family bench.py reports."""
import collections
import csv
import json
import re
import sys


def family(name, grid):
    if "k_band_timeop2<0" in name:
        return "timeop_r1"
    if "k_band_timeop2<1" in name:
        return "timeop_z"
    if "k_band_apply" in name:
        return "aref"
    if "k_dst_reg<1" in name or "k_dst_fft<1" in name:
        return "dst_inverse_transpose"
    if "k_dst_reg<0" in name or "k_dst_fft<0" in name:
        return "dst_inverse"
    if "k_band_pre2" in name:
        return "mg_pre_fine" if ", 128," in name or "<2, 128" in name or "<1, 128" in name else "mg_pre_coarse"
    if "k_band_post2" in name:
        return "mg_post_fine" if re.search(r", 128, 8(, [01]){0,2}>", name) else "mg_post_coarse"
    if "k_mg_tail" in name:
        return "mg_tail"
    if "k_reduce" in name:
        return "reduce"
    return re.sub(r"<.*", "", name)


def main(path, out):
    lines = [l for l in open(path) if l.startswith('"')]
    launches = collections.OrderedDict()
    for r in csv.DictReader(lines):
        key = (int(r["ID"]), r["Kernel Name"], r["Grid Size"])
        launches.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    seq = [(k[1], k[2], v) for k, v in launches.items()]
    starts = [i for i, (n, g, v) in enumerate(seq) if "k_band_timeop2<0" in n]
    a, b = starts[-2], starts[-1]
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for n, g, v in seq[a:b]:
        f = family(n, g)
        fam[f][0] += 1
        fam[f][1] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        fam[f][2] += v.get("gpu__time_duration.sum", 0) / 1e6
    tot = sum(x[2] for x in fam.values())
    res = {"source": path, "note": "ncu serialised replay, one steady-state c2 iteration",
           "iteration_ms_serialised": tot,
           "kernels": {k: {"launches": c, "dram_bytes_per_launch": by / c, "ms_per_launch": ms / c,
                           "share": ms / tot}
                       for k, (c, by, ms) in sorted(fam.items(), key=lambda kv: -kv[1][2])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
