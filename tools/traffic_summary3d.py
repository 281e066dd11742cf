"""Per-kernel-family DRAM traffic of one steady-state 3D (c3) Uzawa iteration
from an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum; serialised, cold-cache replay).  The last complete
iteration (it starts with the M u pass in front of the r1 residual kernel) is
used.  Writes JSON with measured DRAM bytes and the algorithmic bytes per
launch of each family (slab = 8 N n bytes)."""
import collections
import csv
import json
import re
import sys

N, n = 512, 63 ** 3
SLAB = 8.0 * N * n


def family(name):
    if "kz_r1" in name:
        return "timeop_r1"
    if "kz_z" in name:
        return "timeop_z"
    if "kz_apply" in name or "kc3_apply" in name:
        return "mass_or_aref"
    if "k_dst_reg<1" in name or "k_dst_fft<1" in name:
        return "dst_inverse_transpose"
    if "k_dst_reg<0" in name or "k_dst_fft<0" in name:
        return "dst_inverse"
    if "kc3_pre" in name:
        return "mg_pre_fine" if re.search(r", 6>", name) else "mg_pre_coarse"
    if "kc3_post" in name:
        return "mg_post_fine" if re.search(r", 6>", name) else "mg_post_coarse"
    if "k_reduce" in name:
        return "reduce"
    return re.sub(r"<.*", "", name)


# algorithmic bytes per launch in slabs
ALG = {"mg_pre_fine": 1.125, "mg_post_fine": (3.125 + 2.125 + 3.125) / 3, "dst_inverse_transpose": 2.0,
       "dst_inverse": 3.0, "timeop_r1": 4.0, "timeop_z": 5.0, "mass_or_aref": 2.0}


def main(path, out):
    lines = [l for l in open(path) if l.startswith('"')]
    launches = collections.OrderedDict()
    for r in csv.DictReader(lines):
        key = (int(r["ID"]), r["Kernel Name"])
        launches.setdefault(key, {})[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    seq = [(k[1], v) for k, v in launches.items()]
    starts = [i - 1 for i, (nm, v) in enumerate(seq) if "kz_r1" in nm]
    a, b = starts[-2], starts[-1]
    fam = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for nm, v in seq[a:b]:
        f = family(nm)
        fam[f][0] += 1
        fam[f][1] += v.get("dram__bytes_read.sum", 0) + v.get("dram__bytes_write.sum", 0)
        fam[f][2] += v.get("gpu__time_duration.sum", 0) / 1e6
    tot = sum(x[2] for x in fam.values())
    res = {"source": path, "note": "ncu serialised replay, one steady-state c3 iteration "
           "(N = 512, n = 63^3; slab = %.4g bytes)" % SLAB,
           "iteration_ms_serialised": tot,
           "iteration_dram_bytes": sum(x[1] for x in fam.values()),
           "kernels": {k: {"launches": c, "dram_bytes_per_launch": by / c,
                           "algorithmic_bytes_per_launch": ALG[k] * SLAB if k in ALG else None,
                           "traffic_over_algorithmic": (by / c) / (ALG[k] * SLAB) if k in ALG else None,
                           "ms_per_launch": ms / c, "share": ms / tot}
                       for k, (c, by, ms) in sorted(fam.items(), key=lambda kv: -kv[1][2])}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
