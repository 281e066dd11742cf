"""Opcode mix (warp instructions) and stall totals of one kernel block of an
ncu --page source --csv --print-source sass export.  usage: ncu_mix.py file [index|name]"""
import collections
import csv
import sys


def blocks(path):
    out, cur = [], None
    for r in csv.reader(open(path)):
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            out.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(dict(zip(cur["hdr"], r)))
    return out


def main(path, sel=None, points=None):
    bs = blocks(path)
    seen = set()
    for k, b in enumerate(bs):
        if sel is not None and sel != str(k) and sel not in b["name"]:
            continue
        key = (b["name"], len(b["rows"]), sum(float(d["Instructions Executed"] or 0) for d in b["rows"]))
        if key in seen:
            continue
        seen.add(key)
        h = collections.Counter()
        for d in b["rows"]:
            t = d["Source"].strip().split()
            op = t[1] if t[0].startswith("@") else t[0]
            h[op.split(".")[0]] += float(d["Instructions Executed"] or 0)
        tot = sum(h.values())
        print(f"== [{k}] {b['name'][:110]}  warp instr {tot:.4g}" +
              (f"  per point {tot * 32 / float(points):.1f}" if points else ""))
        print("   " + "  ".join(f"{o}={v / tot:.3f}" for o, v in h.most_common(22)))
        cols = [c for c in b["hdr"] if c.startswith("stall_") and "Not Issued" not in c]
        st = {c: sum(float(d[c] or 0) for d in b["rows"]) for c in cols}
        s = sum(st.values()) or 1
        print("   stalls: " + "  ".join(f"{c[6:]}={v / s:.2f}" for c, v in sorted(st.items(), key=lambda x: -x[1]) if v / s >= 0.02))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None, sys.argv[3] if len(sys.argv) > 3 else None)
