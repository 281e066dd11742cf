"""Stall-reason totals per kernel from an ncu --page source --csv --print-source
sass export (columns stall_*), plus shared-memory excess wavefronts."""
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


def num(v):
    try:
        return float(v or 0)
    except ValueError:
        return 0.0


def main(path, which=None):
    for b in blocks(path):
        if which and which not in b["name"]:
            continue
        cols = [h for h in b["hdr"] if h.startswith("stall_") and "Not Issued" not in h]
        tot = {c: sum(num(d[c]) for d in b["rows"]) for c in cols}
        s = sum(tot.values()) or 1
        print(f"== {b['name'][:100]}")
        print("   " + "  ".join(f"{c[6:]}={v / s:.2f}" for c, v in sorted(tot.items(), key=lambda x: -x[1]) if v / s >= 0.01))
        ws = sum(num(d["L1 Wavefronts Shared"]) for d in b["rows"])
        wi = sum(num(d["L1 Wavefronts Shared Ideal"]) for d in b["rows"])
        ins = sum(num(d["Instructions Executed"]) for d in b["rows"])
        print(f"   shared wavefronts {ws:.3g} (ideal {wi:.3g}), warp instructions {ins:.3g}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
