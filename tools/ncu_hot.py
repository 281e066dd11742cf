"""Top SASS lines by warp-stall samples from an ncu --page source --csv
--print-source sass export (first kernel in the file, or the one named)."""
import csv
import sys


def main(path, top=40, which=None):
    rows = list(csv.reader(open(path)))
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = {"name": r[1], "rows": []}
            blocks.append(cur)
        elif r and r[0] == "Address":
            cur["hdr"] = r
        elif cur is not None and "hdr" in cur and len(r) == len(cur["hdr"]):
            cur["rows"].append(dict(zip(cur["hdr"], r)))
    for b in blocks:
        if which and which not in b["name"]:
            continue
        tot = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in b["rows"])
        print(f"== {b['name']}  total samples {tot}")
        rs = sorted(b["rows"], key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))
        for d in rs[:top]:
            print(f"{d['Address'][-5:]} {int(d['Warp Stall Sampling (All Samples)']):6d} "
                  f"{d['Source'].strip()[:70]:70s} wfS={d.get('L1 Wavefronts Shared','')} "
                  f"ideal={d.get('L1 Wavefronts Shared Ideal','')} L2sec={d.get('L2 Theoretical Sectors Global','')}")
        break


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40,
         sys.argv[3] if len(sys.argv) > 3 else None)
