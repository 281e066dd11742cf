"""Opcode histogram (executed warp instructions) of the first kernel in an
ncu --page source --csv --print-source sass export."""
import collections
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "Address":
            hdr = r
            continue
        if r and r[0] == "Kernel Name" and data:
            break
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    cnt, tot = collections.Counter(), 0
    for d in data:
        op = d["Source"].strip().split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        n = int(d["Instructions Executed"] or 0)
        cnt[o.split(".")[0]] += n
        tot += n
    print(f"total warp instructions {tot}")
    for o, n in cnt.most_common(top):
        print(f"  {o:10s} {n:12d} {n / tot:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
