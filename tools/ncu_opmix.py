"""Executed-instruction mix by SASS opcode for one kernel of an ncu
--page source --csv --print-source sass export."""
import collections
import sys

from ncu_stalls import blocks, num


def main(path, which, top=25):
    for b in blocks(path):
        if which not in b["name"]:
            continue
        mix = collections.Counter()
        for d in b["rows"]:
            src = d["Source"].strip()
            if src.startswith("@"):
                src = src.split(None, 1)[1] if " " in src else src
            op = src.split()[0] if src else "?"
            mix[op.split(".")[0]] += num(d["Instructions Executed"])
        tot = sum(mix.values())
        print(f"== {b['name'][:90]}  warp instructions {tot:.3g}")
        for op, v in mix.most_common(top):
            print(f"   {op:10s} {v / tot:6.3f}")
        return


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
