"""Instruction mix and hottest SASS lines of one kernel from an ncu report:
    ncu -i REP --page source --csv --print-source sass > src.csv
    python tools/ncu_sass_hot.py src.csv [kernel-substring]"""
import csv
import sys
from collections import Counter


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    want = sys.argv[2] if len(sys.argv) > 2 else None
    blocks, cur = [], None
    for r in rows:
        if r and r[0] == "Kernel Name":
            cur = [r[1], None, []]
            blocks.append(cur)
        elif r and r[0] == "Address" and cur is not None:
            cur[1] = r
        elif cur is not None and cur[1] is not None and len(r) >= len(cur[1]) - 1:
            cur[2].append(r)
    for name, hdr, data in blocks:
        if want and want not in name:
            continue
        ix = hdr.index("Instructions Executed")
        isamp = hdr.index("Warp Stall Sampling (All Samples)")
        isrc = hdr.index("Source")

        def num(v):
            try:
                return int(float(v or 0))
            except ValueError:
                return 0
        tot = sum(num(r[ix]) for r in data) or 1
        ts = sum(num(r[isamp]) for r in data) or 1
        print(name, "warp instr", tot, "samples", ts)
        op, sp = Counter(), Counter()
        for r in data:
            s = r[isrc].strip().split()
            o = s[0] if s else "?"
            if o.startswith("@") and len(s) > 1:
                o = s[1]
            o = o.split(".")[0]
            op[o] += num(r[ix])
            sp[o] += num(r[isamp])
        for o, c in op.most_common(25):
            print(f"  {o:10s} {100 * c / tot:5.1f}% instr  {100 * sp[o] / ts:5.1f}% samples")
        print("  hottest:")
        for r in sorted(data, key=lambda r: -num(r[isamp]))[:25]:
            print("  ", r[isamp], r[ix], r[0][-5:], r[isrc].strip()[:90])


if __name__ == "__main__":
    main()
