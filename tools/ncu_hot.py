"""Summarise an `ncu --page source --csv --print-source sass` export: the
hottest SASS instructions (by executed count and stall samples) and the
executed-instruction mix.  Usage: python tools/ncu_hot.py file.csv [top]"""
import collections
import csv
import sys


def main():
    path = sys.argv[1]
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    rows = list(csv.reader(open(path)))
    h = rows[1]
    iA, iS, iX, iW = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    recs = []
    for r in rows[2:]:
        if len(r) <= iX:
            continue
        try:
            recs.append((r[iA], r[iS].strip(), int(r[iX] or 0), int(r[iW] or 0)))
        except ValueError:
            continue
    tot = sum(x[2] for x in recs)
    st = sum(x[3] for x in recs)
    print(f"executed warp-instructions {tot}  stall samples {st}")
    mix = collections.Counter()
    for a, s, x, w in recs:
        mix[s.split()[0] if not s.startswith("@") else s.split()[1]] += x
    print("mix:", ", ".join(f"{k} {v / tot:.1%}" for k, v in mix.most_common(25)))
    print("hottest by stall samples:")
    for a, s, x, w in sorted(recs, key=lambda r: -r[3])[:top]:
        print(f"  {w:7d} {x:11d}  {a[-5:]}  {s[:90]}")


if __name__ == "__main__":
    main()
