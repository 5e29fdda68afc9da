"""Stall-reason totals and hottest instructions of one kernel's ncu SASS
source page (ncu -i rep --page source --csv --print-source=sass).

    python tools/stall_breakdown.py sass.csv [top]
"""
import csv
import sys


def main(path, top=25):
    rows = list(csv.reader(open(path)))
    h = rows[1]
    idx = {k: i for i, k in enumerate(h)}
    stall_cols = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
    tot = {k: 0 for k in stall_cols}
    allsum = 0
    body = []
    for r in rows[2:]:
        if len(r) != len(h):
            continue
        s = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
        allsum += s
        for k in stall_cols:
            tot[k] += int(r[idx[k]] or 0)
        body.append((s, r[idx["Address"]], r[idx["Source"]].strip(),
                     {k: int(r[idx[k]] or 0) for k in stall_cols}))
    print(f"total samples {allsum}")
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        if v:
            print(f"  {k:26s} {v:9d} {100.0 * v / allsum:6.2f} %")
    print("hottest instructions:")
    for s, a, src, st in sorted(body, key=lambda b: -b[0])[: int(top)]:
        main_r = sorted(st.items(), key=lambda kv: -kv[1])[:2]
        print(f"  {s:7d} {a[-5:]} {src[:48]:48s} " + " ".join(f"{k[6:]}={v}" for k, v in main_r))


if __name__ == "__main__":
    main(*sys.argv[1:])
