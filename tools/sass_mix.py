"""Per-opcode executed-instruction mix and top stall lines from an ncu
source-page export (ncu -i R --page source --csv --print-source=sass).

    python tools/sass_mix.py export.csv [nodes]
"""
import collections
import csv
import sys


def main(path, nodes=None):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
    istall = hdr.index("Warp Stall Sampling (All Samples)")
    mix = collections.Counter()
    stalls = []
    total = 0
    for r in rows[2:]:
        if len(r) <= ia or not r[ia].isdigit():
            continue
        n = int(r[ia])
        op = r[isrc].strip().split()
        if not op:
            continue
        k = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        k = k.split(".")[0]
        mix[k] += n
        total += n
        stalls.append((int(r[istall] or 0), r[isrc].strip()[:70], n))
    print(f"total warp-instructions {total:.4e}" + (f"  per node (thread-inst) {32 * total / nodes:.1f}" if nodes else ""))
    for k, v in mix.most_common(25):
        print(f"  {k:10s} {v:.4e}  {100 * v / total:5.1f} %" + (f"  {32 * v / nodes:6.1f}/node" if nodes else ""))
    print("top stall samples:")
    for s, src, n in sorted(stalls, reverse=True)[:15]:
        print(f"  {s:7d}  {src}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else None)
