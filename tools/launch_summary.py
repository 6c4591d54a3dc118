"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list by kernel name.

    python tools/launch_summary.py gpurun_out/x.csv [--last N] [--detail REGEX]
"""
import collections
import csv
import re
import sys


def load(f):
    rows = list(csv.reader(open(f)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr) and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            v = float(r[hdr.index("Metric Value")].replace(",", ""))
            unit = r[hdr.index("Metric Unit")]
            v *= {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(unit, 1.0)
            grid = r[hdr.index("Grid Size")] if "Grid Size" in hdr else ""
            out.append((r[hdr.index("Kernel Name")], v, grid))
    return out


def main():
    f = sys.argv[1]
    L = load(f)
    if "--last" in sys.argv:
        L = L[-int(sys.argv[sys.argv.index("--last") + 1]):]
    c = collections.defaultdict(lambda: [0, 0.0])
    for n, v, _ in L:
        k = re.sub(r"\(.*", "", n)[:80]
        c[k][0] += 1
        c[k][1] += v
    tot = sum(v for _, v, _ in L)
    print(f"{len(L)} launches, {tot / 1e3:.2f} ms (serialised, cold-cache)\n")
    print("| kernel | launches | ms | share |\n|---|---|---|---|")
    for k, (n, v) in sorted(c.items(), key=lambda x: -x[1][1]):
        if v / tot >= 0.002:
            print(f"| `{k}` | {n} | {v / 1e3:.2f} | {100 * v / tot:.1f}% |")
    if "--detail" in sys.argv:
        pat = re.compile(sys.argv[sys.argv.index("--detail") + 1])
        print()
        for n, v, g in L:
            if pat.search(n):
                print(f"{v:9.1f} us  grid {g}  {re.sub(r'[(].*', '', n)[:60]}")


if __name__ == "__main__":
    main()
