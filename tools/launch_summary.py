"""Per-kernel share of an `ncu --metrics gpu__time_duration.sum --csv` launch list.

usage: python tools/launch_summary.py profiles/<launches>.csv [first_launch_id]
"""
import collections
import csv
import sys


def short(name):
    base = name.split("(")[0].replace("void ", "")
    return base.split("<")[0].split("::")[-1] or base


def main():
    path = sys.argv[1]
    first = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    t, n = collections.Counter(), collections.Counter()
    for r in csv.reader(open(path)):
        if len(r) < 15 or not r[0].isdigit() or int(r[0]) < first:
            continue
        k = short(r[4])
        t[k] += float(r[14].replace(",", ""))
        n[k] += 1
    tot = sum(t.values())
    for k, v in t.most_common(25):
        print(f"{k:36s} {n[k]:5d} launches {v / 1e6:9.3f} ms {100 * v / tot:5.1f}%")
    print(f"total {tot / 1e6:.3f} ms over {sum(n.values())} launches")


if __name__ == "__main__":
    main()
