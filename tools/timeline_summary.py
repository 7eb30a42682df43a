"""Summarise a tools/qb_timeline.py log: device time per (stream, kernel)."""
import collections
import re
import sys

for f in sys.argv[1:]:
    rows = []
    for line in open(f):
        m = re.match(r"\s*([\d.]+)\s+([\d.]+)\s+(\S+)\s+(.*)", line)
        if m:
            rows.append((float(m.group(1)), float(m.group(2)), m.group(3), m.group(4)))
    agg = collections.defaultdict(lambda: [0, 0.0])
    for s, d, st, name in rows:
        k = name.replace("void ", "").replace("qlra_dev::", "").replace("(anonymous namespace)::", "")
        k = re.sub(r"\(.*", "", k)[:48]
        agg[(st, k)][0] += 1
        agg[(st, k)][1] += d
    print("==", f, "span %.2f ms" % (max(s + d for s, d, _, _ in rows) / 1e3))
    for (st, k), (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
        print(f"  stream {st:>3} {k:48s} n={n:4d} {t / 1000:8.2f} ms")
