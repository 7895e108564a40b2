"""Summarises an ncu --metrics gpu__time_duration.sum --csv launch list:
per-kernel launch count, total device time and share."""
import collections
import csv
import sys


def summarize(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for r in rows[1:]:
        name = r[ki].split("(")[0].split("::")[-1]
        agg[name][0] += 1
        agg[name][1] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
    tot = sum(v[1] for v in agg.values())
    out = ["%-26s %7s %12s %7s" % ("kernel", "launches", "total_us", "share")]
    for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
        out.append("%-26s %7d %12.1f %6.1f%%" % (k, n, t, 100 * t / tot))
    out.append("%-26s %7d %12.1f" % ("TOTAL", sum(v[0] for v in agg.values()), tot))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1]))
