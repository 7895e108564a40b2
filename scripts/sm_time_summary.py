"""Per-kernel SM-time of a frame, from an ncu launch list taken with
    --metrics gpu__time_duration.sum,sm__cycles_active.sum,sm__warps_active.sum
Under concurrent streams a kernel costs the GPU roughly the warp slots it holds,
not its serialised duration (a 10-warp latency-bound chain takes 20 us alone
but leaves the other 9 000 warp slots to other streams). Columns, per frame:
  dur_us      serialised duration (ncu, cold)
  sm_cyc_k    SM-active cycles / 148 SMs, thousands (SMs with >= 1 resident warp)
  warp_cyc_k  warp-slot cycles / (148 SMs x 64 slots), thousands: the
              full-occupancy equivalent (1k cycles ~ 0.5 us at 1.9 GHz)
Usage: python scripts/sm_time_summary.py launches.csv [frames]"""
import collections
import csv
import sys


def summarize(path, frames=1, sms=148, slots=64):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    idi = hdr.index("ID")
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        per[r[idi]][r[mi]] = (float(r[vi].replace(",", "")), r[ui])
        names[r[idi]] = r[ki].split("(")[0].split("::")[-1]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
    for lid, m in per.items():
        dur = m["gpu__time_duration.sum"]
        dus = dur[0] * scale.get(dur[1], 1.0)
        cyc = m.get("sm__cycles_active.sum", (0.0, ""))[0]
        warps = m.get("sm__warps_active.sum", (0.0, ""))[0]
        a = agg[names[lid]]
        a[0] += 1
        a[1] += dus
        if dus > 0:
            a[2] += cyc / sms  # SM-cycles per SM
            a[3] += warps / (sms * slots)
    out = ["%-26s %6s %10s %10s %10s" % ("kernel", "launch", "dur_us", "sm_cyc_k", "warp_cyc_k")]
    tot = [0.0, 0.0, 0.0]
    for k, (n, d, c, w) in sorted(agg.items(), key=lambda x: -x[1][3]):
        out.append("%-26s %6d %10.1f %10.1f %10.1f" % (k, n, d / frames, c / frames / 1e3, w / frames / 1e3))
        tot[0] += d / frames
        tot[1] += c / frames / 1e3
        tot[2] += w / frames / 1e3
    out.append("%-26s %6s %10.1f %10.1f %10.1f" % ("TOTAL per frame", "", *tot))
    return "\n".join(out)


if __name__ == "__main__":
    print(summarize(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 1))
