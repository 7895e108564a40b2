"""Per-opcode executed-instruction mix and stall samples of one kernel from an
ncu report's SASS source page: python scripts/ncu_sass_mix.py rep kernel_regex."""
import collections
import csv
import io
import subprocess
import sys


def main(path, kernel, top=32):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", "regex:" + kernel, "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = next(r for r in rows if "Instructions Executed" in r and "Source" in r)
    ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
    st = hdr.index("Warp Stall Sampling (All Samples)")

    def f(x):
        try:
            return float(x.replace(",", "") or 0)
        except ValueError:
            return 0.0

    data = [r for r in rows if len(r) == len(hdr) and r is not hdr]
    tot = sum(f(r[ie]) for r in data)
    op, stall = collections.Counter(), collections.Counter()
    for r in data:
        parts = r[src].split()
        if not parts:
            continue
        o = (parts[1] if parts[0].startswith("@") and len(parts) > 1 else parts[0]).split(".")[0]
        op[o] += f(r[ie])
        stall[o] += f(r[st])
    stot = sum(stall.values()) or 1
    print("warp instructions executed: %.0f" % tot)
    for o, c in op.most_common(top):
        print("%-10s %12.0f %5.1f%%   stall samples %5.1f%%" % (o, c, 100 * c / tot, 100 * stall[o] / stot))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
