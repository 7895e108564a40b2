"""Top SASS instructions by sampled warp stalls for one kernel (ncu source page)."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=30):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", "regex:" + kernel],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[1]
    si, wi = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
    data = [r for r in rows[2:] if len(r) == len(hdr) and r[wi] != hdr[wi]]
    data = [r for r in data if r[wi].replace(".", "", 1).isdigit() or r[wi] == ""]
    tot = sum(float(r[wi] or 0) for r in data)
    print("total samples", tot)
    for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][wi] or 0))[:top]:
        print("%6.2f%%  [%5d] %s" % (100 * float(r[wi] or 0) / max(tot, 1), idx, r[si].strip()[:90]))


main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 30)
