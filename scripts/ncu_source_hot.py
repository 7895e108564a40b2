"""Top source lines by sampled stalls for one kernel of an ncu report."""
import csv
import io
import subprocess
import sys


def main(path, kernel, top=25):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "-k", "regex:" + kernel, "--print-source",
                          "cuda"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = None
    data = []
    for r in rows:
        if r and r[0] == "#":
            hdr = r
            continue
        if hdr is None and "Source" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(r)
    if not hdr:
        print(raw[:2000])
        return
    def col(name):
        for i, h in enumerate(hdr):
            if h.startswith(name):
                return i
        return None
    si = col("Source")
    wi = col("Warp Stall Sampling (All Samples)")
    li = col("#") if col("#") is not None else 0
    tot = sum(float(r[wi] or 0) for r in data)
    data.sort(key=lambda r: -float(r[wi] or 0))
    for r in data[:top]:
        print("%6.1f%%  %s | %s" % (100 * float(r[wi] or 0) / max(tot, 1), r[li], r[si].strip()[:110]))


main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25)
