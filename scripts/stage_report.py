"""The reference's bench report (pipeline.cpp:323-391, StageTimings
pipeline.cpp:57-82) for the GPU stream: per-stage mean / min / max ms per
composited frame over R repetitions of a synthetic sequence, in the reference's
14-stage schema and text / CSV formats, so the CPU and GPU tables compare
line by line.

  python scripts/stage_report.py [--width 1280 --height 720 --disparities 128
                                  --frames 8 --repetitions 3 --csv out.csv]

Stage mapping (CUDA-event spans -> the 14 stages): paper_2203_02300_b200/report.py.
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2203_02300_b200 import dco  # noqa: E402
from paper_2203_02300_b200.config import Config  # noqa: E402
from paper_2203_02300_b200.report import bench_csv, format_bench_report, stages_from_spans, summarize  # noqa: E402
from paper_2203_02300_b200.synth import StereoVideo  # noqa: E402


def run_once(W, H, cfg, frames):
    """One run_pipeline over the sequence: per-stage mean ms per composited frame."""
    s = dco.Stream(W, H, cfg)
    s.set_timing(True)
    for l8, r8 in frames:
        s.push_gray8(l8, r8, want_result=False)
    spans, n = s.span_times()
    s.close()
    return stages_from_spans(spans, n), sum(spans.values()) / max(n, 1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--width", type=int, default=1280)
    ap.add_argument("--height", type=int, default=720)
    ap.add_argument("--disparities", type=int, default=128)
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--repetitions", type=int, default=3)
    ap.add_argument("--csv", default=None)
    a = ap.parse_args()
    if a.repetitions < 1:
        raise SystemExit("bench: repetitions must be >= 1")
    W, H = a.width, a.height
    cfg = Config(d_max=a.disparities - 1)
    vid = StereoVideo(W, H)
    frames = [tuple(torch.from_numpy(x).cuda() for x in vid.frame(i)) for i in range(a.frames)]
    run_once(W, H, cfg, frames)  # warm-up, excluded from statistics (pipeline.cpp:327)
    samples, totals = [], []
    for _ in range(a.repetitions):
        per, total = run_once(W, H, cfg, frames)
        samples.append(per)
        totals.append(total)
    rows = summarize(samples, totals)
    print(format_bench_report(a.repetitions, rows), end="")
    if a.csv:
        with open(a.csv, "w") as f:
            f.write(bench_csv(rows))


if __name__ == "__main__":
    main()
