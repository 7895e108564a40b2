"""The reference's bench report for the GPU stream: StageTimings'
14-stage schema (pipeline.hpp:27-46, stage names pipeline.cpp:57-75) and
bench()'s mean / min / max aggregation with format_bench_report /
write_bench_csv output (pipeline.cpp:323-391), so CPU and GPU stage tables
compare line by line.

Mapping of the stream's CUDA-event spans (include/dco_gpu.h DCO_SPAN_*):
  adaptive filter area construction <- cross
  initial parallax                  <- cost + aggregate + wta
  parallax optimisation             <- refine
  sparse map                        <- sparse
  bidirectional optical flow        <- flow
  amplitude                         <- (fused into "fusion": one kernel)
  fusion                            <- fusion
  box filter, normalisation, Gaussian filtering, depth contour extraction
                                    <- box, normalize, blur, contour
  densification                     <- assemble + solve
  rendering                         <- composite (includes the virtual layer)
  other                             <- ingest (u8 decode + downsample)
"""

STAGES = [
    ("adaptive filter area construction", ["cross"]),
    ("initial parallax", ["cost", "aggregate", "wta"]),
    ("parallax optimisation", ["refine"]),
    ("sparse map", ["sparse"]),
    ("bidirectional optical flow", ["flow"]),
    ("amplitude", []),
    ("fusion", ["fusion"]),
    ("box filter", ["box"]),
    ("normalisation", ["normalize"]),
    ("Gaussian filtering", ["blur"]),
    ("depth contour extraction", ["contour"]),
    ("densification", ["assemble", "solve"]),
    ("rendering", ["composite"]),
    ("other", ["ingest"]),
]
STAGE_NAMES = [n for n, _ in STAGES]
TOTAL = "frame processing"


def stages_from_spans(spans, frames):
    """Per-frame ms of the 14 stages from the stream's span totals."""
    n = max(frames, 1)
    return [sum(spans[k] for k in keys) / n for _, keys in STAGES]


def summarize(samples, totals):
    """bench()'s aggregation (pipeline.cpp:341-363): samples[rep] = the 14
    per-frame stage means of one repetition, totals[rep] its frame mean.
    -> 15 rows (stage, mean, min, max), the frame total last."""
    if not samples:
        raise ValueError("bench: repetitions must be >= 1")
    rows = []
    for i, name in enumerate(STAGE_NAMES):
        xs = [s[i] for s in samples]
        rows.append((name, sum(xs) / len(xs), min(xs), max(xs)))
    rows.append((TOTAL, sum(totals) / len(totals), min(totals), max(totals)))
    return rows


def format_bench_report(repetitions, rows):
    """format_bench_report, pipeline.cpp:376-391."""
    out = ["repetitions: %d\n" % repetitions, "%-36s %10s %10s %10s\n" % ("stage", "mean(ms)", "min(ms)", "max(ms)")]
    out += ["%-36s %10.2f %10.2f %10.2f\n" % r for r in rows]
    return "".join(out)


def _num(x):
    """std::ostream << double with the default format (6 significant digits)."""
    return "%g" % x


def bench_csv(rows):
    """write_bench_csv's text, pipeline.cpp:366-374."""
    lines = ["stage,mean_ms,min_ms,max_ms\n"]
    lines += ["%s,%s,%s,%s\n" % (r[0], _num(r[1]), _num(r[2]), _num(r[3])) for r in rows]
    return "".join(lines)
