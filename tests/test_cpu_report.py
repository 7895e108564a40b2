"""The bench report schema: paper_2203_02300_b200.report
reproduces the reference's StageTimings stage list (pipeline.cpp:57-75),
bench()'s aggregation (pipeline.cpp:341-363) and format_bench_report /
write_bench_csv byte for byte (pipeline.cpp:366-391), checked against the
reference's own functions in oracle/_ref."""
import numpy as np
import pytest

from paper_2203_02300_b200 import report


def test_stage_names_are_the_references(ref):
    assert report.STAGE_NAMES == ref.STAGES
    assert len(report.STAGES) == 14 and report.STAGE_NAMES[-1] == "other"


def test_spans_cover_every_stream_span():
    from paper_2203_02300_b200.dco import Stream

    mapped = [k for _, keys in report.STAGES for k in keys]
    assert sorted(mapped) == sorted(Stream.SPANS)  # every span lands in exactly one stage


@pytest.mark.parametrize("reps,seed", [(1, 0), (3, 1), (5, 2)])
def test_format_and_csv_match_reference(ref, tmp_path, reps, seed):
    rng = np.random.default_rng(seed)
    samples = [list(rng.random(14) * 10.0 ** rng.integers(-3, 4, 14)) for _ in range(reps)]
    totals = [sum(s) for s in samples]
    rows = report.summarize(samples, totals)
    assert len(rows) == 15 and rows[-1][0] == "frame processing"
    mmm = np.array([r[1:] for r in rows])
    csv = tmp_path / "bench.csv"
    want = ref.format_bench_report(reps, mmm, str(csv))
    assert report.format_bench_report(reps, rows) == want
    assert report.bench_csv(rows) == csv.read_text()


def test_summarize_rejects_empty():
    with pytest.raises(ValueError):
        report.summarize([], [])
