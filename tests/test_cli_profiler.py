"""CLI, profiler report and probe logic on CPU (no kernel launches)."""

import pytest

from paper_1904_12380_b200 import bench_cli, profiler
from paper_1904_12380_b200.bound_probe import MEMORY_BOUND_THRESHOLD, Verdict, _verdict
from paper_1904_12380_b200.errors import ArgumentError
from paper_1904_12380_b200.kernels import KernelVariant


def test_report_round_trip_and_ratios():
    rep = profiler.build_report([("MaxSub", [1000, 2000]), ("Exp", [5000, 7000]),
                                 ("SumScale", [1500, 1600]), ("WholeOp", [8000, 11000])])
    assert [e.name for e in rep.events] == ["WholeOp", "Exp", "SumScale", "MaxSub"]
    assert abs(sum(e.ratio for e in rep.events) - 1.0) < 1e-9
    text = profiler.format_report(rep)
    assert text.startswith(profiler.REPORT_HEADER) and "Place: GPU" in text
    back = profiler.parse_report(text)
    for a, b in zip(rep.events, back.events):
        assert a.name == b.name and a.calls == b.calls
        assert abs(a.total - b.total) <= 1e-3 * a.total
    assert profiler.report_to_csv(rep).splitlines()[0] == "Event,Calls,Total,Min.,Max.,Ave.,Ratio."
    with pytest.raises(ArgumentError):
        profiler.build_report([])
    with pytest.raises(ArgumentError):
        profiler.parse_report("nothing here")


def test_phase_ratio_summary():
    t = [profiler.PhaseTimings(1, 6, 2, 10), profiler.PhaseTimings(2, 5, 2, 10)]
    s = profiler.phase_ratio_summary(t)
    assert s[profiler.PhaseId.WHOLEOP] == 1.0 and abs(s[profiler.PhaseId.EXP] - 0.55) < 1e-9


def test_probe_verdict_threshold():
    assert MEMORY_BOUND_THRESHOLD == 1.3
    assert _verdict(1.3) is Verdict.MEMORY_BOUND_LIKELY
    assert _verdict(1.31) is Verdict.COMPUTE_BOUND_LIKELY


def test_bench_config_validation():
    with pytest.raises(ArgumentError):
        bench_cli.BenchConfig(batch_sizes=())
    with pytest.raises(ArgumentError):
        bench_cli.BenchConfig(variants=(KernelVariant.FULL_VECTORIZED,))  # baseline missing
    with pytest.raises(ArgumentError):
        bench_cli.BenchConfig(output_format="xml")
    c = bench_cli.BenchConfig(variants=tuple(reversed(bench_cli.LADDER)))
    assert c.ladder_variants == bench_cli.LADDER
    assert bench_cli.elem_tolerance(KernelVariant.FULL_VECTORIZED_APPROX_EXP) == 1e-5


def test_cli_usage_errors(monkeypatch):
    assert bench_cli.main(["bogus"]) == 2
    assert bench_cli.main(["verify", "--variant", "NoSuchVariant"]) == 2
    assert bench_cli.main(["verify", "--batch-size", "0"]) == 2
    monkeypatch.setenv("SOFTMAX_KIT_THREADS", "4")
    assert bench_cli.main(["verify"]) == 2


def test_refcheck_matches_reference_oracle_semantics():
    import numpy as np

    from paper_1904_12380_b200 import refcheck

    x = np.array([[1.0, 2.0, 3.0]], np.float32)
    np.testing.assert_allclose(refcheck.softmax_f64(x)[0], [0.09003057, 0.24472847, 0.66524096],
                               atol=1e-8)
    assert refcheck.kahan_sum(np.full(1000, 0.1)) == pytest.approx(100.0, abs=1e-12)
    assert refcheck.max_rowsum_dev(np.array([[0.5, 0.5]])) == 0.0
