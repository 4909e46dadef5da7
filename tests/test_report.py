"""Run reports and sweeps (paper_2405_09157_b200.report, mirroring R/bench.py:22-161)."""
import json

import pytest

from paper_2405_09157_b200 import RunConfig, report


def test_fields_mirror_the_reference():
    assert report.REPORT_FIELDS == ("problem", "n", "d", "eps", "value_primal", "value_dual",
                                    "gap", "iterations_total", "search_steps", "wall_ms",
                                    "termination", "threads")
    assert report.SWEEP_FIELDS[:9] == ("problem", "n", "d", "rep", "status", "wall_ms",
                                       "iterations", "value", "error")


def test_loglog_slope_and_format():
    xs = [1e3, 1e4, 1e5]
    assert abs(report.fit_loglog_slope(xs, [2 * x ** 1.5 for x in xs]) - 1.5) < 1e-12
    r = {k: 1 for k in report.REPORT_FIELDS + report.DEVICE_FIELDS}
    assert json.loads(report.format_report(r))["gbs"] == 1
    assert report.format_report(r, "csv").splitlines()[0].startswith("problem,n,d")
    with pytest.raises(ValueError):
        report.format_report(r, "xml")


def test_sweep_records_failures_and_continues():
    rows = report.sweep("ses", [1], [3], 2, RunConfig())   # n = 1 is rejected by gen_ses
    assert len(rows) == 2 and all(r["status"].startswith("error") for r in rows)
    with pytest.raises(ValueError):
        report.sweep("lp", [10], [2], 1, RunConfig())


@pytest.mark.gpu
def test_gpu_sweep_with_verification():
    rows = report.sweep("ses", [2000, 20000], [10], 1, RunConfig(eps=1e-2))
    rows += report.sweep("svm", [4000], [10], 1, RunConfig(eps=1e-2))
    ok = [r for r in rows if r["rep"] != "mean"]
    assert all(r["status"] == "ok" for r in ok), rows
    for r in ok:
        assert r["gbs"] > 0 and r["passes"] > 0
        assert r["error"] != "" and r["error"] <= 0.05   # independent baseline agrees
    csv = report.sweep_csv(rows)
    assert csv.count("\n") == len(rows) + 1
