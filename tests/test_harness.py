"""Experiment harness (paper_2411_18026_b200/harness.py): report helpers on
CPU (csv_render / CsvTable / fit_exponent as proj/src/report.cpp:14-121),
the three experiments on the GPU."""
import json

import numpy as np
import pytest

from paper_2411_18026_b200 import harness as H


def test_csv_render_and_table(tmp_path):
    assert H.csv_render(3) == "3"
    assert H.csv_render(0.5) == "5.0000000000000000e-01"
    assert H.csv_render("fds") == "fds"
    with pytest.raises(ValueError):
        H.csv_render("a,b")
    t = H.CsvTable(["solver", "n_elements", "seconds"])
    t.row(["fds", 4096, 0.25])
    with pytest.raises(ValueError):
        t.row(["fds", 1])
    p = tmp_path / "x.csv"
    t.save(str(p))
    assert p.read_text() == "solver,n_elements,seconds\nfds,4096,2.5000000000000000e-01\n"


def test_fit_exponent():
    n = [4096, 16384, 65536, 262144]
    assert H.fit_exponent(n, [2e-3 * x for x in n]) == pytest.approx(1.0, abs=1e-12)
    assert H.fit_exponent(n, [x * np.log(x) for x in n]) == pytest.approx(1.0974, abs=1e-3)
    with pytest.raises(ValueError):
        H.fit_exponent([1.0], [1.0])
    with pytest.raises(ValueError):
        H.fit_exponent([2.0, 2.0], [1.0, 3.0])


def test_timing_protocol():
    assert H.timing_repeats(1600) == 3 and H.timing_repeats(1601) == 1
    calls = []
    assert H.median_seconds(lambda: calls.append(1) or len(calls), 3, True) == 3.0
    assert len(calls) == 4


@pytest.mark.gpu
def test_harness_experiments_small(eb, tmp_path):
    rep = H.scaling(1024, 4096, 1.0, 1e-10, 32, 800, str(tmp_path / "s.csv"))
    assert rep["summary"]["fds_exponent"] is not None
    rows = (tmp_path / "s.csv").read_text().splitlines()
    assert rows[0] == "solver,n_elements,levels,ell0,epsilon,seconds"
    assert len(rows) == 1 + 3 + 2
    doc = json.loads((tmp_path / "s.json").read_text())
    assert set(doc) >= {"config", "phases", "max_rank_per_level", "relative_errors",
                        "peak_memory_mib", "summary"}
    rep = H.multi_rhs(2048, 4.0, 6, 1e-10, 32, out=str(tmp_path / "m.csv"))
    assert rep["summary"]["max_deviation_vs_batch"] < 1e-12
    assert len((tmp_path / "m.csv").read_text().splitlines()) == 7
    rep = H.error_table((400,), (1e-8, 1e-10), 2.0, str(tmp_path / "e.csv"))
    assert rep["summary"]["worst_error_over_epsilon"] < 100
