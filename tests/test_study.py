"""Host logic of the GPU study runner (paper_2211_03293_b200/study.py) against
the reference harness's rules (proj/src/harness.cpp); no GPU needed."""
import csv
import json
import math

import numpy as np
import pytest

from paper_2211_03293_b200 import study as St


def test_parse_method_selectors():
    """harness.cpp:89-157 and the selector list :159-163."""
    s = St.parse_method("mri3-10")
    assert (s.family, s.coupling_name, s.fast_table, s.m) == ("mri", "mis-kw3",
                                                             "bogacki-shampine3", 10)
    assert not s.needs_implicit_solver
    s = St.parse_method("imex-mri3-4")
    assert (s.coupling_name, s.fast_table, s.m, s.needs_implicit_solver) == (
        "imex-mri-gark3b", "kutta3", 4, True)
    s = St.parse_method("imex-mri4-2")
    assert (s.coupling_name, s.fast_table, s.m) == ("imex-mri-gark4", "classic-rk4", 2)
    assert St.parse_method("ark-imex").needs_implicit_solver
    assert St.parse_method("erk-cash-karp5").table_name == "cash-karp5"
    assert (St.parse_method("sdc").sweeps, St.parse_method("sdc-3").sweeps) == (4, 3)
    s = St.parse_method("mrsdc-338")
    assert (s.X, s.Y, s.Z, s.sweeps) == (3, 3, 8, 4)
    s = St.parse_method("mri:imex-mri-gark4-explicit:classic-rk4:50")
    assert (s.coupling_name, s.m, s.needs_implicit_solver) == ("imex-mri-gark4-explicit", 50,
                                                              False)
    for bad in ("mri3-x", "nope", "mrsdc-12", "mri:a:b"):
        with pytest.raises((St.ConfigError, ValueError)):
            St.parse_method(bad)
    assert "ark-imex" in St.known_method_selectors()


def test_validate_rules():
    """StudyConfig::validate (harness.cpp:165-186)."""
    ok = St.StudyConfig(methods=["mri3-4"], h_list=[0.1, 0.05], tf=1.0)
    ok.validate()
    for bad in (St.StudyConfig(methods=["mri3-4"], h_list=[0.1, 0.1]),
                St.StudyConfig(methods=["mri3-4"], h_list=[]),
                St.StudyConfig(methods=["mri3-4"], h_list=[0.1], t0=1.0, tf=1.0),
                St.StudyConfig(methods=["mri3-4"], h_list=[0.1], reference_method="analytic"),
                St.StudyConfig(methods=["bogus"], h_list=[0.1])):
        with pytest.raises(St.ConfigError):
            bad.validate()


def test_fitted_slope_rules():
    """fitted_slope (harness.cpp:514-538): exact power laws, the coarsest point
    dropped with >= 4 points, non-finite / non-positive errors skipped."""
    pts = [(0.1 / 2 ** i, 3.0 * (0.1 / 2 ** i) ** 3) for i in range(3)]
    assert St.fitted_slope(pts) == pytest.approx(3.0, rel=1e-12)
    bent = [(1.0, 1.0)] + [(0.1 / 2 ** i, (0.1 / 2 ** i) ** 2) for i in range(3)]
    assert St.fitted_slope(bent) == pytest.approx(2.0, rel=1e-12)
    assert math.isnan(St.fitted_slope([(0.1, 1e-3)]))
    assert St.fitted_slope([(0.1, 1e-3), (0.05, float("nan")), (0.025, 0.0),
                            (0.0125, 1e-3 / 64)]) == pytest.approx(2.0, rel=1e-12)


def test_measure_error():
    """measure_error (harness.cpp:316-324): max norm, or one component block."""
    ref = np.zeros(12)
    st = np.arange(12, dtype=float) * np.where(np.arange(12) % 2 == 0, 1.0, -1.0)
    assert St.measure_error(st, ref) == 11.0
    assert St.measure_error(st, ref, 1, 1, ncell=4) == 7.0  # component 1 = entries 4..7


def test_report_files(tmp_path):
    """write_csv / write_json (harness.cpp:645-705): header, %.17g, null for
    non-finite error and rate."""
    cnt = np.arange(1, 9, dtype=np.uint64)
    rep = St.RunReport(rows=[St.RunRecord("mri3-4", 0.1, 0.0, 1.5e-3, math.nan, 0.25, 10, cnt),
                             St.RunRecord("mri3-4", 0.05, 0.0, math.nan, math.nan, 0.5, 20,
                                          cnt, True, "blew up")],
                       fitted_slopes={"mri3-4": math.nan})
    rep.write_csv(tmp_path / "r.csv")
    rows = list(csv.reader(open(tmp_path / "r.csv")))
    assert rows[0] == ["method", "H", "tolerance", "error", "rate", "wall_s", "steps",
                       "diverged", "n_fast_evals", "n_implicit_evals", "n_explicit_evals",
                       "n_implicit_solves", "n_nonlinear_iters", "n_linear_iters",
                       "n_precond_solves", "n_fast_ivps"]
    assert rows[1][:8] == ["mri3-4", "0.10000000000000001", "0", "0.0015", "nan", "0.25", "10",
                           "0"]
    assert rows[1][8:] == [str(i) for i in range(1, 9)] and rows[2][7] == "1"
    rep.write_json(tmp_path / "r.json", St.StudyConfig(methods=["mri3-4"], h_list=[0.1, 0.05]))
    j = json.load(open(tmp_path / "r.json"))
    assert j["rows"][1]["error"] is None and j["rows"][1]["diverged"] is True
    assert j["rows"][0]["counters"]["fast_ivps"] == 8
    assert j["fitted_slopes"]["mri3-4"] is None


class _FakeCtx:
    """A context stand-in whose 'integration' has error c * H^p exactly: checks
    execute_study's bookkeeping (rows, rates, slopes, divergence)."""
    ncell = 1

    def __init__(self, p=3.0, diverge_below=None):
        self.p, self.div, self.y = p, diverge_below, None

    def upload(self, y):
        self.y = np.array(y, dtype=float)

    def download(self):
        return self.y.copy()

    def reference_solution(self, t0, tf, h):
        pass

    def method(self, *a):
        pass

    def newton_config(self, *a):
        pass

    def mri_integrate(self, t0, tf, H, cnt):
        from paper_2211_03293_b200 import IntegrationError
        if self.div is not None and H < self.div:
            raise IntegrationError("mri_step: non-finite state", 2)
        cnt[7] += int(round((tf - t0) / H))
        self.y = self.y + 5.0 * H ** self.p


def test_execute_study_rates_and_divergence():
    cfg = St.StudyConfig(methods=["mri3-4"], h_list=[0.2, 0.1, 0.05, 0.025], tf=1.0)
    rep = St.run_convergence_study(_FakeCtx(3.0), np.zeros(3), cfg)
    assert [r.H for r in rep.rows] == cfg.h_list
    assert [r.steps for r in rep.rows] == [5, 10, 20, 40]
    assert math.isnan(rep.rows[0].rate)
    for r in rep.rows[1:]:
        assert r.rate == pytest.approx(3.0, rel=1e-9)
    assert rep.fitted_slopes["mri3-4"] == pytest.approx(3.0, rel=1e-9)
    assert int(rep.rows[3].counters[7]) == 40
    rep = St.run_efficiency_study(_FakeCtx(3.0, diverge_below=0.06), np.zeros(3), cfg)
    assert [r.diverged for r in rep.rows] == [False, False, True, True]
    assert "non-finite" in rep.rows[2].note and math.isnan(rep.rows[2].error)
    assert all(math.isnan(r.rate) for r in rep.rows) and rep.fitted_slopes == {}


def test_sdc_families_refused():
    cfg = St.StudyConfig(methods=["sdc"], h_list=[0.1], tf=1.0)
    from paper_2211_03293_b200 import ContractError
    with pytest.raises(ContractError):
        St.run_method(_FakeCtx(), np.zeros(2), St.parse_method("sdc"), cfg, 0.1)
