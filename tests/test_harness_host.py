"""The harness runner (harness.cpp:97-195, :305-343, :518-553) on the CPU
oracle engine: the reference's harness tests (test_harness.cpp:103-136,
:184-300) and the CSV formatting of std::to_chars."""
import math

import numpy as np
import pytest

from _harness_engine import OracleEngine
from paper_2605_23727_b200 import harness as H
from paper_2605_23727_b200.precision import PolicyVariant
from paper_2605_23727_b200.solver import SolveStatus


@pytest.mark.parametrize("v,s", [
    (1e-06, "1e-06"), (0.001, "0.001"), (0.0001, "1e-04"), (100000.0, "1e+05"), (123456.0, "123456"),
    (0.1, "0.1"), (1.5, "1.5"), (2.0, "2"), (-3.25, "-3.25"), (1e22, "1e+22"), (5e-324, "5e-324"),
    (31.41592653589793, "31.41592653589793"), (6.283185307179586, "6.283185307179586"),
    (1e16, "1e+16"), (1.2345678901234568e+17, "123456789012345680"), (0.5, "0.5"), (10.0, "10"),
    (1e-05, "1e-05"), (2.5e-07, "2.5e-07"), (0.0, "0"), (-0.0, "-0"), (math.inf, "inf"), (-math.inf, "-inf"),
    (1.7976931348623157e308, "1.7976931348623157e+308"), (120.0, "120"), (1200000.0, "1200000"),
])
def test_format_double_is_to_chars(v, s):
    assert H.format_double(v) == s
    if math.isfinite(v):
        assert float(H.format_double(v)) == v  # round trip


def test_format_double_golden():
    """libstdc++ std::to_chars outputs (tests/golden/gen_to_chars.cpp)."""
    from pathlib import Path
    lines = (Path(__file__).parent / "golden" / "to_chars.txt").read_text().splitlines()
    for ln in lines:
        a, s = ln.split()
        v = float.fromhex(a) if a.startswith(("0x", "-0x")) else float(a)
        assert H.format_double(v) == s, (a, s)
    assert len(lines) > 2000


def test_initial_conditions():  # test_harness.cpp:103-136
    tc = H.TestCase(test_id=12, benchmark="lco", agents=50)
    a, b = H.initial_conditions(tc), H.initial_conditions(tc)
    assert np.array_equal(a, b) and a.size == 100 and a.min() >= 0.0 and a.max() <= 2.0
    tc.benchmark = "kuramoto"
    k = H.initial_conditions(tc)
    assert k.size == 50 and k.min() >= 0.0 and k.max() < 2.0 * math.pi
    tc.benchmark = "cc"
    c = H.initial_conditions(tc).reshape(50, 4)
    assert np.all((c[:, 0] >= 0.9) & (c[:, 0] <= 1.1))
    assert np.all((c[:, 2] >= -1.29) & (c[:, 2] <= -1.09)) and np.all((c[:, 3] >= -0.72) & (c[:, 3] <= -0.52))
    other = H.TestCase(test_id=13, benchmark="cc", agents=50)
    assert not np.array_equal(H.initial_conditions(other).reshape(50, 4), c)
    with pytest.raises(ValueError):
        H.initial_conditions(H.TestCase(benchmark="nope", agents=2))


def test_gamma_beta_capital_gamma():  # test_metrics.cpp (gamma, beta, capital gamma)
    assert abs(H.gamma_of(1.0, 0.5) - 0.5) <= 1e-15
    assert abs(H.gamma_of(5.0 / 6.0, 0.5) - 7.0 / 12.0) <= 1e-15
    assert H.gamma_of(0.0, 0.5) == 1.0
    with pytest.raises(ValueError):
        H.gamma_of(-0.1, 0.5)
    with pytest.raises(ValueError):
        H.gamma_of(0.5, 1.5)
    assert H.beta_of(1000, 1000) == 1.0 and H.beta_of(900, 1000) == pytest.approx(0.9, rel=1e-15)
    with pytest.raises(ValueError):
        H.beta_of(0, 10)
    assert H.capital_gamma_of(0.75, 1.0) == 0.75
    with pytest.raises(ValueError):
        H.capital_gamma_of(0.75, 0.0)


def tiny_lco_cases():  # test_harness.cpp:23-31: LCO N=6, rel 1e-4 (abs = 1e-2 rel), t_f = 2
    return [H.TestCase(test_id=i, benchmark="lco", agents=6, rel_tol=1e-4, abs_tol=1e-6, t_final=2.0)
            for i in range(4)]


def test_run_one_rows():  # test_harness.cpp:184-213
    eng = OracleEngine()
    for tc in tiny_lco_cases():
        rows, _ = H.run_one(tc, engine=eng)
        assert [r.variant for r in rows] == ["Single", "Mixed1", "Mixed2", "Double", "Reference"]
        for r in rows:
            assert r.test_id == tc.test_id and r.status == SolveStatus.Completed
            if r.variant != "Reference":
                assert r.final_error is not None and r.final_error < 1e-3 and r.beta is not None
        dbl = rows[3]
        assert dbl.rho == 0.0 and dbl.gamma == 1.0 and dbl.beta == 1.0 and dbl.capital_gamma == 1.0
    rows, _ = H.run_one(tiny_lco_cases()[0], H.CampaignSpec(variants=[PolicyVariant.Double]), engine=eng)
    assert [r.variant for r in rows] == ["Double", "Reference"]  # :229-237


def test_results_csv_round_trip_and_resume(tmp_path):  # test_harness.cpp:239-300
    eng = OracleEngine()
    spec = H.CampaignSpec(snapshots=True)
    opt = H.RunOptions(output_dir=str(tmp_path), step_log_csv=True)
    cases = tiny_lco_cases()
    rows = H.run_cases(cases, spec, opt, engine=eng)
    rp, sp = tmp_path / "results.csv", tmp_path / "steps.csv"
    assert rp.exists() and sp.exists()
    back = H.read_results_csv(rp)
    assert len(back) == len(rows) == 5 * len(cases)
    for a, b in zip(back, rows):
        assert H.result_row_to_csv(a) == H.result_row_to_csv(b)
        assert (a.test_id, a.variant, a.status, a.final_error, a.mean_ebs, a.mean_eanalytic, a.beta) == \
            (b.test_id, b.variant, b.status, b.final_error, b.mean_ebs, b.mean_eanalytic, b.beta)
    assert any(r.mean_eanalytic is not None for r in back)  # LCO with snapshots
    assert sp.read_text().splitlines()[0] == H.STEPS_CSV_HEADER
    before, steps_before = rp.read_text(), sp.read_text()

    class Counting(OracleEngine):
        calls = 0

        def dp54_reference(self, *a):
            Counting.calls += 1
            return super().dp54_reference(*a)

    H.run_cases(cases, spec, opt, engine=Counting())  # resume over a complete campaign: no work, same bytes
    assert Counting.calls == 0 and rp.read_text() == before and sp.read_text() == steps_before
    H.write_results_csv(rp, [r for r in back if r.test_id != cases[-1].test_id])
    H.run_cases(cases, spec, opt, engine=Counting())  # exactly the missing case is recomputed
    assert Counting.calls == 1 and rp.read_text() == before
    rp.write_text("nope\n1,2,3\n")
    with pytest.raises(ValueError):
        H.read_results_csv(rp)


def test_run_cases_validation():
    with pytest.raises(ValueError):
        H.run_cases([], engine=OracleEngine())
    with pytest.raises(ValueError):
        H.run_cases(tiny_lco_cases(), H.CampaignSpec(variants=[]), engine=OracleEngine())
    with pytest.raises(ValueError):
        H.run_cases(tiny_lco_cases(), H.CampaignSpec(speedup_r=1.0), engine=OracleEngine())
