"""The harness runner over the device (harness.DeviceEngine) against the same
runner over the CPU oracle: the rows a device campaign writes are the oracle's
rows (counts, statuses, error columns), so results.csv files can be diffed."""
import pytest

from _harness_engine import OracleEngine
from paper_2605_23727_b200 import harness as H

pytestmark = pytest.mark.gpu


def _cases():
    return [H.TestCase(test_id=i, benchmark="lco", agents=6, rel_tol=1e-4, abs_tol=1e-6, t_final=2.0)
            for i in range(3)] + [
        H.TestCase(test_id=7, benchmark="kuramoto", agents=16, rel_tol=1e-5, abs_tol=1e-7, t_final=3.0, sigma=0.5,
                   coupling_k=1.3),
        H.TestCase(test_id=9, benchmark="cc", agents=8, rel_tol=1e-5, abs_tol=1e-7, t_final=4.0, coupling_k=0.1,
                   stimulus_i0=0.228249)]


def _close(a, b, rel):
    if a is None or b is None:
        return a is b
    return abs(a - b) <= rel * max(abs(a), abs(b)) + 1e-300


def test_device_rows_match_oracle_rows(gpu, tmp_path):
    spec = H.CampaignSpec(snapshots=True)
    dev_rows = H.run_cases(_cases(), spec, H.RunOptions(rhs_mode="faithful", output_dir=str(tmp_path),
                                                          step_log_csv=True))
    orc_rows = H.run_cases(_cases(), spec, H.RunOptions(), engine=OracleEngine())
    assert len(dev_rows) == len(orc_rows) == 5 * len(_cases())
    for d, o in zip(dev_rows, orc_rows):
        assert (d.test_id, d.variant, d.status) == (o.test_id, o.variant, o.status)
        # the controller's pow is correctly rounded on the device and ~0.1 % of
        # glibc's calls are 1 ulp off, which can move a step sequence by one step
        assert abs(d.n_accepted - o.n_accepted) <= 1 and abs(d.n_failed - o.n_failed) <= 1
        # binary32 rows: the device's sinf (correctly rounded in binary64) and
        # glibc's differ by an ulp now and then, so the runs are two noise-level
        # realisations; their error columns agree in magnitude, not digits
        rel = 0.05 if d.variant in ("Mixed2", "Double", "Reference") or d.benchmark == "lco" else 0.75
        for k in ("final_error", "mean_ebs", "mean_eanalytic"):
            assert _close(getattr(d, k), getattr(o, k), rel), (d.variant, k, getattr(d, k), getattr(o, k))
        assert d.rho == o.rho
    # the persisted campaign reads back as written
    back = H.read_results_csv(tmp_path / "results.csv")
    assert [H.result_row_to_csv(r) for r in back] == [H.result_row_to_csv(r) for r in dev_rows]


def test_concurrent_variants_rows_equal_sequential_rows(gpu):
    cases = [c for c in _cases() if c.benchmark != "lco"] + [_cases()[0]]
    conc = H.run_cases(cases, H.CampaignSpec(), H.RunOptions(concurrent_variants=True))
    seq = H.run_cases(cases, H.CampaignSpec(), H.RunOptions(concurrent_variants=False))
    assert [H.result_row_to_csv(r) for r in conc] == [H.result_row_to_csv(r) for r in seq]
