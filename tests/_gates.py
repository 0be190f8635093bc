"""The BASELINE.md §2 parity gate for whole solves, device vs oracle (shared
by the full-size config tests)."""
import numpy as np

from paper_2605_23727_b200 import solver as S


def gate(r, o, cfg, dev=None, w=None, rtol_state=1e-5):
    assert r.status == o.status
    att = o.n_accepted + o.n_failed
    assert abs(r.n_accepted - o.n_accepted) <= max(1, 0.01 * o.n_accepted), (r.n_accepted, o.n_accepted)
    assert abs(r.n_failed - o.n_failed) <= max(1, 0.01 * att), (r.n_failed, o.n_failed)
    floor = cfg.abs_tol / cfg.rel_tol
    wrel = lambda a, b: float(np.max(np.abs(a - b) / np.maximum(np.abs(b), floor)))
    rel = wrel(r.final_state, o.final_state)
    print(f"device vs oracle final state: {rel:.3e} (counts {r.n_accepted}/{r.n_failed} vs {o.n_accepted}/{o.n_failed})")
    if rel <= rtol_state:
        return rel
    ref = S.dp54_reference(dev, w.x0, w.t0, w.tf, S.SolverConfig(time_limits_enabled=False), log_capacity=1)
    assert ref.status == S.SolveStatus.Completed
    e_dev, e_orc = wrel(r.final_state, ref.final_state), wrel(o.final_state, ref.final_state)
    print(f"  global error vs DP5(4) 1e-9: device {e_dev:.3e}, oracle {e_orc:.3e}")
    assert e_dev <= 1.5 * e_orc + 1e-7, (e_dev, e_orc)
    return rel
