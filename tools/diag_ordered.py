"""Diagnose MS_RHS_ORDERED vs the oracle split and an independent numpy restatement."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O
from paper_2605_23727_b200.configs import TWO_PI, rng_uniform
from paper_2605_23727_b200.precision import B32, B64, StagePrecision
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec
for n in (31, 64, 65, 128, 300):
    om = rng_uniform(11, 0, n, -1.0, 1.0)
    spec = SystemSpec("kuramoto", n, k_storage="f32", rhs_mode="ordered", omega=om, k_uniform=(11, 2, 0.0, 2.0))
    dev, orc = DeviceSystem(spec), O.OracleSystem(spec)
    x = rng_uniform(3, 1, n, 0.0, TWO_PI)
    K = orc.get_k().astype(np.float32)
    xf = x.astype(np.float32)
    s = np.sin(xf.astype(np.float64)).astype(np.float32); c = np.cos(xf.astype(np.float64)).astype(np.float32)
    for sp in (StagePrecision(B32, B32, B32), StagePrecision(B32, B64, B32), StagePrecision(B64, B64, B32)):
        a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
        SS = np.float32 if sp.sum_prec == B32 else np.float64
        ps = (K * s[None, :]).astype(SS); pc = (K * c[None, :]).astype(SS)
        A = np.add.accumulate(ps, axis=1)[:, -1]; Bv = np.add.accumulate(pc, axis=1)[:, -1]
        mw = SS(1.0 / n)
        coup = mw * (c.astype(SS) * A - s.astype(SS) * Bv)
        FS = np.float32 if sp.f_prec == B32 else np.float64
        WS = np.float32 if (FS == np.float32 and SS == np.float32) else np.float64
        ref = (om.astype(FS).astype(WS) + coup.astype(WS)).astype(np.float64)
        print(n, sp.f_prec.name[-2:], sp.sum_prec.name[-2:], "dev==orc", np.mean(a == b), "dev==np", np.mean(a == ref),
              "orc==np", np.mean(b == ref), "maxdiff dev-orc", float(np.max(np.abs(a - b))))
