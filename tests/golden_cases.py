"""The whole-solve golden cases (BASELINE.json configs at their stated sizes)
whose oracle results are committed under tests/golden/solves/ by
tools/make_golden_solves.py. Shared by that script and the tests that read the
fixtures: the workload definitions live in one place.

Each case names the reference code it pins: the adaptive loop
(solver.cpp:226-347), the stage rows of its policy (precision.cpp:22-42) and
the model's eval_core (systems.cpp:30-189)."""
from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.configs import config2_kuramoto, config3_cc, config4_kuramoto, config5_batch
from paper_2605_23727_b200.precision import PolicyVariant, policy_for

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "tests" / "golden" / "solves"
ORACLE_SOURCES = ("oracle/mixedstep_oracle.cpp", "oracle/mixedstep_oracle.hpp", "oracle/oracle_capi.cpp")

# 16 trajectories of the C5 ensemble whose final states are pinned (counts are
# pinned for all 1024)
C5_SAMPLE = [0, 1, 67, 130, 201, 255, 256, 384, 511, 512, 640, 767, 768, 895, 1000, 1023]


def _c4_mixed2():
    w = config4_kuramoto()
    w.policy = policy_for(PolicyVariant.Mixed2)
    return w


def _c3_full():
    return config3_cc()


CASES = {
    "c2_rtol1e-6_f32": {"build": lambda: config2_kuramoto(rtol=1e-6), "what": "C2 N=4096 t[0,50] rtol 1e-6 K f32"},
    "c2_rtol1e-6_f16": {"build": lambda: config2_kuramoto(rtol=1e-6, k_storage="f16"),
                        "what": "C2 N=4096 t[0,50] rtol 1e-6 K f16"},
    # rtol 1e-8 under binary32 rows is noise-driven: the rounding noise of the
    # RHS sums (~1e-7 relative) exceeds the tolerance, so the step sequence
    # follows the summation order's noise (tests/test_gpu_golden_solves.py)
    "c2_rtol1e-8_f32": {"build": lambda: config2_kuramoto(rtol=1e-8), "what": "C2 N=4096 t[0,50] rtol 1e-8 K f32",
                        "noise": True},
    "c2_rtol1e-8_f16": {"build": lambda: config2_kuramoto(rtol=1e-8, k_storage="f16"),
                        "what": "C2 N=4096 t[0,50] rtol 1e-8 K f16", "noise": True},
    "c3_full": {"build": _c3_full, "what": "C3 CC N=2048 t[0,240] rtol 1e-6 K f32", "log": False},
    "c4_f32": {"build": lambda: config4_kuramoto(), "what": "C4 N=32768 t[0,20] rtol 1e-6 SSS rows, K f32"},
    "c4_f16": {"build": lambda: config4_kuramoto(k_storage="f16"),
               "what": "C4 N=32768 t[0,20] rtol 1e-6 SSS rows, K f16 (pre-rounded in the oracle)"},
    "c4_mixed2": {"build": _c4_mixed2, "what": "C4 N=32768 t[0,20] rtol 1e-6 Mixed2 (DDS rows), K f32"},
    "c5_bf16": {"build": lambda: config5_batch(), "batch": True, "op_round": _abi.MS_K_BF16, "sample": C5_SAMPLE,
                "what": "C5 B=1024 N=2048 t[0,20] rtol 1e-6, K bf16, tensor-core operand rounding (hi+lo bf16)"},
}


def oracle_source_hash() -> str:
    h = hashlib.sha256()
    for p in ORACLE_SOURCES:
        h.update((ROOT / p).read_bytes())
    return h.hexdigest()[:16]


def input_hash(w) -> str:
    """Hash of everything a solve reads besides K's generator parameters."""
    h = hashlib.sha256()
    for a in (w.x0, getattr(w, "omega", None), w.spec.omega, w.spec.cc_k1, w.spec.cc_theta_h, w.spec.cc_k0):
        if a is not None:
            h.update(np.ascontiguousarray(a, dtype=np.float64).tobytes())
    h.update(repr((w.spec.model, w.spec.n_agents, w.spec.k_storage, w.spec.k_uniform, w.t0, w.tf,
                   w.cfg.rel_tol, w.cfg.abs_tol, w.policy.c().per_stage[0].sum_prec,
                   [(r.f_prec, r.sum_prec, r.g_prec) for r in w.policy.c().per_stage])).encode())
    return h.hexdigest()[:16]


def load(name: str) -> dict:
    import json
    d = dict(np.load(OUT / f"{name}.npz"))
    d["meta"] = json.loads(str(d["meta"]))
    return d
