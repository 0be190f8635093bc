"""Seeded synthetic workloads of BASELINE.json ``configs``.

Every draw comes from ``SplitMix64(seed, stream)`` (rng.hpp:13-52) in row-major
order: stream 0 = per-agent parameters (the make_kuramoto / make_cc stream,
systems.cpp:230-231, 251-259), stream 1 = initial conditions
(harness.cpp:305-330), stream 2 = the dense coupling K (new), stream 3 = the CC
per-cell multipliers (new). The reference publishes no dataset; these seeded
inputs with BASELINE.json's shapes and distributions stand in for it.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _abi
from .precision import (B32, B64, DDD, DDS, SSS, PolicyVariant, PrecisionPolicy, custom_policy, policy_for)
from .solver import SolverConfig
from .systems import CcConstants, SystemSpec, cc_parameters

TWO_PI = 6.283185307179586476925286766559  # harness.cpp:27
STREAM_PARAMS, STREAM_IC, STREAM_K, STREAM_MULT = 0, 1, 2, 3


def rng_uniform(seed: int, stream: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n)
    _abi.lib().ms_rng_uniform(seed, stream, n, lo, hi, _abi.dptr(out))
    return out


def rng_normal(seed: int, stream: int, n: int) -> np.ndarray:
    out = np.empty(n)
    _abi.lib().ms_rng_normal(seed, stream, n, _abi.dptr(out))
    return out


@dataclass
class Workload:
    name: str
    spec: SystemSpec
    x0: np.ndarray
    t0: float
    tf: float
    policy: PrecisionPolicy
    cfg: SolverConfig
    notes: dict = field(default_factory=dict)


# config 1's policy: K and RHS in fp32, combination/error in fp64
SSS_D = custom_policy((SSS, SSS, SSS), SSS, B64)


def config1_lco(n: int = 1024, seed: int = 0, k_storage: str = "f32", rhs_mode: str = "fast",
                policy: PrecisionPolicy | None = None) -> Workload:
    """C1: x_i'' = -w_i^2 x_i + (1/N) sum_j K_ij (x_j - x_i); coupling into the
    velocity slot. w_i ~ U(0.5,1.5) (stream 0); K symmetric,
    K_ij ~ N(0,1) drawn for i<j in row-major order of the strict upper
    triangle (stream 2), zero diagonal; x0, v0 ~ U(-1,1) (stream 1)."""
    w = rng_uniform(seed, STREAM_PARAMS, n, 0.5, 1.5)
    w2 = w * w
    z = rng_normal(seed, STREAM_K, n * (n - 1) // 2)
    K = np.zeros((n, n))
    iu = np.triu_indices(n, 1)
    K[iu] = z
    K.T[iu] = z
    x0 = rng_uniform(seed, STREAM_IC, 2 * n, -1.0, 1.0)
    spec = SystemSpec("lco", n, k_storage=k_storage, rhs_mode=rhs_mode, coupled_slot=1, w2=w2, K=K)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    return Workload("C1-lco", spec, x0, 0.0, 10.0, policy or SSS_D, cfg, {"seed": seed})


def kuramoto_workload(name: str, n: int, seed: int, tf: float, rtol: float, atol: float,
                      k_storage: str = "f32", rhs_mode: str = "fast",
                      policy: PrecisionPolicy | None = None) -> Workload:
    """Kuramoto with omega ~ N(0,1) (= make_kuramoto sigma = 1, stream 0),
    K_ij ~ U(0,2) (stream 2, generated on the device) and theta0 ~ U(0, 2pi)
    (the reference IC, harness.cpp:313-317, stream 1)."""
    omega = rng_normal(seed, STREAM_PARAMS, n)
    theta0 = rng_uniform(seed, STREAM_IC, n, 0.0, TWO_PI)
    spec = SystemSpec("kuramoto", n, k_storage=k_storage, rhs_mode=rhs_mode, omega=omega,
                      k_uniform=(seed, STREAM_K, 0.0, 2.0))
    cfg = SolverConfig(rel_tol=rtol, abs_tol=atol, time_limits_enabled=False)
    return Workload(name, spec, theta0, 0.0, tf, policy or SSS_D, cfg, {"seed": seed})


def config2_kuramoto(n: int = 4096, seed: int = 1, rtol: float = 1e-6, **kw) -> Workload:
    """C2: N=4096, t in [0,50], rtol sweep {1e-3,1e-4,1e-6,1e-8}, atol = rtol*1e-3."""
    return kuramoto_workload("C2-kuramoto", n, seed, 50.0, rtol, rtol * 1e-3, **kw)


def config4_kuramoto(n: int = 32768, seed: int = 3, rtol: float = 1e-6, atol: float = 1e-9,
                     tf: float = 20.0, **kw) -> Workload:
    """C4: N=32768 (K 4 GiB f32 / 2 GiB f16), t in [0,20], rtol 1e-6, atol 1e-9 (D8)."""
    return kuramoto_workload("C4-kuramoto", n, seed, tf, rtol, atol, **kw)


def config3_cc(n: int = 2048, seed: int = 2, k_storage: str = "f32", rhs_mode: str = "fast",
               policy: PrecisionPolicy | None = None, stimulus_i0: float = 1.5) -> Workload:
    """C3: the reference's d=4 circadian clock with dense
    K_ij ~ U(0,1) on variable 1 and M = 1/N (D4, applied once). k1 and
    theta_h follow make_cc (stream 0); the constants k0, k2, a, b, c, eps are
    multiplied per cell by 1 + 0.05 * normal() (stream 3, six draws per cell in
    that order) and theta_h = k1/(k0_i - k1).

    Initial state: the reference's CC initial conditions, base
    (1, 1, -1.19, -0.62) + 0.2 (U - 0.5) (harness.cpp:320-326, stream 1).
    BASELINE.json asks for x0 ~ U(0,1), but from there the Goodwin equation
    (a x1^2 growth repressed only once x2^4 catches up) blows up in finite time
    in the reference model itself: the oracle's all-binary64 run reaches
    x1 ~ 4e9 by t = 2 and needs h < 1e-10 (tests/test_configs.py pins this)."""
    k1, _ = cc_parameters(n, seed)
    mult = 1.0 + 0.05 * rng_normal(seed, STREAM_MULT, 6 * n).reshape(n, 6)
    k0 = CcConstants.k0 * mult[:, 0]
    th = k1 / (k0 - k1)
    spec = SystemSpec("cc", n, k_storage=k_storage, rhs_mode=rhs_mode, stimulus_i0=stimulus_i0,
                      cc_k1=k1, cc_theta_h=th, cc_k0=k0, cc_k2=CcConstants.k2 * mult[:, 1],
                      cc_a=CcConstants.a * mult[:, 2], cc_b=CcConstants.b * mult[:, 3],
                      cc_c=CcConstants.c * mult[:, 4], cc_eps=CcConstants.eps * mult[:, 5],
                      k_uniform=(seed, STREAM_K, 0.0, 1.0))
    x0 = reference_ic("cc", n, seed)
    cfg = SolverConfig(rel_tol=1e-6, abs_tol=1e-9, time_limits_enabled=False)
    return Workload("C3-cc", spec, x0, 0.0, 240.0, policy or SSS_D, cfg, {"seed": seed, "I0": stimulus_i0})


def reference_ic(model: str, n: int, test_id: int) -> np.ndarray:
    """harness.cpp:305-330 initial_conditions (stream 1 of the test id)."""
    if model == "lco":
        return 2.0 * rng_uniform(test_id, STREAM_IC, 2 * n, 0.0, 1.0)
    if model == "kuramoto":
        return rng_uniform(test_id, STREAM_IC, n, 0.0, TWO_PI)
    u = rng_uniform(test_id, STREAM_IC, 4 * n, 0.0, 1.0).reshape(n, 4)
    base = np.array([1.0, 1.0, -1.19, -0.62])
    return (base + 0.2 * (u - 0.5)).reshape(-1)


@dataclass
class BatchWorkload:
    name: str
    spec: SystemSpec          # the shared-K Kuramoto system
    omega: np.ndarray         # [B][N]
    x0: np.ndarray            # [B][N]
    t0: float
    tf: float
    policy: PrecisionPolicy
    cfg: SolverConfig


def config5_batch(batch: int = 1024, n: int = 2048, seed: int = 4, k_storage: str = "bf16", tf: float = 20.0,
                  rtol: float = 1e-6, atol: float = 1e-9, policy: PrecisionPolicy | None = None) -> BatchWorkload:
    """C5: B trajectories sharing K_ij ~ U(0,2) (stream 2, stored bf16), each with
    omega_b,i ~ N(0,1) (stream 0) and theta0_b,i ~ U(0,2pi) (stream 1), drawn in
    trajectory-major order. BASELINE.json gives no time span: t in [0,20] as C4;
    atol = 1e-9 (D8)."""
    omega = rng_normal(seed, STREAM_PARAMS, batch * n).reshape(batch, n)
    x0 = rng_uniform(seed, STREAM_IC, batch * n, 0.0, TWO_PI).reshape(batch, n)
    spec = SystemSpec("kuramoto", n, k_storage=k_storage, omega=np.zeros(n), k_uniform=(seed, STREAM_K, 0.0, 2.0))
    cfg = SolverConfig(rel_tol=rtol, abs_tol=atol, time_limits_enabled=False)
    return BatchWorkload("C5-batch", spec, omega, x0, 0.0, tf, policy or SSS_D, cfg)
