"""Coupled systems on the B200 — mirror of proj/include/mixedstep/systems.hpp
(``CoupledSystem`` :60-103, factories :107-119) backed by the C-ABI.

A :class:`DeviceSystem` owns its device memory. The coupling matrix K is
converted to its storage format (f32/f16/bf16) and uploaded once, at creation
(or generated on the device from SplitMix64 for large N), and is read-only
afterwards. ``eval_rhs`` is the drop-in for ``CoupledSystem::eval_rhs``.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _abi
from .precision import StagePrecision

MODEL_IDS = {"lco": _abi.MS_MODEL_LCO, "kuramoto": _abi.MS_MODEL_KURAMOTO, "cc": _abi.MS_MODEL_CC,
             "scalar_exp": _abi.MS_MODEL_SCALAR_EXP, "scalar_zero": _abi.MS_MODEL_SCALAR_ZERO,
             "scalar_nan": _abi.MS_MODEL_SCALAR_NAN}
K_STORAGE = {"scalar": _abi.MS_K_SCALAR, "f32": _abi.MS_K_F32, "f16": _abi.MS_K_F16, "bf16": _abi.MS_K_BF16}
RHS_MODES = {"fast": _abi.MS_RHS_FAST, "faithful": _abi.MS_RHS_FAITHFUL, "ordered": _abi.MS_RHS_ORDERED}
DIMS = {"lco": 2, "kuramoto": 1, "cc": 4, "scalar_exp": 1, "scalar_zero": 1, "scalar_nan": 1}


# reference CcConstants, systems.hpp:32-43
class CcConstants:
    k0 = 2.0
    k2 = 0.144832
    k3 = 2.0
    a = 2.0
    b = 0.7
    c = 0.8
    hill_h = 4
    eps = 0.228249
    k1_mean = 0.339278
    k1_sdev = 0.090909


def _f64(a):
    if a is None:
        return None
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class SystemSpec:
    """Everything ``ms_system_create`` needs (the arguments of the reference
    factories plus the dense-coupling extension)."""
    model: str
    n_agents: int
    k_storage: str = "scalar"
    rhs_mode: str = "fast"
    coupled_slot: int = 0
    coupling_k: float = 1.0
    stimulus_i0: float = 0.0
    m: Optional[np.ndarray] = None
    omega: Optional[np.ndarray] = None
    w2: Optional[np.ndarray] = None
    cc_k1: Optional[np.ndarray] = None
    cc_theta_h: Optional[np.ndarray] = None
    cc_k0: Optional[np.ndarray] = None
    cc_k2: Optional[np.ndarray] = None
    cc_a: Optional[np.ndarray] = None
    cc_b: Optional[np.ndarray] = None
    cc_c: Optional[np.ndarray] = None
    cc_eps: Optional[np.ndarray] = None
    K: Optional[np.ndarray] = None            # host N x N (float64 or float32)
    k_uniform: Optional[tuple] = None         # (seed, stream, lo, hi): device SplitMix64 fill
    device: int = 0
    row_begin: int = 0
    row_end: int = 0

    @property
    def dim(self) -> int:
        return DIMS[self.model]

    def desc(self):
        """Build the C descriptor; returns (desc, keepalive)."""
        keep = []
        d = _abi.SystemDesc()
        d.model = MODEL_IDS[self.model]
        d.n_agents = int(self.n_agents)
        d.coupled_slot = int(self.coupled_slot)
        d.k_storage = K_STORAGE[self.k_storage]
        d.rhs_mode = RHS_MODES[self.rhs_mode]
        d.device = int(self.device)
        d.row_begin = int(self.row_begin)
        d.row_end = int(self.row_end)
        d.coupling_k = float(self.coupling_k)
        d.stimulus_i0 = float(self.stimulus_i0)
        for name in ("m", "omega", "w2", "cc_k1", "cc_theta_h", "cc_k0", "cc_k2", "cc_a", "cc_b", "cc_c", "cc_eps"):
            arr = _f64(getattr(self, name))
            if arr is not None:
                keep.append(arr)
                setattr(d, name, _abi.dptr(arr))
        if self.K is not None:
            K = np.asarray(self.K)
            if K.dtype == np.float32:
                K = np.ascontiguousarray(K)
                d.k_host_dtype = _abi.MS_HOST_F32
            else:
                K = np.ascontiguousarray(K, dtype=np.float64)
                d.k_host_dtype = _abi.MS_HOST_F64
            if K.shape != (self.n_agents, self.n_agents):
                raise ValueError("K must be N x N")
            keep.append(K)
            d.K = K.ctypes.data_as(C.c_void_p)
        return d, keep


class DeviceSystem:
    """A coupled system resident on one B200 (``CoupledSystem`` drop-in)."""

    def __init__(self, spec: SystemSpec):
        L = _abi.lib()
        self.spec = spec
        desc, keep = spec.desc()
        h = C.c_void_p()
        _abi.check(L.ms_system_create(C.byref(desc), C.byref(h)), "ms_system_create")
        self._h = h
        del keep
        if spec.k_uniform is not None:
            seed, stream, lo, hi = spec.k_uniform
            _abi.check(L.ms_system_fill_k_uniform(self._h, seed, stream, lo, hi), "ms_system_fill_k_uniform")

    @property
    def handle(self) -> C.c_void_p:
        if self._h is None:
            raise ValueError("system destroyed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            _abi.lib().ms_system_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # CoupledSystem accessors (systems.hpp:64-71)
    def dim(self) -> int:
        return self.spec.dim

    def agents(self) -> int:
        return self.spec.n_agents

    def size(self) -> int:
        return self.spec.dim * self.spec.n_agents

    def flop_profile(self):
        out = (C.c_int64 * 4)()
        _abi.check(_abi.lib().ms_system_flop_profile(self.handle, out), "flop_profile")
        return tuple(out)

    def get_k(self) -> np.ndarray:
        rows = (self.spec.row_end or self.spec.n_agents) - self.spec.row_begin
        out = np.empty((rows, self.spec.n_agents))
        _abi.check(_abi.lib().ms_system_get_k(self.handle, _abi.dptr(out)), "get_k")
        return out

    def eval_rhs(self, t: float, x, sp: StagePrecision, out: Optional[np.ndarray] = None) -> np.ndarray:
        """CoupledSystem::eval_rhs (systems.hpp:79-86): host in, host out."""
        x = _f64(x)
        if x.shape != (self.size(),):
            raise ValueError("eval_rhs: state length must be d*N")
        if out is None:
            out = np.empty_like(x)
        _abi.check(_abi.lib().ms_eval_rhs(self.handle, float(t), _abi.dptr(x), sp.c(), _abi.dptr(out)),
                   "ms_eval_rhs")
        return out


# ---- reference factories (systems.cpp:209-268) -----------------------------
def _rng_normal(seed: int, stream: int, n: int) -> np.ndarray:
    out = np.empty(n)
    _abi.lib().ms_rng_normal(seed, stream, n, _abi.dptr(out))
    return out


def make_lco(n_agents: int, seed: int = 0, **kw) -> DeviceSystem:
    """Harmonic oscillators coupled through the position slot, M = (1/N, 0)."""
    if n_agents < 1:
        raise ValueError("make_lco: N must be >= 1")
    return DeviceSystem(SystemSpec("lco", n_agents, coupling_k=1.0, **kw))


def kuramoto_omega(n_agents: int, sigma: float, seed: int) -> np.ndarray:
    """omega_i = sigma * normal() from SplitMix64(seed, stream 0) (systems.cpp:230-231)."""
    return sigma * _rng_normal(seed, 0, n_agents)


def make_kuramoto(n_agents: int, sigma: float, coupling_k: float, seed: int, **kw) -> DeviceSystem:
    if n_agents < 1:
        raise ValueError("make_kuramoto: N must be >= 1")
    if sigma < 0.0:
        raise ValueError("make_kuramoto: sigma must be >= 0")
    return DeviceSystem(SystemSpec("kuramoto", n_agents, coupling_k=coupling_k,
                                   omega=kuramoto_omega(n_agents, sigma, seed), **kw))


def cc_parameters(n_agents: int, seed: int):
    """k1 ~ N(0.339278, 0.090909^2) redrawn into (0.05, 1.95), theta_h = k1/(k0-k1)
    (systems.cpp:251-259), from SplitMix64(seed, stream 0)."""
    k1 = np.empty(n_agents)
    # sequential draws with redraw: pull normals in blocks from one generator
    buf = _rng_normal(seed, 0, 4 * n_agents + 64)
    pos = 0
    for i in range(n_agents):
        while True:
            if pos >= buf.size:  # same generator, longer prefix
                buf = _rng_normal(seed, 0, 2 * buf.size)
            v = CcConstants.k1_mean + CcConstants.k1_sdev * buf[pos]
            pos += 1
            if 0.05 < v < 1.95:
                break
        k1[i] = v
    th = k1 / (CcConstants.k0 - k1)
    return k1, th


def make_cc(n_agents: int, coupling_k: float, stimulus_i0: float, seed: int, **kw) -> DeviceSystem:
    if n_agents < 1:
        raise ValueError("make_cc: N must be >= 1")
    k1, th = cc_parameters(n_agents, seed)
    return DeviceSystem(SystemSpec("cc", n_agents, coupling_k=coupling_k, stimulus_i0=stimulus_i0,
                                   cc_k1=k1, cc_theta_h=th, **kw))


def scalar_fixture(kind: str) -> DeviceSystem:
    """The reference test fixtures ScalarExp / ScalarZero / ScalarNan
    (proj/tests/test_support.hpp:21-53) as device systems."""
    return DeviceSystem(SystemSpec("scalar_" + kind, 1))
