"""Precision formats and per-stage policies — mirror of
proj/include/mixedstep/precision.hpp:11-80 and proj/src/precision.cpp:9-42.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass, field

import numpy as np

from . import _abi


class FloatFormat(enum.IntEnum):  # precision.hpp:11
    Binary32 = _abi.MS_BINARY32
    Binary64 = _abi.MS_BINARY64


def machine_epsilon(p: FloatFormat) -> float:  # precision.hpp:14-16
    return 2.0 ** -23 if p == FloatFormat.Binary32 else 2.0 ** -52


def round_to(x, p: FloatFormat):  # precision.hpp:21-24
    if p == FloatFormat.Binary64:
        return x
    with np.errstate(over="ignore"):
        return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def wider_of(a: FloatFormat, b: FloatFormat) -> FloatFormat:  # precision.hpp:26-30
    return FloatFormat.Binary64 if FloatFormat.Binary64 in (a, b) else FloatFormat.Binary32


@dataclass(frozen=True)
class StagePrecision:  # precision.hpp:36-42
    f_prec: FloatFormat
    sum_prec: FloatFormat
    g_prec: FloatFormat

    def c(self) -> _abi.StagePrec:
        return _abi.StagePrec(int(self.f_prec), int(self.sum_prec), int(self.g_prec), 0)


B32, B64 = FloatFormat.Binary32, FloatFormat.Binary64
kAllBinary64 = StagePrecision(B64, B64, B64)
kAllBinary32 = StagePrecision(B32, B32, B32)
SSS, DDS, DDD = kAllBinary32, StagePrecision(B64, B64, B32), kAllBinary64


class PolicyVariant(enum.IntEnum):  # precision.hpp:51
    Single = _abi.MS_SINGLE
    Mixed1 = _abi.MS_MIXED1
    Mixed2 = _abi.MS_MIXED2
    Double = _abi.MS_DOUBLE
    Custom = _abi.MS_CUSTOM


@dataclass(frozen=True)
class PrecisionPolicy:  # precision.hpp:61-74
    variant: PolicyVariant
    per_stage: tuple  # rows for stages k2, k3, k4
    first_step_k1: StagePrecision
    storage: FloatFormat = FloatFormat.Binary64

    def stage(self, ell: int) -> StagePrecision:
        return self.per_stage[ell - 2]

    def lowest_format(self) -> FloatFormat:  # precision.cpp:9-20
        if self.storage == B32:
            return B32
        for sp in (*self.per_stage, self.first_step_k1):
            if B32 in (sp.f_prec, sp.sum_prec, sp.g_prec):
                return B32
        return B64

    def c(self) -> _abi.Policy:
        p = _abi.Policy()
        for i, sp in enumerate(self.per_stage):
            p.per_stage[i] = sp.c()
        p.first_step_k1 = self.first_step_k1.c()
        p.storage = int(self.storage)
        p.variant = int(self.variant)
        return p


def policy_for(v: PolicyVariant) -> PrecisionPolicy:  # precision.cpp:22-42
    rows = {
        PolicyVariant.Single: (SSS, SSS, SSS),
        PolicyVariant.Mixed1: (SSS, SSS, DDS),
        PolicyVariant.Mixed2: (DDS, DDS, DDS),
        PolicyVariant.Double: (DDD, DDD, DDD),
    }
    if v not in rows:
        raise ValueError(f"policy_for: no table row for {v!r}")
    r = rows[v]
    return PrecisionPolicy(v, r, r[2], B32 if v == PolicyVariant.Single else B64)


def custom_policy(rows, first_step_k1=None, storage=FloatFormat.Binary64) -> PrecisionPolicy:
    """Any per-stage assignment, e.g. config 1's
    ``{SSS, SSS, SSS}`` rows with binary64 storage."""
    rows = tuple(rows)
    return PrecisionPolicy(PolicyVariant.Custom, rows, first_step_k1 or rows[2], storage)


def variant_name(v: PolicyVariant) -> str:
    return v.name


def variant_from_name(name: str):
    for v in (PolicyVariant.Single, PolicyVariant.Mixed1, PolicyVariant.Mixed2, PolicyVariant.Double):
        if name in (v.name, v.name.lower()):
            return v
    return None
