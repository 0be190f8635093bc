"""CPU engine with the segment protocol of ms_loop_* (TEST INFRASTRUCTURE).

It replays, in numpy with the same IEEE operation order, what the device
segments do for a row-sharded BS3(2) solve — each rank evaluates only its own
rows of the RHS (through the oracle) and leaves the other rows as NaN, so the
all-gather is what makes the state whole — and lets the multi-process driver
(paper_2605_23727_b200.sharded.ShardedSolver) be tested with gloo on CPU.
"""
from __future__ import annotations

import math

import numpy as np

from paper_2605_23727_b200.precision import B32, DDD
from paper_2605_23727_b200.sharded import Exchange
from paper_2605_23727_b200.solver import FlopTally, SolveResult, SolveStatus, StepRecord

A21, A32 = 0.5, 0.75
A41, A42, A43 = 2.0 / 9.0, 1.0 / 3.0, 4.0 / 9.0
BT = (7.0 / 24.0, 0.25, 1.0 / 3.0, 0.125)


def seq_sum(v):
    return float(np.cumsum(v)[-1]) if v.size else 0.0


class ShardCpuEngine:
    def __init__(self, orc, row0: int, row1: int, d: int):
        self.orc = orc
        self.r0, self.r1, self.d = row0, row1, d

    # ---- helpers -------------------------------------------------------------------
    def _rhs(self, x, sp, out):
        full = self.orc.eval_rhs(0.0, x, sp)
        out[:] = np.nan
        a, b = self.r0 * self.d, self.r1 * self.d
        out[a:b] = full[a:b]
        self.evals += 1
        return Exchange(True, out, a, b - a, out.size)

    def begin(self, x0, t0, tf, policy, cfg, cap):
        self.x0 = np.array(x0, dtype=np.float64)
        self.n = self.x0.size
        self.t0, self.tf, self.pol, self.cfg = t0, tf, policy, cfg
        self.store32 = policy.storage == B32
        self.k = [np.zeros(self.n) for _ in range(5)]
        self.t, self.done_, self.status = t0, False, SolveStatus.Completed
        self.n_acc = self.n_fail = self.evals = 0
        self.need_k1 = False
        self.log = []
        eps = 2.0 ** -23 if policy.lowest_format() == B32 else 2.0 ** -52
        self.h_min = cfg.h_min_factor * eps

    def segment_count(self, lst):
        return 4 if lst == 0 else 4

    def done(self):
        return self.done_

    def _loop_check(self):  # solver.cpp:273-314
        c = self.cfg
        if self.n_acc + self.n_fail >= c.max_iterations:
            self.status, self.done_ = SolveStatus.MaxIterations, True
        elif self.n_fail >= c.max_failed_steps:
            self.status, self.done_ = SolveStatus.MaxFailedSteps, True
        elif self.h <= self.h_min:
            self.status, self.done_ = SolveStatus.StepTooSmall, True
        if self.done_:
            return
        self.last = False
        self.h_att = self.h
        if self.t + 1.01 * self.h >= self.tf:
            self.h_att, self.last = self.tf - self.t, True

    def run_segment(self, lst, idx):
        c = self.cfg
        none = Exchange(False, None, 0, 0, 0)
        if lst == 0:
            if idx == 0:
                return self._rhs(self.x0, DDD, self.k[1])
            if idx == 1:
                f0 = self.k[1]
                self.cap = (self.tf - self.t0) / 10.0
                self.skip2 = False
                if not np.all(np.isfinite(f0)):
                    self.h, self.skip2 = math.nan, True
                    return none
                sk = c.abs_tol + c.rel_tol * np.abs(self.x0)
                inv_n = 1.0 / self.n
                d0 = math.sqrt(seq_sum((self.x0 / sk) ** 2) * inv_n)
                self.d1 = math.sqrt(seq_sum((f0 / sk) ** 2) * inv_n)
                if self.d1 < 1e-12:
                    self.h, self.skip2 = self.cap, True
                    return none
                self.h1 = 0.01 * d0 / self.d1 if d0 >= 1e-8 else 1e-6
                return self._rhs(self.x0 + self.h1 * f0, DDD, self.k[2])
            if idx == 2:
                if not self.skip2:
                    f0, f1 = self.k[1], self.k[2]
                    if not np.all(np.isfinite(f1)):
                        h2 = self.h1 * 1e-3
                    else:
                        sk = c.abs_tol + c.rel_tol * np.abs(self.x0)
                        d2 = math.sqrt(seq_sum(((f1 - f0) / sk) ** 2) * (1.0 / self.n)) / self.h1
                        der = max(self.d1, d2)
                        h2 = self.cap if der < 1e-12 else math.pow(0.01 / der, 1.0 / 4.0)
                    self.h = min(100.0 * self.h1, h2, self.cap)
                if not math.isfinite(self.h):
                    self.status, self.done_ = SolveStatus.NonFinite, True
                    return none
                self.x = self.x0.astype(np.float32).astype(np.float64) if self.store32 else self.x0.copy()
                return self._rhs(self.x, self.pol.first_step_k1, self.k[0])
            if idx == 3:
                if self.done_:
                    return none
                if not np.all(np.isfinite(self.k[0])):
                    self.status, self.done_ = SolveStatus.NonFinite, True
                    return none
                self._loop_check()
                return none
        if self.done_:
            return none
        k1, k2, k3 = self.k[0], self.k[1], self.k[2]
        h, x = self.h_att, self.x
        if idx == 0:
            if self.need_k1:
                self.evals += 1  # elided recompute (k1 row == k4 row), still counted
                self.need_k1 = False
            self.nf = False
            return self._rhs(x + h * (A21 * k1), self.pol.stage(2), self.k[1])
        if idx == 1:
            self.nf = not np.all(np.isfinite(k2))
            if self.nf:
                return none
            return self._rhs(x + h * (A32 * k2), self.pol.stage(3), self.k[2])
        if idx == 2:
            self.nf = self.nf or not np.all(np.isfinite(k3))
            if self.nf:
                return none
            self.xn = x + h * (((A41 * k1) + (A42 * k2)) + (A43 * k3))
            if self.store32:
                hf = np.float32(h)
                acc = x.astype(np.float32)
                for a, km in ((A41, k1), (A42, k2), (A43, k3)):
                    acc = acc + np.float32(hf * np.float32(a)) * km.astype(np.float32)
                self.xs = acc.astype(np.float64)
            else:
                self.xs = self.xn
            return self._rhs(self.xs, self.pol.stage(4), self.k[4])
        # finalize (solver.cpp:188-214, 321-342)
        k4 = self.k[4]
        err, acc = math.nan, False
        if self.nf or not np.all(np.isfinite(k4)):
            hn = h * c.fac_min * 0.5
        else:
            xt = x + h * ((((BT[0] * k1) + (BT[1] * k2)) + (BT[2] * k3)) + (BT[3] * k4))
            if not (np.all(np.isfinite(self.xn)) and np.all(np.isfinite(xt)) and np.all(np.isfinite(self.xs))):
                hn = h * c.fac_min * 0.5
            else:
                w = np.maximum(np.maximum(np.abs(x), np.abs(self.xn)), c.abs_tol / c.rel_tol)
                err = float(np.max(np.abs(self.xn - xt) / w))
                acc = err <= c.rel_tol
                if err <= 0.0:
                    hn = h * c.fac_max
                else:
                    fac = c.safety * math.pow(c.rel_tol / err, c.controller_exponent)
                    hn = h * min(max(fac, c.fac_min), c.fac_max)
        self.log.append(StepRecord(self.t, h, err, acc))
        if acc:
            self.n_acc += 1
            self.x = self.xs
            tn = self.t + h
            self.t = self.tf if self.last else (float(np.float32(tn)) if self.store32 else tn)
            self.k[0] = k4.copy()
            self.h = hn
            if self.t >= self.tf:
                self.status, self.done_ = SolveStatus.Completed, True
        else:
            self.n_fail += 1
            self.h = hn
            self.need_k1 = True
        if not self.done_:
            self._loop_check()
        return none

    def end(self):
        return SolveResult(self.status, self.x.copy(), self.t, self.n_acc, self.n_fail, list(self.log),
                           FlopTally(0, 0, self.evals), 0.0, len(self.log))
