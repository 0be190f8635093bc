"""Device eval_rhs (the all-pairs hot path, systems.cpp:30-64) against the CPU
oracle on the same seeded inputs, through the C-ABI.

FAITHFUL mode sums in the reference's exact order: transcendental-free paths
(LCO) must be bit-identical; sin/atan paths may differ by the libm-vs-device
ulp of G only. FAST mode reorders the j-sum (blocked warp tree, Kuramoto
sin/cos split): it is held to the worst-case bound of reordering a sum in the
accumulation format, TOL = 2 N eps_SS mw sum_j |G_ij| + 4 eps_WS |out|.
"""
import itertools

import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200.configs import TWO_PI, rng_uniform
from paper_2605_23727_b200.precision import B32, B64, StagePrecision
from paper_2605_23727_b200.systems import DeviceSystem, SystemSpec

pytestmark = pytest.mark.gpu

ALL_ROWS = [StagePrecision(f, s, g) for f, s, g in itertools.product((B32, B64), repeat=3)]


def eps(fmt):
    return 2.0 ** -23 if fmt == B32 else 2.0 ** -52


def pair(spec):
    return DeviceSystem(spec), O.OracleSystem(spec)


def kur_spec(n, k_storage="f32", mode="fast", seed=11, coupling_k=1.0):
    om = rng_uniform(seed, 0, n, -1.0, 1.0)
    kw = {} if k_storage == "scalar" else {"k_uniform": (seed, 2, 0.0, 2.0)}
    return SystemSpec("kuramoto", n, k_storage=k_storage, rhs_mode=mode, omega=om, coupling_k=coupling_k, **kw)


def reorder_tol(sp, n, out, gabs_rowsum):
    ws = B32 if (sp.f_prec == B32 and sp.sum_prec == B32) else B64
    tol = 2.0 * n * eps(sp.sum_prec) * gabs_rowsum / n + 4.0 * eps(ws) * np.abs(out)
    if sp.g_prec == B32:
        tol = tol + 4.0 * eps(B32) * gabs_rowsum / n  # product rounded in GS
    return tol + 1e-300


@pytest.mark.parametrize("n", [1, 2, 17, 100, 513])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
def test_lco_reference_form_faithful_bitwise(gpu, n, sp):
    """make_lco (systems.cpp:209-218) + eval_core order: bit-identical."""
    spec = SystemSpec("lco", n, rhs_mode="faithful", coupling_k=1.0)
    dev, orc = pair(spec)
    x = rng_uniform(99, 0, 2 * n, -2.0, 2.0)
    assert np.array_equal(dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp))


@pytest.mark.parametrize("k_storage", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
def test_lco_config1_dense_faithful_bitwise(gpu, k_storage, sp):
    """C1 form (coupling on the velocity slot, w_i^2, dense symmetric K)."""
    from paper_2605_23727_b200.configs import config1_lco
    w = config1_lco(n=96, k_storage=k_storage, rhs_mode="faithful")
    dev, orc = pair(w.spec)
    assert np.array_equal(dev.get_k(), orc.get_k())
    assert np.array_equal(dev.eval_rhs(0.0, w.x0, sp), orc.eval_rhs(0.0, w.x0, sp))


@pytest.mark.parametrize("n", [1, 7, 64, 300])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
def test_kuramoto_faithful(gpu, n, sp):
    """Order-faithful Kuramoto: only the sin of G can differ (<= 1 ulp of G per pair)."""
    spec = kur_spec(n, "f32", "faithful")
    dev, orc = pair(spec)
    x = rng_uniform(5, 1, n, 0.0, TWO_PI)
    a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
    gsum = np.abs(orc.get_k()).sum(axis=1)
    ws = B32 if (sp.f_prec == B32 and sp.sum_prec == B32) else B64
    # a differing sin moves one term by <= 2 ulp(GS); the sequential sum can
    # then round differently at each later add (<= N ulp(SS) of the row scale)
    tol = (2.0 * eps(sp.g_prec) + 2.0 * n * eps(sp.sum_prec)) * gsum / n + 4.0 * eps(ws) * np.abs(b)
    assert np.all(np.abs(a - b) <= tol + 1e-300), float(np.max(np.abs(a - b) / (tol + 1e-300)))


@pytest.mark.parametrize("k_storage", ["scalar", "f32", "f16", "bf16"])
@pytest.mark.parametrize("n", [1, 3, 64, 1000, 4096])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
def test_kuramoto_fast_split(gpu, k_storage, n, sp):
    """Fast path (sin/cos split, blocked sum) vs the oracle's split semantics."""
    if n == 4096 and k_storage == "bf16" and sp.g_prec == B64:
        pytest.skip("covered by the other storage formats")
    spec = kur_spec(n, k_storage, "fast", coupling_k=1.3)
    dev, orc = pair(spec)
    x = rng_uniform(6, 1, n, 0.0, 50.0)
    a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
    gsum = (np.abs(orc.get_k()).sum(axis=1) if k_storage != "scalar" else np.full(n, 1.3 * n)) * 2.0
    tol = reorder_tol(sp, n, b, gsum)
    assert np.all(np.abs(a - b) <= tol), float(np.max(np.abs(a - b) / tol))


@pytest.mark.parametrize("mode", ["fast", "faithful"])
@pytest.mark.parametrize("k_storage", ["scalar", "f32", "f16"])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
def test_cc(gpu, mode, k_storage, sp):
    from paper_2605_23727_b200.configs import config3_cc
    w = config3_cc(n=200, k_storage=k_storage if k_storage != "scalar" else "f32", rhs_mode=mode)
    spec = w.spec
    if k_storage == "scalar":
        spec.k_storage, spec.k_uniform, spec.coupling_k = "scalar", None, 0.8
    dev, orc = pair(spec)
    x = w.x0
    a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
    n = spec.n_agents
    K = orc.get_k() if k_storage != "scalar" else np.full((n, n), 0.8)
    pref = 2.0 * 2.0 * 2.0  # |k0 th a/(th+x2^4)| <= k0 a
    gsum = np.abs(K).sum(axis=1) * 1.6 * pref
    tol = np.repeat(reorder_tol(sp, n, b[0::4], gsum), 4)
    tol = np.maximum(tol, 4.0 * eps(B32 if sp.f_prec == B32 else B64) * (np.abs(b) + 1.0))
    assert np.all(np.abs(a - b) <= tol), float(np.max(np.abs(a - b) / tol))
    # uncoupled slots are F alone: identical formula, identical order
    for s in (1, 2, 3):
        assert np.array_equal(a[s::4], b[s::4])


def test_device_k_generation_bit_identical(gpu):
    for ks in ("f32", "f16", "bf16"):
        spec = kur_spec(333, ks)
        dev, orc = pair(spec)
        assert np.array_equal(dev.get_k(), orc.get_k())


def test_host_k_upload_bit_identical(gpu):
    n = 77
    K = rng_uniform(3, 2, n * n, -3.0, 3.0).reshape(n, n)
    for ks in ("f32", "f16", "bf16"):
        for host in (K, K.astype(np.float32)):
            spec = SystemSpec("kuramoto", n, k_storage=ks, omega=np.zeros(n), K=host)
            dev, orc = pair(spec)
            assert np.array_equal(dev.get_k(), orc.get_k())


def test_row_sharded_rhs_is_bitwise_the_unsharded_rows(gpu):
    """Each row's reduction order depends only on N: a row-range handle
    (one rank of a row-sharded K) reproduces the full evaluation bitwise."""
    n = 1000
    full = DeviceSystem(kur_spec(n, "f32"))
    x = rng_uniform(8, 1, n, 0.0, TWO_PI)
    ref = full.eval_rhs(0.0, x, StagePrecision(B32, B32, B32))
    for r0, r1 in ((0, 250), (250, 500), (500, 999), (999, 1000)):
        spec = kur_spec(n, "f32")
        spec.row_begin, spec.row_end = r0, r1
        part = DeviceSystem(spec)
        got = part.eval_rhs(0.0, x, StagePrecision(B32, B32, B32))
        assert np.array_equal(got[r0:r1], ref[r0:r1])


@pytest.mark.parametrize("k_storage", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("n", [1000, 4096, 8200])
@pytest.mark.parametrize("sp", [StagePrecision(B32, B32, B32), StagePrecision(B64, B64, B32),
                                StagePrecision(B64, B64, B64)], ids=str)
def test_tma_sweep_bitwise_equals_register_sweep(gpu, k_storage, n, sp, monkeypatch):
    """The TMA-fed K sweep (k_rhs_tma) and the register-fed one (k_rhs_fast)
    assign columns to lanes identically: rows must agree bit for bit."""
    spec = kur_spec(n, k_storage, "fast", coupling_k=1.0)
    dev = DeviceSystem(spec)
    x = rng_uniform(6, 1, n, 0.0, 50.0)
    monkeypatch.setenv("MS_SWEEP", "ldg")
    a = dev.eval_rhs(0.0, x, sp)
    monkeypatch.setenv("MS_SWEEP", "tma")
    b = dev.eval_rhs(0.0, x, sp)
    assert np.array_equal(a, b)
    # and sharded row ranges of the TMA sweep reproduce the full rows
    spec.row_begin, spec.row_end = 3, n - 5
    part = DeviceSystem(spec)
    c = part.eval_rhs(0.0, x, sp)
    assert np.array_equal(c[3:n - 5], b[3:n - 5])


@pytest.mark.parametrize("k_storage", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("n", [1000, 4096])
@pytest.mark.parametrize("sp", [StagePrecision(B32, B32, B32), StagePrecision(B64, B64, B32),
                                StagePrecision(B64, B64, B64)], ids=str)
def test_tile_sweep_bitwise_equals_register_sweep(gpu, k_storage, n, sp, monkeypatch):
    """The 2D-tensor-tiled sweep (one-lane k_rhs_multi, MS_SWEEP=tile) keeps the
    lanes' column order: rows agree bit for bit with the register sweep, also
    on a row-sharded handle."""
    spec = kur_spec(n, k_storage, "fast", coupling_k=1.0)
    dev = DeviceSystem(spec)
    x = rng_uniform(7, 1, n, 0.0, 50.0)
    monkeypatch.setenv("MS_SWEEP", "ldg")
    a = dev.eval_rhs(0.0, x, sp)
    monkeypatch.setenv("MS_SWEEP", "tile")
    b = dev.eval_rhs(0.0, x, sp)
    assert np.array_equal(a, b)
    spec.row_begin, spec.row_end = 5, n - 3
    part = DeviceSystem(spec)
    c = part.eval_rhs(0.0, x, sp)
    assert np.array_equal(c[5:n - 3], b[5:n - 3])


@pytest.mark.parametrize("model", ["lco", "lco_c1", "cc"])
@pytest.mark.parametrize("k_storage", ["scalar", "f32", "f16"])
@pytest.mark.parametrize("sp", [StagePrecision(B32, B32, B32), StagePrecision(B64, B64, B32),
                                StagePrecision(B64, B64, B64)], ids=str)
def test_fused_eval_bitwise_equals_prep_plus_sweep(gpu, model, k_storage, sp, monkeypatch):
    """k_eval_fused (prep + sweep in one launch, small systems) against the
    two-kernel path: identical RHS rows, bit for bit."""
    from paper_2605_23727_b200.systems import SystemSpec
    n = 700
    kw = dict(k_storage=k_storage, rhs_mode="fast", coupling_k=1.3)
    if k_storage != "scalar":
        kw["k_uniform"] = (5, 2, 0.0, 2.0)
    if model == "lco_c1":
        spec = SystemSpec("lco", n, coupled_slot=1, **kw)
    elif model == "kuramoto":
        spec = SystemSpec("kuramoto", n, omega=rng_uniform(1, 0, n, -1.0, 1.0), **kw)
    elif model == "cc":
        from paper_2605_23727_b200.systems import cc_parameters
        k1, th = cc_parameters(n, 3)
        spec = SystemSpec("cc", n, cc_k1=k1, cc_theta_h=th, stimulus_i0=0.2, **kw)
    else:
        spec = SystemSpec(model, n, **kw)
    dev = DeviceSystem(spec)
    x = rng_uniform(9, 1, n * spec.dim, -1.0, 1.0)
    monkeypatch.setenv("MS_FUSE", "off")
    a = dev.eval_rhs(0.0, x, sp)
    monkeypatch.delenv("MS_FUSE")
    b = dev.eval_rhs(0.0, x, sp)
    assert np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("k_storage", ["f32", "f16", "bf16"])
@pytest.mark.parametrize("n", [1000, 4096, 8200])
@pytest.mark.parametrize("sp", [StagePrecision(B32, B32, B32), StagePrecision(B64, B64, B32),
                                StagePrecision(B64, B64, B64)], ids=str)
def test_small_split_sweep_bitwise_equals_register_sweep(gpu, k_storage, n, sp, monkeypatch):
    """The small split-Kuramoto sweep (MS_SWEEP=small: column values staged in
    shared memory, one row per warp, unrolled) against k_rhs_fast."""
    spec = kur_spec(n, k_storage, "fast", coupling_k=1.0)
    dev = DeviceSystem(spec)
    x = rng_uniform(8, 1, n, 0.0, 50.0)
    monkeypatch.setenv("MS_SWEEP", "ldg")
    a = dev.eval_rhs(0.0, x, sp)
    monkeypatch.setenv("MS_SWEEP", "small")
    b = dev.eval_rhs(0.0, x, sp)
    assert np.array_equal(a, b)


@pytest.mark.parametrize("sweep", ["tma", "ldg"])
@pytest.mark.parametrize("case", ["tiny_k", "tiny_theta", "normal"])
@pytest.mark.parametrize("ks", ["f32", "bf16"])
def test_packed_ftz_products_equal_scalar_products(gpu, monkeypatch, sweep, case, ks):
    """The split sweeps' packed FMUL2.FTZ path (ms_common.cuh mac2) against
    the scalar products (MS_SWEEP_PK=off), bit for bit, including inputs where
    a flushing multiply WOULD differ: K entries that are binary32-subnormal
    (the system is flagged at creation, ms_system::k_tiny) and column values
    sin(theta) ~ 1e-30 whose products with K ~ 1e-10 are subnormal (the prep
    flags them, Ctl::pk_off). Rows with omega = 0 expose the subnormal sums in
    the output."""
    from paper_2605_23727_b200.precision import SSS
    n = 96
    om = rng_uniform(5, 0, n, -1.0, 1.0)
    om[:8] = 0.0
    theta = rng_uniform(5, 1, n, 0.0, TWO_PI)
    K = rng_uniform(5, 2, n * n, 0.0, 2.0).reshape(n, n)
    if case == "tiny_k":
        K[:8] = 1e-39 * (1.0 + rng_uniform(5, 3, 8 * n, 0.0, 1.0).reshape(8, n))
    elif case == "tiny_theta":
        K[:8] = 1e-10
        theta = 1e-30 * (1.0 + np.arange(n) / n)
    spec = SystemSpec("kuramoto", n, k_storage=ks, rhs_mode="fast", omega=om, K=K)
    dev = DeviceSystem(spec)
    monkeypatch.setenv("MS_SWEEP", sweep)
    packed = dev.eval_rhs(0.0, theta, SSS)
    monkeypatch.setenv("MS_SWEEP_PK", "off")
    scalar = dev.eval_rhs(0.0, theta, SSS)
    assert np.array_equal(packed, scalar)
    if case != "normal":
        assert np.any(packed[:8] != 0.0)  # the subnormal sums reached the output
    orc = O.OracleSystem(spec)
    ref = orc.eval_rhs(0.0, theta, SSS)
    gsum = np.abs(orc.get_k()).sum(axis=1)
    assert np.all(np.abs(packed - ref) <= reorder_tol(SSS, n, ref, gsum) * 4 + 1e-44)


@pytest.mark.parametrize("n", [1, 31, 300, 4097])
@pytest.mark.parametrize("sp", ALL_ROWS, ids=str)
@pytest.mark.parametrize("ks", ["f32", "f16"])
def test_kuramoto_ordered_mode_is_the_oracle_split(gpu, n, sp, ks):
    """MS_RHS_ORDERED: the split Kuramoto summed in ascending j (k_rhs_seq) is
    the oracle's split form: equal up to the libm ulp of sin/cos (device:
    binary64 sincos rounded once; oracle: glibc). One differing s_j or c_j
    moves every row's binary64 sum by ~K ulp(s_j); binary32 sums absorb it,
    so there nearly every row is bit-identical."""
    spec = kur_spec(n, k_storage=ks, mode="ordered")
    dev, orc = pair(spec)
    x = rng_uniform(3, 1, n, 0.0, TWO_PI)
    a, b = dev.eval_rhs(0.0, x, sp), orc.eval_rhs(0.0, x, sp)
    gsum = np.abs(orc.get_k()).sum(axis=1)
    tol = 8 * eps(sp.g_prec) * gsum / max(n, 1) * 2 + 4 * eps(sp.sum_prec) * np.abs(b) + 1e-300
    assert np.all(np.abs(a - b) <= tol), float(np.max(np.abs(a - b) / tol))
    if sp.sum_prec == B32 and sp.f_prec == B32:  # binary32 output absorbs the ulp
        assert np.mean(a == b) >= 0.9
