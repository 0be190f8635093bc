"""The C-ABI boundary: the in-tree sm_100a library loads, exports every symbol
include/mixedstep_b200.h declares, its structs match the Python bindings, and
its host-side pieces agree with the oracle. No compute call runs here."""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import _oracle as O
from paper_2605_23727_b200 import _abi
from paper_2605_23727_b200.precision import PolicyVariant, policy_for
from paper_2605_23727_b200.solver import SolverConfig

HEADER = Path(__file__).resolve().parent.parent / "include" / "mixedstep_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ms_[a-z0-9_]+)\s*\(", text)))


def test_library_loads_and_exports_every_declared_symbol():
    L = _abi.lib()
    syms = declared_symbols()
    assert len(syms) >= 24
    missing = [s for s in syms if not hasattr(L, s)]
    assert not missing, missing
    bound = {name for name, _, _ in _abi.SIGNATURES}
    assert set(syms) == bound, set(syms) ^ bound
    assert L.ms_abi_version() == 3


def test_struct_layouts_match():
    out = (C.c_int64 * 8)()
    assert _abi.lib().ms_abi_sizes(out) == 0
    py = [_abi.StagePrec, _abi.Policy, _abi.SolverConfigC, _abi.StepRecordC, _abi.SystemDesc, _abi.SolveResultC,
          _abi.StepOutcomeC, _abi.ExchangeC]
    assert list(out) == [C.sizeof(t) for t in py]


def test_default_config_matches_reference_defaults():  # solver.hpp:39-61
    c = _abi.SolverConfigC()
    _abi.lib().ms_default_config(C.byref(c))
    ref = SolverConfig().c()
    for name, _ in _abi.SolverConfigC._fields_:
        assert getattr(c, name) == getattr(ref, name), name


def test_policy_for_matches_oracle():  # precision.cpp:22-42
    for v in range(4):
        a, b = _abi.Policy(), _abi.Policy()
        assert _abi.lib().ms_policy_for(v, C.byref(a)) == 0
        assert O.lib().orc_policy_for(v, C.byref(b)) == 0
        assert bytes(a) == bytes(b)
        assert bytes(policy_for(PolicyVariant(v)).c()) == bytes(a)
        assert _abi.lib().ms_policy_lowest_format(C.byref(a)) == O.lib().orc_policy_lowest_format(C.byref(b))
    bad = _abi.Policy()
    assert _abi.lib().ms_policy_for(9, C.byref(bad)) == _abi.MS_EINVAL


def test_input_generators_bitwise_equal_oracle():  # rng.hpp:13-52
    for seed, stream in ((0, 0), (3, 1), (4, 2), (123456789, 3)):
        a = np.empty(5000)
        _abi.lib().ms_rng_uniform(seed, stream, 5000, -1.0, 1.0, _abi.dptr(a))
        assert np.array_equal(a, O.rng_uniform(seed, stream, 5000, -1.0, 1.0))
        b = np.empty(5001)
        _abi.lib().ms_rng_normal(seed, stream, 5001, _abi.dptr(b))
        assert np.array_equal(b, O.rng_normal(seed, stream, 5001))


def test_compute_without_gpu_fails_loudly():
    """The product path has no CPU fallback: with no device visible every
    compute entry point reports MS_ECUDA (a GPU box skips this check)."""
    L = _abi.lib()
    if L.ms_device_count() > 0:
        pytest.skip("a CUDA device is visible")
    from paper_2605_23727_b200.systems import SystemSpec, DeviceSystem
    with pytest.raises(_abi.CudaError):
        DeviceSystem(SystemSpec("kuramoto", 8, omega=np.zeros(8)))
    out = C.c_double()
    a = np.zeros(3)
    assert L.ms_estimate_error(3, _abi.dptr(a), _abi.dptr(a), _abi.dptr(a), 1e-8, 1e-6, C.byref(out)) == _abi.MS_ECUDA


def test_invalid_descriptors_are_rejected_before_device_work():
    from paper_2605_23727_b200.systems import SystemSpec, DeviceSystem
    with pytest.raises(ValueError):
        DeviceSystem(SystemSpec("kuramoto", 0, omega=np.zeros(1)))
    with pytest.raises(ValueError):
        DeviceSystem(SystemSpec("kuramoto", 4))  # omega missing


def test_library_sass_has_no_packed_fma():
    """The arithmetic contract forbids contracting a product into a sum. The
    sweeps accumulate with packed add.rn.f32x2 (FADD2) fed by scalar mul.rn;
    ptxas contracts mul.rn.f32x2 + add.rn.f32x2 into FFMA2 even under
    -fmad=false, so no packed multiply may reach a packed add: no FFMA2 in
    the shipped SASS."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", str(_abi.LIB_PATH)], capture_output=True, text=True, check=True).stdout
    assert "FADD2" in sass  # the packed accumulation is in use
    assert "FFMA2" not in sass
