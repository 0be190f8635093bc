"""B200-native mixed-precision Bogacki-Shampine 3(2) integrator for densely
coupled ODE systems (the hot path of arxiv/paper_2605_23727 "mixedstep").

The compute path is ``libmixedstep_b200.so`` (sm_100a kernels behind the C-ABI
of ``include/mixedstep_b200.h``); this package is the host-side mirror of the
reference's model/solver/precision API over that ABI.
"""
from .precision import (B32, B64, DDD, DDS, SSS, FloatFormat, PolicyVariant, PrecisionPolicy, StagePrecision,
                        custom_policy, kAllBinary32, kAllBinary64, machine_epsilon, policy_for, round_to,
                        variant_from_name, variant_name, wider_of)
from .solver import (FlopTally, SolveResult, SolverConfig, SolveStatus, StepOutcome, StepRecord, adjust_step,
                     bs32_step, dp54_reference, estimate_error, initial_step, kSchemeFlopsBs32, solve, solve_device,
                     status_name)
from .systems import (CcConstants, DeviceSystem, SystemSpec, make_cc, make_kuramoto, make_lco, scalar_fixture)

__all__ = [n for n in dir() if not n.startswith("_")]
