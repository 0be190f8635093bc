"""The harness engine protocol on the CPU oracle (TEST INFRASTRUCTURE): lets
paper_2605_23727_b200.harness run cases without a GPU, and gives the GPU tests
the oracle's rows to diff the device rows against."""
import _oracle as O


class OracleEngine:
    def __init__(self, rhs_mode: str = "faithful"):
        self.rhs_mode = rhs_mode

    def build_system(self, tc):  # harness.cpp:332-343
        if tc.benchmark == "lco":
            return O.OracleSystem.make_lco(tc.agents, tc.test_id)
        if tc.benchmark == "kuramoto":
            return O.OracleSystem.make_kuramoto(tc.agents, tc.sigma, tc.coupling_k, tc.test_id)
        if tc.benchmark == "cc":
            return O.OracleSystem.make_cc(tc.agents, tc.coupling_k, tc.stimulus_i0, tc.test_id)
        raise ValueError(tc.benchmark)

    def solve(self, sys, x0, tf, policy, cfg):
        return O.solve(sys, x0, 0.0, tf, policy, cfg)

    def dp54_reference(self, sys, x0, tf, cfg):
        return O.dp54_reference(sys, x0, 0.0, tf, cfg)

    def release(self, sys):
        pass
