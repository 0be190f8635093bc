"""C5 contraction: signed error of the tensor-core sums against the exact
(binary64) sums of the same rounded operands, along the sum's own sign
(negative = shrunk toward zero, the truncation bias of DESIGN 10.10), for the
accumulation window selected by MS_TC_WINDOW (32 = one accumulator over all of K)."""
import json
import os
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import _oracle as O  # noqa: E402
from paper_2605_23727_b200 import _abi  # noqa: E402
from paper_2605_23727_b200.batch import DeviceBatch  # noqa: E402
from paper_2605_23727_b200.configs import config5_batch  # noqa: E402
from paper_2605_23727_b200.precision import B32, StagePrecision  # noqa: E402
from paper_2605_23727_b200.systems import DeviceSystem  # noqa: E402

SSS = StagePrecision(B32, B32, B32)
w = config5_batch()
dev = DeviceSystem(w.spec)
bat = DeviceBatch(dev, w.omega, tensor_cores=True)
got = bat.eval_rhs(w.x0, SSS)
orc = O.OracleSystem(w.spec)
K = np.asarray(orc.get_k(), dtype=np.float64)  # the bf16-rounded K as stored
n = K.shape[0]


def bf16(v):
    u = np.asarray(v, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return r.astype(np.uint32).view(np.float32)


res = []
for b in range(0, 1024, 64):
    th = np.asarray(w.x0[b], dtype=np.float32)
    s = np.sin(th.astype(np.float64)).astype(np.float32)
    c = np.cos(th.astype(np.float64)).astype(np.float32)
    sh, ch = bf16(s), bf16(c)
    sl, cl = bf16(s - sh), bf16(c - ch)
    A = K @ (sh.astype(np.float64) + sl.astype(np.float64))
    Bv = K @ (ch.astype(np.float64) + cl.astype(np.float64))
    exact = w.omega[b] + (1.0 / n) * (c.astype(np.float64) * A - s.astype(np.float64) * Bv)
    coup_exact = exact - w.omega[b]
    coup_got = got[b] - w.omega[b]
    d = coup_got - coup_exact
    res.append((np.mean(d * np.sign(coup_exact)), np.sqrt(np.mean(d * d)), np.mean(np.abs(coup_exact))))
r = np.array(res)
print(json.dumps({"window": os.environ.get("MS_TC_WINDOW"),
                  "signed_bias_along_coupling": float(r[:, 0].mean()), "rms_error": float(np.sqrt((r[:, 1] ** 2).mean())),
                  "mean_abs_coupling": float(r[:, 2].mean()),
                  "relative_bias": float(r[:, 0].mean() / r[:, 2].mean())}))
