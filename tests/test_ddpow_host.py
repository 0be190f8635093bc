"""The controller's pow (csrc/ms_ddpow.cuh) is compiled for the host here and
checked to be correctly rounded, and to agree with glibc's pow (the
reference's, solver.cpp:416, 448) wherever glibc itself is correctly rounded.
The same source is compiled into the device controller."""
import math
import random
import subprocess
import tempfile
from decimal import Decimal, getcontext
from pathlib import Path

CSRC = Path(__file__).resolve().parent.parent / "paper_2605_23727_b200" / "csrc"
PROG = r'''
#include "ms_ddpow.cuh"
#include <cstdio>
int main() {
  double x, y;
  while (scanf("%lf %lf", &x, &y) == 2)
    printf("%a %a %a\n", msb::pow_cr(x, y), std::pow(x, y), msb::pow_cr_general(x, y));
}
'''


def test_pow_cr_is_correctly_rounded_and_matches_glibc():
    getcontext().prec = 80
    with tempfile.TemporaryDirectory() as d:
        src, exe = Path(d) / "t.cpp", Path(d) / "t"
        src.write_text(PROG)
        subprocess.run(["/usr/bin/g++", "-O2", "-ffp-contract=off", "-I", str(CSRC), str(src), "-o", str(exe)],
                       check=True)
        rnd = random.Random(11)
        xs = [(10 ** rnd.uniform(-4, 7), 1.0 / 3.0) for _ in range(2000)]
        xs += [(10 ** rnd.uniform(-8, 10), 0.25) for _ in range(1000)]
        xs += [(10 ** rnd.uniform(-8, 10), 0.2) for _ in range(1000)]
        xs += [(10 ** rnd.uniform(-12, 12), 1.0 / q) for q in (2, 6, 7, 8) for _ in range(300)]
        xs += [(10 ** rnd.uniform(-3, 6), 0.3) for _ in range(300)]  # not 1/q: general path
        out = subprocess.run([str(exe)], input="\n".join(f"{x!r} {y!r}" for x, y in xs), capture_output=True,
                             text=True, check=True).stdout.split("\n")
    agree_when_glibc_cr = 0
    glibc_cr = 0
    for (x, y), line in zip(xs, out):
        a, b, g = (float.fromhex(v) for v in line.split())
        assert a == g, (x, y)  # the 1/q root path is the general dd path, bit for bit
        ex = Decimal(x) ** Decimal(y)
        cands = [math.nextafter(a, -math.inf), a, math.nextafter(a, math.inf)]
        assert min(cands, key=lambda c: abs(Decimal(c) - ex)) == a, (x, y)
        cb = [math.nextafter(b, -math.inf), b, math.nextafter(b, math.inf)]
        if min(cb, key=lambda c: abs(Decimal(c) - ex)) == b:
            glibc_cr += 1
            agree_when_glibc_cr += a == b
    assert agree_when_glibc_cr == glibc_cr
    assert glibc_cr >= 0.995 * len(xs)
