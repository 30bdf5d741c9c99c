"""Pin of the division-free x/3 used for quadrature points (tm_common.cuh div3):
multiply by fl(1/3), exact FMA residual, one FMA correction.  Checked against the
IEEE quotient x/3 on random doubles over a wide exponent range, by a small C
program (the same operations, -ffp-contract=off, libm fma)."""
import os
import subprocess
import tempfile

SRC = r"""
#include <stdio.h>
#include <math.h>
#include <stdint.h>
#include <string.h>
static uint64_t s = 88172645463325252ull;
static uint64_t xr(void) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return s; }
int main(void) {
    const double T = 0.33333333333333331483;
    long long bad = 0, n = 20000000LL;
    for (long long i = 0; i < n; i++) {
        uint64_t b = xr();
        b = (b & 0x800FFFFFFFFFFFFFull) | ((uint64_t)(1023 - 200 + (xr() % 400)) << 52);
        double x;
        memcpy(&x, &b, 8);
        volatile double q = x * T;
        volatile double r = fma(-q, 3.0, x);
        volatile double q2 = fma(r, T, q);
        volatile double ref = x / 3.0;
        if (q2 != ref) bad++;
    }
    printf("%lld\n", bad);
    return 0;
}
"""


def test_div3_equals_ieee_quotient():
    with tempfile.TemporaryDirectory() as d:
        c, exe = os.path.join(d, "d3.c"), os.path.join(d, "d3")
        open(c, "w").write(SRC)
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-o", exe, c, "-lm"])
        assert int(subprocess.check_output([exe]).decode().strip()) == 0
