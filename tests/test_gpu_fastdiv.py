"""The kernels divide by a ray's direction components through a factored
float64 division (wc_common.cuh recip_of / div_by: div.rn.f64's divisor-only
reciprocal refinement done once per divisor, its quotient steps and range
tests per division, the plain division outside that range).  Bit-exact
parity of every traversal and raytrace buffer rests on it being exactly
a / b: checked here over 2^31 hashed operand pairs per seed."""

import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("seed", [1, 0x5EED5EED])
def test_factored_division_is_exact(seed):
    import paper_2309_10212_b200 as wc

    wc._lib.ensure_device(0)
    bad = C.c_int64(-1)
    ex = np.zeros(2, np.float64)
    wc._lib.call("wc_check_fastdiv", 1 << 31, seed, C.byref(bad), wc._lib.ptr(ex))
    assert bad.value == 0, f"{bad.value} quotients differ from a / b, e.g. a={ex[0]!r} b={ex[1]!r}"
