"""Device pow used by shade ((1-alpha)**ratio, kernels.py:348).

The reference evaluates it with glibc's pow.  That pow is not correctly rounded:
it misrounds ~7e-4 of these inputs by 1 ulp (verified against 50-digit decimal
arithmetic).  The device pow is double-double and correctly rounded, so it
agrees with glibc everywhere glibc is right and differs by exactly 1 ulp where
glibc is wrong."""

from decimal import Decimal, getcontext

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def test_shade_pow_is_correctly_rounded_and_within_1ulp_of_libm():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.device import ptr

    import math

    rng = np.random.default_rng(0)
    n = 1 << 18
    alpha = np.concatenate([rng.uniform(1e-4, 1.0, n // 2), 10 ** rng.uniform(-6, 0, n // 2)])
    x = np.maximum(1.0 - alpha, 1e-12)
    y = np.concatenate([rng.uniform(1e-3, 16.0, n // 2), rng.uniform(0.5, 1.5, n // 2)])
    # glibc pow through math.pow (what numba's `**` lowers to); np.power may use an
    # AVX-512 SVML kernel on the GPU host and is not the reference's pow
    want = np.array([math.pow(a, b) for a, b in zip(x.tolist(), y.tolist())])
    tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    out = torch.empty_like(tx)
    N.call("vcb_debug_pow", n, ptr(tx), ptr(ty), ptr(out), 0)
    got = out.cpu().numpy()
    ulps = np.abs(got.view(np.int64) - want.view(np.int64))
    rate = float((ulps != 0).mean())
    print(f"device pow vs libm: {rate:.2e} differ, max {ulps.max()} ulp")
    assert ulps.max() <= 1, f"max {ulps.max()} ulp from libm"
    assert rate <= 1e-2
    getcontext().prec = 50
    check = np.concatenate([np.flatnonzero(ulps)[:300], rng.choice(n, 300, replace=False)])
    wrong = 0
    for i in check:
        cr = float(Decimal(float(x[i])) ** Decimal(float(y[i])))
        wrong += got[i] != cr
    # the device pow is the correctly rounded one wherever it departs from libm
    assert wrong <= 1, f"{wrong}/{check.size} device results not correctly rounded"


def test_shade_pow_fast_phase_equals_accurate_phase():
    """The pow's fast phase + rounding test returns exactly what its double-double phase
    returns (both correctly rounded), over the shade's input range and beyond it:
    2^22 random (1 - alpha, ratio) pairs plus values near 1, tiny bases and exponents
    up to the fast phase's |y| <= 16 bound and past it."""
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2504_18001_b200 import _native as N
    from paper_2504_18001_b200.device import ptr

    rng = np.random.default_rng(5)
    n = 1 << 22
    q = n // 4
    x = np.concatenate([1.0 - rng.uniform(1e-4, 1.0 - 1e-12, q), 1.0 - 10 ** rng.uniform(-16, -1, q),
                        10 ** rng.uniform(-300, 0, q), rng.uniform(0.5, 2.0, q)])
    y = np.concatenate([rng.uniform(1e-3, 4.0, q), rng.uniform(0.01, 16.0, q), rng.uniform(-2.0, 2.0, q),
                        rng.uniform(-40.0, 40.0, q)])
    tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    fast, acc = torch.empty_like(tx), torch.empty_like(tx)
    N.call("vcb_debug_pow", n, ptr(tx), ptr(ty), ptr(fast), 0)
    N.call("vcb_debug_pow_accurate", n, ptr(tx), ptr(ty), ptr(acc), 0)
    f, a = fast.cpu().numpy(), acc.cpu().numpy()
    bad = np.flatnonzero(f.view(np.int64) != a.view(np.int64))
    assert bad.size == 0, f"{bad.size} differ, e.g. pow({x[bad[0]]!r}, {y[bad[0]]!r}): {f[bad[0]]!r} vs {a[bad[0]]!r}"
