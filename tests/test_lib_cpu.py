"""CPU-side checks of libsf.so: it loads, exports every symbol include/sf.h declares,
its host-only logic (FD weights, slab plan, sparse ownership) is right, and compute
calls fail loudly (no CPU fallback) when no GPU is present."""
import ctypes
import math
import os
import re
from fractions import Fraction

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sf():
    import paper_1707_03776_b200 as m
    return m


def header_symbols():
    src = open(os.path.join(ROOT, "include", "sf.h")).read()
    return sorted(set(re.findall(r"^SF_API\s+[\w\s\*]*?\b(sf_\w+)\s*\(", src, flags=re.M)))


def test_library_exports_every_declared_symbol():
    L = sf().lib()
    declared = header_symbols()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(L, name), name
    assert sorted(sf().EXPORTS) == declared
    assert L.sf_version() >= 1


def test_fd_weights_closed_form_and_oracle_independent():
    """libsf's host weights (closed form) vs exact rationals from Fornberg-free
    Vandermonde solves (Fraction arithmetic), orders 2..16."""
    for so in range(2, 17, 2):
        r = so // 2
        # exact: symmetric moment system sum_{j=-r..r} w_|j| j^(2i) = 2 [i == 1], i = 0..r
        A = [[Fraction((1 if i == 0 else 0) if j == 0 else 2 * j ** (2 * i)) for j in range(r + 1)]
             for i in range(r + 1)]
        b = [Fraction(2 if i == 1 else 0) for i in range(r + 1)]
        # Gaussian elimination in exact arithmetic
        n = r + 1
        M = [row[:] + [b[i]] for i, row in enumerate(A)]
        for c in range(n):
            piv = next(i for i in range(c, n) if M[i][c] != 0)
            M[c], M[piv] = M[piv], M[c]
            for i in range(n):
                if i != c and M[i][c] != 0:
                    f = M[i][c] / M[c][c]
                    M[i] = [x - f * y for x, y in zip(M[i], M[c])]
        exact = [M[i][n] / M[i][i] for i in range(n)]
        got = sf().fd_weights(so)
        np.testing.assert_allclose(got, [float(x) for x in exact], rtol=1e-13, atol=1e-15)


def test_fd_weights_errors():
    with pytest.raises(sf().SfError) as e:
        sf().fd_weights(5)
    assert e.value.status == "SF_ERR_ORDER"


@pytest.mark.parametrize("n0,so,P", [(1024, 16, 8), (1027, 16, 8), (336, 8, 3), (64, 2, 7), (33, 16, 4)])
def test_slab_plan_partitions(n0, so, P):
    x = 0
    for p in range(P):
        x0, nl = sf().slab_plan(n0, so, p, P)
        assert x0 == x and nl >= so // 2
        assert abs(nl - n0 / P) < 1
        x += nl
    assert x == n0


def test_slab_plan_too_thin():
    with pytest.raises(sf().SfError) as e:
        sf().slab_plan(30, 16, 0, 8)
    assert e.value.status == "SF_ERR_SHAPE"


def test_sparse_owner_base_plane():
    n0, so, P, h = 100, 8, 4, 10.0
    for c in [0.0, 249.0, 250.0, 255.0, 499.9, 500.0, 990.0]:
        own = sf().sparse_owner(n0, so, P, h, c)
        base = min(int(math.floor(c / h)), n0 - 2)
        x0, nl = sf().slab_plan(n0, so, own, P)
        assert x0 <= base < x0 + nl
    with pytest.raises(sf().SfError):
        sf().sparse_owner(n0, so, P, h, 990.01)


def test_compute_fails_loudly_without_gpu():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    L = sf().lib()

    class D(ctypes.Structure):
        _fields_ = sf()._lib.SfDesc._fields_

    d = sf()._lib.SfDesc()
    d.ndim = 3
    for a in range(3):
        d.shape[a] = 8
    d.h, d.space_order, d.nt, d.dt = 10.0, 4, 10, 1e-3
    m = np.ones(512, np.float32)
    d.m = m.ctypes.data
    h = ctypes.c_void_p()
    code = L.sf_create(ctypes.byref(d), ctypes.byref(h))
    assert code == 7  # SF_ERR_CUDA
    assert b"CUDA" in L.sf_last_error() or b"device" in L.sf_last_error()
