"""Pins of the oracle's discrete operators (SURVEY.md §8(c) "Operators (a1, a2)").

grad (D+), div (sum of D-), symgrad (Eq. 3) and div2 as
defined in DESIGN.md reading R6.  The pins are mathematical facts, not a
retyping of the stencils:
  * adjointness  <grad u, p> = -<u, div p>,  <E v, q>_F = -<v, div2 q>
    (Frobenius product with both off-diagonal entries counted), on random
    fields including axes of size 1 and 2;
  * exactness on polynomials: grad of a linear field, E(grad u) = Hessian of
    a quadratic in the interior;
  * hand-derived boundary values of E for a linear v (Neumann reading);
  * the operator norm of K(u,v) = (grad u - v, E v) by power iteration
    stays below 16, the bound used by the step-size check tau*sigma*16 <= 1.
"""
import numpy as np
import pytest

import oracle

SHAPES = [(5, 4, 3), (1, 6, 7), (2, 1, 5), (1, 1, 9), (7, 2, 1), (1, 1, 1), (6, 6, 6)]
OFFW = np.array([1, 1, 1, 2, 2, 2], dtype=np.float64)  # Frobenius weights for xx,yy,zz,xy,xz,yz


def rnd(rng, *shape):
    return rng.standard_normal(shape)


@pytest.mark.parametrize("shape", SHAPES)
def test_grad_div_adjoint(shape):
    nx, ny, nz = shape
    rng = np.random.default_rng(1)
    for _ in range(5):
        u = rnd(rng, nz, ny, nx)
        p = rnd(rng, 3, nz, ny, nx)
        lhs = np.sum(oracle.grad(u) * p)
        rhs = -np.sum(u * oracle.div(p))
        scale = np.linalg.norm(u) * np.linalg.norm(p)
        assert abs(lhs - rhs) <= 1e-12 * scale


@pytest.mark.parametrize("shape", SHAPES)
def test_symgrad_div2_adjoint(shape):
    nx, ny, nz = shape
    rng = np.random.default_rng(2)
    for _ in range(5):
        v = rnd(rng, 3, nz, ny, nx)
        q = rnd(rng, 6, nz, ny, nx)
        lhs = np.sum(OFFW[:, None, None, None] * oracle.symgrad(v) * q)
        rhs = -np.sum(v * oracle.div2(q))
        scale = np.linalg.norm(v) * np.linalg.norm(q)
        assert abs(lhs - rhs) <= 1e-12 * scale


def coords(nx, ny, nz):
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    return x.astype(float), y.astype(float), z.astype(float)


def test_grad_of_linear_field():
    nx, ny, nz = 6, 5, 4
    x, y, z = coords(nx, ny, nz)
    u = 2.0 * x - 3.0 * y + 0.5 * z
    g = oracle.grad(u)
    # forward difference is exact; Neumann: zero on the last plane of each axis
    np.testing.assert_array_equal(g[0][:, :, :-1], 2.0)
    np.testing.assert_array_equal(g[0][:, :, -1], 0.0)
    np.testing.assert_array_equal(g[1][:, :-1, :], -3.0)
    np.testing.assert_array_equal(g[1][:, -1, :], 0.0)
    np.testing.assert_array_equal(g[2][:-1], 0.5)
    np.testing.assert_array_equal(g[2][-1], 0.0)


def test_symgrad_of_gradient_is_hessian_in_interior():
    nx, ny, nz = 7, 6, 8
    x, y, z = coords(nx, ny, nz)
    # Hessian of u: xx=2a, yy=2b, zz=2c, xy=d, xz=e, yz=f
    a, b, c, d, e, f = 0.5, -1.0, 0.25, 2.0, -0.75, 1.5
    u = a * x * x + b * y * y + c * z * z + d * x * y + e * x * z + f * y * z
    H = oracle.symgrad(oracle.grad(u))
    inner = (slice(1, nz - 1), slice(1, ny - 1), slice(1, nx - 1))
    expect = [2 * a, 2 * b, 2 * c, d, e, f]
    for m in range(6):
        np.testing.assert_allclose(H[m][inner], expect[m], rtol=0, atol=1e-12)


def test_symgrad_boundary_values_closed_form():
    # v = (y, 0, 0):  E_xx = D-_x v_x = y at x=0, -y at x=n-1, else 0
    #                 E_xy = 1/2 D-_y v_x : D-_y y = y-(y-1)=1 interior, y=0 -> 0 (=v[0]=0), y=n-1 -> -(n-2)
    #                 E_xz = 1/2 D-_z v_x : v_x constant in z -> +y at z=0, -y at z=n-1
    nx, ny, nz = 5, 6, 4
    x, y, z = coords(nx, ny, nz)
    v = np.stack([y, 0 * y, 0 * y])
    E = oracle.symgrad(v)
    exx = np.where(x == 0, y, np.where(x == nx - 1, -y, 0.0))
    dy = np.where(y == 0, 0.0, np.where(y == ny - 1, -(ny - 2.0), 1.0))
    exz = np.where(z == 0, y, np.where(z == nz - 1, -y, 0.0))
    np.testing.assert_array_equal(E[0], exx)
    np.testing.assert_array_equal(E[1], 0.0)
    np.testing.assert_array_equal(E[2], 0.0)
    np.testing.assert_array_equal(E[3], 0.5 * dy)
    np.testing.assert_array_equal(E[4], 0.5 * exz)
    np.testing.assert_array_equal(E[5], 0.0)


def test_div2_of_constant_diagonal_tensor():
    # q_xx = 1 everywhere: (div2 q)_x = D+_x q_xx = 0 (constant, Neumann) ; others 0
    # q_xy = y: (div2 q)_x = D+_y q_xy = 1 except last y-plane, (div2 q)_y = D+_x q_xy = 0
    nx, ny, nz = 4, 5, 3
    x, y, z = coords(nx, ny, nz)
    q = np.zeros((6, nz, ny, nx))
    q[0] = 1.0
    q[3] = y
    w = oracle.div2(q)
    np.testing.assert_array_equal(w[0], np.where(y < ny - 1, 1.0, 0.0))
    np.testing.assert_array_equal(w[1], 0.0)
    np.testing.assert_array_equal(w[2], 0.0)


def knorm2(shape, iters=300, seed=0):
    nx, ny, nz = shape
    rng = np.random.default_rng(seed)
    u = rnd(rng, nz, ny, nx)
    v = rnd(rng, 3, nz, ny, nx)
    lam = 0.0
    for _ in range(iters):
        n = np.sqrt(np.sum(u * u) + np.sum(v * v))
        u, v = u / n, v / n
        p = oracle.grad(u) - v
        q = oracle.symgrad(v)
        # K^T (p, q) = (-div p, -p - div2 q)  (q-space inner product counts off-diagonals twice)
        u2 = -oracle.div(p)
        v2 = -p - oracle.div2(q)
        lam = np.sum(u * u2) + np.sum(v * v2)
        u, v = u2, v2
    return lam


def test_operator_norm_below_16():
    for shape, lo in [((4, 4, 4), 12.0), ((8, 8, 8), 14.5)]:
        L2 = knorm2(shape)
        assert lo < L2 < 16.0, (shape, L2)
