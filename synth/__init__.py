"""Seeded synthetic inputs shared by the tests, the bench and smoke().

This module holds the *problem instance*, never the method: it builds the
per-mode matrices A_d (cubic B-spline bases or dense Gaussians) and L_d
(second differences), x_true and the noise, and the gridded data
y = (A_1 (x) ... (x) A_D) x_true + sigma * noise that BASELINE.json's configs
describe.  The method itself (G_d = A_d^T A_d, the operator apply, the
right-hand side, CG) lives in ``oracle/`` (CPU, test infrastructure) and in
``paper_1001_5460_b200`` (CUDA); neither is imported here.

Readings of the paper used here:
  Z5  centred cardinal cubic B-spline, samples t_i = i (n-1)/(m-1)
  Z6  m_d = oversampling * n_d exactly
  Z7  L_d is the (n_d-2) x n_d second difference [1,-2,1]
  Z9  counter-based generator keyed by (seed, stream, linear index):
      stream 0 = x_true (unknown index), 1 = noise (data index),
      2+d = dense Gaussian A_d entries (row-major index k*n_d + a)
  Z18 dense A_d entries N(0, 1/64)

The counter generator is SplitMix64's output function applied to
key + idx * GAMMA (mod 2^64); the CUDA generator in the product implements
the same integer recipe independently (gen_normal_kernel in
paper_1001_5460_b200/csrc/tca_kernels.cu).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

GAMMA = 0x9E3779B97F4A7C15
_M1 = 0xBF58476D1CE4E5B9
_M2 = 0x94D049BB133111EB
_MASK = (1 << 64) - 1

STREAM_XTRUE = 0
STREAM_NOISE = 1
STREAM_DENSE_A = 2  # + d (0-based mode index)

NOISE_SIGMA = 0.01


# --------------------------------------------------------------------------
# counter-based generator (Z9)
# --------------------------------------------------------------------------
def _mix64_scalar(z: int) -> int:
    z &= _MASK
    z = ((z ^ (z >> 30)) * _M1) & _MASK
    z = ((z ^ (z >> 27)) * _M2) & _MASK
    return z ^ (z >> 31)


def stream_key(seed: int, stream: int) -> int:
    """64-bit key of (seed, stream): mix64(seed * GAMMA + stream)."""
    return _mix64_scalar((seed * GAMMA + stream) & _MASK)


def _mix64_vec(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= np.uint64(_M1)
        z ^= z >> np.uint64(27)
        z *= np.uint64(_M2)
        z ^= z >> np.uint64(31)
    return z


def counter_u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """u64 = mix64(key(seed, stream) + idx * GAMMA), elementwise, wrapping."""
    idx = np.asarray(idx, dtype=np.uint64)
    key = np.uint64(stream_key(seed, stream))
    with np.errstate(over="ignore"):
        z = key + idx * np.uint64(GAMMA)
    return _mix64_vec(z)


def counter_uniform(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Uniform in (0,1): ((u64 >> 11) + 0.5) * 2^-53."""
    u = counter_u64(seed, stream, idx)
    return ((u >> np.uint64(11)).astype(np.float64) + 0.5) * (2.0 ** -53)


def counter_normal(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Standard normal number idx of a stream (Box-Muller, cosine branch).

    normal[j] = sqrt(-2 ln u[2j]) * cos(2 pi u[2j+1]).
    """
    idx = np.asarray(idx, dtype=np.uint64)
    u1 = counter_uniform(seed, stream, idx * np.uint64(2))
    u2 = counter_uniform(seed, stream, idx * np.uint64(2) + np.uint64(1))
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)


def normals(seed: int, stream: int, count: int, offset: int = 0) -> np.ndarray:
    return counter_normal(seed, stream, np.arange(offset, offset + count, dtype=np.uint64))


# --------------------------------------------------------------------------
# per-mode matrices (Z5, Z7, Z18)
# --------------------------------------------------------------------------
def cubic_bspline(u):
    """Centred cardinal cubic B-spline beta^3(u)."""
    a = np.abs(np.asarray(u, dtype=np.float64))
    out = np.zeros_like(a)
    m1 = a < 1.0
    m2 = (a >= 1.0) & (a < 2.0)
    out[m1] = 2.0 / 3.0 - a[m1] ** 2 + a[m1] ** 3 / 2.0
    out[m2] = (2.0 - a[m2]) ** 3 / 6.0
    return out


def sample_positions(n: int, m: int) -> np.ndarray:
    """t_i = i (n-1)/(m-1), i = 0..m-1 (Z5)."""
    if m == 1:
        return np.zeros(1)
    return np.arange(m, dtype=np.float64) * (n - 1) / (m - 1)


def bspline_matrix(n: int, m: int) -> np.ndarray:
    """A[i,k] = beta^3(t_i - k), shape m x n, row-major fp64 (Z5)."""
    t = sample_positions(n, m)
    return cubic_bspline(t[:, None] - np.arange(n, dtype=np.float64)[None, :])


def gaussian_matrix(n: int, m: int, seed: int, mode: int) -> np.ndarray:
    """Dense A_d with i.i.d. N(0, 1/64) entries (Z18), stream 2+mode."""
    vals = normals(seed, STREAM_DENSE_A + mode, m * n)
    return (vals / 8.0).reshape(m, n)


def second_difference(n: int) -> np.ndarray:
    """L[k, k:k+3] = [1, -2, 1], shape (n-2) x n (Z7); empty for n < 3."""
    rows = max(n - 2, 0)
    L = np.zeros((rows, n))
    for k in range(rows):
        L[k, k] = 1.0
        L[k, k + 1] = -2.0
        L[k, k + 2] = 1.0
    return L


def laplacian_1d(n: int) -> np.ndarray:
    """One-dimensional second-order finite-difference factor of the separable
    Poisson operator (Eq. 9; reading Z25): tridiag(-1, 2, -1)
    with homogeneous Dirichlet ends (the truncated band, Z15), grid step 1."""
    T = 2.0 * np.eye(n)
    i = np.arange(n - 1)
    T[i, i + 1] = -1.0
    T[i + 1, i] = -1.0
    return T


# Fig. 1c's Poisson workload shape: X 128, Y 129, Z 130
POISSON_SHAPE = (128, 129, 130)


# --------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Config:
    index: int
    n: tuple
    m: tuple
    basis: str          # "bspline" | "gauss"
    lam: float
    rtol: float         # > 0: stop at relative residual; <= 0: fixed iterations
    max_iters: int
    dtypes: tuple = ("f64",)
    note: str = ""

    @property
    def order(self) -> int:
        return len(self.n)

    @property
    def N(self) -> int:
        return int(np.prod(self.n))

    @property
    def Mdata(self) -> int:
        return int(np.prod(self.m))


CONFIGS = {
    0: Config(0, (12, 12, 12), (20, 20, 20), "bspline", 1e-2, 1e-12, 2000,
              note="order-3 B-spline fit"),
    1: Config(1, (48, 48, 48), (64, 64, 64), "gauss", 1e-3, 1e-10, 5000,
              note="order-3 dense-mode system"),
    2: Config(2, (32, 32, 32, 16), (64, 64, 64, 32), "bspline", 1e-2, 0.0, 200,
              note="order-4 B-spline fit, 2x"),
    3: Config(3, (128, 128, 128, 15), (256, 256, 256, 30), "bspline", 1e-3, 0.0, 500,
              dtypes=("f64", "f32"), note="order-4 paper-scale (~30M unknowns)"),
    4: Config(4, (256, 256, 256, 32), (384, 384, 384, 48), "bspline", 1e-3, 0.0, 100,
              note="order-4 scaling system, 1.5x"),
}


def mode_matrices(cfg_or_n, m=None, basis="bspline", seed=1):
    """Return (A list, L list) for a config or explicit shapes."""
    if isinstance(cfg_or_n, Config):
        n, m, basis = cfg_or_n.n, cfg_or_n.m, cfg_or_n.basis
    else:
        n = tuple(cfg_or_n)
    A, L = [], []
    for d, (nd, md) in enumerate(zip(n, m)):
        if basis == "bspline":
            A.append(bspline_matrix(nd, md))
        elif basis == "gauss":
            A.append(gaussian_matrix(nd, md, seed, d))
        else:
            raise ValueError(basis)
        L.append(second_difference(nd))
    return A, L


def x_true(n, seed=1) -> np.ndarray:
    N = int(np.prod(n))
    return normals(seed, STREAM_XTRUE, N).reshape(n)


def noise(m, seed=1) -> np.ndarray:
    M = int(np.prod(m))
    return normals(seed, STREAM_NOISE, M).reshape(m)


def forward_model(A, x):
    """(A_1 (x) ... (x) A_D) x for a row-major tensor x (numpy tensordot per mode)."""
    y = np.asarray(x, dtype=np.float64)
    for d, Ad in enumerate(A):
        y = np.moveaxis(np.tensordot(Ad, y, axes=([1], [d])), 0, d)
    return np.ascontiguousarray(y)


def data(A, n, m, seed=1, sigma=NOISE_SIGMA, xt=None):
    """y = (kron A) x_true + sigma * noise, the config's gridded data."""
    if xt is None:
        xt = x_true(n, seed)
    return forward_model(A, xt) + sigma * noise(m, seed)


def data_at(A, n, m, k, seed=1, sigma=NOISE_SIGMA):
    """y at the data multi-indices k (shape (S, D)), computed point by point
    from x_true and the noise stream (position keyed, no full-size arrays)."""
    k = np.atleast_2d(np.asarray(k, dtype=np.int64))
    D = len(n)
    out = np.empty(k.shape[0])
    strides_n = np.array([int(np.prod(n[d + 1:])) for d in range(D)], dtype=np.int64)
    strides_m = np.array([int(np.prod(m[d + 1:])) for d in range(D)], dtype=np.int64)
    for s in range(k.shape[0]):
        supp = [np.nonzero(A[d][k[s, d]])[0] for d in range(D)]
        grids = np.meshgrid(*supp, indexing="ij")
        lin = sum(g.astype(np.int64) * strides_n[d] for d, g in enumerate(grids)).ravel()
        w = np.ones(lin.shape[0])
        for d, g in enumerate(grids):
            w = w * A[d][k[s, d], g.ravel()]
        xv = counter_normal(seed, STREAM_XTRUE, lin.astype(np.uint64))
        out[s] = np.sum(w * xv) + sigma * counter_normal(
            seed, STREAM_NOISE, np.array([int(np.dot(k[s], strides_m))], dtype=np.uint64))[0]
    return out


STREAM_SCATTER = 6   # scattered sample coordinates (reading Z27)
# the paper's scattered workload: 128^3 x 16 grid, ~9e6 samples
SCATTER_SHAPE = (128, 128, 128, 16)
SCATTER_K = 9_000_000


def scattered_positions(n, K, seed=1) -> np.ndarray:
    """K x D sample coordinates, uniform on [0, n_d - 1] per mode (coefficient
    grid units, Z27): t[k, d] = (n_d - 1) * u(seed, STREAM_SCATTER, k D + d)."""
    D = len(n)
    u = counter_uniform(seed, STREAM_SCATTER, np.arange(K * D, dtype=np.uint64)).reshape(K, D)
    return u * (np.asarray(n, dtype=np.float64) - 1.0)[None, :]


def random_tensor(shape, seed, stream=7) -> np.ndarray:
    """Generic seeded N(0,1) test tensor (streams >= 7 are test-only)."""
    return normals(seed, stream, int(np.prod(shape))).reshape(shape)
