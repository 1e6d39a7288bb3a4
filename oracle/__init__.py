"""CPU oracle for the tca hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline and
--impl reference) may import this package.  The product package
(paper_1001_5460_b200) never imports it and shares no code with it.

The arithmetic is in tca_oracle.c (plain C loops, fp64); this module only
builds it with gcc, loads it with ctypes and marshals numpy arrays.  Every
function cites the passage of PAPER.md it follows (see the C file header).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tca_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, BREAKDOWN, NONFINITE, NOT_CONVERGED = 0, 7, 8, 9

_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build(force: bool = False) -> str:
    """Compile tca_oracle.c -> liboracle.so (gcc -O2 -fopenmp)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-Wall",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            L.orc_gram.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, _dp]
            L.orc_transpose.argtypes = [ctypes.c_int64, ctypes.c_int64, _dp, _dp]
            L.orc_mode_product.argtypes = [ctypes.c_int, _i64p, _dp, ctypes.c_int,
                                           ctypes.c_int64, _dp, _dp]
            L.orc_apply.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp),
                                    ctypes.POINTER(_dp), ctypes.c_double, _dp, _dp]
            L.orc_rhs.argtypes = [ctypes.c_int, _i64p, _i64p, ctypes.POINTER(_dp), _dp, _dp]
            L.orc_apply_point.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp),
                                          ctypes.POINTER(_dp), ctypes.c_double, _dp, _i64p]
            L.orc_apply_point.restype = ctypes.c_double
            L.orc_rhs_point.argtypes = [ctypes.c_int, _i64p, _i64p, ctypes.POINTER(_dp),
                                        _dp, _i64p]
            L.orc_rhs_point.restype = ctypes.c_double
            L.orc_dot.argtypes = [ctypes.c_int64, _dp, _dp]
            L.orc_dot.restype = ctypes.c_double
            L.orc_cg.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp), ctypes.POINTER(_dp),
                                 ctypes.c_double, _dp, _dp, ctypes.c_double, ctypes.c_int, _dp,
                                 ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
            L.orc_cg.restype = ctypes.c_int
            L.orc_num_threads.restype = ctypes.c_int
            L.orc_cholesky.argtypes = [ctypes.c_int64, _dp, _dp]
            L.orc_cholesky.restype = ctypes.c_int
            L.orc_geomean_eig.argtypes = [ctypes.c_int64, _dp]
            L.orc_geomean_eig.restype = ctypes.c_double
            L.orc_precond_factors.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp), ctypes.POINTER(_dp),
                                              ctypes.c_double, ctypes.POINTER(_dp), _dp]
            L.orc_precond_factors.restype = ctypes.c_int
            L.orc_precond_apply.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp), _dp, _dp]
            L.orc_pcg.argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp), ctypes.POINTER(_dp),
                                  ctypes.c_double, _dp, _dp, ctypes.c_double, ctypes.c_int, _dp,
                                  ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
            L.orc_pcg.restype = ctypes.c_int
            for nm in ("orc_cg_x0", "orc_pcg_x0", "orc_cgsr_x0"):
                getattr(L, nm).argtypes = [ctypes.c_int, _i64p, ctypes.POINTER(_dp), ctypes.POINTER(_dp),
                                           ctypes.c_double, _dp, _dp, ctypes.c_int, ctypes.c_double, ctypes.c_int,
                                           _dp, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)]
                getattr(L, nm).restype = ctypes.c_int
            L.orc_cgsr.argtypes = L.orc_cg.argtypes
            L.orc_cgsr.restype = ctypes.c_int
            L.orc_jacobi.argtypes = L.orc_cg.argtypes
            L.orc_jacobi.restype = ctypes.c_int
            for nm in ("orc_scattered_data", "orc_scattered_rhs", "orc_scattered_forward"):
                getattr(L, nm).argtypes = [ctypes.c_int, _i64p, ctypes.c_int64, _dp, _dp, _dp]
            _lib = L
    return _lib


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _p(a):
    return a.ctypes.data_as(_dp)


def _i64(v):
    a = np.ascontiguousarray(v, dtype=np.int64)
    return a, a.ctypes.data_as(_i64p)


def _ptr_array(mats):
    arr = (_dp * len(mats))()
    for i, M in enumerate(mats):
        arr[i] = ctypes.cast(None, _dp) if M is None else _p(M)
    return arr


def num_threads() -> int:
    return lib().orc_num_threads()


def gram(A) -> np.ndarray:
    """G = A^T A by explicit loops."""
    A = _f64(A)
    m, n = A.shape
    G = np.empty((n, n))
    lib().orc_gram(m, n, _p(A), _p(G))
    return G


def mode_product(X, d: int, M) -> np.ndarray:
    """Y = X x_d M (Eq. 4 one-dimensional transformation along mode d)."""
    X, M = _f64(X), _f64(M)
    s = list(X.shape)
    rows = M.shape[0]
    assert M.shape[1] == s[d]
    out_shape = s.copy()
    out_shape[d] = rows
    Y = np.empty(out_shape)
    sa, sp = _i64(s)
    lib().orc_mode_product(len(s), sp, _p(X), d, rows, _p(M), _p(Y))
    return Y


class Operator:
    """M = (kron_d G_d) + lam * sum_d (mode-d R_d), G_d = A_d^T A_d, R_d = L_d^T L_d.

    A: list of m_d x n_d arrays; L: list of (n_d-2) x n_d arrays or None.
    """

    def __init__(self, A, L=None, lam=0.0):
        self.A = [_f64(a) for a in A]
        self.D = len(self.A)
        self.n = tuple(a.shape[1] for a in self.A)
        self.m = tuple(a.shape[0] for a in self.A)
        self.lam = float(lam)
        self.G = [gram(a) for a in self.A]
        if L is None:
            self.R = [None] * self.D
        else:
            self.R = [None if (l is None or l.shape[0] == 0) else gram(l) for l in L]
        self._na, self._np = _i64(self.n)
        self._ma, self._mp = _i64(self.m)
        self._G = _ptr_array(self.G)
        self._R = _ptr_array(self.R)
        self._A = _ptr_array(self.A)

    @classmethod
    def from_gram(cls, G, R, lam):
        """Operator given by its factors: M = (kron_d G_d) + lam sum_d (mode-d R_d).
        G None: no Kronecker-product term (Eq. 9's separable Poisson form); R a list
        of n_d x n_d matrices (None entries: no term for that mode)."""
        self = cls.__new__(cls)
        self.D = len(R)
        self.n = tuple(r.shape[0] for r in R)
        self.m = self.n
        self.lam = float(lam)
        self.G = [_f64(g) for g in G] if G is not None else [None] * self.D
        self.R = [None if r is None else _f64(r) for r in R]
        self.A = [np.eye(k) for k in self.n]
        self._na, self._np = _i64(self.n)
        self._ma, self._mp = _i64(self.m)
        self._G = _ptr_array(self.G)
        self._R = _ptr_array(self.R)
        self._A = _ptr_array(self.A)
        return self

    @property
    def N(self):
        return int(np.prod(self.n))

    def apply(self, x) -> np.ndarray:
        x = _f64(x).reshape(self.n)
        y = np.empty(self.n)
        lib().orc_apply(self.D, self._np, self._G, self._R, self.lam, _p(x), _p(y))
        return y

    def rhs(self, ydata) -> np.ndarray:
        ydata = _f64(ydata).reshape(self.m)
        b = np.empty(self.n)
        lib().orc_rhs(self.D, self._np, self._mp, self._A, _p(ydata), _p(b))
        return b

    def apply_point(self, x, idx) -> float:
        x = _f64(x)
        ia, ip = _i64(idx)
        return lib().orc_apply_point(self.D, self._np, self._G, self._R, self.lam, _p(x), ip)

    def apply_points(self, x, idxs) -> np.ndarray:
        x = _f64(x)
        return np.array([self.apply_point(x, i) for i in np.atleast_2d(idxs)])

    def rhs_point(self, ydata, idx) -> float:
        ydata = _f64(ydata)
        ia, ip = _i64(idx)
        return lib().orc_rhs_point(self.D, self._np, self._mp, self._A, _p(ydata), ip)

    def _krylov(self, fn, b, rtol, max_iters, x0):
        b = _f64(b).reshape(self.n)
        x = np.zeros(self.n) if x0 is None else _f64(x0).reshape(self.n).copy()
        hist = np.zeros(max_iters + 1)
        it = ctypes.c_int(0)
        rf = ctypes.c_double(0.0)
        st = fn(self.D, self._np, self._G, self._R, self.lam, _p(b), _p(x), 1 if x0 is None else 0,
                float(rtol), int(max_iters), _p(hist), ctypes.byref(it), ctypes.byref(rf))
        return x, it.value, st, hist[: it.value + 1]

    def cg(self, b, rtol: float, max_iters: int, x0=None):
        """Fig. 2 CG from x0 = 0, or from x0 (R := B - A*C; stop reference <b, b>,
        reading Z28).  Returns (x, iters, status, rho_history)."""
        return self._krylov(lib().orc_cg_x0, b, rtol, max_iters, x0)

    def cgsr(self, b, rtol: float, max_iters: int, x0=None):
        """Single-reduction (Chronopoulos-Gear) CG from x0 = 0 or x0 (reading Z24).
        Returns (x, iters, status, rr_history)."""
        return self._krylov(lib().orc_cgsr_x0, b, rtol, max_iters, x0)

    def jacobi(self, b, threshold: float, max_iters: int):
        """Tensor Jacobi (Fig. 1) from U = 0, stopping when R+*R <= threshold.
        Returns (u, iters, status, rr_history)."""
        b = _f64(b).reshape(self.n)
        u = np.empty(self.n)
        hist = np.zeros(max_iters + 1)
        it = ctypes.c_int(0)
        rf = ctypes.c_double(0.0)
        st = lib().orc_jacobi(self.D, self._np, self._G, self._R, self.lam, _p(b), _p(u),
                              float(threshold), int(max_iters), _p(hist), ctypes.byref(it), ctypes.byref(rf))
        return u, it.value, st, hist[: it.value + 1]

    # ---- Kronecker-factor preconditioner (reading Z22)
    def precond_factors(self):
        """(F_d list, eps_d list): F_d = G_d + eps_d R_d, eps_d = lam / prod_{e!=d} gbar_e."""
        F = [np.empty((k, k)) for k in self.n]
        eps = np.empty(self.D)
        st = lib().orc_precond_factors(self.D, self._np, self._G, self._R, self.lam,
                                       _ptr_array(F), _p(eps))
        if st != 0:
            raise ValueError("G_d not positive definite")
        return F, list(eps)

    def precond_apply(self, r) -> np.ndarray:
        """z = P^-1 r = (F_1^-1 (x) ... (x) F_D^-1) r by per-mode Cholesky solves."""
        F, _ = self.precond_factors()
        C = [cholesky(f) for f in F]
        r = _f64(r).reshape(self.n)
        z = np.empty(self.n)
        lib().orc_precond_apply(self.D, self._np, _ptr_array(C), _p(r), _p(z))
        return z

    def pcg(self, b, rtol: float, max_iters: int, x0=None):
        """Preconditioned CG from x0 = 0 or x0.  Returns (x, iters, status, rr_history)."""
        return self._krylov(lib().orc_pcg_x0, b, rtol, max_iters, x0)


def cholesky(F) -> np.ndarray:
    """Lower C with F = C C^T (plain loops); raises if F is not SPD."""
    F = _f64(F)
    n = F.shape[0]
    C = np.empty((n, n))
    if lib().orc_cholesky(n, _p(F), _p(C)) != 0:
        raise ValueError("not positive definite")
    return C


def geomean_eig(G) -> float:
    """det(G)^(1/n): the geometric mean of the eigenvalues of an SPD G."""
    G = _f64(G)
    return lib().orc_geomean_eig(G.shape[0], _p(G))


def dot(a, b) -> float:
    a, b = _f64(a).ravel(), _f64(b).ravel()
    assert a.size == b.size
    return lib().orc_dot(a.size, _p(a), _p(b))


def cg_fig2(apply, b, rtol: float, max_iters: int):
    """Fig. 2 step by step for any SPD apply (numpy vectors),
    with readings Z1-Z3, Z12 as in orc_cg; dots through orc_dot.  Returns
    (x, iterations, status, rho history)."""
    b = _f64(b)
    r = b.copy()                       # R := B - A*0
    x = np.zeros_like(b)               # C := 0
    p = r.copy()                       # P := R
    rho = dot(r, r)                    # rho := R+*R
    rho0, hist, k, status = rho, [rho], 0, OK
    if not np.isfinite(rho):
        return x, 0, NONFINITE, np.array(hist)
    while rho > 0.0 and k < max_iters:
        q = apply(p)                   # Q := A*(P*D)
        pq = dot(p, q)
        if not np.isfinite(pq):
            status = NONFINITE
            break
        if not pq > 0.0:
            status = BREAKDOWN
            break
        alpha = rho / pq               # alpha := rho / (P+*Q)
        x = x + alpha * p              # C := C + alpha*P*D
        r = r - alpha * q              # R := R - alpha*Q
        rho1 = dot(r, r)               # rho1 := R+*R
        k += 1
        hist.append(rho1)
        if not np.isfinite(rho1):
            status = NONFINITE
            break
        if rho1 == 0.0 or (rtol > 0.0 and rho1 <= rtol * rtol * rho0):   # Z12; Z1, Z2
            break
        if k == max_iters:
            if rtol > 0.0:
                status = NOT_CONVERGED
            break
        p = r + (rho1 / rho) * p       # P := R + (rho1/rho)*P
        rho = rho1
    return x, k, status, np.array(hist)


class ScatteredOperator:
    """Scattered-data normal operator (Sec. 4; reading Z27):
    M x = sum_k w_k <w_k, x> + lam * sum_d (mode-d R_d) x,  w_k = (x)_d a_{k,d},
    a_{k,d}[i] = beta3(t[k, d] - i) (the cubic B-spline of Z5), R_d = L_d^T L_d.
    n: grid shape; t: K x D sample coordinates in grid units; L: list or None."""

    def __init__(self, n, t, L=None, lam=0.0):
        self.n = tuple(int(v) for v in n)
        self.D = len(self.n)
        self.t = _f64(t).reshape(-1, self.D)
        self.K = self.t.shape[0]
        self.lam = float(lam)
        self._na, self._np = _i64(self.n)
        R = [None] * self.D if L is None else [None if (l is None or l.shape[0] == 0) else gram(l) for l in L]
        self._reg = Operator.from_gram(None, [r if r is not None else np.zeros((k, k)) for r, k in zip(R, self.n)],
                                       self.lam)

    @property
    def N(self):
        return int(np.prod(self.n))

    def data(self, x) -> np.ndarray:
        """sum_k w_k <w_k, x>"""
        x = _f64(x).reshape(self.n)
        y = np.zeros(self.n)
        lib().orc_scattered_data(self.D, self._np, self.K, _p(self.t), _p(x), _p(y))
        return y

    def apply(self, x) -> np.ndarray:
        return self.data(x) + self._reg.apply(x)

    def rhs(self, yk) -> np.ndarray:
        yk = _f64(yk).ravel()
        assert yk.size == self.K
        b = np.empty(self.n)
        lib().orc_scattered_rhs(self.D, self._np, self.K, _p(self.t), _p(yk), _p(b))
        return b

    def forward(self, x) -> np.ndarray:
        x = _f64(x).reshape(self.n)
        yk = np.empty(self.K)
        lib().orc_scattered_forward(self.D, self._np, self.K, _p(self.t), _p(x), _p(yk))
        return yk

    def cg(self, b, rtol: float, max_iters: int):
        x, k, st, hist = cg_fig2(lambda v: self.apply(v.reshape(self.n)), _f64(b).reshape(self.n), rtol, max_iters)
        return x, k, st, hist
