"""Thin ctypes binding of libtca.so (include/tca.h) -- argument marshalling only.

Every numerical step runs in the library's CUDA kernels.  There is no CPU
fallback: importing this module raises ImportError when libtca.so is missing,
and every call raises TcaError when the library reports a failure.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtca.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"libtca.so not found at {LIB_PATH}: build it with "
        "`python -m paper_1001_5460_b200.build` (there is no CPU fallback)")

_lib = ctypes.CDLL(LIB_PATH)

TCA_F64, TCA_F32 = 0, 1
OK, ERR_INVALID_ARG, ERR_SHAPE, ERR_NOT_SPD, ERR_OOM, ERR_CUDA, ERR_NCCL, \
    ERR_BREAKDOWN, ERR_NONFINITE, NOT_CONVERGED = range(10)

EXPORTED = ["tca_operator_create", "tca_operator_query", "tca_apply", "tca_rhs",
            "tca_cg_solve", "tca_solve_host", "tca_solve_host_batch", "tca_operator_destroy", "tca_generate_normal",
            "tca_forward_model", "tca_status_string", "tca_last_error", "tca_version",
            "tca_operator_set_timing", "tca_operator_get_timing", "tca_kernel_launches",
            "tca_operator_apply_path", "tca_operator_cg_engine", "tca_operator_cg_fused_step", "tca_operator_cg_deferred_x", "tca_operator_create_scattered", "tca_shard_layout", "tca_nccl_get_unique_id",
            "tca_nccl_comm_create", "tca_nccl_comm_destroy", "tca_local_group_create",
            "tca_local_group_destroy", "tca_pcg_solve", "tca_precond_apply", "tca_precond_info",
            "tca_cgsr_solve", "tca_operator_create_gram", "tca_jacobi_solve"]

_vp = ctypes.c_void_p
_i64p = ctypes.POINTER(ctypes.c_int64)
_dpp = ctypes.POINTER(ctypes.POINTER(ctypes.c_double))


def _report(rep):
    return dict(iterations=rep.iterations, converged=bool(rep.converged), status=rep.status, rho0=rep.rho0,
                rho_final=rep.rho_final, relres_final=rep.relres_final, seconds=rep.seconds)


class CgReport(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32),
                ("status", ctypes.c_int32), ("pad", ctypes.c_int32),
                ("rho0", ctypes.c_double), ("rho_final", ctypes.c_double),
                ("relres_final", ctypes.c_double), ("seconds", ctypes.c_double),
                ("rho_history", ctypes.POINTER(ctypes.c_double)),
                ("history_capacity", ctypes.c_int32), ("pad2", ctypes.c_int32)]


class Dist(ctypes.Structure):
    """tca_dist: mode-1 sharding over nranks (exactly one transport)."""
    _fields_ = [("rank", ctypes.c_int), ("nranks", ctypes.c_int), ("nccl_comm", _vp),
                ("local_group", _vp)]


_lib.tca_operator_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _i64p, _i64p, _dpp,
                                     _dpp, ctypes.c_double, ctypes.c_int,
                                     ctypes.POINTER(Dist), _vp]
_lib.tca_operator_query.argtypes = [_vp, _i64p, _i64p, _i64p, _i64p,
                                    ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_size_t)]
_lib.tca_apply.argtypes = [_vp, _vp, _vp, _vp]
_lib.tca_rhs.argtypes = [_vp, _vp, _vp, _vp]
_lib.tca_cg_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int32,
                              ctypes.POINTER(CgReport), _vp]
_lib.tca_solve_host.argtypes = [_vp, _vp, _vp, ctypes.c_double, ctypes.c_int32,
                                ctypes.POINTER(CgReport), _vp]
_lib.tca_solve_host_batch.argtypes = [_vp, ctypes.c_int, ctypes.POINTER(_vp), ctypes.POINTER(_vp), ctypes.c_double,
                                      ctypes.c_int32, ctypes.POINTER(CgReport), _vp]
_lib.tca_operator_destroy.argtypes = [_vp]
_lib.tca_operator_destroy.restype = None
_lib.tca_generate_normal.argtypes = [_vp, ctypes.c_int, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_uint64, ctypes.c_uint32, ctypes.c_double, _vp]
_lib.tca_forward_model.argtypes = [_vp, _vp, _vp, ctypes.c_double, ctypes.c_uint64, _vp]
_lib.tca_status_string.argtypes = [ctypes.c_int]
_lib.tca_status_string.restype = ctypes.c_char_p
_lib.tca_last_error.restype = ctypes.c_char_p
_lib.tca_version.restype = ctypes.c_char_p
_lib.tca_operator_set_timing.argtypes = [_vp, ctypes.c_int]
_lib.tca_operator_get_timing.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), _i64p,
                                         ctypes.c_int]
_lib.tca_kernel_launches.restype = ctypes.c_int64
_lib.tca_shard_layout.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.POINTER(ctypes.c_double),
                                  ctypes.c_int, ctypes.c_int, _i64p]
_lib.tca_shard_layout.restype = ctypes.c_int
_lib.tca_nccl_get_unique_id.argtypes = [_vp]
_lib.tca_nccl_get_unique_id.restype = ctypes.c_int
_lib.tca_nccl_comm_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _vp, ctypes.c_int]
_lib.tca_nccl_comm_create.restype = ctypes.c_int
_lib.tca_nccl_comm_destroy.argtypes = [_vp]
_lib.tca_nccl_comm_destroy.restype = None
_lib.tca_local_group_create.argtypes = [ctypes.POINTER(_vp), ctypes.c_int]
_lib.tca_local_group_create.restype = ctypes.c_int
_lib.tca_local_group_destroy.argtypes = [_vp]
_lib.tca_local_group_destroy.restype = None
_lib.tca_operator_apply_path.argtypes = [_vp]
_lib.tca_operator_cg_engine.argtypes = [_vp]
_lib.tca_operator_cg_fused_step.argtypes = [_vp]
_lib.tca_operator_cg_fused_step.restype = ctypes.c_int
_lib.tca_operator_cg_deferred_x.argtypes = [_vp]
_lib.tca_operator_cg_deferred_x.restype = ctypes.c_int
_lib.tca_pcg_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int32, _vp, _vp]
_lib.tca_precond_apply.argtypes = [_vp, _vp, _vp, _vp]
_lib.tca_cgsr_solve.argtypes = [_vp, _vp, _vp, ctypes.c_int, ctypes.c_double, ctypes.c_int32, _vp, _vp]
_lib.tca_jacobi_solve.argtypes = [_vp, _vp, _vp, ctypes.c_double, ctypes.c_int32, _vp, _vp]
_lib.tca_operator_create_gram.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _i64p, _dpp, _dpp, ctypes.c_double,
                                          ctypes.c_int, _vp, _vp]
_lib.tca_precond_info.argtypes = [_vp, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_int), _vp]
_lib.tca_operator_create_scattered.argtypes = [ctypes.POINTER(_vp), ctypes.c_int, _i64p, ctypes.c_int64,
                                               ctypes.POINTER(ctypes.c_double),
                                               _dpp, ctypes.c_double, ctypes.c_int, _vp]
_lib.tca_operator_apply_path.restype = ctypes.c_int
_lib.tca_operator_cg_engine.restype = ctypes.c_int
for _name in ("tca_operator_create", "tca_operator_query", "tca_apply", "tca_rhs",
              "tca_cg_solve", "tca_solve_host", "tca_solve_host_batch", "tca_generate_normal", "tca_forward_model",
              "tca_operator_set_timing", "tca_operator_get_timing"):
    getattr(_lib, _name).restype = ctypes.c_int


class TcaError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.tca_last_error().decode()
        super().__init__(f"{where}: {_lib.tca_status_string(status).decode()}: {msg}")


def _check(st, where, allow=()):
    if st != OK and st not in allow:
        raise TcaError(st, where)
    return st


def version() -> str:
    return _lib.tca_version().decode()


def _dtype_code(dtype) -> int:
    if dtype in ("f64", "float64", np.float64, TCA_F64):
        return TCA_F64
    if dtype in ("f32", "float32", np.float32, TCA_F32):
        return TCA_F32
    raise ValueError(f"unsupported dtype {dtype!r}")


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    if stream is None:
        torch = _torch()
        if not torch.cuda.is_available():
            return 0  # legacy stream; the library reports the missing device itself
        return torch.cuda.current_stream().cuda_stream
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream


def _dev_ptr(t, numel, tdtype, name):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if t.dtype != tdtype:
        raise ValueError(f"{name} has dtype {t.dtype}, operator uses {tdtype}")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, expected {numel}")
    return ctypes.c_void_p(t.data_ptr())


class Operator:
    """M = (kron_d A_d^T A_d) + lam * sum_d (mode-d L_d^T L_d) on the GPU.

    A: list of m_d x n_d host arrays; L: list of (n_d-2) x n_d arrays or None.
    """

    def __init__(self, A, L=None, lam=0.0, dtype="f64", stream=None, dist=None):
        self._h = _vp()
        A = [np.ascontiguousarray(a, dtype=np.float64) for a in A]
        D = len(A)
        self.order = D
        self.n = tuple(int(a.shape[1]) for a in A)
        self.m = tuple(int(a.shape[0]) for a in A)
        self.lam = float(lam)
        self.dtype_code = _dtype_code(dtype)
        self.dtype = "f64" if self.dtype_code == TCA_F64 else "f32"
        n_arr = (ctypes.c_int64 * D)(*self.n)
        m_arr = (ctypes.c_int64 * D)(*self.m)
        dp = ctypes.POINTER(ctypes.c_double)
        A_arr = (dp * D)(*[a.ctypes.data_as(dp) for a in A])
        keep = [A]
        L_arr = None
        if L is not None:
            Ls = [None if l is None else np.ascontiguousarray(l, dtype=np.float64) for l in L]
            keep.append(Ls)
            L_arr = (dp * D)(*[ctypes.cast(None, dp) if l is None or l.size == 0
                               else l.ctypes.data_as(dp) for l in Ls])
        dist_p = None
        if dist is not None:
            dist_p = ctypes.byref(dist)
        st = _lib.tca_operator_create(ctypes.byref(self._h), D, n_arr, m_arr, A_arr, L_arr,
                                      self.lam, self.dtype_code, dist_p,
                                      _vp(_stream_ptr(stream)))
        _check(st, "tca_operator_create")
        self._finish()

    @classmethod
    def from_gram(cls, G, R, lam=1.0, dtype="f64", stream=None, dist=None):
        """M = (kron_d G_d) + lam * sum_d (mode-d R_d) from its factors
        (tca_operator_create_gram).  G None: no Kronecker-product term (Eq. 9's
        separable Poisson operator); R: list of n_d x n_d arrays (None: no term)."""
        self = cls.__new__(cls)
        self._h = _vp()
        Rs = [None if r is None else np.ascontiguousarray(r, dtype=np.float64) for r in R]
        Gs = None if G is None else [np.ascontiguousarray(g, dtype=np.float64) for g in G]
        D = len(Rs)
        self.order = D
        self.n = tuple(int(r.shape[0]) if r is not None else int(Gs[d].shape[0]) for d, r in enumerate(Rs))
        self.m = self.n
        self.lam = float(lam)
        self.dtype_code = _dtype_code(dtype)
        self.dtype = "f64" if self.dtype_code == TCA_F64 else "f32"
        dp = ctypes.POINTER(ctypes.c_double)
        n_arr = (ctypes.c_int64 * D)(*self.n)
        R_arr = (dp * D)(*[ctypes.cast(None, dp) if r is None else r.ctypes.data_as(dp) for r in Rs])
        G_arr = None if Gs is None else (dp * D)(*[g.ctypes.data_as(dp) for g in Gs])
        st = _lib.tca_operator_create_gram(ctypes.byref(self._h), D, n_arr, G_arr, R_arr, self.lam,
                                           self.dtype_code, None if dist is None else ctypes.byref(dist),
                                           _vp(_stream_ptr(stream)))
        _check(st, "tca_operator_create_gram")
        self._finish()
        return self

    @classmethod
    def scattered(cls, n, t, L=None, lam=0.0, dtype="f64", stream=None):
        """Scattered-data operator (tca_operator_create_scattered, reading Z27):
        M x = sum_k w_k <w_k, x> + lam sum_d (mode-d L_d^T L_d) x for the K x D
        sample coordinates t (grid units, in [0, n_d - 1]).  Its "data" are the K
        sample values: rhs / forward_model / solve_host use shape (K,)."""
        self = cls.__new__(cls)
        self._h = _vp()
        n = tuple(int(v) for v in n)
        D = len(n)
        t = np.ascontiguousarray(t, dtype=np.float64).reshape(-1, D)
        K = t.shape[0]
        self.order = D
        self.n = n
        self.lam = float(lam)
        self.dtype_code = _dtype_code(dtype)
        self.dtype = "f64" if self.dtype_code == TCA_F64 else "f32"
        dp = ctypes.POINTER(ctypes.c_double)
        Ls = None if L is None else [None if l is None else np.ascontiguousarray(l, dtype=np.float64) for l in L]
        L_arr = None if Ls is None else (dp * D)(*[ctypes.cast(None, dp) if l is None else l.ctypes.data_as(dp)
                                                   for l in Ls])
        n_arr = (ctypes.c_int64 * D)(*n)
        st = _lib.tca_operator_create_scattered(ctypes.byref(self._h), D, n_arr, K, t.ctypes.data_as(dp), L_arr,
                                                self.lam, self.dtype_code, _vp(_stream_ptr(stream)))
        _check(st, "tca_operator_create_scattered")
        self.m = (K,)
        self._finish()
        self.K = K
        self.local_m = (K,)
        self.Mloc = K
        return self

    def _finish(self):
        q = self.query()
        self.own_lo, self.own_hi, self.data_lo, self.data_hi = q[:4]
        self.banded_mask, self.half_bandwidth, self.device_bytes = q[4:]
        self.local_n = (self.own_hi - self.own_lo,) + self.n[1:]
        self.local_m = (self.data_hi - self.data_lo,) + self.m[1:]
        self.N = int(np.prod(self.local_n))
        self.Mloc = int(np.prod(self.local_m))

    @property
    def torch_dtype(self):
        torch = _torch()
        return torch.float64 if self.dtype_code == TCA_F64 else torch.float32

    def query(self):
        vals = [ctypes.c_int64() for _ in range(4)]
        mask = ctypes.c_int()
        hb = (ctypes.c_int * 4)()
        nb = ctypes.c_size_t()
        _check(_lib.tca_operator_query(self._h, *[ctypes.byref(v) for v in vals],
                                       ctypes.byref(mask), hb, ctypes.byref(nb)),
               "tca_operator_query")
        return [v.value for v in vals] + [mask.value, tuple(hb[: self.order]), nb.value]

    @property
    def apply_path(self):
        """'fused' (one-pass banded kernel), 'ksum' (Kronecker-sum stencil, factor-form
        operators without a product term) or 'multipass' (generic per-mode kernels)."""
        return {1: "fused", 2: "ksum"}.get(_lib.tca_operator_apply_path(self._h), "multipass")

    @property
    def tiny_engine(self):
        """True when cg_solve runs the single-block engine (tca_tiny.cu: the whole
        solve in one kernel launch, vectors in shared memory) on this operator."""
        return _lib.tca_operator_cg_engine(self._h) == 1

    @property
    def cg_engine(self):
        """Which engine cg_solve runs: 'tiny' (one block, tca_tiny.cu), 'grid' (one
        cooperative grid, tca_grid.cu) or 'general' (graph-replayed kernels)."""
        return {1: "tiny", 2: "grid"}.get(_lib.tca_operator_cg_engine(self._h), "general")

    @property
    def cg_deferred_x(self):
        """True when CG / PCG solves defer the x update into the next apply (a
        streaming warp beside the operator), False otherwise, None
        before the first solve."""
        v = _lib.tca_operator_cg_deferred_x(self._h)
        return None if v < 0 else bool(v)

    @property
    def cg_fused_step(self):
        """True when CG / PCG solves run the fused step B1' (one kernel per iteration
        forms P, updates C and applies the operator), False otherwise, None before
        the first solve."""
        v = _lib.tca_operator_cg_fused_step(self._h)
        return None if v < 0 else bool(v)

    def set_timing(self, enable=True):
        _check(_lib.tca_operator_set_timing(self._h, 1 if enable else 0), "set_timing")

    def get_timing(self, reset=True):
        """(summed apply device ms, number of timed applies) since the last reset."""
        ms = ctypes.c_double()
        cnt = ctypes.c_int64()
        _check(_lib.tca_operator_get_timing(self._h, ctypes.byref(ms), ctypes.byref(cnt),
                                            1 if reset else 0), "get_timing")
        return ms.value, cnt.value

    def close(self):
        if self._h:
            _lib.tca_operator_destroy(self._h)
            self._h = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def empty(self, shape="unknowns"):
        torch = _torch()
        shp = self.local_n if shape == "unknowns" else self.local_m
        return torch.empty(shp, dtype=self.torch_dtype, device="cuda")

    def apply(self, x, y=None, stream=None):
        """y = M x (device tensors of the local unknown shape)."""
        if y is None:
            y = self.empty()
        _check(_lib.tca_apply(self._h, _dev_ptr(x, self.N, self.torch_dtype, "x"),
                              _dev_ptr(y, self.N, self.torch_dtype, "y"),
                              _vp(_stream_ptr(stream))), "tca_apply")
        return y

    def rhs(self, ydata, b=None, stream=None):
        """b = (kron_d A_d^T) ydata."""
        if b is None:
            b = self.empty()
        _check(_lib.tca_rhs(self._h, _dev_ptr(ydata, self.Mloc, self.torch_dtype, "ydata"),
                            _dev_ptr(b, self.N, self.torch_dtype, "b"),
                            _vp(_stream_ptr(stream))), "tca_rhs")
        return b

    def cg_solve(self, b, x=None, rtol=0.0, max_iters=100, history=False, stream=None,
                 raise_on=("breakdown", "nonfinite"), x0=None):
        """Fig. 2 CG from x0 = 0, or from the device tensor x0 (warm start: R := B - A*C).
        Returns (x, report dict)."""
        return self._solve(_lib.tca_cg_solve, "tca_cg_solve", b, x, rtol, max_iters, history, stream, raise_on, x0)

    def pcg_solve(self, b, x=None, rtol=0.0, max_iters=100, history=False, stream=None,
                  raise_on=("breakdown", "nonfinite"), x0=None):
        """CG preconditioned with the Kronecker-factor P (tca_pcg_solve).  Returns (x, report dict)."""
        return self._solve(_lib.tca_pcg_solve, "tca_pcg_solve", b, x, rtol, max_iters, history, stream, raise_on,
                           x0)

    def jacobi_solve(self, b, x=None, threshold=1e-4, max_iters=100000, history=False, stream=None):
        """Tensor Jacobi (Fig. 1, tca_jacobi_solve): x <- U with R+*R <= threshold."""
        return self._solve(_lib.tca_jacobi_solve, "tca_jacobi_solve", b, x, threshold, max_iters, history, stream,
                           ("nonfinite",))

    def cgsr_solve(self, b, x=None, rtol=0.0, max_iters=100, history=False, stream=None,
                   raise_on=("breakdown", "nonfinite"), x0=None):
        """Single-reduction (Chronopoulos-Gear) CG (tca_cgsr_solve).  Returns (x, report dict)."""
        return self._solve(_lib.tca_cgsr_solve, "tca_cgsr_solve", b, x, rtol, max_iters, history, stream, raise_on,
                           x0)

    def _solve(self, fn, name, b, x, rtol, max_iters, history, stream, raise_on, x0=None):
        if x is None:
            x = self.empty()
        if x0 is not None:   # the C ABI's x0_zero = 0: x holds the start on entry
            _dev_ptr(x0, self.N, self.torch_dtype, "x0")
            x.copy_(x0)
        rep = CgReport()
        hist = None
        if history:
            hist = np.zeros(max_iters + 1)
            rep.rho_history = hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
            rep.history_capacity = max_iters + 1
        args = [self._h, _dev_ptr(b, self.N, self.torch_dtype, "b"), _dev_ptr(x, self.N, self.torch_dtype, "x")]
        if fn is not _lib.tca_jacobi_solve:
            args.append(0 if x0 is not None else 1)   # x0_zero
        st = fn(*args, float(rtol), int(max_iters), ctypes.byref(rep), _vp(_stream_ptr(stream)))
        allow = [NOT_CONVERGED]
        if "breakdown" not in raise_on:
            allow.append(ERR_BREAKDOWN)
        if "nonfinite" not in raise_on:
            allow.append(ERR_NONFINITE)
        _check(st, name, allow=allow)
        out = _report(rep)
        if hist is not None:
            out["rho_history"] = hist[: rep.iterations + 1]
        return x, out

    def precond_apply(self, r, z=None, stream=None):
        """z = P^-1 r with the PCG preconditioner (device tensors of the local shape)."""
        if z is None:
            z = self.empty()
        _check(_lib.tca_precond_apply(self._h, _dev_ptr(r, self.N, self.torch_dtype, "r"),
                                      _dev_ptr(z, self.N, self.torch_dtype, "z"),
                                      _vp(_stream_ptr(stream))), "tca_precond_apply")
        return z

    def precond_info(self):
        """(eps_d list, lower bandwidth of each Cholesky factor)."""
        eps = (ctypes.c_double * self.order)()
        bw = (ctypes.c_int * self.order)()
        _check(_lib.tca_precond_info(self._h, eps, bw, _vp(0)), "tca_precond_info")
        return list(eps), list(bw)

    def solve_host_batch(self, ydata_hosts, x_hosts, rtol=0.0, max_iters=100, stream=None):
        """Pipelined end-to-end solves (tca_solve_host_batch): item i's host data
        ydata_hosts[i] -> rhs -> CG -> x_hosts[i], the host<->device copies of
        neighbouring items overlapping the compute.  Returns one report per item."""
        if len(ydata_hosts) != len(x_hosts):
            raise ValueError("ydata_hosts and x_hosts differ in length")
        for lst, numel, name in ((ydata_hosts, self.Mloc, "ydata_hosts"), (x_hosts, self.N, "x_hosts")):
            for t in lst:
                if t.is_cuda or not t.is_contiguous() or t.dtype != self.torch_dtype or t.numel() != numel:
                    raise ValueError(f"{name}: expected contiguous host tensors of {numel} {self.torch_dtype}")
        n = len(ydata_hosts)
        ys = (_vp * max(n, 1))(*[_vp(t.data_ptr()) for t in ydata_hosts])
        xs = (_vp * max(n, 1))(*[_vp(t.data_ptr()) for t in x_hosts])
        reps = (CgReport * max(n, 1))()
        st = _lib.tca_solve_host_batch(self._h, n, ys, xs, float(rtol), int(max_iters), reps,
                                       _vp(_stream_ptr(stream)))
        _check(st, "tca_solve_host_batch", allow=[NOT_CONVERGED])
        return [_report(r) for r in reps[:n]]

    def solve_host(self, ydata_host, x_host, rtol=0.0, max_iters=100, stream=None):
        """End-to-end solve from host buffers (torch CPU tensors, pinned recommended)."""
        torch = _torch()
        for t, numel, name in ((ydata_host, self.Mloc, "ydata_host"), (x_host, self.N, "x_host")):
            if t.is_cuda or not t.is_contiguous() or t.dtype != self.torch_dtype or t.numel() != numel:
                raise ValueError(f"{name}: expected a contiguous host tensor of {numel} {self.torch_dtype}")
        rep = CgReport()
        st = _lib.tca_solve_host(self._h, _vp(ydata_host.data_ptr()), _vp(x_host.data_ptr()),
                                 float(rtol), int(max_iters), ctypes.byref(rep),
                                 _vp(_stream_ptr(stream)))
        _check(st, "tca_solve_host", allow=[NOT_CONVERGED])
        del torch
        return _report(rep)

    def forward_model(self, x=None, ydata=None, sigma=0.01, seed=1, stream=None):
        """ydata = (kron A_d) x + sigma * noise(seed); x None -> x_true(seed) generated on device."""
        if ydata is None:
            ydata = self.empty("data")
        xp = None if x is None else _dev_ptr(x, int(np.prod(self.n)), self.torch_dtype, "x")
        _check(_lib.tca_forward_model(self._h, xp,
                                      _dev_ptr(ydata, self.Mloc, self.torch_dtype, "ydata"),
                                      float(sigma), int(seed), _vp(_stream_ptr(stream))),
               "tca_forward_model")
        return ydata


def kernel_launches() -> int:
    """Process-wide count of CUDA kernel launches issued by libtca."""
    return int(_lib.tca_kernel_launches())


def generate_normal(out, seed, stream_id, offset=0, scale=1.0, stream=None):
    """out[i] = scale * normal(seed, stream_id, offset + i) on the device."""
    torch = _torch()
    code = TCA_F64 if out.dtype == torch.float64 else TCA_F32
    _check(_lib.tca_generate_normal(_dev_ptr(out, out.numel(), out.dtype, "out"), code,
                                    out.numel(), int(offset), int(seed), int(stream_id),
                                    float(scale), _vp(_stream_ptr(stream))),
           "tca_generate_normal")
    return out


def shard_layout(n1, A1, rank, nranks):
    """(own_lo, own_hi, data_lo, data_hi) of a mode-1 shard (host-only library call)."""
    A1 = np.ascontiguousarray(A1, dtype=np.float64)
    m1, n1_ = A1.shape
    assert n1_ == n1
    out = (ctypes.c_int64 * 4)()
    _check(_lib.tca_shard_layout(n1, m1, A1.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                 rank, nranks, out), "tca_shard_layout")
    return tuple(int(v) for v in out)


class NcclComm:
    """NCCL communicator of the library (bootstrap: rank 0's unique id is broadcast
    by the caller, e.g. over torch.distributed)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(_lib.tca_nccl_get_unique_id(buf), "tca_nccl_get_unique_id")
        return buf.raw

    def __init__(self, nranks, uid: bytes, rank):
        self.handle = _vp()
        buf = ctypes.create_string_buffer(uid, 128)
        _check(_lib.tca_nccl_comm_create(ctypes.byref(self.handle), nranks, buf, rank),
               "tca_nccl_comm_create")
        self.nranks, self.rank = nranks, rank

    def dist(self):
        return Dist(self.rank, self.nranks, self.handle, None)

    def close(self):
        if self.handle:
            _lib.tca_nccl_comm_destroy(self.handle)
            self.handle = _vp()


class LocalGroup:
    """In-process shard group (local transport): shards driven by host threads."""

    def __init__(self, nranks):
        self.handle = _vp()
        _check(_lib.tca_local_group_create(ctypes.byref(self.handle), nranks),
               "tca_local_group_create")
        self.nranks = nranks

    def dist(self, rank):
        return Dist(rank, self.nranks, None, self.handle)

    def close(self):
        if self.handle:
            _lib.tca_local_group_destroy(self.handle)
            self.handle = _vp()


def exported_symbols():
    """Names from include/tca.h that the loaded library exports."""
    return [n for n in EXPORTED if hasattr(_lib, n)]
