"""Thin ctypes binding of libdd (include/dd_api.h): argument marshalling only.

Every step of the hot path runs in libdd's CUDA kernels; torch is used for device memory
and streams.  There is no CPU fallback: if libdd.so is missing or fails to load, every
entry point raises.
Vectors are torch float64 tensors of shape (ncols, n_Γ), contiguous — i.e. the library's
n_Γ x ncols column-major layout (one right-hand side per row of the tensor).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdd.so")

DD_OK, DD_EINVAL, DD_ECUDA, DD_ENOMEM, DD_ENOTSPD, DD_ENOCONV, DD_ENCCL, DD_EUNSUPPORTED = range(8)
STATUS_NAMES = ["DD_OK", "DD_EINVAL", "DD_ECUDA", "DD_ENOMEM", "DD_ENOTSPD", "DD_ENOCONV", "DD_ENCCL", "DD_EUNSUPPORTED"]
KCLASS = ["gemm_dst", "gemm_schur", "polesum_pcg", "other"]

EXPORTS = ["dd_setup", "dd_setup_ex", "dd_interface_size", "dd_apply_schur", "dd_apply_precond", "dd_pcg_solve",
           "dd_pcg_solve_host", "dd_destroy", "dd_last_error", "dd_profile_enable", "dd_profile_read",
           "dd_launch_count", "dd_query_config", "dd_test_dgemm", "dd_last_solve_ms", "dd_nccl_unique_id",
           "dd_inner_iterations", "dd_bulk_solve", "dd_bulk_pcg_solve", "dd_set_schur_mode"]


class DDError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES[status] if 0 <= status < len(STATUS_NAMES) else status}: {msg}")
        self.status = status


class _Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("cells_per_side", ctypes.c_int), ("gamma_face", ctypes.c_int)]


class _Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("mode", ctypes.c_int)]


class _Frac(ctypes.Structure):
    _fields_ = [("t", ctypes.c_double), ("shifted", ctypes.c_int), ("mode", ctypes.c_int), ("fc0", ctypes.c_double),
                ("n_fpoles", ctypes.c_int), ("fpoles", ctypes.c_void_p), ("fresidues", ctypes.c_void_p)]


DD_FRAC_DENSE, DD_FRAC_RA = 0, 1


@dataclass
class Frac:
    """Fractional perturbation γ L^t (dd_frac): t in (-1, 1); shifted: L = -Δ_Γ + I_Γ;
    mode 'dense' (F formed at setup) or 'ra' (F x = M r_F(L) M x, r_F = fra ≈ λ^t, Remark 1)."""
    t: float = -0.5
    shifted: bool = False
    mode: str = "dense"
    fra: object = None           # RationalApprox-like (c0, poles, residues) in the pair (A_Γ, M_Γ) convention


_lib = None


def load():
    """Load libdd.so (fails loudly: the product path has no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"libdd.so not built ({LIB_PATH}); run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_double
    lib.dd_setup.argtypes = [ctypes.POINTER(_Mesh), I, P, P, I, P, P, P, I, I, P, ctypes.POINTER(_Dist), ctypes.POINTER(P)]
    lib.dd_setup.restype = I
    lib.dd_setup_ex.argtypes = [ctypes.POINTER(_Mesh), ctypes.POINTER(_Frac), I, P, P, I, P, P, P, I, I, P,
                                ctypes.POINTER(_Dist), ctypes.POINTER(P)]
    lib.dd_setup_ex.restype = I
    lib.dd_interface_size.argtypes = [P]; lib.dd_interface_size.restype = I
    lib.dd_apply_schur.argtypes = [P, I, P, P, P]; lib.dd_apply_schur.restype = I
    lib.dd_apply_precond.argtypes = [P, I, P, P, P]; lib.dd_apply_precond.restype = I
    lib.dd_pcg_solve.argtypes = [P, I, P, P, P, D, I, I, P, P, P]; lib.dd_pcg_solve.restype = I
    lib.dd_pcg_solve_host.argtypes = [P, I, P, P, P, D, I, I, P, P, P]; lib.dd_pcg_solve_host.restype = I
    lib.dd_destroy.argtypes = [P]; lib.dd_destroy.restype = I
    lib.dd_last_error.argtypes = []; lib.dd_last_error.restype = ctypes.c_char_p
    lib.dd_profile_enable.argtypes = [P, I]; lib.dd_profile_enable.restype = I
    lib.dd_set_schur_mode.argtypes = [P, I]; lib.dd_set_schur_mode.restype = I
    lib.dd_profile_read.argtypes = [P, P, P]; lib.dd_profile_read.restype = I
    lib.dd_launch_count.argtypes = [P]; lib.dd_launch_count.restype = ctypes.c_longlong
    lib.dd_query_config.argtypes = [P, P, P, P, P]; lib.dd_query_config.restype = I
    lib.dd_last_solve_ms.argtypes = [P, P]; lib.dd_last_solve_ms.restype = I
    lib.dd_nccl_unique_id.argtypes = [P]; lib.dd_nccl_unique_id.restype = I
    lib.dd_inner_iterations.argtypes = [P, P]; lib.dd_inner_iterations.restype = I
    lib.dd_bulk_solve.argtypes = [P, I, P, P, P, D, I, I, P, P]; lib.dd_bulk_solve.restype = I
    lib.dd_bulk_pcg_solve.argtypes = [P, I, P, P, P, D, I, P, P]; lib.dd_bulk_pcg_solve.restype = I
    lib.dd_test_dgemm.argtypes = [I, I, I, P, I, P, I, P, I, I, P]; lib.dd_test_dgemm.restype = I
    _lib = lib
    return lib


def _check(status: int, allow=()):
    if status != DD_OK and status not in allow:
        raise DDError(status, load().dd_last_error().decode())
    return status


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


@dataclass
class SolveResult:
    x: object
    iters: np.ndarray
    rel_res: np.ndarray
    hist: np.ndarray | None
    status: int


class Solver:
    """Handle on libdd for one mesh and a list of parameter sets.

    params: sequence of (K, mu_inv); ras: matching RationalApprox-like objects with
    attributes c0, poles, residues (all parameter sets padded to the same pole count with
    zero residues).
    """

    def __init__(self, dim: int, N: int, params, ras, max_cols: int, device: int = 0, stream=None, dist=None,
                 frac: Frac = None):
        """dist: None, or (rank, world, mode, unique_id_bytes) with mode DD_SHARD_COLUMNS (0) or
        DD_SHARD_POLES (1); the 128-byte unique id comes from nccl_unique_id() on rank 0.
        frac: None (Eq.(2): t = -1/2, unshifted, dense F) or a Frac."""
        import torch
        self._torch = torch
        lib = load()
        self.dim, self.N = dim, N
        self.n_param = len(params)
        m = max(len(r.poles) for r in ras)
        K = _f64([p[0] for p in params]); mu = _f64([p[1] for p in params])
        poles = np.full((self.n_param, m), -1.0); res = np.zeros((self.n_param, m))
        for j, r in enumerate(ras):
            poles[j, :len(r.poles)] = r.poles; res[j, :len(r.residues)] = r.residues
        poles, res = _f64(poles), _f64(res)
        c0 = _f64([r.c0 for r in ras])
        self.device = torch.device("cuda", device)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        mesh = _Mesh(dim, N, 0)
        h = ctypes.c_void_p()
        dptr = None
        if dist is not None:
            rank, world, mode, uid = dist
            # uid None: no communicator (pole split: this rank's partial sums; see dd_api.h dd_dist)
            self._uid = ctypes.create_string_buffer(bytes(uid), 128) if uid is not None else None
            self._dist = _Dist(int(rank), int(world),
                               ctypes.cast(self._uid, ctypes.c_void_p) if uid is not None else None, int(mode))
            dptr = ctypes.byref(self._dist)
        fr = frac if frac is not None else Frac()
        self.frac = fr
        fpol = _f64(fr.fra.poles if fr.fra is not None else [])
        fres = _f64(fr.fra.residues if fr.fra is not None else [])
        self._fkeep = (fpol, fres)
        mode = {"dense": DD_FRAC_DENSE, "ra": DD_FRAC_RA}.get(fr.mode, -1)
        cfr = _Frac(float(fr.t), int(bool(fr.shifted)), mode,
                    float(fr.fra.c0) if fr.fra is not None else 0.0, int(fpol.size),
                    fpol.ctypes.data if fpol.size else None, fres.ctypes.data if fres.size else None)
        st = lib.dd_setup_ex(ctypes.byref(mesh), ctypes.byref(cfr), self.n_param, K.ctypes.data, mu.ctypes.data, m,
                             poles.ctypes.data, res.ctypes.data, c0.ctypes.data, int(max_cols), int(device),
                             ctypes.c_void_p(self.stream.cuda_stream), dptr, ctypes.byref(h))
        _check(st)
        self._h = h
        self.max_cols = int(max_cols)
        self.n_gamma = lib.dd_interface_size(h)

    # ------------------------------------------------------------------ helpers
    def _cols(self, col_param):
        t = self._torch
        if isinstance(col_param, t.Tensor):
            return col_param.to(device=self.device, dtype=t.int32).contiguous()
        return t.as_tensor(np.asarray(col_param, dtype=np.int32), device=self.device)

    def _vec(self, a):
        t = self._torch
        if not isinstance(a, t.Tensor):
            a = t.as_tensor(_f64(a), device=self.device)
        assert a.dtype == t.float64 and a.is_contiguous() and a.device == self.device
        assert a.dim() == 2 and a.shape[1] == self.n_gamma
        return a

    # ------------------------------------------------------------------ API
    def apply_schur(self, x, col_param, y=None):
        x = self._vec(x); cp = self._cols(col_param)
        y = self._torch.empty_like(x) if y is None else y
        _check(load().dd_apply_schur(self._h, x.shape[0], _ptr(cp), _ptr(x), _ptr(y)))
        return y

    def apply_precond(self, r, col_param, z=None):
        r = self._vec(r); cp = self._cols(col_param)
        z = self._torch.empty_like(r) if z is None else z
        _check(load().dd_apply_precond(self._h, r.shape[0], _ptr(cp), _ptr(r), _ptr(z)))
        return z

    def pcg_solve(self, b, col_param, x=None, rtol=1e-10, maxit=500, norm_kind=0, want_hist=False):
        b = self._vec(b); cp = self._cols(col_param)
        x = self._torch.empty_like(b) if x is None else x
        nc = b.shape[0]
        iters = np.zeros(nc, dtype=np.int32); rel = np.zeros(nc)
        hist = np.full(maxit + 1, np.nan) if want_hist else None
        st = load().dd_pcg_solve(self._h, nc, _ptr(cp), _ptr(b), _ptr(x), float(rtol), int(maxit), int(norm_kind),
                                 iters.ctypes.data, rel.ctypes.data, hist.ctypes.data if want_hist else None)
        _check(st, allow=(DD_ENOCONV, DD_ENOTSPD))
        if hist is not None:
            hist = hist[: int(iters[0]) + 1] if nc else hist[:0]
        return SolveResult(x, iters, rel, hist, st)

    def bulk_solve(self, b, col_param, x=None, rtol=1e-10, maxit=500, norm_kind=0):
        """Full DD solve on bulk right-hand sides: b is (ncols, n^d + n^(d-1)) — interior nodes
        x-major (2D: (i, j); 3D: (i, j, k)), then the Γ nodes (include/dd_api.h dd_bulk_solve)."""
        t = self._torch
        n = self.N - 1
        if not isinstance(b, t.Tensor):
            b = t.as_tensor(_f64(b), device=self.device)
        assert b.dtype == t.float64 and b.is_contiguous() and b.device == self.device
        assert b.dim() == 2 and b.shape[1] == (n * n + n if self.dim == 2 else n ** 3 + n * n)
        ncols = b.shape[0]
        x = t.empty_like(b) if x is None else x
        cp = self._cols(col_param)
        iters = np.zeros(ncols, dtype=np.int32); rel = np.zeros(ncols)
        st = load().dd_bulk_solve(self._h, ncols, _ptr(cp), _ptr(b), _ptr(x), float(rtol), int(maxit), int(norm_kind),
                                  iters.ctypes.data, rel.ctypes.data)
        _check(st, allow=(DD_ENOCONV,))
        return SolveResult(x, iters, rel, None, st)

    def bulk_pcg_solve(self, b, col_param, x=None, rtol=1e-10, maxit=500):
        """PCG on the bulk system with the Eq.(5) DD preconditioner (dd_bulk_pcg_solve)."""
        t = self._torch
        n = self.N - 1
        if not isinstance(b, t.Tensor):
            b = t.as_tensor(_f64(b), device=self.device)
        assert b.dtype == t.float64 and b.is_contiguous() and b.device == self.device
        assert b.dim() == 2 and b.shape[1] == (n * n + n if self.dim == 2 else n ** 3 + n * n)
        ncols = b.shape[0]
        x = t.empty_like(b) if x is None else x
        cp = self._cols(col_param)
        iters = np.zeros(ncols, dtype=np.int32); rel = np.zeros(ncols)
        st = load().dd_bulk_pcg_solve(self._h, ncols, _ptr(cp), _ptr(b), _ptr(x), float(rtol), int(maxit),
                                      iters.ctypes.data, rel.ctypes.data)
        _check(st, allow=(DD_ENOCONV,))
        return SolveResult(x, iters, rel, None, st)

    def pcg_solve_host(self, b: np.ndarray, col_param, rtol=1e-10, maxit=500, norm_kind=0, x_out=None):
        b = np.ascontiguousarray(b, dtype=np.float64)
        nc = b.shape[0]
        cp = np.ascontiguousarray(np.asarray(col_param, dtype=np.int32))
        x = np.empty_like(b) if x_out is None else x_out
        iters = np.zeros(nc, dtype=np.int32); rel = np.zeros(nc)
        st = load().dd_pcg_solve_host(self._h, nc, cp.ctypes.data, b.ctypes.data, x.ctypes.data, float(rtol),
                                      int(maxit), int(norm_kind), iters.ctypes.data, rel.ctypes.data, None)
        _check(st, allow=(DD_ENOCONV, DD_ENOTSPD))
        return SolveResult(x, iters, rel, None, st)

    def set_schur_mode(self, mode: str):
        """2D: "grouped" (default for dense F; one GEMM with H_p = K_p G + γ_p F per parameter set),
        "assembled" (one GEMM with [F | G]) or "factored" (K1 + K2 per apply)."""
        _check(load().dd_set_schur_mode(self._h, {"factored": 0, "assembled": 1, "grouped": 2}.get(mode, -1)))

    def profile(self, on: bool):
        _check(load().dd_profile_enable(self._h, 1 if on else 0))

    def profile_read(self):
        ms = np.zeros(4); n = np.zeros(4, dtype=np.int64)
        _check(load().dd_profile_read(self._h, ms.ctypes.data, n.ctypes.data))
        return {k: (float(ms[i]), int(n[i])) for i, k in enumerate(KCLASS)}

    def last_solve_ms(self) -> float:
        v = ctypes.c_double()
        _check(load().dd_last_solve_ms(self._h, ctypes.byref(v)))
        return v.value

    def inner_iterations(self) -> int:
        v = ctypes.c_int()
        _check(load().dd_inner_iterations(self._h, ctypes.byref(v)))
        return v.value

    def launch_count(self) -> int:
        return int(load().dd_launch_count(self._h))

    def query_config(self):
        v = [ctypes.c_int() for _ in range(4)]
        _check(load().dd_query_config(self._h, *[ctypes.byref(a) for a in v]))
        return {"splitk_dst": v[0].value, "splitk_schur": v[1].value, "polesum_warps": v[2].value,
                "graph_while": v[3].value}

    def close(self):
        if getattr(self, "_h", None):
            load().dd_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(load().dd_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return buf.raw


def test_dgemm(A, B, splitk=1):
    """C = A @ B with libdd's DMMA GEMM (test hook).  A: (M, K) row-major torch fp64 cuda;
    B given as (N, K) row-major torch tensor = K x N column-major.  Returns C as (N, M)."""
    import torch
    M, K = A.shape
    N = B.shape[0]
    Kp = (K + 15) // 16 * 16
    Mp = (M + 63) // 64 * 64; Np = (N + 63) // 64 * 64
    Ap = torch.zeros(Mp, Kp, dtype=torch.float64, device=A.device); Ap[:M, :K] = A
    Bp = torch.zeros(Np, Kp, dtype=torch.float64, device=A.device); Bp[:N, :K] = B
    C = torch.zeros(N, M, dtype=torch.float64, device=A.device)
    st = torch.cuda.current_stream(A.device).cuda_stream
    _check(load().dd_test_dgemm(M, N, Kp, _ptr(Ap), Kp, _ptr(Bp), Kp, _ptr(C), M, int(splitk), ctypes.c_void_p(st)))
    return C
