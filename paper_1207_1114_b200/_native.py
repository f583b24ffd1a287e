"""ctypes binding of the FastPFP C-ABI (include/fastpfp.h) — argument marshalling only.

Every step of the method runs in the library's sm_100a kernels; this module converts numpy arrays /
torch tensors into pointers, checks status codes and packs reports. It never falls back to a CPU
implementation: if libfastpfp.so is missing or no sm_100 device is present it raises.
"""
from __future__ import annotations

import ctypes as C
import os
import re
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FASTPFP_LIB") or os.path.join(HERE, "lib", "libfastpfp.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "fastpfp.h")

OK, EINVAL, ESYM, ENONFINITE, ESTATE, ENOMEM, ECUDA, ENCCL, ENODEV, EPOISONED, EUNSUPPORTED = range(11)
OPT_SLACK_MODE, OPT_PRECISION, OPT_RESCALE, OPT_STREAM, OPT_CHECK_EVERY, OPT_PROFILE = 1, 2, 3, 4, 5, 6
OPT_GEMM_CTA_GROUP = 7
OPT_PROJ_KERNEL = 8
OPT_METHOD = 9
OPT_NCCL_TIMEOUT_MS = 10
METHOD_FASTPFP, METHOD_PG, METHOD_FASTGA = 0, 1, 2
PREC_TF32X3, PREC_TF32, PREC_FP32_SIMT, PREC_INT8_OZAKI = 0, 1, 2, 3


class FastPFPError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[{status}] {msg}")
        self.status = status


class Report(C.Structure):
    _fields_ = [
        ("iterations", C.c_int32), ("converged", C.c_int32), ("degenerate", C.c_int32),
        ("total_sweeps", C.c_int32), ("last_rho", C.c_double), ("last_delta", C.c_double),
        ("last_mu", C.c_double), ("trace_capacity", C.c_int32), ("reserved", C.c_int32),
        ("rho_trace", C.POINTER(C.c_double)), ("sweeps_trace", C.POINTER(C.c_int32)),
        ("delta_trace", C.POINTER(C.c_double)), ("mu_trace", C.POINTER(C.c_double)),
    ]


class Stats(C.Structure):
    _fields_ = [
        ("launches", C.c_int64), ("gemm_launches", C.c_int64), ("proj_launches", C.c_int64),
        ("outer_iterations", C.c_int64), ("sweeps", C.c_int64), ("gemm_ms", C.c_double),
        ("proj_ms", C.c_double), ("gemm_flops", C.c_double), ("onchip_launches", C.c_int64),
        ("onchip_tiles", C.c_int32), ("reserved", C.c_int32),
    ]


_lib = None


def declared_symbols() -> List[str]:
    """Function names declared in include/fastpfp.h."""
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^(?:const\s+)?(?:int|void|char)\s*\**\s*(fastpfp_\w+)\s*\(",
                                 src, flags=re.M)))


def _nccl_hint():
    """Point the library's NCCL loader at torch's bundled libnccl (the one the process uses)."""
    if os.environ.get("FASTPFP_NCCL_LIB"):
        return
    try:
        import nvidia.nccl as nv
        for base in list(getattr(nv, "__path__", [])):
            cand = os.path.join(base, "lib", "libnccl.so.2")
            if os.path.exists(cand):
                os.environ["FASTPFP_NCCL_LIB"] = cand
                return
    except Exception:
        pass


def lib():
    """Load libfastpfp.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    _nccl_hint()
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1207_1114_b200.build` "
                          "(there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    H, I64, I32, D, FP, VP = C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_void_p, C.c_void_p
    sig = {
        "fastpfp_create": (C.c_int, [I64, I64, I64, C.POINTER(H)]),
        "fastpfp_create_dist": (C.c_int, [I64, I64, I64, C.c_int, C.c_int, VP, C.POINTER(H)]),
        "fastpfp_nccl_unique_id": (C.c_int, [VP, I64]),
        "fastpfp_set_graphs": (C.c_int, [H, FP, FP, FP, FP, C.c_int]),
        "fastpfp_set_x0": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_set_ga_schedule": (C.c_int, [H, D, D, D]),
        "fastpfp_reset": (C.c_int, [H]),
        "fastpfp_iterate": (C.c_int, [H, D, D, D, D, I32, I32, FP, C.POINTER(Report)]),
        "fastpfp_copy_x": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_copy_y": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_set_y": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_discretize": (C.c_int, [H, VP]),
        "fastpfp_objective": (C.c_int, [H, D, C.POINTER(D)]),
        "fastpfp_set_option": (C.c_int, [H, C.c_int, I64]),
        "fastpfp_get_option": (C.c_int, [H, C.c_int, C.POINTER(I64)]),
        "fastpfp_dist_collectives": (C.c_int, [H, VP, I64, C.POINTER(I64)]),
        "fastpfp_get_stats": (C.c_int, [H, C.POINTER(Stats)]),
        "fastpfp_reset_stats": (C.c_int, [H]),
        "fastpfp_destroy": (None, [H]),
        "fastpfp_last_error": (C.c_char_p, [H]),
        "fastpfp_status_string": (C.c_char_p, [C.c_int]),
        "fastpfp_abi_version": (C.c_int, []),
        "fastpfp_device_arch": (C.c_int, []),
        "fastpfp_project": (C.c_int, [FP, I64, D, I32, C.POINTER(I32), C.POINTER(D), I64]),
        "fastpfp_batched_create": (C.c_int, [I64, I64, I64, I64, C.POINTER(H)]),
        "fastpfp_batched_set_graphs": (C.c_int, [H, FP, FP, FP, FP, C.c_int]),
        "fastpfp_batched_set_x0": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_batched_iterate": (C.c_int, [H, D, D, D, D, I32, I32, FP, VP, VP, VP]),
        "fastpfp_batched_copy_x": (C.c_int, [H, FP, C.c_int]),
        "fastpfp_batched_discretize": (C.c_int, [H, VP]),
        "fastpfp_batched_set_option": (C.c_int, [H, C.c_int, I64]),
        "fastpfp_batched_get_stats": (C.c_int, [H, C.POINTER(Stats)]),
        "fastpfp_batched_destroy": (None, [H]),
        "fastpfp_batched_last_error": (C.c_char_p, [H]),
        "fastpfp_gemm_nt": (C.c_int, [FP, FP, FP, I64, I64, I64, C.c_int, C.c_int, I64]),
        "fastpfp_gemm_nt_blocked": (C.c_int, [FP, FP, FP, I64, I64, I64, I32, C.c_int, I64]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    _lib = L
    return L


def _ptr(x):
    """(pointer, is_device, keepalive) for a numpy array or torch tensor (float32, C-contiguous)."""
    if x is None:
        return None, 0, None
    if hasattr(x, "data_ptr") and hasattr(x, "is_cuda"):
        if x.dtype.__repr__() != "torch.float32":
            raise TypeError("float32 tensor required")
        if not x.is_contiguous():
            raise ValueError("contiguous tensor required")
        return (x.data_ptr(), 1 if x.is_cuda else 0, x)
    a = np.ascontiguousarray(x, dtype=np.float32)
    return a.ctypes.data, 0, a


def _check(st: int, h=None, err_fn="fastpfp_last_error"):
    if st != OK:
        L = lib()
        msg = (getattr(L, err_fn)(h) or b"").decode() if h else ""
        raise FastPFPError(st, f"{L.fastpfp_status_string(st).decode()}: {msg}")


@dataclass
class IterReport:
    iterations: int
    converged: bool
    degenerate: bool
    total_sweeps: int
    last_rho: float
    last_delta: float
    last_mu: float
    rho: List[float] = field(default_factory=list)
    sweeps: List[int] = field(default_factory=list)
    delta: List[float] = field(default_factory=list)
    mu: List[float] = field(default_factory=list)


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for Solver(..., dist=(rank, world, uid)) (create on rank 0)."""
    buf = C.create_string_buffer(128)
    _check(lib().fastpfp_nccl_unique_id(buf, 128))
    return buf.raw


class Solver:
    """One FastPFP problem instance on the current CUDA device (fastpfp_create ... destroy).

    dist=(rank, world, uid) creates the row-sharded handle (fastpfp_create_dist): this rank owns
    rows [rank*n/world, (rank+1)*n/world) of A, B and X."""

    def __init__(self, n: int, n_prime: int, d: int = 0, dist=None):
        L = lib()
        h = C.c_void_p()
        self.rank, self.world = 0, 1
        if dist is None:
            _check(L.fastpfp_create(n, n_prime, d, C.byref(h)))
        else:
            rank, world, uid = dist
            ub = C.create_string_buffer(bytes(uid), 128)
            _check(L.fastpfp_create_dist(n, n_prime, d, int(rank), int(world), ub, C.byref(h)))
            self.rank, self.world = int(rank), int(world)
        self._h = h
        self.n_glob = n
        self.n, self.n_prime, self.d = n // self.world, n_prime, d

    # -- lifecycle --------------------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            lib().fastpfp_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- calls ------------------------------------------------------------------------------
    def set_option(self, key: int, value: int):
        _check(lib().fastpfp_set_option(self._h, key, int(value)), self._h)

    def get_option(self, key: int) -> int:
        v = C.c_int64()
        _check(lib().fastpfp_get_option(self._h, key, C.byref(v)), self._h)
        return v.value

    def set_graphs(self, A, Ap, B=None, Bp=None):
        pa, da, ka = _ptr(A)
        pp, dp, kp = _ptr(Ap)
        pb, db, kb = _ptr(B)
        pbp, dbp, kbp = _ptr(Bp)
        dev = da
        if any(x is not None and d != dev for x, d in ((Ap, dp), (B, db), (Bp, dbp))):
            raise ValueError("all inputs must live on the same side (host or device)")
        self._check_shape(A, (self.n, self.n_glob)); self._check_shape(Ap, (self.n_prime, self.n_prime))
        if self.d > 0:
            self._check_shape(B, (self.n, self.d)); self._check_shape(Bp, (self.n_prime, self.d))
        _check(lib().fastpfp_set_graphs(self._h, pa, pp, pb, pbp, dev), self._h)

    def set_x0(self, X0=None):
        p, dev, keep = _ptr(X0)
        if X0 is not None:
            self._check_shape(X0, (self.n, self.n_prime))
        _check(lib().fastpfp_set_x0(self._h, p, dev), self._h)

    def reset(self):
        _check(lib().fastpfp_reset(self._h), self._h)

    def set_ga_schedule(self, beta0=0.5, rate=1.075, beta_max=10.0):
        _check(lib().fastpfp_set_ga_schedule(self._h, float(beta0), float(rate), float(beta_max)),
               self._h)

    def iterate(self, alpha, lam, eps1, eps2, max_iter1, max_iter2, want_x=True, trace=None):
        trace = max_iter1 if trace is None else trace
        rep = Report()
        bufs = None
        if trace > 0:
            bufs = (np.zeros(trace), np.zeros(trace, np.int32), np.zeros(trace), np.zeros(trace))
            rep.trace_capacity = trace
            rep.rho_trace = bufs[0].ctypes.data_as(C.POINTER(C.c_double))
            rep.sweeps_trace = bufs[1].ctypes.data_as(C.POINTER(C.c_int32))
            rep.delta_trace = bufs[2].ctypes.data_as(C.POINTER(C.c_double))
            rep.mu_trace = bufs[3].ctypes.data_as(C.POINTER(C.c_double))
        X = np.empty((self.n, self.n_prime), np.float32) if want_x else None
        _check(lib().fastpfp_iterate(self._h, float(alpha), float(lam), float(eps1), float(eps2),
                                     int(max_iter1), int(max_iter2),
                                     X.ctypes.data if X is not None else None, C.byref(rep)),
               self._h)
        k = rep.iterations
        out = IterReport(k, bool(rep.converged), bool(rep.degenerate), rep.total_sweeps,
                         rep.last_rho, rep.last_delta, rep.last_mu)
        if bufs is not None:
            kk = min(k, trace)
            out.rho = bufs[0][:kk].tolist(); out.sweeps = bufs[1][:kk].tolist()
            out.delta = bufs[2][:kk].tolist(); out.mu = bufs[3][:kk].tolist()
        return X, out

    def copy_x(self, out=None):
        if out is None:
            out = np.empty((self.n, self.n_prime), np.float32)
        p, dev, keep = _ptr(out) if hasattr(out, "data_ptr") else (out.ctypes.data, 0, out)
        _check(lib().fastpfp_copy_x(self._h, p, dev), self._h)
        return out

    def _y_shape(self):
        m = max(self.n_glob, self.n_prime)
        return (self.n if self.world > 1 else m, m)     # sharded: local rows x m

    def copy_y(self):
        out = np.empty(self._y_shape(), np.float32)
        _check(lib().fastpfp_copy_y(self._h, out.ctypes.data, 0), self._h)
        return out

    def set_y(self, Y):
        """Load the slacked matrix (checkpoint/resume; after set_x0, which zeroes Y)."""
        self._check_shape(Y, self._y_shape())
        p, dev, keep = _ptr(Y)
        _check(lib().fastpfp_set_y(self._h, p, dev), self._h)

    def collectives(self):
        """[(kind, nccl dtype, nccl op, count)] issued by the last call of a sharded handle."""
        cnt = C.c_int64()
        _check(lib().fastpfp_dist_collectives(self._h, None, 0, C.byref(cnt)), self._h)
        buf = np.zeros((max(cnt.value, 1), 4), np.int64)
        _check(lib().fastpfp_dist_collectives(self._h, buf.ctypes.data, cnt.value, C.byref(cnt)), self._h)
        return [tuple(int(x) for x in row) for row in buf[:cnt.value]]

    def stats(self) -> dict:
        st = Stats()
        _check(lib().fastpfp_get_stats(self._h, C.byref(st)), self._h)
        return {k: getattr(st, k) for k, _ in Stats._fields_}

    def reset_stats(self):
        _check(lib().fastpfp_reset_stats(self._h), self._h)

    def discretize(self):
        out = np.empty(self.n_glob, np.int32)
        _check(lib().fastpfp_discretize(self._h, out.ctypes.data), self._h)
        return out

    def objective(self, lam):
        f = C.c_double()
        _check(lib().fastpfp_objective(self._h, float(lam), C.byref(f)), self._h)
        return f.value

    @staticmethod
    def _check_shape(x, shape):
        if tuple(x.shape) != tuple(shape):
            raise ValueError(f"expected shape {shape}, got {tuple(x.shape)}")


def project(Y, eps2: float, max_iter2: int, stream: int = 0):
    """In-place projection sweeps on a dense m x m float32 CUDA tensor (fastpfp_project)."""
    sweeps = C.c_int32()
    delta = C.c_double()
    _check(lib().fastpfp_project(Y.data_ptr(), Y.shape[0], float(eps2), int(max_iter2),
                                 C.byref(sweeps), C.byref(delta), int(stream)))
    return sweeps.value, delta.value


def gemm_nt(P, Q, C_out, precision: int = PREC_TF32X3, cta_group: int = 2, stream: int = 0):
    """C = P Q^T on dense float32 CUDA tensors (fastpfp_gemm_nt)."""
    M, K = P.shape
    N = Q.shape[0]
    _check(lib().fastpfp_gemm_nt(P.data_ptr(), Q.data_ptr(), C_out.data_ptr(), M, N, K,
                                 int(precision), int(cta_group), int(stream)))
    return C_out


def gemm_nt_blocked(P, Q, C_out, q_blocks: int, precision: int = PREC_TF32X3, stream: int = 0):
    """C = P Q^T with Q re-laid as [q_blocks][N][K/q_blocks] (fastpfp_gemm_nt_blocked): the
    row-sharded GEMM2's 3-D TMA K-loop, on one GPU."""
    M, K = P.shape
    N = Q.shape[0]
    _check(lib().fastpfp_gemm_nt_blocked(P.data_ptr(), Q.data_ptr(), C_out.data_ptr(), M, N, K,
                                         int(q_blocks), int(precision), int(stream)))
    return C_out


@dataclass
class BatchReport:
    iterations: np.ndarray
    converged: np.ndarray
    sweeps: np.ndarray


class BatchedSolver:
    """Many independent small pairs (n, n' <= 128), one CTA per pair (fastpfp_batched_*)."""

    def __init__(self, batch: int, n: int, n_prime: int, d: int = 0):
        L = lib()
        h = C.c_void_p()
        _check(L.fastpfp_batched_create(batch, n, n_prime, d, C.byref(h)))
        self._h = h
        self.batch, self.n, self.n_prime, self.d = batch, n, n_prime, d

    def _ck(self, st):
        _check(st, self._h, "fastpfp_batched_last_error")

    def close(self):
        if getattr(self, "_h", None):
            lib().fastpfp_batched_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key: int, value: int):
        self._ck(lib().fastpfp_batched_set_option(self._h, key, int(value)))

    def set_graphs(self, A, Ap, B=None, Bp=None):
        pa, da, ka = _ptr(A)
        pp, dp, kp = _ptr(Ap)
        pb, db, kb = _ptr(B)
        pbp, dbp, kbp = _ptr(Bp)
        Solver._check_shape(A, (self.batch, self.n, self.n))
        Solver._check_shape(Ap, (self.batch, self.n_prime, self.n_prime))
        if self.d > 0:
            Solver._check_shape(B, (self.batch, self.n, self.d))
            Solver._check_shape(Bp, (self.batch, self.n_prime, self.d))
        self._ck(lib().fastpfp_batched_set_graphs(self._h, pa, pp, pb, pbp, da))

    def set_x0(self, X0=None):
        p, dev, keep = _ptr(X0)
        if X0 is not None:
            Solver._check_shape(X0, (self.batch, self.n, self.n_prime))
        self._ck(lib().fastpfp_batched_set_x0(self._h, p, dev))

    def iterate(self, alpha, lam, eps1, eps2, max_iter1, max_iter2, want_x=True):
        it = np.zeros(self.batch, np.int32)
        cv = np.zeros(self.batch, np.int32)
        sw = np.zeros(self.batch, np.int32)
        X = np.empty((self.batch, self.n, self.n_prime), np.float32) if want_x else None
        self._ck(lib().fastpfp_batched_iterate(self._h, float(alpha), float(lam), float(eps1),
                                               float(eps2), int(max_iter1), int(max_iter2),
                                               X.ctypes.data if X is not None else None,
                                               it.ctypes.data, cv.ctypes.data, sw.ctypes.data))
        return X, BatchReport(it, cv.astype(bool), sw)

    def copy_x(self, out=None):
        if out is None:
            out = np.empty((self.batch, self.n, self.n_prime), np.float32)
        p, dev, keep = _ptr(out) if hasattr(out, "data_ptr") else (out.ctypes.data, 0, out)
        self._ck(lib().fastpfp_batched_copy_x(self._h, p, dev))
        return out

    def discretize(self):
        out = np.empty((self.batch, self.n), np.int32)
        self._ck(lib().fastpfp_batched_discretize(self._h, out.ctypes.data))
        return out

    def stats(self) -> dict:
        st = Stats()
        self._ck(lib().fastpfp_batched_get_stats(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in Stats._fields_}
