"""Python binding of libnewtonmd.so (include/ns.h) -- argument marshalling only.

Every step of the Newton step runs in the CUDA kernels of the library; this
module only converts torch CUDA tensors / numpy arrays into pointers and
checks shapes.  There is NO CPU fallback: importing works without a GPU, but
every call needs the built library and a CUDA device and raises otherwise.

Names follow the C ABI: ``NewtonSystem.step`` is ``ns_newton_series_step``,
``step_batched`` is ``ns_newton_series_step_batched``, ``eval_diff`` is
``ns_eval_diff``, ``toeplitz_solve`` is ``ns_toeplitz_solve``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnewtonmd.so")

NS_REUSE_QR = 1
NS_NO_RESIDUAL = 2
NS_LEDGER = 4
NS_TILED_BS = 8
NS_QR_ONCE = 16
NS_NO_STAGGER = 32

STATUS = {0: "NS_OK", 1: "NS_EINVAL", 2: "NS_EPREC", 3: "NS_EDIM", 4: "NS_EMONO", 5: "NS_ESINGULAR",
          6: "NS_ENONFINITE", 7: "NS_ENOMEM", 8: "NS_ECUDA", 9: "NS_ENCCL", 10: "NS_ESTATE"}

# every symbol include/ns.h declares (checked by tests/test_abi.py)
EXPORTS = ["ns_system_create", "ns_system_destroy", "ns_newton_series_step",
           "ns_newton_series_step_batched", "ns_eval_diff", "ns_nnz", "ns_jacobian_pattern",
           "ns_toeplitz_solve", "ns_get_r_diag", "ns_md_op", "ns_get_status", "ns_get_ledger",
           "ns_reset_ledger", "ns_last_launch_count", "ns_strerror", "ns_build_info",
           "ns_fp64_peak_probe", "ns_md_latency_probe", "ns_barrier_probe", "ns_set_partition",
           "ns_newton_series_step_from", "ns_get_trace", "ns_get_qr_trace", "ns_set_window",
           "ns_get_stage_norms", "ns_run_newton", "ns_get_stage_trace",
           "ns_set_residual_sample", "ns_fabry_ratio", "ns_nccl_unique_id", "ns_comm_init",
           "ns_exchange_plan", "ns_comm_status", "ns_pack_rows", "ns_get_batch_trace"]


class NSError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: {STATUS.get(code, code)}")
        self.code = code


class _Desc(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("degree", ctypes.c_int32), ("precision", ctypes.c_int32),
                ("n_monomials", ctypes.c_int32), ("max_batch", ctypes.c_int32),
                ("eq_ptr", ctypes.c_void_p), ("mono_ptr", ctypes.c_void_p), ("var_idx", ctypes.c_void_p),
                ("coeff", ctypes.c_void_p), ("rhs", ctypes.c_void_p), ("is_complex", ctypes.c_int32)]


class StepInfo(ctypes.Structure):
    _fields_ = [("status_bits", ctypes.c_uint32), ("qr_cached", ctypes.c_int32)]


class IterLog(ctypes.Structure):
    _fields_ = [("iter", ctypes.c_int32), ("k_lo", ctypes.c_int32), ("dc", ctypes.c_int32), ("qr", ctypes.c_int32),
                ("norm_b", ctypes.c_double), ("norm_r", ctypes.c_double), ("norm_dx", ctypes.c_double),
                ("ms", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class RunInfo(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int32), ("converged", ctypes.c_int32), ("qr_count", ctypes.c_int32),
                ("k_lo", ctypes.c_int32)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class Ledger(ctypes.Structure):
    _fields_ = [("ms_convolution", ctypes.c_double), ("ms_qr", ctypes.c_double),
                ("ms_stage", ctypes.c_double), ("ms_residual", ctypes.c_double), ("ms_total", ctypes.c_double),
                ("steps", ctypes.c_int64), ("qr_count", ctypes.c_int64),
                ("md_fma_convolution", ctypes.c_int64), ("md_fma_qr", ctypes.c_int64),
                ("md_fma_stage", ctypes.c_int64), ("md_fma_residual", ctypes.c_int64),
                ("flops_per_md_fma", ctypes.c_double), ("fp64_flops", ctypes.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def lib() -> ctypes.CDLL:
    """Load libnewtonmd.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2301_12659_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, u32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_uint32
    sig = {
        "ns_system_create": ([ctypes.POINTER(_Desc), ctypes.c_int, ctypes.POINTER(vp)], ctypes.c_int),
        "ns_system_destroy": ([vp], None),
        "ns_newton_series_step": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, u32, vp], ctypes.c_int),
        "ns_newton_series_step_batched": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp,
                                           u32, vp], ctypes.c_int),
        "ns_eval_diff": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "ns_set_partition": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "ns_get_trace": ([vp, vp, i32, vp], i32),
        "ns_get_qr_trace": ([vp, vp, i32], i32),
        "ns_get_stage_trace": ([vp, vp], i32),
        "ns_get_batch_trace": ([vp, vp, i32], i32),
        "ns_set_residual_sample": ([vp, vp, ctypes.c_int], ctypes.c_int),
        "ns_fabry_ratio": ([vp, vp, vp, vp], ctypes.c_int),
        "ns_nccl_unique_id": ([vp], ctypes.c_int),
        "ns_comm_init": ([vp, ctypes.c_int, ctypes.c_int, vp], ctypes.c_int),
        "ns_exchange_plan": ([ctypes.POINTER(_Desc), ctypes.c_int, vp, vp], ctypes.c_int),
        "ns_pack_rows": ([vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, ctypes.c_int, vp], ctypes.c_int),
        "ns_comm_status": ([vp, vp], ctypes.c_int),
        "ns_newton_series_step_from": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp, vp, u32, vp],
                                       ctypes.c_int),
        "ns_set_window": ([vp, ctypes.c_int, ctypes.c_int], ctypes.c_int),
        "ns_get_stage_norms": ([vp, vp], ctypes.c_int),
        "ns_run_newton": ([vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, ctypes.c_int, ctypes.c_double, u32, vp,
                           ctypes.POINTER(IterLog), ctypes.POINTER(RunInfo)], ctypes.c_int),
        "ns_nnz": ([vp], i32),
        "ns_jacobian_pattern": ([vp, vp, vp], ctypes.c_int),
        "ns_toeplitz_solve": ([vp, vp, vp, vp, vp, vp], ctypes.c_int),
        "ns_get_r_diag": ([vp, vp, vp], ctypes.c_int),
        "ns_md_op": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp], ctypes.c_int),
        "ns_get_status": ([vp, ctypes.POINTER(StepInfo)], ctypes.c_int),
        "ns_get_ledger": ([vp, ctypes.POINTER(Ledger)], ctypes.c_int),
        "ns_reset_ledger": ([vp], ctypes.c_int),
        "ns_last_launch_count": ([vp], i32),
        "ns_strerror": ([ctypes.c_int], ctypes.c_char_p),
        "ns_build_info": ([], ctypes.c_char_p),
        "ns_fp64_peak_probe": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "ns_md_latency_probe": ([ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)], ctypes.c_int),
        "ns_barrier_probe": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double)],
                             ctypes.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(code: int, what: str):
    if code != 0:
        raise NSError(code, what)


def _ptr(t) -> int | None:
    if t is None:
        return None
    return t.data_ptr()


def _stream_ptr(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return stream.cuda_stream


def _require_cuda(t, name, shape=None):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError(f"{name} must be a contiguous float64 CUDA tensor")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")


class NewtonSystem:
    """Handle of one monomial system (ns_system_create).

    eq_ptr [n+1], mono_ptr [M+1], var_idx: int32 CSR (host arrays);
    coeff [K][M] or None; rhs [K][n][D+1] float64 host array.
    """

    def __init__(self, eq_ptr, mono_ptr, var_idx, coeff, rhs, dim: int, degree: int, precision: int,
                 max_batch: int = 1, device: int = 0, is_complex: bool = False):
        L = lib()
        self._keep = [np.ascontiguousarray(eq_ptr, np.int32), np.ascontiguousarray(mono_ptr, np.int32),
                      np.ascontiguousarray(var_idx, np.int32),
                      None if coeff is None else np.ascontiguousarray(coeff, np.float64),
                      np.ascontiguousarray(rhs, np.float64)]
        e, m, v, c, r = self._keep
        desc = _Desc(dim, degree, precision, len(m) - 1, max_batch,
                     e.ctypes.data, m.ctypes.data, v.ctypes.data,
                     None if c is None else c.ctypes.data, r.ctypes.data, 1 if is_complex else 0)
        h = ctypes.c_void_p()
        _check(L.ns_system_create(ctypes.byref(desc), device, ctypes.byref(h)), "ns_system_create")
        self._h = h
        self.n, self.D, self.K, self.max_batch, self.device = dim, degree, precision, max_batch, device
        self.d = degree + 1
        self.C = 2 if is_complex else 1
        self._xshape = ((2,) if is_complex else ()) + (precision, dim, degree + 1)
        self.nnz = int(L.ns_nnz(h))

    @classmethod
    def from_system(cls, sysobj, max_batch: int = 1, device: int = 0):
        """Build from a synth.System-like object (duck typed)."""
        return cls(sysobj.eq_ptr, sysobj.mono_ptr, sysobj.var_idx, sysobj.coeff, sysobj.rhs,
                   sysobj.n, sysobj.D, sysobj.K, max_batch=max_batch, device=device,
                   is_complex=getattr(sysobj, "is_complex", False))

    def close(self):
        if getattr(self, "_h", None):
            lib().ns_system_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- the hot path
    def step(self, x, residual_out=None, flags: int = 0, stream=None):
        """ns_newton_series_step: x [K][n][d] ([2][K][n][d] complex) CUDA float64, updated in place."""
        _require_cuda(x, "x", self._xshape)
        if residual_out is not None:
            _require_cuda(residual_out, "residual_out", (self.K, 3))
        _check(lib().ns_newton_series_step(self._h, self.K, self.n, self.D, _ptr(x), _ptr(residual_out),
                                           flags, _stream_ptr(stream)), "ns_newton_series_step")

    def step_batched(self, x, rhs=None, residual_out=None, flags: int = 0, stream=None):
        """ns_newton_series_step_batched: x [B][K][n][d]."""
        B = x.shape[0]
        _require_cuda(x, "x", (B,) + self._xshape)
        if rhs is not None:
            _require_cuda(rhs, "rhs", (B,) + self._xshape)
        if residual_out is not None:
            _require_cuda(residual_out, "residual_out", (B, self.K, 3))
        _check(lib().ns_newton_series_step_batched(self._h, self.K, self.n, self.D, B, _ptr(x), _ptr(rhs),
                                                   _ptr(residual_out), flags, _stream_ptr(stream)),
               "ns_newton_series_step_batched")

    # ---- staggered Newton (NEXT-1)
    def set_window(self, k_lo: int, dc: int):
        """ns_set_window: following steps solve stages [k_lo, dc) on series truncated at t^dc."""
        _check(lib().ns_set_window(self._h, k_lo, dc), "ns_set_window")

    def stage_norms(self) -> np.ndarray:
        """ns_get_stage_norms: [4][K][d] md norms sum_i |v_k,i| of b, b - A dx, dx, x (last step)."""
        out = np.zeros((4, self.K, self.d), np.float64)
        _check(lib().ns_get_stage_norms(self._h, out.ctypes.data), "ns_get_stage_norms")
        return out

    def run_newton(self, x, max_iter: int = 24, eps: float = 0.0, flags: int = 0, stream=None):
        """ns_run_newton: staggered Newton from x (updated in place).  Returns (info, log)."""
        _require_cuda(x, "x", (self.K, self.n, self.d))
        log = (IterLog * max(1, max_iter))()
        info = RunInfo()
        _check(lib().ns_run_newton(self._h, self.K, self.n, self.D, _ptr(x), max_iter, eps, flags,
                                   _stream_ptr(stream), log, ctypes.byref(info)), "ns_run_newton")
        return info.as_dict(), [log[i].as_dict() for i in range(info.iterations)]

    # ---- NEXT-4: residual sampling and Fabry ratios
    def set_residual_sample(self, rows=None):
        """ns_set_residual_sample: residuals of the listed equations only (None/empty: all)."""
        r = np.ascontiguousarray([] if rows is None else rows, np.int32)
        _check(lib().ns_set_residual_sample(self._h, r.ctypes.data if len(r) else None, len(r)),
               "ns_set_residual_sample")

    def fabry_ratio(self, x, stream=None):
        """ns_fabry_ratio: z [K][n] = c_{D-1} / c_D per series of x."""
        import torch
        _require_cuda(x, "x", (self.K, self.n, self.d))
        z = torch.empty((self.K, self.n), dtype=torch.float64, device=x.device)
        _check(lib().ns_fabry_ratio(self._h, _ptr(x), _ptr(z), _stream_ptr(stream)), "ns_fabry_ratio")
        return z

    # ---- one system over N GPUs: library-owned NCCL communicator (C4)
    def comm_init(self, nranks: int, rank: int, uid: bytes):
        """ns_comm_init: from now on step() shards eval/diff by equations and
        replicates the rows over NCCL inside the library (collective)."""
        buf = ctypes.create_string_buffer(bytes(uid), 128)
        _check(lib().ns_comm_init(self._h, nranks, rank, buf), "ns_comm_init")

    def pack_rows(self, lo: int, hi: int, b, A, A0, block, unpack: bool = False, stream=None):
        """ns_pack_rows: rows [lo, hi) of (b, A, A0) <-> one replication block."""
        _check(lib().ns_pack_rows(self._h, lo, hi, _ptr(b), _ptr(A), _ptr(A0), _ptr(block), 1 if unpack else 0,
                                  _stream_ptr(stream)), "ns_pack_rows")

    def comm_status(self) -> int:
        e = ctypes.c_int32()
        lib().ns_comm_status(self._h, ctypes.byref(e))
        return e.value

    # ---- sharded eval/diff (C4), caller-driven variant
    def set_partition(self, eq_lo: int, eq_hi: int):
        """ns_set_partition: this handle's eval/diff computes rows [eq_lo, eq_hi)."""
        _check(lib().ns_set_partition(self._h, eq_lo, eq_hi), "ns_set_partition")

    def step_from(self, x, b, A, A0, residual_out=None, flags: int = 0, stream=None):
        """ns_newton_series_step_from: QR + stage loop + residual + x += dx for given (b, A, A0)."""
        _require_cuda(x, "x", (self.K, self.n, self.d))
        _require_cuda(b, "b", (self.K, self.d, self.n))
        _require_cuda(A, "A", (self.K, self.d, self.nnz))
        _require_cuda(A0, "A0", (self.K, self.n, self.n))
        if residual_out is not None:
            _require_cuda(residual_out, "residual_out", (self.K, 3))
        _check(lib().ns_newton_series_step_from(self._h, self.K, self.n, self.D, _ptr(x), _ptr(b), _ptr(A),
                                                _ptr(A0), _ptr(residual_out), flags, _stream_ptr(stream)),
               "ns_newton_series_step_from")

    # ---- debug / parity entry points
    def eval_diff(self, x, stream=None):
        import torch
        _require_cuda(x, "x", (self.K, self.n, self.d))
        dev = x.device
        b = torch.empty((self.K, self.d, self.n), dtype=torch.float64, device=dev)
        A = torch.empty((self.K, self.d, self.nnz), dtype=torch.float64, device=dev)
        A0 = torch.empty((self.K, self.n, self.n), dtype=torch.float64, device=dev)
        _check(lib().ns_eval_diff(self._h, _ptr(x), _ptr(b), _ptr(A), _ptr(A0), _stream_ptr(stream)),
               "ns_eval_diff")
        return b, A, A0

    def toeplitz_solve(self, b, A, A0, stream=None):
        import torch
        _require_cuda(b, "b", (self.K, self.d, self.n))
        _require_cuda(A, "A", (self.K, self.d, self.nnz))
        _require_cuda(A0, "A0", (self.K, self.n, self.n))
        dx = torch.empty((self.K, self.d, self.n), dtype=torch.float64, device=b.device)
        _check(lib().ns_toeplitz_solve(self._h, _ptr(b), _ptr(A), _ptr(A0), _ptr(dx), _stream_ptr(stream)),
               "ns_toeplitz_solve")
        return dx

    def r_diag(self, stream=None):
        import torch
        out = torch.empty((self.K, self.n), dtype=torch.float64, device=f"cuda:{self.device}")
        _check(lib().ns_get_r_diag(self._h, _ptr(out), _stream_ptr(stream)), "ns_get_r_diag")
        return out

    def pattern(self):
        rp = np.zeros(self.n + 1, np.int32)
        ci = np.zeros(max(self.nnz, 1), np.int32)
        _check(lib().ns_jacobian_pattern(self._h, rp.ctypes.data, ci.ctypes.data), "ns_jacobian_pattern")
        return rp, ci[:self.nnz]

    def status(self) -> StepInfo:
        info = StepInfo()
        _check(lib().ns_get_status(self._h, ctypes.byref(info)), "ns_get_status")
        return info

    def ledger(self) -> dict:
        led = Ledger()
        _check(lib().ns_get_ledger(self._h, ctypes.byref(led)), "ns_get_ledger")
        return led.as_dict()

    def reset_ledger(self):
        _check(lib().ns_reset_ledger(self._h), "ns_reset_ledger")

    def trace(self):
        """Job trace of the last eval/diff (env NS_TRACE=1 at create): (times [J][3] ns, jobs [J][4])."""
        cap = 1 << 22
        t = np.zeros((cap, 3), np.int64)
        jb = np.zeros((cap, 4), np.int32)
        nj = int(lib().ns_get_trace(self._h, t.ctypes.data, cap, jb.ctypes.data))
        if nj < 0:
            raise RuntimeError("no trace (create the handle with NS_TRACE=1)")
        return t[:nj], jb[:nj]

    def stage_trace(self):
        """Stamps of the last split stage loop (env NS_STAGE_TRACE=1 at create): critical chain
        [d][4] ns, bulk pend_k completion [d] ns."""
        t = np.zeros(5 * self.d, np.int64)
        if int(lib().ns_get_stage_trace(self._h, t.ctypes.data)) < 0:
            raise RuntimeError("no stage trace (create the handle with NS_STAGE_TRACE=1)")
        return t[:4 * self.d].reshape(self.d, 4), t[4 * self.d:]

    def batch_trace(self):
        """Phase stamps of the last batched step (env NS_BATCH_TRACE=1 at create): [CTAs][8] ns."""
        t = np.zeros((4096, 8), np.int64)
        g = int(lib().ns_get_batch_trace(self._h, t.ctypes.data, 4096))
        if g < 0:
            raise RuntimeError("no batch trace (create the handle with NS_BATCH_TRACE=1)")
        return t[:g]

    def last_launch_count(self) -> int:
        return int(lib().ns_last_launch_count(self._h))


def md_op(precision: int, op: str, a, b=None, c=None, stream=None):
    """Run one md primitive elementwise on planar [K][n] CUDA arrays (row a0 tests).
    op in add, mul, fma (c + a*b, c in/out), div, sqrt, sub.  Returns c."""
    import torch
    code = {"add": 0, "mul": 1, "fma": 2, "div": 3, "sqrt": 4, "sub": 5}[op]
    _require_cuda(a, "a")
    n = a.shape[1]
    if c is None:
        c = torch.zeros_like(a)
    _check(lib().ns_md_op(precision, code, n, _ptr(a), _ptr(b), _ptr(c), _stream_ptr(stream)), "ns_md_op")
    return c


def exchange_plan(eq_ptr, mono_ptr, var_idx, dim: int, degree: int, precision: int, nranks: int):
    """ns_exchange_plan (host only, no GPU): equation bounds [nranks+1] of the
    partition and each rank's replication block size in doubles [nranks]."""
    e = np.ascontiguousarray(eq_ptr, np.int32)
    m = np.ascontiguousarray(mono_ptr, np.int32)
    v = np.ascontiguousarray(var_idx, np.int32)
    desc = _Desc(dim, degree, precision, len(m) - 1, 1, e.ctypes.data, m.ctypes.data, v.ctypes.data, None, None)
    b = np.zeros(nranks + 1, np.int32)
    c = np.zeros(nranks, np.int64)
    _check(lib().ns_exchange_plan(ctypes.byref(desc), nranks, b.ctypes.data, c.ctypes.data), "ns_exchange_plan")
    return b, c


def nccl_unique_id() -> bytes:
    """ns_nccl_unique_id: 128 bytes for ns_comm_init (rank 0; broadcast by the caller)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().ns_nccl_unique_id(buf), "ns_nccl_unique_id")
    return buf.raw


def build_info() -> str:
    return lib().ns_build_info().decode()


def fp64_peak_probe(device: int = 0, op: str = "dfma") -> dict:
    """Measured FP64 pipe rate (G instructions/s) of DFMA or DADD chains on all SMs."""
    g, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().ns_fp64_peak_probe(device, 0 if op == "dfma" else 1, ctypes.byref(g), ctypes.byref(ms)),
           "ns_fp64_peak_probe")
    return {"ginstr_per_s": g.value, "ms": ms.value}


def md_latency_probe(precision: int, op: str = "fma") -> float:
    """SM cycles per md operation in a dependent chain (one warp)."""
    v = ctypes.c_double()
    code = {"fma": 0, "add": 1, "mul": 2, "recip": 3, "sqrt": 4}[op]
    _check(lib().ns_md_latency_probe(precision, code, ctypes.byref(v)), "ns_md_latency_probe")
    return v.value


def barrier_probe(blocks: int, threads: int = 128, device: int = 0) -> float:
    """Microseconds per grid barrier of the cooperative kernels."""
    v = ctypes.c_double()
    _check(lib().ns_barrier_probe(device, blocks, threads, ctypes.byref(v)), "ns_barrier_probe")
    return v.value
