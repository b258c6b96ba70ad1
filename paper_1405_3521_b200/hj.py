"""Thin Python binding of the C ABI in include/hj.h (argument marshalling only).

Every step of the hot path runs in libhj.so's CUDA kernels.  PyTorch provides
device memory and the CUDA stream.  There is no CPU fallback: if the library or
a CUDA device is missing, every call raises.

Problems are passed as duck-typed objects with the fields of
``hj_workloads.Problem`` (grid, dynamics, controls, cost, lam, h, ...).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_LIB_PATH = os.environ.get("HJ_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "_lib", "libhj.so")
_lib = None

HJ_OK, HJ_ERR_INVALID, HJ_ERR_CUDA, HJ_ERR_NOT_CONVERGED, HJ_ERR_UNSUPPORTED, HJ_ERR_WORKSPACE = range(6)
HJ_F32, HJ_F64 = 0, 1
MAX_CONTROLS = 128
MAX_SUBDOMAINS = 64          # sets of a uint64 membership mask (pieces + exit set)


class HJError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"hj status {status}: {msg}")
        self.status = status


class hj_grid(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int32), ("periodic", ctypes.c_int32 * 3),
                ("n", ctypes.c_int64 * 3), ("lo", ctypes.c_double * 3),
                ("hi", ctypes.c_double * 3)]


class hj_problem(ctypes.Structure):
    _fields_ = [("dynamics", ctypes.c_int32), ("cost", ctypes.c_int32),
                ("n_controls", ctypes.c_int32), ("sweep_kernel", ctypes.c_int32),
                ("controls", (ctypes.c_double * 3) * MAX_CONTROLS),
                ("A", (ctypes.c_double * 3) * 3), ("b", ctypes.c_double * 3),
                ("dubins_v", ctypes.c_double), ("dubins_w", ctypes.c_double),
                ("vdp_mu", ctypes.c_double), ("lam", ctypes.c_double), ("h", ctypes.c_double),
                ("l0", ctypes.c_double), ("lq", ctypes.c_double), ("ln", ctypes.c_double),
                ("lr", ctypes.c_double), ("v_out", ctypes.c_double)]


class hj_fields(ctypes.Structure):
    _fields_ = [("speed", ctypes.c_void_p), ("piece", ctypes.c_void_p), ("g", ctypes.c_void_p)]


class hj_report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("residual", ctypes.c_double),
                ("converged", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("node_updates", ctypes.c_int64), ("device_ms", ctypes.c_double),
                ("launches", ctypes.c_int64), ("evaluated_updates", ctypes.c_int64)]

    def as_dict(self):
        return dict(iterations=self.iterations, residual=self.residual,
                    converged=bool(self.converged), node_updates=self.node_updates,
                    device_ms=self.device_ms, launches=self.launches,
                    evaluated_updates=self.evaluated_updates)


class hj_subdomain(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_int64 * 3), ("hi", ctypes.c_int64 * 3),
                ("n_nodes", ctypes.c_int64), ("box_nodes", ctypes.c_int64),
                ("work", ctypes.c_double)]


EXPORTS = ["hj_last_error", "hj_version", "hj_solve_workspace_bytes", "hj_solve",
           "hj_coarse_feedback", "hj_label_subdomains", "hj_partition_plan",
           "hj_assign_subdomains", "hj_solve_partitioned", "hj_ra_workspace_bytes",
           "hj_ra_subdomains"]


# hj.h HJ_SWEEP_*
SWEEP_KERNELS = {"auto": 0, "generic": 1, "local_scalar": 2, "local_packed": 3, "field2d": 4,
                 "dubins": 5, "local_tb": 6, "local_coop": 7,
                 "field_coop": 8, "dubins_coop": 9, "field_col": 10, "field_lat": 11}


def lib():
    """Load libhj.so (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python __graft_entry__.py` / build()")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
        G, P, F = ctypes.POINTER(hj_grid), ctypes.POINTER(hj_problem), ctypes.POINTER(hj_fields)
        R, S = ctypes.POINTER(hj_report), ctypes.POINTER(hj_subdomain)
        L.hj_last_error.restype = ctypes.c_char_p
        L.hj_version.restype = ctypes.c_char_p
        L.hj_solve_workspace_bytes.argtypes = [G, i32, i64]
        L.hj_solve_workspace_bytes.restype = ctypes.c_size_t
        L.hj_solve.argtypes = [G, P, F, i32, vp, ctypes.c_double, i64, vp, ctypes.c_size_t, vp, R]
        L.hj_coarse_feedback.argtypes = [G, P, F, i32, vp, vp, vp, vp]
        L.hj_label_subdomains.argtypes = [G, P, F, i32, vp, vp, ctypes.c_double, i64, G,
                                          ctypes.POINTER(i32), i32, i32, vp, vp, vp, vp, vp, vp,
                                          vp]
        L.hj_partition_plan.argtypes = [G, vp, i32, i32, i64, S, ctypes.POINTER(ctypes.c_size_t),
                                        vp]
        L.hj_assign_subdomains.argtypes = [i32, S, i32, ctypes.POINTER(i32)]
        L.hj_solve_partitioned.argtypes = [G, P, F, i32, vp, i32, S, ctypes.c_uint64,
                                           ctypes.c_double, i64, vp, vp, ctypes.c_size_t, vp, R]
        L.hj_ra_workspace_bytes.argtypes = [G, i32, i64]
        L.hj_ra_workspace_bytes.restype = ctypes.c_size_t
        dbl = ctypes.c_double
        L.hj_ra_subdomains.argtypes = [G, P, F, i32, i32, dbl, dbl, dbl, dbl, i64, G,
                                       ctypes.POINTER(i32), i32, vp, vp, vp, vp, vp, vp,
                                       ctypes.c_size_t, vp, R]
        for name in EXPORTS[2:]:
            if not name.endswith("_bytes"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status):
    if status != HJ_OK:
        raise HJError(status, lib().hj_last_error().decode())


def _torch_dtype(dtype):
    return {"f32": torch.float32, "f64": torch.float64}[dtype]


def _code(dtype):
    return {"f32": HJ_F32, "f64": HJ_F64}[dtype]


def _stream(stream):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def make_grid(grid) -> hj_grid:
    g = hj_grid()
    g.dim = grid.dim
    for d in range(3):
        g.n[d] = grid.n[d] if d < grid.dim else 1
        g.lo[d] = grid.lo[d] if d < grid.dim else 0.0
        g.hi[d] = grid.hi[d] if d < grid.dim else 1.0
        g.periodic[d] = int(grid.periodic[d]) if d < grid.dim else 0
    return g


def make_problem(prob) -> hj_problem:
    p = hj_problem()
    p.dynamics = prob.dynamics
    p.cost = prob.cost
    K = prob.controls.shape[0]
    if not 1 <= K <= MAX_CONTROLS:
        raise ValueError(f"{K} controls (max {MAX_CONTROLS})")
    p.n_controls = K
    for k in range(K):
        for c in range(3):
            p.controls[k][c] = float(prob.controls[k, c])
    A = np.asarray(prob.A, np.float64).reshape(3, 3)
    for i in range(3):
        p.b[i] = float(prob.b[i])
        for j in range(3):
            p.A[i][j] = float(A[i, j])
    p.dubins_v, p.dubins_w, p.vdp_mu = prob.dubins_v, prob.dubins_w, prob.vdp_mu
    p.lam, p.h = prob.lam, prob.h
    p.l0, p.lq, p.ln, p.lr = prob.l0, prob.lq, prob.ln, prob.lr
    p.v_out = prob.v_out
    return p


class DeviceProblem:
    """hj_grid / hj_problem structs plus the problem's node fields on the device."""

    def __init__(self, prob, dtype="f32", device="cuda", piece=None, speed=None, g=None,
                 sweep_kernel="auto", reuse_buffers=False):
        self.prob = prob
        # reuse_buffers: outputs and workspaces are cached on this object and reused by
        # the next call (no allocator traffic in a timed loop; results alias)
        self.reuse = reuse_buffers
        self._bufs = {}
        self.dtype = dtype
        self.grid = make_grid(prob.grid)
        self.cprob = make_problem(prob)
        self.cprob.sweep_kernel = SWEEP_KERNELS[sweep_kernel]
        td = _torch_dtype(dtype)
        self.piece = piece if piece is not None else torch.as_tensor(
            np.ascontiguousarray(prob.piece, np.int8)).to(device)
        if speed is None and prob.speed is not None:
            speed = torch.as_tensor(np.asarray(prob.speed)).to(device=device, dtype=td)
        if g is None and prob.g is not None:
            g = torch.as_tensor(np.asarray(prob.g)).to(device=device, dtype=td)
        self.speed, self.g = speed, g
        self.fields = hj_fields(speed.data_ptr() if speed is not None else None,
                                self.piece.data_ptr(),
                                g.data_ptr() if g is not None else None)
        self.N = prob.grid.size
        self.device = device


def _buf(dp, name, numel, dtype):
    """A device tensor for `name`: fresh, or the cached one when dp.reuse_buffers."""
    if not getattr(dp, "reuse", False):
        return torch.empty(numel, dtype=dtype, device=dp.device)
    t = dp._bufs.get(name)
    if t is None or t.numel() < numel or t.dtype != dtype:
        t = torch.empty(numel, dtype=dtype, device=dp.device)
        dp._bufs[name] = t
    return t[:numel]


def hj_version() -> str:
    return lib().hj_version().decode()


def hj_solve(dp: DeviceProblem, tol=None, max_iter=None, V=None, workspace=None, stream=None,
             allow_not_converged=False):
    """Value iteration on the whole grid.  Returns (V, report dict)."""
    prob = dp.prob
    tol = prob.tol if tol is None else tol
    max_iter = prob.max_iter if max_iter is None else max_iter
    L = lib()
    if V is None:
        V = _buf(dp, "V", dp.N, _torch_dtype(dp.dtype))
    need = L.hj_solve_workspace_bytes(ctypes.byref(dp.grid), _code(dp.dtype), max_iter)
    if workspace is None or workspace.numel() < need:
        workspace = _buf(dp, "ws", need, torch.uint8)
    rep = hj_report()
    st = L.hj_solve(ctypes.byref(dp.grid), ctypes.byref(dp.cprob), ctypes.byref(dp.fields),
                    _code(dp.dtype), V.data_ptr(), float(tol), int(max_iter), workspace.data_ptr(),
                    workspace.numel(), _stream(stream), ctypes.byref(rep))
    if not (allow_not_converged and st == HJ_ERR_NOT_CONVERGED):
        _check(st)
    return V, rep.as_dict()


def hj_coarse_feedback(dp: DeviceProblem, V, stream=None):
    astar = torch.empty(dp.N, dtype=torch.int32, device=dp.device)
    margin = torch.empty(dp.N, dtype=torch.float64, device=dp.device)
    _check(lib().hj_coarse_feedback(ctypes.byref(dp.grid), ctypes.byref(dp.cprob),
                                    ctypes.byref(dp.fields), _code(dp.dtype), V.data_ptr(),
                                    astar.data_ptr(), margin.data_ptr(), _stream(stream)))
    return astar, margin


def hj_label_subdomains(coarse: DeviceProblem, Vc, n_max, fine: DeviceProblem, ratio, band, m,
                        Vexit=None, exit_tol=0.0, stream=None):
    """Labels (piece, -1 unlabelled, -2 exit set when Vexit is given) and the fine uint64
    membership mask (returned as an int64 tensor holding the bits)."""
    Nc, Nf = coarse.N, fine.N
    label = _buf(coarse, "label", Nc, torch.int32)
    margin = _buf(coarse, "margin", Nc, torch.float64)
    geo = _buf(coarse, "geo", Nc, torch.float64)
    steps = _buf(coarse, "steps", Nc, torch.int32)
    mask = _buf(fine, "mask", Nf, torch.int64)   # uint64 bits
    r = (ctypes.c_int32 * 3)(*[int(ratio[d]) if d < len(ratio) else 1 for d in range(3)])
    _check(lib().hj_label_subdomains(
        ctypes.byref(coarse.grid), ctypes.byref(coarse.cprob), ctypes.byref(coarse.fields),
        _code(coarse.dtype), Vc.data_ptr(), Vexit.data_ptr() if Vexit is not None else None,
        float(exit_tol), int(n_max), ctypes.byref(fine.grid), r, int(band), int(m),
        fine.piece.data_ptr(), label.data_ptr(), margin.data_ptr(), geo.data_ptr(),
        steps.data_ptr(), mask.data_ptr(), _stream(stream)))
    return dict(label=label, margin=margin, geo=geo, steps=steps, mask=mask,
                n_sets=m + (1 if Vexit is not None else 0))


def _check_mask(mask, N):
    if mask.dtype != torch.int64 or mask.numel() < N or not mask.is_cuda:
        raise ValueError("fine_mask must be a CUDA int64 tensor (the uint64 set bits) of N nodes")


def hj_partition_plan(fine: DeviceProblem, mask, m, max_iter=None, stream=None):
    max_iter = fine.prob.max_iter if max_iter is None else max_iter
    _check_mask(mask, fine.N)
    plan = (hj_subdomain * m)()
    ws = ctypes.c_size_t()
    _check(lib().hj_partition_plan(ctypes.byref(fine.grid), mask.data_ptr(), int(m),
                                   _code(fine.dtype), int(max_iter), plan, ctypes.byref(ws),
                                   _stream(stream)))
    return plan, ws.value


def hj_assign_subdomains(plan, n_ranks):
    m = len(plan)
    owner = (ctypes.c_int32 * m)()
    _check(lib().hj_assign_subdomains(m, plan, int(n_ranks), owner))
    return list(owner)


def hj_solve_partitioned(fine: DeviceProblem, mask, m, plan, ws_bytes, solve_set=None, tol=None,
                         max_iter=None, Vbar=None, workspace=None, stream=None):
    prob = fine.prob
    tol = prob.tol if tol is None else tol
    max_iter = prob.max_iter if max_iter is None else max_iter
    solve_set = ((1 << m) - 1) if solve_set is None else solve_set
    _check_mask(mask, fine.N)
    if Vbar is None:
        Vbar = _buf(fine, "Vbar", fine.N, _torch_dtype(fine.dtype))
    if workspace is None or workspace.numel() < ws_bytes:
        workspace = _buf(fine, "pws", max(ws_bytes, 1), torch.uint8)
    reps = (hj_report * m)()
    _check(lib().hj_solve_partitioned(
        ctypes.byref(fine.grid), ctypes.byref(fine.cprob), ctypes.byref(fine.fields),
        _code(fine.dtype), mask.data_ptr(), int(m), plan, ctypes.c_uint64(solve_set), float(tol),
        int(max_iter), Vbar.data_ptr(), workspace.data_ptr(), workspace.numel(), _stream(stream),
        reps))
    return Vbar, [reps[k].as_dict() if (solve_set >> k) & 1 else None for k in range(m)]


def hj_ra_subdomains(coarse: DeviceProblem, m, C=1.0, M=1.0, q=0.5, fine: DeviceProblem = None,
                     ratio=None, band=0, tol=None, max_iter=None, stream=None):
    """The paper's RA reconstruction on the coarse grid, prolonged
    to the fine grid when `fine` is given.  Returns dict(Vaux (m x N_c), Vmin,
    coarse_mask, mask (fine, or None), reports)."""
    prob = coarse.prob
    tol = prob.tol if tol is None else tol
    max_iter = prob.max_iter if max_iter is None else max_iter
    L = lib()
    Nc = coarse.N
    td = _torch_dtype(coarse.dtype)
    Vaux = _buf(coarse, "ra_Vaux", m * Nc, td)
    Vmin = _buf(coarse, "ra_Vmin", Nc, td)
    cmask = _buf(coarse, "ra_cmask", Nc, torch.int64)
    need = L.hj_ra_workspace_bytes(ctypes.byref(coarse.grid), _code(coarse.dtype), int(max_iter))
    ws = _buf(coarse, "ra_ws", need, torch.uint8)
    fmask = None
    r = (ctypes.c_int32 * 3)(1, 1, 1)
    if fine is not None:
        fmask = _buf(fine, "mask", fine.N, torch.int64)
        for d in range(len(ratio)):
            r[d] = int(ratio[d])
    reps = (hj_report * m)()
    _check(L.hj_ra_subdomains(
        ctypes.byref(coarse.grid), ctypes.byref(coarse.cprob), ctypes.byref(coarse.fields),
        _code(coarse.dtype), int(m), float(C), float(M), float(q), float(tol), int(max_iter),
        ctypes.byref(fine.grid) if fine is not None else None, r, int(band),
        fine.piece.data_ptr() if fine is not None else None, Vaux.data_ptr(), Vmin.data_ptr(),
        cmask.data_ptr(), fmask.data_ptr() if fmask is not None else None, ws.data_ptr(),
        ws.numel(), _stream(stream), reps))
    return dict(Vaux=Vaux.view(m, Nc), Vmin=Vmin, coarse_mask=cmask, mask=fmask,
                reports=[reps[i].as_dict() for i in range(m)])

