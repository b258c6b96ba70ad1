"""oracle — TEST INFRASTRUCTURE ONLY.

Plain, slow, fp64 CPU oracle of the hot path (PAPER.md eq. (Tdef)/(SL), the RA/ISA
algorithms of §3-§4, and the north_star's trajectory labelling), used to prove the
CUDA path right.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this package.  It never imports
paper_1405_3521_b200 and the product never imports it.

The arithmetic lives in ``hj_oracle.c`` (plain C, compiled with -O2
-ffp-contract=off); this module only marshals numpy arrays into it.

Pinned against closed forms / brute force in tests/test_oracle_pins.py; every
function below is pinned (see DESIGN.md §4 for the pin list).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hj_oracle.c")
_LIB = os.path.join(_HERE, "_hj_oracle.so")
_lock = threading.Lock()
_lib = None

DYN_AFFINE, DYN_DUBINS, DYN_VANDERPOL = 0, 1, 2
COST_KRUZKOV, COST_DISCOUNTED = 0, 1
INTERIOR, TARGET, GHOST = 0, 1, 2


def build(force: bool = False) -> str:
    """Compile the C oracle (gcc, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        # -fopenmp: the per-node loops run on the host's cores (Jacobi: every node reads
        # only the previous iterate, so the result does not depend on the thread count)
        cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-fPIC",
               "-shared", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


class _Prob(ctypes.Structure):
    _fields_ = [
        ("dim", ctypes.c_int),
        ("n", ctypes.c_long * 3),
        ("lo", ctypes.c_double * 3),
        ("hi", ctypes.c_double * 3),
        ("periodic", ctypes.c_int * 3),
        ("dynamics", ctypes.c_int),
        ("K", ctypes.c_int),
        ("ctrl", ctypes.POINTER(ctypes.c_double)),
        ("A", ctypes.c_double * 9),
        ("b", ctypes.c_double * 3),
        ("speed", ctypes.POINTER(ctypes.c_double)),
        ("dub_v", ctypes.c_double),
        ("dub_w", ctypes.c_double),
        ("vdp_mu", ctypes.c_double),
        ("cost", ctypes.c_int),
        ("lam", ctypes.c_double),
        ("h", ctypes.c_double),
        ("l0", ctypes.c_double),
        ("lq", ctypes.c_double),
        ("ln", ctypes.c_double),
        ("lr", ctypes.c_double),
        ("v_out", ctypes.c_double),
        ("piece", ctypes.POINTER(ctypes.c_byte)),
        ("g", ctypes.POINTER(ctypes.c_double)),
    ]


_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_lp = ctypes.POINTER(ctypes.c_long)
_up = ctypes.POINTER(ctypes.c_ulonglong)    # uint64 membership masks
_bp = ctypes.POINTER(ctypes.c_byte)


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            P = ctypes.POINTER(_Prob)
            lib.or_spacing.argtypes = [P, ctypes.c_int]
            lib.or_spacing.restype = ctypes.c_double
            lib.or_beta.argtypes = [P]
            lib.or_beta.restype = ctypes.c_double
            lib.or_interp_field.argtypes = [P, _dp, _dp, ctypes.c_double]
            lib.or_interp_field.restype = ctypes.c_double
            lib.or_bracket.argtypes = [P, _dp, _dp, ctypes.c_int]
            lib.or_bracket.restype = ctypes.c_double
            lib.or_min_bracket.argtypes = [P, _dp, _dp, _ip, _dp]
            lib.or_min_bracket.restype = ctypes.c_double
            lib.or_classes.argtypes = [P, _up, ctypes.c_int, _bp]
            lib.or_apply_T.argtypes = [P, _bp, _dp, _dp]
            lib.or_apply_T.restype = ctypes.c_double
            lib.or_apply_T_range.argtypes = [P, _bp, _dp, _dp, ctypes.c_long, ctypes.c_long]
            lib.or_apply_T_range.restype = ctypes.c_double
            lib.or_initial.argtypes = [P, _bp, _dp]
            lib.or_value_iteration.argtypes = [P, _bp, _dp, ctypes.c_double, ctypes.c_long, _dp]
            lib.or_value_iteration.restype = ctypes.c_long
            lib.or_feedback.argtypes = [P, _dp, _ip, _dp]
            lib.or_label_nodes.argtypes = [P, _dp, _lp, ctypes.c_long, ctypes.c_long, _ip, _lp,
                                           _dp, _dp]
            lib.or_prolong.argtypes = [_lp, _lp, _ip, ctypes.c_int, _lp, ctypes.c_long, _ip,
                                       ctypes.c_int, ctypes.c_int, _bp, _up]
            lib.or_exit_labels.argtypes = [ctypes.c_long, _ip, _dp, _dp, ctypes.c_double]
            lib.or_prolong_mask.argtypes = [_lp, _lp, _ip, ctypes.c_int, _lp, ctypes.c_long, _up,
                                            ctypes.c_int, _bp, _up]
            lib.or_ra_masks.argtypes = [ctypes.c_long, ctypes.c_int, ctypes.POINTER(_dp), _dp, _bp,
                                        ctypes.c_double, _up]
            lib.or_solve_subdomain.argtypes = [P, _up, ctypes.c_int, _dp, ctypes.c_double,
                                               ctypes.c_long, _dp]
            lib.or_solve_subdomain.restype = ctypes.c_long
            lib.or_assemble.argtypes = [ctypes.c_long, ctypes.c_int, _up,
                                        ctypes.POINTER(_dp), ctypes.c_double, _dp]
            _lib = lib
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


class OracleProblem:
    """Holds the ctypes struct plus the numpy arrays it points into."""

    def __init__(self, prob):
        g = prob.grid
        self.prob = prob
        self.dim = g.dim
        self.N = g.size
        self._ctrl = np.ascontiguousarray(prob.controls, dtype=np.float64)
        self._speed = None if prob.speed is None else np.ascontiguousarray(prob.speed, np.float64)
        self._piece = np.ascontiguousarray(prob.piece, dtype=np.int8)
        self._g = None if prob.g is None else np.ascontiguousarray(prob.g, np.float64)
        s = _Prob()
        s.dim = g.dim
        for d in range(3):
            s.n[d] = g.n[d] if d < g.dim else 1
            s.lo[d] = g.lo[d] if d < g.dim else 0.0
            s.hi[d] = g.hi[d] if d < g.dim else 1.0
            s.periodic[d] = int(g.periodic[d]) if d < g.dim else 0
        s.dynamics = prob.dynamics
        s.K = prob.n_controls
        s.ctrl = _ptr(self._ctrl, _dp)
        A = np.asarray(prob.A, np.float64).reshape(3, 3)
        for i in range(9):
            s.A[i] = A.reshape(-1)[i]
        for i in range(3):
            s.b[i] = float(prob.b[i])
        s.speed = _ptr(self._speed, _dp) if self._speed is not None else _dp()
        s.dub_v, s.dub_w, s.vdp_mu = prob.dubins_v, prob.dubins_w, prob.vdp_mu
        s.cost = prob.cost
        s.lam, s.h = prob.lam, prob.h
        s.l0, s.lq, s.ln, s.lr = prob.l0, prob.lq, prob.ln, prob.lr
        s.v_out = prob.v_out
        s.piece = _ptr(self._piece, _bp)
        s.g = _ptr(self._g, _dp) if self._g is not None else _dp()
        self.s = s
        self.ref = ctypes.byref(s)
        self.lib = _load()

    # -- building blocks ----------------------------------------------------
    def spacing(self, d):
        return self.lib.or_spacing(self.ref, d)

    def beta(self):
        return self.lib.or_beta(self.ref)

    def interp(self, field, gi):
        field = np.ascontiguousarray(field, np.float64)
        gi3 = np.zeros(3)
        gi3[: len(gi)] = gi
        return self.lib.or_interp_field(self.ref, _ptr(field, _dp), _ptr(gi3, _dp),
                                        float(self.prob.v_out))

    def bracket(self, V, gi, k):
        V = np.ascontiguousarray(V, np.float64)
        gi3 = np.zeros(3)
        gi3[: len(gi)] = gi
        return self.lib.or_bracket(self.ref, _ptr(V, _dp), _ptr(gi3, _dp), int(k))

    def min_bracket(self, V, gi):
        V = np.ascontiguousarray(V, np.float64)
        gi3 = np.zeros(3)
        gi3[: len(gi)] = gi
        a = ctypes.c_int()
        m = ctypes.c_double()
        v = self.lib.or_min_bracket(self.ref, _ptr(V, _dp), _ptr(gi3, _dp), ctypes.byref(a),
                                    ctypes.byref(m))
        return v, a.value, m.value

    def classes(self, mask=None, k=0):
        cls = np.empty(self.N, np.int8)
        mp = _ptr(np.ascontiguousarray(mask, np.uint64), _up) if mask is not None else _up()
        self._keep = mask
        self.lib.or_classes(self.ref, mp, int(k), _ptr(cls, _bp))
        return cls

    def apply_T(self, V, cls=None):
        cls = self.classes() if cls is None else np.ascontiguousarray(cls, np.int8)
        V = np.ascontiguousarray(V, np.float64)
        out = np.empty_like(V)
        res = self.lib.or_apply_T(self.ref, _ptr(cls, _bp), _ptr(V, _dp), _ptr(out, _dp))
        return out, res

    def apply_T_rows(self, V, cls, out, row0, row1):
        """T(V) on the node rows [row0, row1) of axis 1 only (written into `out`); for
        timing the oracle on a bounded sample.  Returns the sup-norm change there."""
        n0 = self.prob.grid.n[0]
        return self.lib.or_apply_T_range(self.ref, _ptr(cls, _bp), _ptr(V, _dp), _ptr(out, _dp),
                                         int(row0 * n0), int(row1 * n0))

    def initial(self, cls=None):
        cls = self.classes() if cls is None else np.ascontiguousarray(cls, np.int8)
        V = np.empty(self.N)
        self.lib.or_initial(self.ref, _ptr(cls, _bp), _ptr(V, _dp))
        return V

    # -- the path -----------------------------------------------------------
    def solve(self, tol=None, max_iter=None, cls=None):
        """Value iteration from V^0 (R6).  Returns (V, iterations, last residual)."""
        cls = self.classes() if cls is None else np.ascontiguousarray(cls, np.int8)
        tol = self.prob.tol if tol is None else tol
        max_iter = self.prob.max_iter if max_iter is None else max_iter
        V = np.empty(self.N)
        res = ctypes.c_double()
        it = self.lib.or_value_iteration(self.ref, _ptr(cls, _bp), _ptr(V, _dp), float(tol),
                                         int(max_iter), ctypes.byref(res))
        return V, int(it), res.value

    def feedback(self, V):
        V = np.ascontiguousarray(V, np.float64)
        a = np.empty(self.N, np.int32)
        m = np.empty(self.N)
        self.lib.or_feedback(self.ref, _ptr(V, _dp), _ptr(a, _ip), _ptr(m, _dp))
        return a, m

    def label(self, V, nodes, n_max):
        V = np.ascontiguousarray(V, np.float64)
        nodes = np.ascontiguousarray(nodes, np.int64)
        cnt = len(nodes)
        lab = np.empty(cnt, np.int32)
        st = np.empty(cnt, np.int64)
        mar = np.empty(cnt)
        geo = np.empty(cnt)
        self.lib.or_label_nodes(self.ref, _ptr(V, _dp), _ptr(nodes, _lp), cnt, int(n_max),
                                _ptr(lab, _ip), _ptr(st, _lp), _ptr(mar, _dp), _ptr(geo, _dp))
        return lab, st, mar, geo

    def solve_subdomain(self, mask, k, tol=None, max_iter=None):
        mask = np.ascontiguousarray(mask, np.uint64)
        tol = self.prob.tol if tol is None else tol
        max_iter = self.prob.max_iter if max_iter is None else max_iter
        V = np.empty(self.N)
        res = ctypes.c_double()
        it = self.lib.or_solve_subdomain(self.ref, _ptr(mask, _up), int(k), _ptr(V, _dp),
                                         float(tol), int(max_iter), ctypes.byref(res))
        return V, int(it), res.value


def prolong(coarse_grid, fine_grid, ratio, band, coarse_label, m, fine_piece, exit_set=False):
    """ISA step 2 with the overlap band (R9; R9b with exit_set: label -2 -> set m, -1 ->
    all m + 1 sets).  Returns the uint64 membership mask."""
    lib = _load()
    dim = fine_grid.dim
    nc = np.ones(3, np.int64)
    nf = np.ones(3, np.int64)
    per = np.zeros(3, np.int32)
    rr = np.ones(3, np.int64)
    for d in range(dim):
        nc[d], nf[d], per[d], rr[d] = coarse_grid.n[d], fine_grid.n[d], fine_grid.periodic[d], ratio[d]
    lab = np.ascontiguousarray(coarse_label, np.int32)
    fp = np.ascontiguousarray(fine_piece, np.int8)
    out = np.empty(fine_grid.size, np.uint64)
    lib.or_prolong(_ptr(nc, _lp), _ptr(nf, _lp), _ptr(per, _ip), dim, _ptr(rr, _lp), int(band),
                   _ptr(lab, _ip), int(m), int(bool(exit_set)), _ptr(fp, _bp), _ptr(out, _up))
    return out


def exit_labels(labels, Vc, Vexit, tol):
    """Reading R9b: unlabelled (-1) coarse nodes with Vc >= Vexit - tol -> -2 (exit set)."""
    lib = _load()
    lab = np.array(labels, np.int32, copy=True)
    Vc = np.ascontiguousarray(Vc, np.float64)
    Vexit = np.ascontiguousarray(Vexit, np.float64)
    lib.or_exit_labels(len(lab), _ptr(lab, _ip), _ptr(Vc, _dp), _ptr(Vexit, _dp), float(tol))
    return lab


def prolong_mask(coarse_grid, fine_grid, ratio, band, coarse_mask, m, fine_piece):
    """ISA step 2 from coarse membership masks (RA output), with the band (R9)."""
    lib = _load()
    dim = fine_grid.dim
    nc = np.ones(3, np.int64)
    nf = np.ones(3, np.int64)
    per = np.zeros(3, np.int32)
    rr = np.ones(3, np.int64)
    for d in range(dim):
        nc[d], nf[d], per[d], rr[d] = coarse_grid.n[d], fine_grid.n[d], fine_grid.periodic[d], ratio[d]
    cm = np.ascontiguousarray(coarse_mask, np.uint64)
    fp = np.ascontiguousarray(fine_piece, np.int8)
    out = np.empty(fine_grid.size, np.uint64)
    lib.or_prolong_mask(_ptr(nc, _lp), _ptr(nf, _lp), _ptr(per, _ip), dim, _ptr(rr, _lp),
                        int(band), _ptr(cm, _up), int(m), _ptr(fp, _bp), _ptr(out, _up))
    return out


def ra(problem, m, C, M, q, tol=None, max_iter=None):
    """The paper's reconstruction algorithm RA on one grid:
    1) V_i = T_i(V_i), the problem with only piece i as the target (dG := X_i);
    2) V = min_i V_i;  3) Sigma_i = X_i + {j : |V_i(j) - V(j)| <= 2 (C dx^q + M dx)}.
    dx = the largest grid spacing.  Returns (V_i list, V, mask, iterations)."""
    import dataclasses
    lib = _load()
    piece = np.asarray(problem.piece, np.int8)
    Vs, its = [], []
    for i in range(m):
        pi = np.where(piece == i, np.int8(i), np.int8(-1)).astype(np.int8)
        V, it, _ = OracleProblem(dataclasses.replace(problem, piece=pi)).solve(tol, max_iter)
        Vs.append(V)
        its.append(it)
    Vmin = np.minimum.reduce(Vs)
    dx = max(problem.grid.spacing(d) for d in range(problem.grid.dim))
    thr = 2.0 * (C * dx ** q + M * dx)
    arrs = [np.ascontiguousarray(v, np.float64) for v in Vs]
    ptrs = (_dp * m)(*[_ptr(a, _dp) for a in arrs])
    mask = np.empty(problem.grid.size, np.uint64)
    lib.or_ra_masks(problem.grid.size, int(m), ptrs, _ptr(np.ascontiguousarray(Vmin), _dp),
                    _ptr(np.ascontiguousarray(piece), _bp), float(thr), _ptr(mask, _up))
    return Vs, Vmin, mask, its


def ra_masks(Vs, V, piece, thr):
    """RA step 3 alone on given arrays: bit i of mask[j] set iff
    piece[j] == i or |V_i(j) - V(j)| <= thr."""
    lib = _load()
    m = len(Vs)
    arrs = [np.ascontiguousarray(v, np.float64) for v in Vs]
    ptrs = (_dp * m)(*[_ptr(a, _dp) for a in arrs])
    V = np.ascontiguousarray(V, np.float64)
    piece = np.ascontiguousarray(piece, np.int8)
    mask = np.empty(len(V), np.uint64)
    lib.or_ra_masks(len(V), int(m), ptrs, _ptr(V, _dp), _ptr(piece, _bp), float(thr),
                    _ptr(mask, _up))
    return mask


def threads():
    """OpenMP threads the oracle's node loops use (OMP_NUM_THREADS, else all cores)."""
    n = os.environ.get("OMP_NUM_THREADS")
    return int(n) if n and n.isdigit() else (os.cpu_count() or 1)


def assemble(mask, Vks, v_out):
    """ISA step 4: min over the sub-domains containing each node."""
    lib = _load()
    mask = np.ascontiguousarray(mask, np.uint64)
    arrs = [np.ascontiguousarray(v, np.float64) for v in Vks]
    ptrs = (_dp * len(arrs))(*[_ptr(a, _dp) for a in arrs])
    out = np.empty(len(mask))
    lib.or_assemble(len(mask), len(arrs), _ptr(mask, _up), ptrs, float(v_out), _ptr(out, _dp))
    return out


EXIT_TOL_FACTOR = 10.0     # R9b: exit test threshold = 10 x the coarse tolerance


def exit_solution(coarse_problem):
    """Vexit: the coarse problem with no target node (reading R9b)."""
    import dataclasses
    pe = dataclasses.replace(coarse_problem,
                             piece=np.full(coarse_problem.grid.size, -1, np.int8))
    V, _, _ = OracleProblem(pe).solve()
    return V


def isa(fine_problem, coarse_problem, ratio, band, m, n_max, exit_set=True):
    """The full oracle pipeline: coarse solve -> labels (-> exit set, R9b) -> prolong ->
    sub-domain solves -> assembly (§4 ISA with the north_star labelling)."""
    oc = OracleProblem(coarse_problem)
    Vc, itc, _ = oc.solve()
    lab, steps, mar, geo = oc.label(Vc, np.arange(oc.N), n_max)
    Vexit = None
    if exit_set:
        Vexit = exit_solution(coarse_problem)
        lab = exit_labels(lab, Vc, Vexit, EXIT_TOL_FACTOR * coarse_problem.tol)
    sets = m + (1 if exit_set else 0)
    mask = prolong(coarse_problem.grid, fine_problem.grid, ratio, band, lab, m,
                   fine_problem.piece, exit_set=exit_set)
    of = OracleProblem(fine_problem)
    Vks = []
    iters = []
    for k in range(sets):
        V, it, _ = of.solve_subdomain(mask, k)
        Vks.append(V)
        iters.append(it)
    Vbar = assemble(mask, Vks, fine_problem.v_out)
    return dict(Vc=Vc, coarse_iters=itc, labels=lab, label_margin=mar, label_geo=geo,
                label_steps=steps, mask=mask, Vk=Vks, iters=iters, Vbar=Vbar, Vexit=Vexit,
                n_sets=sets)
