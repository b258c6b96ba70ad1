"""Pins of the CPU oracle against things other than itself (closed forms, brute
force, textbook special cases, invariants).  No GPU.  Each test names the
PAPER.md passage or DESIGN.md reading it pins.  A plausible mistake anywhere in
oracle/hj_oracle.c (a dropped cost term, a wrong sign, an index transposition,
beta = 1/(1+h) vs exp(-h), a wrong interpolation weight, an off-by-one in the
stopping rule, a prolongation radius off by one) fails at least one of them.
"""
import collections
import math

import numpy as np
import pytest
from scipy import ndimage

import hj_workloads as W
import oracle


def mk_problem(grid, controls, piece, cost=W.COST_KRUZKOV, lam=1.0, h=None, **kw):
    h = grid.spacing(0) if h is None else h
    n_p = int(piece.max()) + 1 if piece.max() >= 0 else 0
    return W.Problem(grid=grid, dynamics=kw.pop("dynamics", W.DYN_AFFINE), controls=controls,
                     cost=cost, lam=lam, h=h, tol=kw.pop("tol", 1e-13),
                     max_iter=kw.pop("max_iter", 100000), piece=piece, n_pieces=n_p, **kw)


def bfs_distance(shape, targets):
    """4-neighbour lattice distance to the nearest target node (plain BFS)."""
    ny, nx = shape
    d = np.full(shape, -1, np.int64)
    q = collections.deque()
    for j, i in zip(*np.nonzero(targets)):
        d[j, i] = 0
        q.append((j, i))
    while q:
        j, i = q.popleft()
        for dj, di in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            a, b = j + dj, i + di
            if 0 <= a < ny and 0 <= b < nx and d[a, b] < 0:
                d[a, b] = d[j, i] + 1
                q.append((a, b))
    return d


# ---------------------------------------------------------------------------
# P1  lattice-exact Kruzkov problem: V = 1 - beta^d, d = BFS distance.
#     Pins Tdef (line 241) bracket beta*I + (1-beta), beta = 1/(1+lambda h),
#     the index layout (non-square grid, distinct nx, ny), the stopping rule.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("lam", [1.0, 0.7])
def test_p1_lattice_kruzkov_bfs(lam):
    grid = W.Grid((13, 9), (-1.0, -0.5), (1.4, 1.1), (False, False))
    assert abs(grid.spacing(0) - grid.spacing(1)) < 1e-15
    rng = np.random.default_rng(11)
    piece = np.full(grid.size, -1, np.int8)
    idx = rng.choice(grid.size, 4, replace=False)
    piece[idx] = np.arange(4)
    p = mk_problem(grid, W.axis_controls(), piece, lam=lam)
    o = oracle.OracleProblem(p)
    V, it, res = o.solve()
    d = bfs_distance((9, 13), (piece >= 0).reshape(9, 13)).reshape(-1)
    beta = 1.0 / (1.0 + lam * p.h)
    np.testing.assert_allclose(V, 1.0 - beta ** d, rtol=0, atol=1e-13)
    # stopping rule R6: nodes at distance n are final after n sweeps; the
    # (max d + 1)-th sweep is the first with a zero change.
    assert it == d.max() + 1 and res == 0.0
    assert abs(o.beta() - beta) < 1e-16


def test_p1_feedback_and_labels_bfs():
    grid = W.Grid((15, 11), (0.0, 0.0), (1.4, 1.0), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    for k, (i, j) in enumerate([(1, 1), (12, 2), (7, 9)]):
        piece[j * 15 + i] = k
    p = mk_problem(grid, W.axis_controls(), piece)
    o = oracle.OracleProblem(p)
    V, _, _ = o.solve()
    a, margin = o.feedback(V)
    ctrl = W.axis_controls()
    per_piece = []
    for k in range(3):
        per_piece.append(bfs_distance((11, 15), (piece == k).reshape(11, 15)).reshape(-1))
    dmin = np.min(per_piece, axis=0)
    for n in range(grid.size):
        if piece[n] >= 0:
            assert a[n] == -1
            continue
        i, j = n % 15, n // 15
        step = ctrl[a[n]]
        t = (j + int(step[1])) * 15 + (i + int(step[0]))
        assert dmin[t] == dmin[n] - 1          # feedback descends the BFS distance
    labels, steps, mm, geo = o.label(V, np.arange(grid.size), n_max=100)
    for n in range(grid.size):
        assert per_piece[labels[n]][n] == dmin[n]   # reached a nearest piece
        assert steps[n] == dmin[n]


# ---------------------------------------------------------------------------
# P2  closed form of the eikonal minimum time problem (config 1 geometry):
#     T(x) = min_k |x-c_k| - r_k, v = 1 - exp(-T); O(dx) decay (Theorem 3.1).
# ---------------------------------------------------------------------------
def _c1_T(grid):
    x, y = grid.mesh()
    T = np.min([np.hypot(x - cx, y - cy) - 0.05 for cx, cy in
                [(-0.5, -0.5), (0.5, -0.5), (-0.5, 0.5), (0.5, 0.5)]], axis=0).reshape(-1)
    return np.maximum(T, 0.0)


def test_p2_eikonal_closed_form_and_refinement():
    errs = []
    for n in (26, 51, 101, 201):
        p = W.make(1, scale=(n - 1) / 100).fine
        o = oracle.OracleProblem(p)
        V, it, res = o.solve(tol=1e-12)
        assert res < 1e-12
        T = _c1_T(p.grid)
        assert np.all(V >= 0) and np.all(V <= 1)
        # undo the implicit-Euler discount (beta = 1/(1+h) per Tdef): discrete time
        Td = -np.log1p(-V) * p.h / math.log1p(p.h)
        err = np.abs(Td - T).max()
        assert err <= 1.5 * p.grid.spacing(0) + 1e-3, (n, err)
        errs.append(err)
    assert errs[-1] < errs[0] / 4


# ---------------------------------------------------------------------------
# P3  f == 0: each node is its own foot, the recursion V = beta V + h l(x) has
#     the closed form V = h l(x) / (1 - beta) (pins the discounted bracket, the
#     running cost formula, beta).
# ---------------------------------------------------------------------------
def test_p3_stationary_discounted_closed_form():
    grid = W.Grid((9, 7), (-1.0, -0.6), (1.0, 1.4), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    piece[0] = 0
    ctrl = np.zeros((1, 3))
    ctrl[0, 2] = 0.3   # |a|^2 = 0.09 enters via lr
    p = mk_problem(grid, ctrl, piece, cost=W.COST_DISCOUNTED, lam=0.8, h=0.05, l0=0.5, lq=2.0,
                   ln=0.25, lr=3.0, v_out=1e3, tol=1e-14, max_iter=10 ** 6)
    o = oracle.OracleProblem(p)
    V, it, res = o.solve()
    x, y = grid.mesh()
    x, y = x.reshape(-1), y.reshape(-1)
    r2 = x * x + y * y
    ell = 0.5 + 2.0 * r2 + 0.25 * np.sqrt(r2) + 3.0 * 0.09
    beta = 1.0 / (1.0 + 0.8 * 0.05)
    exp = 0.05 * ell / (1.0 - beta)
    exp[0] = 0.0
    np.testing.assert_allclose(V, exp, rtol=1e-11, atol=0)


# ---------------------------------------------------------------------------
# P4  Example 2.1: lambda = 0, l = 1, g = 0 on the
#     square's boundary: v = 1 - max(|x1|,|x2|); and Theorem 2.1: the min of
#     the auxiliary solutions with g_i = g + gamma off Gamma_i recovers v.
# ---------------------------------------------------------------------------
def test_p4_paper_example_2_1_and_min_decomposition():
    n = 41
    grid = W.Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    edges = W.box_edge_pieces(grid, 4)
    base = dict(cost=W.COST_DISCOUNTED, lam=0.0, l0=1.0, v_out=50.0, tol=1e-12,
                max_iter=10 ** 5)
    ctrl = W.unit_circle_controls(64)
    p = mk_problem(grid, ctrl, np.where(edges >= 0, 0, -1).astype(np.int8), **base)
    V, it, res = oracle.OracleProblem(p).solve()
    x, y = grid.mesh()
    v = (1.0 - np.maximum(np.abs(x), np.abs(y))).reshape(-1)
    dx = grid.spacing(0)
    assert np.abs(V - v).max() <= 2 * dx
    gamma = 0.5
    Vi = []
    for i in range(4):
        g = np.where((edges >= 0) & (edges != i), gamma, 0.0)
        pi = mk_problem(grid, ctrl, edges, g=g, **base)
        Vk, _, _ = oracle.OracleProblem(pi).solve()
        assert np.all(Vk >= V - 1e-9)          # comparison principle: v_i >= v
        Vi.append(Vk)
    Vmin = np.min(Vi, axis=0)
    assert np.abs(Vmin - V).max() <= 2 * dx     # Theorem 2.1 (discrete, O(dx))
    # independent sub-domain of edge 0 (y = -1) contains the lower triangle
    lower = (y.reshape(-1) < -np.abs(x.reshape(-1)) - 2 * dx)
    assert np.all(np.abs(Vi[0] - V)[lower] <= 1e-9)


# ---------------------------------------------------------------------------
# P5/P6  monotonicity, contraction (Tdef is a monotone contraction, §3)
#        and the Kruzkov bound 0 <= v <= 1.
# ---------------------------------------------------------------------------
def test_p5_monotone_contraction():
    p = W.make(2, scale=32 / 1024).fine
    o = oracle.OracleProblem(p)
    cls = o.classes()
    rng = np.random.default_rng(5)
    beta = o.beta()
    for t in range(20):
        Vv = rng.uniform(0, 1, p.grid.size)
        Wv = Vv + rng.uniform(0, 0.3, p.grid.size)
        TV, _ = o.apply_T(Vv, cls)
        TW, _ = o.apply_T(Wv, cls)
        assert np.all(TV <= TW + 1e-15)
        interior = cls == oracle.INTERIOR
        assert np.abs(TV - TW)[interior].max() <= beta * np.abs(Vv - Wv).max() + 1e-15
    V, it, res = o.solve()
    assert V.min() >= 0.0 and V.max() <= 1.0


# ---------------------------------------------------------------------------
# P10  multilinear interpolation: node values reproduced, affine fields exact,
#      periodic axis wraps (R4).
# ---------------------------------------------------------------------------
def test_p10_interpolation():
    grid = W.Grid((7, 5, 6), (-1.0, 0.0, 0.0), (2.0, 1.0, 2 * np.pi), (False, False, True))
    piece = np.full(grid.size, -1, np.int8)
    p = mk_problem(grid, np.zeros((1, 3)), piece, dynamics=W.DYN_DUBINS)
    o = oracle.OracleProblem(p)
    rng = np.random.default_rng(3)
    F = rng.normal(size=grid.size)
    for t in range(20):
        i, j, k = rng.integers(0, 7), rng.integers(0, 5), rng.integers(0, 6)
        assert o.interp(F, [i, j, k]) == F[i + 7 * (j + 5 * k)]
    x, y, th = grid.mesh()
    Aff = (0.3 + 1.7 * x - 0.4 * y).reshape(-1)
    for t in range(50):
        gi = [rng.uniform(0, 6), rng.uniform(0, 4), rng.uniform(0, 6)]
        exp = 0.3 + 1.7 * (-1 + gi[0] * 0.5) - 0.4 * (gi[1] * 0.25)
        assert abs(o.interp(Aff, gi) - exp) < 1e-13
    # periodic wrap: halfway between theta node 5 and node 0
    G = np.zeros(grid.size)
    G.reshape(6, 5, 7)[5] = 2.0
    G.reshape(6, 5, 7)[0] = 4.0
    assert abs(o.interp(G, [3, 2, 5.5]) - 3.0) < 1e-14
    assert abs(o.interp(G, [3, 2, -0.5]) - 3.0) < 1e-14
    # outside the box on a non-periodic axis -> v_out; within 1e-6 cells: clamped (R3)
    assert o.interp(G, [6.000002, 2, 1]) == p.v_out
    assert o.interp(G, [-2e-6, 2, 1]) == p.v_out
    assert o.interp(G, [6.0000005, 2, 1]) == o.interp(G, [6.0, 2, 1])
    assert o.interp(G, [-5e-7, 2, 1]) == o.interp(G, [0.0, 2, 1])


# ---------------------------------------------------------------------------
# P11  dynamics by direct substitution, recovered through the bracket on an
#      affine V (interpolation is exact there): affine (Zermelo, regulator),
#      Dubins, Van der Pol (SPEC.md example: f((.5,.5),a) = (.5, a - .125)).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["zermelo", "regulator", "dubins", "vdp"])
def test_p11_dynamics_through_bracket(kind):
    if kind == "dubins":
        grid = W.Grid((41, 41, 16), (-3.0, -3.0, 0.0), (3.0, 3.0, 2 * np.pi), (False, False, True))
    else:
        grid = W.Grid((41, 41), (-2.0, -2.0), (2.0, 2.0), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    A = np.zeros((3, 3))
    if kind == "zermelo":
        ctrl, dyn = W.unit_circle_controls(8), W.DYN_AFFINE
        A[0, 1] = 0.5
    elif kind == "regulator":
        ctrl, dyn = W.interval_controls(5, axis=1), W.DYN_AFFINE
        A[0, 1], A[1, 0] = 1.0, -0.5
    elif kind == "dubins":
        ctrl, dyn = W.interval_controls(3), W.DYN_DUBINS
    else:
        ctrl, dyn = W.interval_controls(3), W.DYN_VANDERPOL
    h = 0.01
    p = mk_problem(grid, ctrl, piece, h=h, A=A, dynamics=dyn, cost=W.COST_DISCOUNTED, lam=0.0,
                   vdp_mu=1.0, v_out=0.0)
    o = oracle.OracleProblem(p)
    xs = grid.mesh()
    gi = [10.0, 30.0] + ([3.0] if grid.dim == 3 else [])
    pt = [grid.lo[d] + gi[d] * grid.spacing(d) for d in range(grid.dim)]
    for k in range(len(ctrl)):
        a = ctrl[k]
        if kind == "zermelo":
            f = [a[0] + 0.5 * pt[1], a[1]]
        elif kind == "regulator":
            f = [pt[1], a[1] - 0.5 * pt[0]]
        elif kind == "dubins":
            f = [math.cos(pt[2]), math.sin(pt[2]), a[0]]
        else:
            f = [pt[1], (1 - pt[0] ** 2) * pt[1] - pt[0] + a[0]]
        for d in range(grid.dim):
            # lambda = 0, l = 0 -> bracket = I[x_d](x + h f) = x_d + h f_d (the heading
            # field is linear in its index away from the periodic wrap)
            val = o.bracket(xs[d].reshape(-1), gi, k)
            assert abs(val - (pt[d] + h * f[d])) < 1e-12, (kind, k, d)
    if kind == "vdp":
        # SPEC.md example: f((0.5,0.5), a) = (0.5, a - 0.125)
        g2 = W.Grid((5, 5), (-1.0, -1.0), (1.0, 1.0), (False, False))
        p2 = mk_problem(g2, np.array([[0.3, 0, 0]]), np.full(25, -1, np.int8), h=0.01,
                        dynamics=W.DYN_VANDERPOL, cost=W.COST_DISCOUNTED, lam=0.0, v_out=0.0)
        o2 = oracle.OracleProblem(p2)
        xx, yy = g2.mesh()
        assert abs(o2.bracket(xx.reshape(-1), [3, 3], 0) - (0.5 + 0.01 * 0.5)) < 1e-14
        assert abs(o2.bracket(yy.reshape(-1), [3, 3], 0) - (0.5 + 0.01 * (0.3 - 0.125))) < 1e-14


# ---------------------------------------------------------------------------
# P12  Dubins special case reducing to a ray-disk intersection: with the single
#      control a = 0 the car moves straight, T = first hitting time of the disk.
# ---------------------------------------------------------------------------
def test_p12_dubins_straight_rays():
    grid = W.Grid((61, 61, 16), (-3.0, -3.0, 0.0), (3.0, 3.0, 2 * np.pi), (False, False, True))
    c, r = (0.4, -0.3), 0.6
    piece = W.ball_pieces(grid, [c], [r])
    p = mk_problem(grid, np.zeros((1, 3)), piece, dynamics=W.DYN_DUBINS, h=grid.spacing(0),
                   tol=1e-12)
    V, it, res = oracle.OracleProblem(p).solve()
    x, y, th = [a.reshape(-1) for a in grid.mesh()]
    ux, uy = np.cos(th), np.sin(th)
    px, py = x - c[0], y - c[1]
    bproj = px * ux + py * uy
    perp2 = px * px + py * py - bproj * bproj
    disc = r * r - perp2
    with np.errstate(invalid="ignore"):
        t_hit = -bproj - np.sqrt(disc)
    hit = (disc > 0) & (t_hit >= 0)
    dx = grid.spacing(0)
    clear_hit = hit & (np.sqrt(np.maximum(perp2, 0)) < r - 4 * dx) & (piece < 0)
    away = (~hit) & (piece < 0) & (bproj > 4 * dx) & (px * px + py * py > (r + 4 * dx) ** 2)
    # (moving away from the disk and clear of it: no foot ever sees a target node)
    clear_miss = (~hit) & (piece < 0) & (np.sqrt(np.maximum(perp2, 0)) > r + 4 * dx)
    T = np.where(hit, t_hit, np.inf)
    Td = -np.log1p(-np.minimum(V, 1 - 1e-16)) * p.h / math.log1p(p.h)
    assert np.all(np.abs(Td - T)[clear_hit] <= 0.1 + 0.05 * T[clear_hit])
    assert np.all(V[away] > 1.0 - 1e-12)
    assert np.all(V[clear_miss] > 0.99)          # only interpolation diffusion leaks in


# ---------------------------------------------------------------------------
# P13  constant drift landing exactly on nodes (b = (1,0), h = dx): the
#      discounted recursion V_i = h l(x_i) + beta V_{i+1} from the right edge.
# ---------------------------------------------------------------------------
def test_p13_drift_recursion():
    grid = W.Grid((21, 5), (-1.0, 0.0), (1.0, 0.4), (False, False))
    piece = np.full((5, 21), -1, np.int8)
    piece[:, -1] = 0
    b = np.array([1.0, 0.0, 0.0])
    p = mk_problem(grid, np.zeros((1, 3)), piece.reshape(-1), b=b, cost=W.COST_DISCOUNTED,
                   lam=0.5, l0=0.2, lq=1.0, v_out=100.0, tol=1e-14)
    V, it, _ = oracle.OracleProblem(p).solve()
    V = V.reshape(5, 21)
    x, y = grid.mesh()
    beta = 1 / (1 + 0.5 * p.h)
    for j in range(5):
        exp = np.zeros(21)
        for i in range(19, -1, -1):
            exp[i] = p.h * (0.2 + x[j, i] ** 2 + y[j, i] ** 2) + beta * exp[i + 1]
        np.testing.assert_allclose(V[j], exp, rtol=1e-12, atol=1e-14)


# ---------------------------------------------------------------------------
# P7  labels vs the additively weighted Voronoi partition (north_star: exact
#     sub-domains of the eikonal problem), at nodes clear of the cell walls.
# ---------------------------------------------------------------------------
def test_p7_labels_weighted_voronoi():
    n = 61
    grid = W.Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    centres = [(-0.5, -0.4), (0.45, -0.5), (-0.3, 0.55), (0.5, 0.4)]
    radii = [0.05, 0.25, 0.12, 0.18]
    piece = W.ball_pieces(grid, centres, radii)
    p = mk_problem(grid, W.unit_circle_controls(64), piece, tol=1e-12)
    o = oracle.OracleProblem(p)
    V, _, _ = o.solve()
    lab, steps, mm, geo = o.label(V, np.arange(grid.size), n_max=4 * n)
    x, y = [a.reshape(-1) for a in grid.mesh()]
    w = np.array([np.hypot(x - cx, y - cy) - r for (cx, cy), r in zip(centres, radii)])
    order = np.sort(w, axis=0)
    vor = np.argmin(w, axis=0)
    clear = (order[1] - order[0]) > 4 * grid.spacing(0)
    assert clear.sum() > 0.8 * grid.size
    assert np.all(lab[clear] == vor[clear])
    assert np.all(lab >= 0)


# ---------------------------------------------------------------------------
# P8  prolongation with the overlap band vs an independent brute force
#     (scipy binary dilation of each label's nodes placed on the fine lattice).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("band", [0, 3])
def test_p8_prolongation_bruteforce(band):
    rng = np.random.default_rng(8)
    cg = W.Grid((9, 7), (0.0, 0.0), (1.0, 0.75), (False, False))
    R = (4, 4)
    fg = W.Grid((33, 25), (0.0, 0.0), (1.0, 0.75), (False, False))
    m = 5
    lab = rng.integers(-1, m, size=cg.size).astype(np.int32)
    fpiece = np.full(fg.size, -1, np.int8)
    fpiece[rng.choice(fg.size, 10, replace=False)] = rng.integers(0, m, 10)
    mask = oracle.prolong(cg, fg, R, band, lab, m, fpiece).reshape(25, 33)
    L = lab.reshape(7, 9)
    for k in range(m):
        seed = np.zeros((25, 33), bool)
        seed[::4, ::4] = (L == k) | (L < 0)
        rad = 4 + band
        dil = ndimage.binary_dilation(seed, structure=np.ones((2 * rad + 1, 2 * rad + 1), bool))
        dil |= (fpiece.reshape(25, 33) == k)
        assert np.array_equal(((mask >> k) & 1).astype(bool), dil), k


def test_p8_prolongation_periodic_axis():
    cg = W.Grid((3, 3, 4), (0, 0, 0), (1, 1, 2 * np.pi), (False, False, True))
    fg = W.Grid((5, 5, 8), (0, 0, 0), (1, 1, 2 * np.pi), (False, False, True))
    lab = np.full(cg.size, 1, np.int32)
    lab.reshape(4, 3, 3)[3] = 0          # theta layer 3 (fine layer 6) labelled 0
    mask = oracle.prolong(cg, fg, (2, 2, 2), 0, lab, 2, np.full(fg.size, -1, np.int8))
    bit0 = (mask.reshape(8, 5, 5) & 1).astype(bool)
    # fine layers within 2 of layer 6 around the circle: 4,5,6,7,0
    assert [bool(bit0[t].all()) for t in range(8)] == [True, False, False, False, True, True,
                                                         True, True]


# ---------------------------------------------------------------------------
# P9  independence invariant (Proposition 2.3 / 4.1): solving each sub-domain
#     alone and assembling by min reproduces the global solution.
# ---------------------------------------------------------------------------
def test_p9_isa_reproduces_global_solution():
    cfg = W.make(1)
    res = oracle.isa(cfg.fine, cfg.coarse, cfg.ratio, cfg.band, cfg.m, cfg.n_max_steps)
    o = oracle.OracleProblem(cfg.fine)
    V, _, _ = o.solve()
    mask = res["mask"]
    assert np.all(mask != 0)                             # coverage
    for k in range(cfg.m):
        inside = ((mask >> k) & 1).astype(bool)
        assert np.all(res["Vk"][k][inside] >= V[inside] - 1e-9)  # restriction only adds cost
    assert np.abs(res["Vbar"] - V).max() < 10 * cfg.fine.tol
    assert np.all(res["labels"] >= 0)
    # each sub-domain is strictly smaller than the domain
    frac = [((mask >> k) & 1).mean() for k in range(cfg.m)]
    assert max(frac) < 0.4          # cf. PAPER.md Table 1: 33% at a 20^2 coarse grid


# ---------------------------------------------------------------------------
# P14  the paper's RA reconstruction on the eikonal problem:
#      every auxiliary V_i is the single-piece Kruzkov distance 1 - exp(-(|x-c_i| - r_i))
#      up to the scheme's O(dx) error; min_i V_i is a supersolution of the joint problem
#      and agrees with its solution to O(dx); each Sigma_i contains the exact independent
#      sub-domain of piece i (the additively weighted Voronoi cell, PAPER Prop. 3.1 with
#      the paper's constants C = M = 1, q = 1/2 for the distance function, line 519).
# ---------------------------------------------------------------------------
def test_p14_ra_eikonal():
    n = 41
    grid = W.Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    centres = [(-0.5, -0.5), (0.5, -0.5), (-0.5, 0.5), (0.5, 0.5)]
    radii = [0.1] * 4
    piece = W.ball_pieces(grid, centres, radii)
    p = mk_problem(grid, W.unit_circle_controls(32), piece, tol=1e-12)
    Vs, Vmin, mask, its = oracle.ra(p, 4, 1.0, 1.0, 0.5)
    x, y = [a.reshape(-1) for a in grid.mesh()]
    dx = grid.spacing(0)
    w = np.array([np.hypot(x - cx, y - cy) - r for (cx, cy), r in zip(centres, radii)])
    for i in range(4):
        exact = 1.0 - np.exp(-np.maximum(w[i], 0.0))
        assert np.abs(Vs[i] - exact).max() < 3 * dx, i
        assert np.all(Vs[i][piece == i] == 0.0)
    Vj, _, _ = oracle.OracleProblem(p).solve()
    assert (Vmin - Vj).min() >= -1e-12            # min_i V_i >= the joint solution
    assert (Vmin - Vj).max() <= 2 * dx
    vor = np.argmin(w, axis=0)
    for i in range(4):
        inside = ((mask >> i) & 1).astype(bool)
        assert np.all(inside[vor == i]), i         # exact sub-domain contained in Sigma_i
        assert np.all(inside[piece == i])
    # the threshold really selects: the sets are proper subsets with the paper's constants
    # (in Kruzkov units |v_i - v| <= |T_i - T|, so the paper's distance-function constants
    # keep containment but select loosely: ~90 % of the square here)
    thr = 2 * (dx ** 0.5 + dx)
    for i in range(4):
        sel = np.abs(Vs[i] - Vmin) <= thr
        assert np.array_equal(((mask >> i) & 1).astype(bool), sel | (piece == i))
        assert 0.25 < sel.mean() < 0.95
        assert not sel[vor == (3 - i)].all()      # the opposite corner's cell is cut


def test_p14_prolong_mask_matches_label_prolongation():
    """Mask prolongation of single-bit masks (label k -> bit k, -1 -> all bits) is the
    pinned label prolongation (P8)."""
    rng = np.random.default_rng(14)
    cg = W.Grid((9, 7), (0.0, 0.0), (1.0, 0.75), (False, False))
    fg = W.Grid((33, 25), (0.0, 0.0), (1.0, 0.75), (False, False))
    m = 5
    lab = rng.integers(-1, m, size=cg.size).astype(np.int32)
    fpiece = np.full(fg.size, -1, np.int8)
    fpiece[rng.choice(fg.size, 10, replace=False)] = rng.integers(0, m, 10)
    cmask = np.where(lab < 0, (1 << m) - 1, 1 << np.maximum(lab, 0)).astype(np.uint64)
    for band in (0, 2):
        a = oracle.prolong(cg, fg, (4, 4), band, lab, m, fpiece)
        b = oracle.prolong_mask(cg, fg, (4, 4), band, cmask, m, fpiece)
        assert np.array_equal(a, b)


# ---------------------------------------------------------------------------
# P15  the speed field c(x) of f = c(x) u_a (config 2's dynamics, §2 line 36).
#  (a) c == 2 on the lattice with h = dx/2: every foot lands on a neighbour node, so the
#      Kruzkov values are the BFS ones, V = 1 - beta^d (a speed ignored or squared puts
#      the feet half a cell or two cells away).
#  (b) c depending on x only, target = the left edge: the minimum time is the 1-D
#      travel time T(x) = int_0^x ds / c(s) = 2 ln(1 + x/2) for c = 1 + x/2, and the
#      discrete times converge to it at O(dx) (Theorem 3.1).
# ---------------------------------------------------------------------------
def test_p15a_constant_speed_lattice():
    grid = W.Grid((13, 9), (-1.0, -0.5), (1.4, 1.1), (False, False))
    rng = np.random.default_rng(15)
    piece = np.full(grid.size, -1, np.int8)
    piece[rng.choice(grid.size, 3, replace=False)] = np.arange(3)
    speed = np.full(grid.size, 2.0)
    p = mk_problem(grid, W.axis_controls(), piece, h=grid.spacing(0) / 2, speed=speed)
    V, it, res = oracle.OracleProblem(p).solve()
    d = bfs_distance((9, 13), (piece >= 0).reshape(9, 13)).reshape(-1)
    beta = 1.0 / (1.0 + p.h)
    np.testing.assert_allclose(V, 1.0 - beta ** d, rtol=0, atol=1e-13)
    assert it == d.max() + 1


def test_p15b_variable_speed_travel_time():
    errs = []
    for n in (21, 41, 81):
        grid = W.Grid((n, (n - 1) // 4 + 1), (0.0, 0.0), (1.0, 0.25), (False, False))
        x, y = [a.reshape(-1) for a in grid.mesh()]
        piece = np.where(np.isclose(x, 0.0), 0, -1).astype(np.int8)
        speed = 1.0 + 0.5 * x
        p = mk_problem(grid, W.unit_circle_controls(64), piece, h=grid.spacing(0) / 1.5,
                       speed=speed, tol=1e-12)
        V, it, res = oracle.OracleProblem(p).solve()
        Td = -np.log1p(-V) * p.h / math.log1p(p.h)
        T = 2.0 * np.log1p(0.5 * x)
        err = np.abs(Td - T).max()
        assert err <= 2.0 * grid.spacing(0), (n, err)
        errs.append(err)
    assert errs[-1] < errs[0] / 2.5
    # the speed really enters: constant speed 1 would give T = x (0.19 off at x = 1)
    assert abs(T.max() - 1.0) > 0.15


# ---------------------------------------------------------------------------
# P16  the control minimisation of the bracket (R7): best = min_k bracket_k, argmin =
#      the LOWEST index attaining it, margin = second smallest bracket - smallest (>= 0),
#      by brute force over the pinned bracket (P1-P13) at every node; and an exact tie
#      (two lattice moves to the same BFS level) that has margin 0 and the lower index.
# ---------------------------------------------------------------------------
def test_p16_min_bracket_brute_force():
    cfg = W.make(2, scale=24 / 1024, ratio=1)      # 25^2, 64 controls, speed field
    p = cfg.fine
    o = oracle.OracleProblem(p)
    rng = np.random.default_rng(16)
    V = rng.uniform(0, 1, p.grid.size)
    a, margin = o.feedback(V)
    n0 = p.grid.n[0]
    for idx in range(p.grid.size):
        if p.piece[idx] >= 0:
            assert a[idx] == -1 and margin[idx] == np.inf
            continue
        gi = [idx % n0, idx // n0]
        b = np.array([o.bracket(V, gi, k) for k in range(p.n_controls)])
        srt = np.sort(b)
        assert a[idx] == int(np.nonzero(b == srt[0])[0][0])
        assert margin[idx] == srt[1] - srt[0] and margin[idx] >= 0
        best, arg, mm = o.min_bracket(V, gi)
        assert best == srt[0] and arg == a[idx] and mm == margin[idx]


def test_p16_exact_tie_lowest_index():
    grid = W.Grid((7, 7), (0.0, 0.0), (1.0, 1.0), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    piece[0] = 0                                      # target at node (0, 0)
    ctrl = W.axis_controls()                          # +x, +y, -x, -y
    p = mk_problem(grid, ctrl, piece)
    o = oracle.OracleProblem(p)
    V, _, _ = o.solve()
    a, margin = o.feedback(V)
    # node (i, j), i, j >= 1: -x and -y both reach BFS level i + j - 1 (an exact tie)
    for j in range(1, 7):
        for i in range(1, 7):
            assert a[j * 7 + i] == 2 and margin[j * 7 + i] == 0.0
    # on the axis y = 0 the move -x is unique: the best bracket is 1 - beta^i (level
    # i - 1), the next best 1 - beta^(i+2) (+x or +y to level i + 1; -y leaves the box)
    beta = 1.0 / (1.0 + p.h)
    for i in range(1, 6):
        assert a[i] == 2
        assert abs(margin[i] - (beta ** i - beta ** (i + 2))) < 1e-14


# ---------------------------------------------------------------------------
# P17  the trajectory bookkeeping of the labelling (R8): a plain re-simulation with the
#      feedback taken AT y_s (o.min_bracket at the off-grid point), the speed
#      interpolated at y_s, y_{s+1} = y_s + h f / dx, the label of the nearest node,
#      gives the oracle's labels and step counts exactly, its minimum control margin
#      along the path exactly, and its "geo" output = the smallest distance of a
#      nearest-node rounding (positions y_0..y_S) or of a box test (y_1..y_S) to its
#      threshold.  A feedback taken at the nearest node instead moves differently (the
#      test asserts that it would on this problem).
# ---------------------------------------------------------------------------
def _simulate(o, p, V, start, n_max):
    g = p.grid
    n = g.n
    gi = [float(start % n[0]), float(start // n[0])]
    dx = [g.spacing(0), g.spacing(1)]
    mm, geo, differs = np.inf, np.inf, False
    s = 0
    while True:
        # distance of the rounding floor(g + 1/2) to its threshold (a half-integer)
        for d in range(2):
            geo = min(geo, abs(gi[d] - (math.floor(gi[d]) + 0.5)))
        r = [min(int(math.floor(gi[d] + 0.5)), n[d] - 1) for d in range(2)]
        pc = p.piece[r[0] + n[0] * r[1]]
        if pc >= 0:
            return int(pc), s, mm, geo, differs
        if s >= n_max:
            return -1, s, mm, geo, differs
        _, a, margin = o.min_bracket(V, gi)
        _, a_node, _ = o.min_bracket(V, r)
        differs |= (a_node != a)
        mm = min(mm, margin)
        c = o.interp(p.speed, gi) if p.speed is not None else 1.0
        x = [g.lo[d] + gi[d] * dx[d] for d in range(2)]
        u = p.controls[a]
        out = False
        for d in range(2):
            f = c * u[d] + p.b[d]
            for e in range(2):
                f += p.A[d, e] * x[e]
            gi[d] = gi[d] + p.h * f / dx[d]
            geo = min(geo, abs(gi[d]), abs((n[d] - 1) - gi[d]))
            out |= gi[d] < 0.0 or gi[d] > n[d] - 1
        s += 1
        if out:
            return -1, s, mm, geo, differs


@pytest.mark.parametrize("idx", [2, 3])
def test_p17_trajectory_bruteforce(idx):
    cfg = W.make(idx, scale=32 / (1024 if idx == 2 else 4096), ratio=1)
    p = cfg.fine
    o = oracle.OracleProblem(p)
    V, _, _ = o.solve()
    rng = np.random.default_rng(17)
    nodes = rng.choice(np.nonzero(p.piece < 0)[0], 60, replace=False)
    lab, st, mar, geo = o.label(V, nodes, cfg.n_max_steps)
    any_differs = False
    for t, start in enumerate(nodes):
        el, es, em, eg, differs = _simulate(o, p, V, int(start), cfg.n_max_steps)
        any_differs |= differs
        assert (lab[t], st[t]) == (el, es), (start, lab[t], st[t], el, es)
        assert mar[t] == em
        assert abs(geo[t] - eg) <= 1e-12, (geo[t], eg)
    assert any_differs       # the nearest node's feedback would have steered elsewhere
    assert np.all(mar >= 0) and np.all(geo >= 0) and np.isfinite(geo).all()


# ---------------------------------------------------------------------------
# P18  the trajectory step budget n_max (R8): on the lattice, a node at BFS distance d
#      from the target is labelled after exactly d steps; a budget of d - 1 steps ends
#      unlabelled (-1) after d - 1 steps.
# ---------------------------------------------------------------------------
def test_p18_step_budget():
    grid = W.Grid((11, 5), (0.0, 0.0), (1.0, 0.4), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    piece[0] = 0
    p = mk_problem(grid, W.axis_controls(), piece)
    o = oracle.OracleProblem(p)
    V, _, _ = o.solve()
    d = bfs_distance((5, 11), (piece >= 0).reshape(5, 11)).reshape(-1)
    nodes = np.nonzero(d >= 2)[0]
    for t, node in enumerate(nodes):
        lab, st, _, _ = o.label(V, [node], d[node])
        assert lab[0] == 0 and st[0] == d[node]
        lab, st, _, _ = o.label(V, [node], d[node] - 1)
        assert lab[0] == -1 and st[0] == d[node] - 1


# ---------------------------------------------------------------------------
# P19  the sub-domain solve (ISA step 3, R10): nodes outside S_k are ghosts holding
#      v_out — a target node of another piece outside S_k included — and every target
#      node inside S_k keeps g.  On the lattice the restricted solution is the BFS
#      distance through S_k's nodes only: V = 1 - beta^d_S, V = 1 where no path exists.
# ---------------------------------------------------------------------------
def bfs_restricted(shape, targets, allowed):
    d = bfs_distance(shape, targets & allowed)
    ny, nx = shape
    # re-run on the allowed nodes only (a plain BFS that never enters a ghost node)
    d = np.full(shape, -1, np.int64)
    q = collections.deque()
    for j, i in zip(*np.nonzero(targets & allowed)):
        d[j, i] = 0
        q.append((j, i))
    while q:
        j, i = q.popleft()
        for dj, di in ((1, 0), (-1, 0), (0, 1), (0, -1)):
            a, b = j + dj, i + di
            if 0 <= a < ny and 0 <= b < nx and allowed[a, b] and d[a, b] < 0:
                d[a, b] = d[j, i] + 1
                q.append((a, b))
    return d


def test_p19_subdomain_ghosts_and_targets():
    nx, ny = 12, 8
    grid = W.Grid((nx, ny), (0.0, 0.0), (1.1, 0.7), (False, False))
    piece = np.full((ny, nx), -1, np.int8)
    piece[1, 1] = 0                 # piece 0 inside S_0
    piece[6, 2] = 1                 # piece 1 inside S_0: keeps g = 0
    piece[2, 9] = 1                 # piece 1 outside S_0: a ghost of S_0
    allowed = np.ones((ny, nx), bool)
    allowed[:, 7] = False           # a wall column ...
    allowed[5, 7] = True            # ... with one gap
    allowed[2, 8:] = False          # and the far piece-1 node's row cut off
    allowed[2, 9] = False
    mask = allowed.reshape(-1).astype(np.uint64)     # bit 0 = S_0
    mask[piece.reshape(-1) == 1] |= 2
    p = mk_problem(grid, W.axis_controls(), piece.reshape(-1), tol=1e-14)
    o = oracle.OracleProblem(p)
    V, it, _ = o.solve_subdomain(mask, 0)
    d = bfs_restricted((ny, nx), piece >= 0, allowed).reshape(-1)
    beta = 1.0 / (1.0 + p.h)
    exp = np.where(d >= 0, 1.0 - beta ** np.maximum(d, 0), 1.0)
    np.testing.assert_allclose(V, exp, rtol=0, atol=1e-13)
    assert V[2 * nx + 9] == p.v_out and V[6 * nx + 2] == 0.0


# ---------------------------------------------------------------------------
# P20  RA step 3 ("if |V_i(j) - V(j)| <= 2(C dx^q + M dx)"): the
#      comparison includes equality, and the piece's own nodes are always in its set.
# ---------------------------------------------------------------------------
def test_p20_ra_threshold_inclusive():
    V = np.array([0.0, 0.0, 0.5, 0.25, 0.75])
    V0 = np.array([0.25, 0.25 + 2 ** -40, 0.25, 0.25, 0.25])   # |.| = thr, > thr, thr, 0, thr
    V1 = np.array([1.0, 1.0, 1.0, 1.0, 0.75])
    piece = np.array([-1, -1, -1, 1, -1], np.int8)
    mask = oracle.ra_masks([V0, V1], V, piece, 0.25)
    assert list(mask & 1) == [1, 0, 1, 1, 0]
    assert list((mask >> 1) & 1) == [0, 0, 0, 1, 1]


# ---------------------------------------------------------------------------
# P21  the box tolerance of R3 only decides feet that lie ON the box in exact
#      arithmetic: on every edge node of a unit-circle control problem, the brackets
#      with the tabulated controls (cos(pi/2) = 6e-17 ...) equal the brackets with the
#      controls' exact-zero components snapped to 0, and every foot that is outside
#      the box in exact arithmetic reads v_out.
# ---------------------------------------------------------------------------
def test_p21_box_tolerance_only_moves_exact_box_feet():
    n = 17
    grid = W.Grid((n, n), (-1.0, -1.0), (1.0, 1.0), (False, False))
    piece = np.full(grid.size, -1, np.int8)
    piece[n * (n // 2) + n // 2] = 0
    ctrl = W.unit_circle_controls(16)
    snapped = np.where(np.abs(ctrl) < 1e-12, 0.0, ctrl)
    assert np.any((ctrl != snapped))
    p = mk_problem(grid, ctrl, piece)
    ps = mk_problem(grid, snapped, piece)
    o, os_ = oracle.OracleProblem(p), oracle.OracleProblem(ps)
    V = np.random.default_rng(21).uniform(0, 0.5, grid.size)
    beta = o.beta()
    for idx in range(grid.size):
        i, j = idx % n, idx // n
        if 0 < i < n - 1 and 0 < j < n - 1:
            continue
        for k in range(16):
            b, bs = o.bracket(V, [i, j], k), os_.bracket(V, [i, j], k)
            assert abs(b - bs) <= 1e-15, (i, j, k)     # (a 6e-17 weight moves 1 ulp)
            foot = np.array([i, j]) + snapped[k, :2]     # h = dx: one cell per unit
            if np.any(foot < 0) or np.any(foot > n - 1):
                assert b == beta * p.v_out + (1 - beta)


# ---------------------------------------------------------------------------
# P22  the exit set (reading R9b): the box boundary is a piece of Gamma of its own
#      (Theorem 2.1 decomposes all of Gamma; exit cost v_out, Tdef line 243).
#  (a) the exit test: an unlabelled node joins the exit set iff Vc >= Vexit - tol
#      (inclusive), labelled nodes never;
#  (b) prolongation: label -2 -> the exit set (bit m) only, -1 -> the m pieces' sets, by
#      brute-force dilation;
#  (c) Kruzkov with no target: Vexit = 1 = "never reached" everywhere (to rounding);
#  (d) Proposition 4.1 still holds with the exit set on the regulator geometry
#      (config 5, reduced): the assembled field is never below the whole-grid solution
#      and within O(dx) of it, the exit set is used, and it shrinks the sets.
# ---------------------------------------------------------------------------
def test_p22a_exit_test_inclusive():
    lab = np.array([-1, -1, -1, 3, -1, 0], np.int32)
    Vc = np.array([0.5, 0.5, 0.75, 0.0, 1.0, 2.0])
    Vexit = np.array([0.75, 0.75 + 2 ** -30, 0.75, 9.0, 1.0, 2.0])
    out = oracle.exit_labels(lab, Vc, Vexit, 0.25)
    assert list(out) == [-2, -1, -2, 3, -2, 0]


def test_p22b_prolong_exit_set_bruteforce():
    rng = np.random.default_rng(22)
    cg = W.Grid((9, 7), (0.0, 0.0), (1.0, 0.75), (False, False))
    fg = W.Grid((33, 25), (0.0, 0.0), (1.0, 0.75), (False, False))
    m = 4
    lab = rng.integers(-2, m, size=cg.size).astype(np.int32)
    fpiece = np.full(fg.size, -1, np.int8)
    fpiece[rng.choice(fg.size, 8, replace=False)] = rng.integers(0, m, 8)
    band = 2
    mask = oracle.prolong(cg, fg, (4, 4), band, lab, m, fpiece, exit_set=True).reshape(25, 33)
    L = lab.reshape(7, 9)
    for k in range(m + 1):
        seed = np.zeros((25, 33), bool)
        member = ((L == k) | (L == -1)) if k < m else (L == -2)
        seed[::4, ::4] = member
        rad = 4 + band
        dil = ndimage.binary_dilation(seed, structure=np.ones((2 * rad + 1, 2 * rad + 1), bool))
        if k < m:
            dil |= (fpiece.reshape(25, 33) == k)
        got = ((mask >> np.uint64(k)) & np.uint64(1)).astype(bool)
        assert np.array_equal(got, dil), k
    assert int(mask.max()) < (1 << (m + 1))


def test_p22c_kruzkov_exit_solution_is_one():
    cfg = W.make(2, scale=32 / 1024, ratio=1)
    Ve = oracle.exit_solution(cfg.coarse)
    assert np.abs(Ve - 1.0).max() <= 1e-15       # beta * 1 + (1 - beta), rounded


def test_p22d_isa_with_exit_set_proposition_4_1():
    cfg = W.make(5, scale=128 / 16384, ratio=4)
    cfg.band = 4      # (the band this pin was written for; R13b's two coarse cells = 8 here
                      # cover most of the 129^2 box either way)
    V, _, _ = oracle.OracleProblem(cfg.fine).solve()
    res = oracle.isa(cfg.fine, cfg.coarse, cfg.ratio, cfg.band, cfg.m, cfg.n_max_steps,
                     exit_set=True)
    r9 = oracle.isa(cfg.fine, cfg.coarse, cfg.ratio, cfg.band, cfg.m, cfg.n_max_steps,
                    exit_set=False)
    assert res["n_sets"] == cfg.m + 1 and (res["labels"] == -2).sum() > 0
    d = res["Vbar"] - V
    dxc = cfg.coarse.grid.spacing(0)
    assert d.min() >= -10 * cfg.fine.tol and d.max() <= dxc
    cover = lambda r: sum(int(((r["mask"] >> np.uint64(k)) & np.uint64(1)).sum())
                          for k in range(r["n_sets"]))
    assert cover(res) < 0.9 * cover(r9)
