/*
 * oracle/hj_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, fp64 CPU implementation of what the hot path computes, written
 * from PAPER.md (arxiv 1405.3521, Festa, "Domains of dependence / independent
 * sub-domains for HJ equations") and the BASELINE.json north_star.  It shares no
 * code, header, helper or constant with paper_1405_3521_b200/ and must only be
 * loaded by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs.  The product path never calls it.
 *
 * Readings R1..R13 are listed in DESIGN.md §3; the ones used here are cited inline.
 *
 * Indexing: node (i0,i1,i2) has flat index i0 + n0*(i1 + n1*i2)  (axis 0 fastest).
 * Positions: x_d = lo_d + i_d*dx_d, dx_d = (hi-lo)/(n-1) (or /n when periodic).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#define OR_DYN_AFFINE 0
#define OR_DYN_DUBINS 1
#define OR_DYN_VANDERPOL 2
#define OR_COST_KRUZKOV 0
#define OR_COST_DISCOUNTED 1

/* Reading R3: a foot is outside the closed box when it lies more than OR_BOX_EPS
 * cells beyond it; feet within OR_BOX_EPS are clamped onto the boundary (feet whose
 * offset is zero in exact arithmetic, e.g. cos(pi/2), stay inside in any precision). */
#define OR_BOX_EPS 1e-6

#define OR_INTERIOR 0
#define OR_TARGET 1
#define OR_GHOST 2

typedef struct {
    int dim;
    long n[3];
    double lo[3], hi[3];
    int periodic[3];
    int dynamics;
    int K;
    const double *ctrl;      /* K x 3 control table                        */
    double A[9], b[3];       /* affine drift: f = c(x) u_a + A x + b        */
    const double *speed;     /* c(x) node field, NULL == 1                  */
    double dub_v, dub_w, vdp_mu;
    int cost;
    double lam, h;
    double l0, lq, ln, lr;   /* l(x,a) = l0 + lq|x|^2 + ln|x| + lr|a|^2     */
    double v_out;            /* value of a foot outside the box (R3)        */
    const signed char *piece;/* target piece of each node, -1 = none       */
    const double *g;         /* g(x_i) on target nodes, NULL == 0           */
} or_problem;

static long or_size(const or_problem *p) {
    long s = 1;
    for (int d = 0; d < p->dim; ++d) s *= p->n[d];
    return s;
}

double or_spacing(const or_problem *p, int d) {
    double span = p->hi[d] - p->lo[d];
    return p->periodic[d] ? span / (double)p->n[d] : span / (double)(p->n[d] - 1);
}

/* beta = 1/(1+lambda h): PAPER.md §3 eq. (Tdef), line 241. */
double or_beta(const or_problem *p) { return 1.0 / (1.0 + p->lam * p->h); }

static void or_unflatten(const or_problem *p, long idx, long ii[3]) {
    ii[0] = ii[1] = ii[2] = 0;
    for (int d = 0; d < p->dim; ++d) {
        ii[d] = idx % p->n[d];
        idx /= p->n[d];
    }
}

static long or_flatten(const or_problem *p, const long ii[3]) {
    long idx = 0;
    for (int d = p->dim - 1; d >= 0; --d) idx = idx * p->n[d] + ii[d];
    return idx;
}

/* Multilinear interpolation I[V] at index-space point gi (R4): the operator
 * "I" of PAPER.md §3 line 247 ("linear n-dimensional interpolation").
 * A point outside the closed box on a non-periodic axis returns v_out (R3:
 * "+infinity, x_i in Phi", Tdef line 243).  Returns the corner weights too. */
double or_interp_field(const or_problem *p, const double *F, const double gi[3],
                       double outside_value) {
    long i0[3] = {0, 0, 0}, i1[3] = {0, 0, 0};
    double w[3] = {0, 0, 0};
    for (int d = 0; d < p->dim; ++d) {
        double g = gi[d];
        long n = p->n[d];
        if (p->periodic[d]) {
            double f = floor(g);
            w[d] = g - f;
            long c = (long)f % n;
            if (c < 0) c += n;
            i0[d] = c;
            i1[d] = (c + 1) % n;
        } else {
            if (g < -OR_BOX_EPS || g > (double)(n - 1) + OR_BOX_EPS) return outside_value;
            if (g < 0.0) g = 0.0;
            if (g > (double)(n - 1)) g = (double)(n - 1);
            long c = (long)floor(g);
            if (c > n - 2) c = n - 2;
            w[d] = g - (double)c;
            i0[d] = c;
            i1[d] = c + 1;
        }
    }
    double acc = 0.0;
    for (int corner = 0; corner < (1 << p->dim); ++corner) {
        long ii[3] = {0, 0, 0};
        double wt = 1.0;
        for (int d = 0; d < p->dim; ++d) {
            if (corner & (1 << d)) {
                ii[d] = i1[d];
                wt *= w[d];
            } else {
                ii[d] = i0[d];
                wt *= 1.0 - w[d];
            }
        }
        acc += wt * F[or_flatten(p, ii)];
    }
    return acc;
}

/* speed c at an index-space point: the node field interpolated (R8), 1 if absent */
static double or_speed_at(const or_problem *p, const double gi[3]) {
    if (!p->speed) return 1.0;
    return or_interp_field(p, p->speed, gi, 1.0);
}

/* dynamics f(x, a_k) (§2 line 36 "y' = f(y,a)"; configs in DESIGN.md) */
void or_dynamics(const or_problem *p, const double x[3], double c, int k, double f[3]) {
    const double *a = p->ctrl + 3 * k;
    f[0] = f[1] = f[2] = 0.0;
    if (p->dynamics == OR_DYN_AFFINE) {
        for (int d = 0; d < p->dim; ++d) {
            double s = c * a[d] + p->b[d];
            for (int e = 0; e < p->dim; ++e) s += p->A[3 * d + e] * x[e];
            f[d] = s;
        }
    } else if (p->dynamics == OR_DYN_DUBINS) {
        f[0] = p->dub_v * cos(x[2]);
        f[1] = p->dub_v * sin(x[2]);
        f[2] = p->dub_w * a[0];
    } else { /* Van der Pol, §4.1 */
        f[0] = x[1];
        f[1] = p->vdp_mu * (1.0 - x[0] * x[0]) * x[1] - x[0] + a[0];
    }
}

/* running cost l(x,a) (§2 (H0) line 57) */
double or_running_cost(const or_problem *p, const double x[3], int k) {
    const double *a = p->ctrl + 3 * k;
    double x2 = 0.0, a2 = a[0] * a[0] + a[1] * a[1] + a[2] * a[2];
    for (int d = 0; d < p->dim; ++d)
        if (!p->periodic[d]) x2 += x[d] * x[d];
    return p->l0 + p->lq * x2 + p->ln * sqrt(x2) + p->lr * a2;
}

static void or_position(const or_problem *p, const double gi[3], double x[3]) {
    x[0] = x[1] = x[2] = 0.0;
    for (int d = 0; d < p->dim; ++d) x[d] = p->lo[d] + gi[d] * or_spacing(p, d);
}

/* The bracket of the SL operator for control k at index-space point gi
 * (PAPER.md eq. (Tdef), with the sign reading R1):
 *     beta * I[V](x + h f(x,a_k)) + c(x,a_k),
 * c = 1 - beta for the Kruzkov minimum-time problem, h l(x,a_k) when discounted. */
double or_bracket(const or_problem *p, const double *V, const double gi[3], int k) {
    double x[3], f[3], foot[3] = {0, 0, 0};
    or_position(p, gi, x);
    or_dynamics(p, x, or_speed_at(p, gi), k, f);
    for (int d = 0; d < p->dim; ++d) foot[d] = gi[d] + p->h * f[d] / or_spacing(p, d);
    double beta = or_beta(p);
    double cost = (p->cost == OR_COST_KRUZKOV) ? (1.0 - beta) : p->h * or_running_cost(p, x, k);
    return beta * or_interp_field(p, V, foot, p->v_out) + cost;
}

/* min over the control set and the lowest-index argmin; margin = second best
 * minus best (R7). */
double or_min_bracket(const or_problem *p, const double *V, const double gi[3], int *argmin,
                      double *margin) {
    double best = INFINITY, second = INFINITY;
    int arg = -1;
    for (int k = 0; k < p->K; ++k) {
        double v = or_bracket(p, V, gi, k);
        if (v < best) {
            second = best;
            best = v;
            arg = k;
        } else if (v < second) {
            second = v;
        }
    }
    if (argmin) *argmin = arg;
    if (margin) *margin = second - best;
    return best;
}

static double or_node_g(const or_problem *p, long idx) { return p->g ? p->g[idx] : 0.0; }

/* Node classes for a (possibly masked) solve: a node outside the sub-domain mask
 * is a ghost holding v_out (R10); a target node holds g (Tdef line 242). */
void or_classes(const or_problem *p, const unsigned long long *mask, int k, signed char *cls) {
    long N = or_size(p);
#pragma omp parallel for schedule(static)
    for (long i = 0; i < N; ++i) {
        int in = mask ? (int)((mask[i] >> k) & 1ull) : 1;
        if (!in) cls[i] = OR_GHOST;
        else cls[i] = (p->piece[i] >= 0) ? OR_TARGET : OR_INTERIOR;
    }
}

/* One Jacobi application V_new = T(V) (PAPER.md eq. (SL) line 235 / (Tdef)) on the nodes
 * [lo, hi) of the flat index (the whole grid in or_apply_T; a bounded sample of rows for
 * bench.py's timing of the oracle).  Returns the sup-norm change on those nodes. */
double or_apply_T_range(const or_problem *p, const signed char *cls, const double *V,
                        double *Vn, long lo, long hi) {
    double res = 0.0;
    /* every node is computed independently from V (Jacobi) and max is exact, so the
     * result does not depend on the thread count */
#pragma omp parallel for schedule(static) reduction(max : res)
    for (long idx = lo; idx < hi; ++idx) {
        double v;
        if (cls[idx] == OR_GHOST) {
            v = p->v_out;
        } else if (cls[idx] == OR_TARGET) {
            v = or_node_g(p, idx);
        } else {
            long ii[3];
            double gi[3];
            or_unflatten(p, idx, ii);
            for (int d = 0; d < 3; ++d) gi[d] = (double)ii[d];
            v = or_min_bracket(p, V, gi, NULL, NULL);
        }
        Vn[idx] = v;
        double dv = fabs(v - V[idx]);
        if (dv > res) res = dv;
    }
    return res;
}

double or_apply_T(const or_problem *p, const signed char *cls, const double *V, double *Vn) {
    return or_apply_T_range(p, cls, V, Vn, 0, or_size(p));
}

/* V^0: g on target nodes, v_out elsewhere (R6). */
void or_initial(const or_problem *p, const signed char *cls, double *V) {
    long N = or_size(p);
    for (long i = 0; i < N; ++i) V[i] = (cls[i] == OR_TARGET) ? or_node_g(p, i) : p->v_out;
}

/* Value iteration V^{n+1} = T(V^n) until ||V^{n+1}-V^n||_inf < tol (§3
 * line 248 and the stopping remark, line 341-345; R6).  Returns the iteration
 * count (number of applications of T); *res_out = last sup-norm change. */
long or_value_iteration(const or_problem *p, const signed char *cls, double *V, double tol,
                        long max_iter, double *res_out) {
    long N = or_size(p);
    double *W = (double *)malloc(sizeof(double) * N);
    or_initial(p, cls, V);
    long it = 0;
    double res = INFINITY;
    while (it < max_iter) {
        res = or_apply_T(p, cls, V, W);
        memcpy(V, W, sizeof(double) * N);
        ++it;
        if (res < tol) break;
    }
    free(W);
    if (res_out) *res_out = res;
    return it;
}

/* Discrete optimal feedback at every node (north_star "coarse feedback"). */
void or_feedback(const or_problem *p, const double *V, int *astar, double *margin) {
    long N = or_size(p);
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < N; ++idx) {
        long ii[3];
        double gi[3];
        or_unflatten(p, idx, ii);
        for (int d = 0; d < 3; ++d) gi[d] = (double)ii[d];
        if (p->piece[idx] >= 0) {
            astar[idx] = -1;
            margin[idx] = INFINITY;
            continue;
        }
        or_min_bracket(p, V, gi, &astar[idx], &margin[idx]);
    }
}

/* Trajectory labelling of one start node (R8): follow y_{s+1} = y_s + h f(y_s, a*(y_s))
 * with the discrete optimal feedback evaluated at y_s; the label is the piece of
 * the node nearest to y_s (floor(g+1/2)) the first time it is a target node;
 * -1 if y leaves the box or n_max steps pass.  Reports the number of steps, the
 * smallest control margin met along the way and the smallest distance of a
 * rounding / box decision to its threshold (index units). */
int or_label_trajectory(const or_problem *p, const double *V, long start, long n_max,
                        long *steps_out, double *min_margin, double *min_geo) {
    long ii[3];
    double gi[3] = {0, 0, 0};
    or_unflatten(p, start, ii);
    for (int d = 0; d < p->dim; ++d) gi[d] = (double)ii[d];
    double mm = INFINITY, mg = INFINITY;
    int label = -1;
    long s = 0;
    for (;; ++s) {
        long r[3] = {0, 0, 0};
        for (int d = 0; d < p->dim; ++d) {
            double t = gi[d] + 0.5;
            double fl = floor(t);
            double dist = t - fl;
            if (1.0 - dist < dist) dist = 1.0 - dist;
            if (dist < mg) mg = dist;
            long c = (long)fl;
            if (p->periodic[d]) {
                c %= p->n[d];
                if (c < 0) c += p->n[d];
            } else if (c > p->n[d] - 1) {
                c = p->n[d] - 1;
            }
            r[d] = c;
        }
        int pc = p->piece[or_flatten(p, r)];
        if (pc >= 0) {
            label = pc;
            break;
        }
        if (s >= n_max) break;
        int a;
        double margin;
        or_min_bracket(p, V, gi, &a, &margin);
        if (margin < mm) mm = margin;
        double x[3], f[3];
        or_position(p, gi, x);
        or_dynamics(p, x, or_speed_at(p, gi), a, f);
        int out = 0;
        for (int d = 0; d < p->dim; ++d) {
            gi[d] = gi[d] + p->h * f[d] / or_spacing(p, d);
            if (p->periodic[d]) {
                double n = (double)p->n[d];
                gi[d] = gi[d] - n * floor(gi[d] / n);
            } else {
                double lo_gap = gi[d], hi_gap = (double)(p->n[d] - 1) - gi[d];
                double gap = fabs(lo_gap) < fabs(hi_gap) ? fabs(lo_gap) : fabs(hi_gap);
                if (gap < mg) mg = gap;
                if (gi[d] < 0.0 || gi[d] > (double)(p->n[d] - 1)) out = 1;
            }
        }
        if (out) {
            ++s;
            break;
        }
    }
    if (steps_out) *steps_out = s;
    if (min_margin) *min_margin = mm;
    if (min_geo) *min_geo = mg;
    return label;
}

void or_label_nodes(const or_problem *p, const double *V, const long *nodes, long count,
                    long n_max, int *labels, long *steps, double *margins, double *geo) {
#pragma omp parallel for schedule(dynamic, 64)
    for (long t = 0; t < count; ++t)
        labels[t] = or_label_trajectory(p, V, nodes[t], n_max, &steps[t], &margins[t], &geo[t]);
}

/* Prolongation of coarse labels to the fine grid with an overlap band (R9,
 * ISA step 2, §4): fine node i is in sub-domain k iff some
 * coarse node I labelled k has |i_d - R_d I_d| <= R_d + band on every axis
 * (periodic axes measured around the circle).  Coarse nodes labelled -1 count
 * for every sub-domain ("automatically included in each approximation", §4.1
 * line 587).  Target nodes of piece k on the fine grid are always in k. */
/* Prolongation of coarse sub-domain memberships (bit k of coarse_mask = coarse node in
 * the k-th set) to the fine grid with the overlap band (R9): fine node i is in S_k iff a
 * coarse node I with bit k has |i_d - R_d I_d| <= R_d + band on every axis; fine target
 * nodes of piece k are always in S_k. */
void or_prolong_mask(const long nc[3], const long nf[3], const int periodic[3], int dim,
                     const long ratio[3], long band, const unsigned long long *coarse_mask,
                     int m, const signed char *fine_piece, unsigned long long *fine_mask) {
    unsigned long long all = (m >= 64) ? ~0ull : ((1ull << m) - 1ull);
    long Nf = 1;
    for (int d = 0; d < dim; ++d) Nf *= nf[d];
#pragma omp parallel for schedule(static)
    for (long idx = 0; idx < Nf; ++idx) {
        long ii[3] = {0, 0, 0}, t = idx;
        for (int d = 0; d < dim; ++d) {
            ii[d] = t % nf[d];
            t /= nf[d];
        }
        long lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int d = 0; d < dim; ++d) {
            long reach = ratio[d] + band;
            /* candidate coarse indices I with |ii - R I| <= reach */
            lo[d] = (long)ceil((double)(ii[d] - reach) / (double)ratio[d]);
            hi[d] = (long)floor((double)(ii[d] + reach) / (double)ratio[d]);
        }
        unsigned long long bits = 0;
        long I[3];
        for (I[2] = lo[2]; I[2] <= hi[2]; ++I[2])
            for (I[1] = lo[1]; I[1] <= hi[1]; ++I[1])
                for (I[0] = lo[0]; I[0] <= hi[0]; ++I[0]) {
                    long J[3] = {0, 0, 0};
                    int ok = 1;
                    for (int d = 0; d < dim; ++d) {
                        long c = I[d];
                        if (periodic[d]) {
                            c %= nc[d];
                            if (c < 0) c += nc[d];
                        } else if (c < 0 || c > nc[d] - 1) {
                            ok = 0;
                        }
                        J[d] = c;
                    }
                    if (!ok) continue;
                    long cidx = 0;
                    for (int d = dim - 1; d >= 0; --d) cidx = cidx * nc[d] + J[d];
                    bits |= coarse_mask[cidx];
                }
        if (fine_piece[idx] >= 0) bits |= 1ull << fine_piece[idx];
        fine_mask[idx] = bits & all;
    }
}

/* ISA step 2 from trajectory labels (R8, R9, R9b): label k -> bit k; label -1 (the
 * trajectory left the box or ran out of steps) -> every piece's set ("automatically
 * included in each approximation"); label -2 (exit set,
 * or_exit_labels) -> bit m only. */
void or_prolong(const long nc[3], const long nf[3], const int periodic[3], int dim,
                const long ratio[3], long band, const int *coarse_label, int m, int exit_set,
                const signed char *fine_piece, unsigned long long *fine_mask) {
    int sets = m + (exit_set ? 1 : 0);
    unsigned long long pieces = (m >= 64) ? ~0ull : ((1ull << m) - 1ull);
    long Nc = 1;
    for (int d = 0; d < dim; ++d) Nc *= nc[d];
    unsigned long long *cm = (unsigned long long *)malloc(sizeof(unsigned long long) * (size_t)Nc);
    for (long j = 0; j < Nc; ++j) {
        int l = coarse_label[j];
        if (l >= 0) cm[j] = 1ull << l;
        else if (l == -2) cm[j] = exit_set ? (1ull << m) : 0ull;
        else cm[j] = pieces;
    }
    or_prolong_mask(nc, nf, periodic, dim, ratio, band, cm, sets, fine_piece, fine_mask);
    free(cm);
}

/* Exit set (reading R9b): the box boundary is a piece of Gamma of its own (exit cost
 * v_out, Tdef line 243; Theorem 2.1 decomposes all of Gamma).  An unlabelled node (-1)
 * whose value needs no target — Vc >= Vexit - tol, Vexit the solution with no target
 * node (RA's test of line 325 for that piece, with a solver-level threshold) — belongs
 * to the exit piece's set: label -2. */
void or_exit_labels(long N, int *labels, const double *Vc, const double *Vexit, double tol) {
    for (long j = 0; j < N; ++j)
        if (labels[j] == -1 && Vc[j] >= Vexit[j] - tol) labels[j] = -2;
}

/* RA step 3: Sigma_i = X_i plus every node j with
 * |V_i(j) - V(j)| <= thr, thr = 2 (C dx^q + M dx); bit i of mask[j]. */
void or_ra_masks(long N, int m, const double *const *Vi, const double *V,
                 const signed char *piece, double thr, unsigned long long *mask) {
#pragma omp parallel for schedule(static)
    for (long j = 0; j < N; ++j) {
        unsigned long long bits = 0;
        for (int i = 0; i < m; ++i)
            if (piece[j] == i || fabs(Vi[i][j] - V[j]) <= thr) bits |= 1ull << i;
        mask[j] = bits;
    }
}

/* ISA step 3 for one sub-domain (§4): value iteration
 * restricted to the mask of sub-domain k (outside = ghost, R10). */
long or_solve_subdomain(const or_problem *p, const unsigned long long *mask, int k, double *V,
                        double tol, long max_iter, double *res_out) {
    long N = or_size(p);
    signed char *cls = (signed char *)malloc(N);
    or_classes(p, mask, k, cls);
    long it = or_value_iteration(p, cls, V, tol, max_iter, res_out);
    free(cls);
    return it;
}

/* ISA step 4 (§4): Vbar(j) = min { V_k(j) : x_j in S_k }. */
void or_assemble(long N, int m, const unsigned long long *mask, const double *const *Vk,
                 double v_out,
                 double *Vbar) {
#pragma omp parallel for schedule(static)
    for (long j = 0; j < N; ++j) {
        double v = v_out;
        int any = 0;
        for (int k = 0; k < m; ++k)
            if ((mask[j] >> k) & 1ull) {
                if (!any || Vk[k][j] < v) v = Vk[k][j];
                any = 1;
            }
        Vbar[j] = v;
    }
}
