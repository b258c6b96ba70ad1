// hj_label.cu — discrete optimal feedback, trajectory labelling of the coarse
// nodes and prolongation of the labels to the fine grid with an overlap band
// (north_star "reconstruction of independent sub-domains"; PAPER.md Definition
// 2.2 line 150-152, Proposition 2.3, ISA steps 1-2 line 396-418;
// readings R7, R8, R9).  Decisions are taken in fp64 whatever the V dtype.
#include <algorithm>

#include "hj_host.cuh"

namespace hj {

// control sets up to this size are labelled one thread per trajectory (a warp per
// trajectory would leave most lanes without a control)
#ifndef HJ_LABEL_THREAD_MAX_K
#define HJ_LABEL_THREAD_MAX_K 16
#endif

// min over controls of the Tdef bracket at index-space point g (fp64), lowest
// index argmin, second-best gap.
template <typename Ts, int DIM>
__device__ double min_bracket(const DevProblem<double, Ts> &P, const Ts *__restrict__ V,
                              const int64_t o[3], const int64_t vn[3], const double g[3],
                              int *arg, double *margin) {
    double x[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[d] = fma(g[d], P.dx[d], P.lo[d]);
    const int64_t zero[3] = {0, 0, 0};
    double cs = 1.0;
    if (P.speed && P.dyn == HJ_DYN_AFFINE)
        cs = interp<double, Ts, DIM>(P.speed, o, vn, P.n, P.periodic, zero, g, 1.0);
    double base = (P.cost == HJ_COST_KRUZKOV) ? P.kcost : P.h * cost_state(P, x);
    double best = INFINITY, second = INFINITY;
    int a = -1;
    for (int k = 0; k < P.K; ++k) {
        double f[3];
        dynamics(P, x, cs, k, f);
        double foot[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) foot[d] = fma(P.hdx[d], f[d], g[d]);
        double I = interp<double, Ts, DIM>(V, o, vn, P.n, P.periodic, zero, foot, P.v_out);
        double ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(P.h * P.lr, P.csq[k], base);
        double v = fma(P.beta, I, ck);
        if (v < best) {
            second = best;
            best = v;
            a = k;
        } else if (v < second) {
            second = v;
        }
    }
    *arg = a;
    *margin = second - best;
    return best;
}

template <typename Ts, int DIM>
__global__ void k_feedback(const DevProblem<double, Ts> P, const Ts *__restrict__ V,
                           const int8_t *__restrict__ piece, int64_t N, int32_t *astar,
                           double *margin) {
    const int64_t o[3] = {0, 0, 0};
    const int64_t vn[3] = {P.n[0], P.n[1], P.n[2]};
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < N;
         t += (int64_t)gridDim.x * blockDim.x) {
        if (piece[t] >= 0) {
            astar[t] = -1;
            if (margin) margin[t] = INFINITY;
            continue;
        }
        double g[3] = {(double)(t % P.n[0]), (double)((t / P.n[0]) % P.n[1]),
                       (double)(t / (P.n[0] * P.n[1]))};
        int a;
        double m;
        min_bracket<Ts, DIM>(P, V, o, vn, g, &a, &m);
        astar[t] = a;
        if (margin) margin[t] = m;
    }
}

// The discrete optimal feedback trajectory of one coarse node (R8), one warp per node:
// the controls of every feedback evaluation split over the lanes (k = lane, lane+32, ...)
// and combined exactly: smallest bracket, lowest index among equal ones, and the
// second smallest value of the multiset (so margin = second - best is the serial
// scan's).  Every lane then takes the same step, so the warp never diverges.
struct BestPair {
    double best, second;
    int arg;
};

__device__ __forceinline__ BestPair warp_best(BestPair a) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        BestPair b;
        b.best = __shfl_xor_sync(0xffffffffu, a.best, o);
        b.second = __shfl_xor_sync(0xffffffffu, a.second, o);
        b.arg = __shfl_xor_sync(0xffffffffu, a.arg, o);
        const bool a_wins = a.best < b.best || (a.best == b.best && a.arg >= 0 &&
                                                (b.arg < 0 || a.arg < b.arg));
        const BestPair &w = a_wins ? a : b;
        const BestPair &l = a_wins ? b : a;
        BestPair r;
        r.best = w.best;
        r.arg = w.arg;
        r.second = fmin(w.second, l.best);
        a = r;
    }
    return a;
}

// dynamics() with the control's components u[0..2] from shared memory: the lanes of
// a warp take different controls, and a lane-divergent read of the kernel-parameter
// control table would serialise (one constant-bank address per pass)
// (ct, st: cos and sin of the heading x[2], computed once per trajectory step for the
// Dubins car — the same values dynamics() computes per control)
template <typename Ts>
__device__ __forceinline__ void dynamics_u(const DevProblem<double, Ts> &P, const double x[3],
                                           double c, const double *u, double f[3], double ct,
                                           double st) {
    if (P.dyn == HJ_DYN_AFFINE) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d >= P.dim) {
                f[d] = 0.0;
                continue;
            }
            double s = fma(c, u[d], P.b[d]);
            for (int e = 0; e < P.dim; ++e) s = fma(P.A[3 * d + e], x[e], s);
            f[d] = s;
        }
    } else if (P.dyn == HJ_DYN_DUBINS) {
        f[0] = P.dub_v * ct;
        f[1] = P.dub_v * st;
        f[2] = P.dub_w * u[0];
    } else {
        f[0] = x[1];
        f[1] = fma(P.vdp_mu * (1.0 - x[0] * x[0]), x[1], u[0] - x[0]);
        f[2] = 0.0;
    }
}

template <typename Ts, int DIM>
__device__ __forceinline__ BestPair lane_bracket(const DevProblem<double, Ts> &P,
                                                 const Ts *__restrict__ V, const int64_t o[3],
                                                 const int64_t vn[3], const double g[3],
                                                 int lane, const double (*uctl)[4], double ct,
                                                 double st) {
    double x[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[d] = fma(g[d], P.dx[d], P.lo[d]);
    const int64_t zero[3] = {0, 0, 0};
    double cs = 1.0;
    if (P.speed && P.dyn == HJ_DYN_AFFINE)
        cs = interp<double, Ts, DIM>(P.speed, o, vn, P.n, P.periodic, zero, g, 1.0);
    const double base = (P.cost == HJ_COST_KRUZKOV) ? P.kcost : P.h * cost_state(P, x);
    BestPair r{INFINITY, INFINITY, -1};
    for (int k = lane; k < P.K; k += 32) {
        double f[3];
        dynamics_u(P, x, cs, uctl[k], f, ct, st);
        double foot[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) foot[d] = fma(P.hdx[d], f[d], g[d]);
        const double I = interp<double, Ts, DIM>(V, o, vn, P.n, P.periodic, zero, foot, P.v_out);
        const double ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(P.h * P.lr, uctl[k][3], base);
        const double v = fma(P.beta, I, ck);
        if (v < r.best) {
            r.second = r.best;
            r.best = v;
            r.arg = k;
        } else if (v < r.second) {
            r.second = v;
        }
    }
    return warp_best(r);
}

// Bilinear interpolation of a whole 2-D non-periodic grid at index-space point (x0, x1):
// interp<double, Ts, 2> with a zero origin and the full grid as the view, the same
// operations in the same order (bit-identical), 32-bit indices.
template <typename Ts>
__device__ __forceinline__ double interp2_grid(const Ts *__restrict__ V, int n0, int n1, double x0,
                                               double x1, double v_out) {
    const double hi0 = (double)(n0 - 1), hi1 = (double)(n1 - 1), lo = -0.0;
    if (!(x0 >= lo - (double)BOX_EPS && x0 <= hi0 + (double)BOX_EPS)) return v_out;
    if (!(x1 >= lo - (double)BOX_EPS && x1 <= hi1 + (double)BOX_EPS)) return v_out;
    x0 = x0 < lo ? lo : (x0 > hi0 ? hi0 : x0);
    x1 = x1 < lo ? lo : (x1 > hi1 ? hi1 : x1);
    const double f0 = floor(x0), f1 = floor(x1);
    int c0 = (int)f0, c1 = (int)f1;
    double w0 = x0 - f0, w1 = x1 - f1;
    if (c0 > n0 - 2) {
        c0 = n0 - 2;
        w0 = 1.0;
    }
    if (c1 > n1 - 2) {
        c1 = n1 - 2;
        w1 = 1.0;
    }
    const Ts *p = V + (c0 + n0 * c1);
    const double a = lerp<double>((double)p[0], (double)p[1], w0);
    const double b = lerp<double>((double)p[n0], (double)p[n0 + 1], w0);
    return lerp<double>(a, b, w1);
}

// lane_bracket for the 2-D affine class on a non-periodic grid (the labelling of the
// local-class configs): state x and speed cs of the step passed in, the dynamics and
// interpolation written out — the same arithmetic, bit for bit.
template <typename Ts>
__device__ __forceinline__ BestPair lane_bracket_2d(const DevProblem<double, Ts> &P,
                                                    const Ts *__restrict__ V, const double g[3],
                                                    const double x[3], double cs, int lane,
                                                    const double (*uctl)[4]) {
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    const double base = kruz ? P.kcost : P.h * cost_state(P, x);
    const int n0 = (int)P.n[0], n1 = (int)P.n[1];
    BestPair r{INFINITY, INFINITY, -1};
    for (int k = lane; k < P.K; k += 32) {
        const double *u = uctl[k];
        double f0 = fma(cs, u[0], P.b[0]);
        f0 = fma(P.A[0], x[0], f0);
        f0 = fma(P.A[1], x[1], f0);
        double f1 = fma(cs, u[1], P.b[1]);
        f1 = fma(P.A[3], x[0], f1);
        f1 = fma(P.A[4], x[1], f1);
        const double I = interp2_grid<Ts>(V, n0, n1, fma(P.hdx[0], f0, g[0]),
                                          fma(P.hdx[1], f1, g[1]), P.v_out);
        const double ck = kruz ? base : fma(P.h * P.lr, u[3], base);
        const double v = fma(P.beta, I, ck);
        if (v < r.best) {
            r.second = r.best;
            r.best = v;
            r.arg = k;
        } else if (v < r.second) {
            r.second = v;
        }
    }
    return warp_best(r);
}

// The bracket of one trajectory point by one thread, controls in index order (the
// serial scan warp_best reproduces: smallest value, lowest index among equal ones, the
// second smallest of the multiset) — for small control sets (the Dubins car's 3), where a
// warp per trajectory would leave most lanes idle.
template <typename Ts, int DIM>
__device__ __forceinline__ BestPair thread_bracket(const DevProblem<double, Ts> &P,
                                                   const Ts *__restrict__ V, const int64_t o[3],
                                                   const int64_t vn[3], const double g[3],
                                                   const double x[3], double cs,
                                                   const double (*uctl)[4], double ct, double st) {
    const int64_t zero[3] = {0, 0, 0};
    const double base = (P.cost == HJ_COST_KRUZKOV) ? P.kcost : P.h * cost_state(P, x);
    BestPair r{INFINITY, INFINITY, -1};
    for (int k = 0; k < P.K; ++k) {
        double f[3];
        dynamics_u(P, x, cs, uctl[k], f, ct, st);
        double foot[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) foot[d] = fma(P.hdx[d], f[d], g[d]);
        const double I = interp<double, Ts, DIM>(V, o, vn, P.n, P.periodic, zero, foot, P.v_out);
        const double ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(P.h * P.lr, uctl[k][3], base);
        const double v = fma(P.beta, I, ck);
        if (v < r.best) {
            r.second = r.best;
            r.best = v;
            r.arg = k;
        } else if (v < r.second) {
            r.second = v;
        }
    }
    return r;
}

// The trajectory's own arithmetic — the state x(y_s), the speed c(y_s), f(y_s, a) and the
// step y_{s+1} = y_s + h f / dx (R8) — in the plain left-to-right order of the recursion,
// every product and sum rounded on its own (no contraction).  The positions, and so every
// nearest-node and box decision, are then a function of the argmins alone: any IEEE fp64
// evaluation of the same recursion that takes the same controls lands on the same bits
// (only the Dubins car's cos/sin may differ by an ulp between libraries).  The brackets,
// which only pick the control, keep their fused form.
__device__ __forceinline__ double rn_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double rn_mul(double a, double b) { return __dmul_rn(a, b); }

// multilinear interpolation of a whole-grid node field at index point g: corner weights
// prod_d (w_d or 1 - w_d) accumulated corner by corner (corner bit d = upper node on d)
template <typename Ts, int DIM>
__device__ double traj_interp(const DevProblem<double, Ts> &P, const Ts *__restrict__ F,
                              const double g[3], double outside) {
    int64_t i0[3] = {0, 0, 0}, i1[3] = {0, 0, 0};
    double w[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        double x = g[d];
        const int64_t n = P.n[d];
        if (P.periodic[d]) {
            const double f = floor(x);
            w[d] = __dsub_rn(x, f);
            int64_t c = (int64_t)f % n;
            if (c < 0) c += n;
            i0[d] = c;
            i1[d] = (c + 1) % n;
        } else {
            const double hi = (double)(n - 1);
            if (x < -(double)BOX_EPS || x > hi + (double)BOX_EPS) return outside;
            x = x < 0.0 ? 0.0 : (x > hi ? hi : x);
            int64_t c = (int64_t)floor(x);
            if (c > n - 2) c = n - 2;
            w[d] = __dsub_rn(x, (double)c);
            i0[d] = c;
            i1[d] = c + 1;
        }
    }
    double acc = 0.0;
#pragma unroll
    for (int corner = 0; corner < (1 << DIM); ++corner) {
        int64_t idx = 0;
        double wt = 1.0;
#pragma unroll
        for (int d = DIM - 1; d >= 0; --d) idx = idx * P.n[d] + ((corner >> d) & 1 ? i1[d] : i0[d]);
#pragma unroll
        for (int d = 0; d < DIM; ++d)
            wt = rn_mul(wt, (corner >> d) & 1 ? w[d] : __dsub_rn(1.0, w[d]));
        acc = rn_add(acc, rn_mul(wt, (double)F[idx]));
    }
    return acc;
}

// f(x, a) with the control's components u (§2 line 36; DESIGN.md configs)
template <typename Ts>
__device__ __forceinline__ void traj_dynamics(const DevProblem<double, Ts> &P, const double x[3],
                                              double c, const double *u, double f[3], double ct,
                                              double st) {
    f[0] = f[1] = f[2] = 0.0;
    if (P.dyn == HJ_DYN_AFFINE) {
        for (int d = 0; d < P.dim; ++d) {
            double s = rn_add(rn_mul(c, u[d]), P.b[d]);
            for (int e = 0; e < P.dim; ++e) s = rn_add(s, rn_mul(P.A[3 * d + e], x[e]));
            f[d] = s;
        }
    } else if (P.dyn == HJ_DYN_DUBINS) {
        f[0] = rn_mul(P.dub_v, ct);
        f[1] = rn_mul(P.dub_v, st);
        f[2] = rn_mul(P.dub_w, u[0]);
    } else {
        f[0] = x[1];
        f[1] = rn_add(__dsub_rn(rn_mul(rn_mul(P.vdp_mu, __dsub_rn(1.0, rn_mul(x[0], x[0]))), x[1]),
                                x[0]),
                      u[0]);
    }
}

// THREAD: one thread per coarse node (small control sets), else one warp per node.
template <typename Ts, int DIM, bool THREAD = false>
__global__ void __launch_bounds__(256)
    k_label_warp(const DevProblem<double, Ts> P, const Ts *__restrict__ V,
                 const int8_t *__restrict__ piece, int64_t N, int64_t n_max, int32_t *label,
                 double *margin_out, double *geo_out, int32_t *steps_out,
                 const Ts *__restrict__ Vexit, double exit_tol) {
    const int64_t o[3] = {0, 0, 0};
    const int64_t vn[3] = {P.n[0], P.n[1], P.n[2]};
    const int lane = THREAD ? 0 : (int)(threadIdx.x & 31);
    const int64_t warps = THREAD ? (int64_t)gridDim.x * blockDim.x
                                 : (int64_t)gridDim.x * (blockDim.x >> 5);
    __shared__ double uctl[HJ_MAX_CONTROLS][4];    // a_k (3 components), |a_k|^2
    for (int i = threadIdx.x; i < P.K * 4; i += blockDim.x)
        uctl[i >> 2][i & 3] = (i & 3) == 3 ? P.csq[i >> 2] : P.ctrl[i >> 2][i & 3];
    __syncthreads();
    const bool fast2 = DIM == 2 && !P.periodic[0] && !P.periodic[1] && P.dyn == HJ_DYN_AFFINE &&
                       P.n[0] * P.n[1] < ((int64_t)1 << 31);
    for (int64_t t = THREAD ? blockIdx.x * (int64_t)blockDim.x + threadIdx.x
                            : blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5);
         t < N; t += warps) {
        double g[3] = {(double)(t % P.n[0]), (double)((t / P.n[0]) % P.n[1]),
                       (double)(t / (P.n[0] * P.n[1]))};
        double mm = INFINITY, mg = INFINITY;
        int lab = -1;
        int64_t s = 0;
        for (;; ++s) {
            int64_t r[3] = {0, 0, 0};
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
                double q = g[d] + 0.5;
                double fl = floor(q);
                double dist = q - fl;
                dist = fmin(dist, 1.0 - dist);
                mg = fmin(mg, dist);
                int64_t c = (int64_t)fl;
                if (P.periodic[d]) {
                    c %= P.n[d];
                    if (c < 0) c += P.n[d];
                } else if (c > P.n[d] - 1) {
                    c = P.n[d] - 1;
                }
                r[d] = c;
            }
            int pc = piece[r[0] + P.n[0] * (r[1] + P.n[1] * r[2])];
            if (pc >= 0) {
                lab = pc;
                break;
            }
            if (s >= n_max) break;
            double x[3] = {0, 0, 0};
#pragma unroll
            for (int d = 0; d < DIM; ++d) x[d] = rn_add(P.lo[d], rn_mul(g[d], P.dx[d]));
            double cs = 1.0;
            if (P.speed && P.dyn == HJ_DYN_AFFINE) cs = traj_interp<Ts, DIM>(P, P.speed, g, 1.0);
            double ct = 0.0, st = 0.0;
            if (P.dyn == HJ_DYN_DUBINS) {
                ct = cos(x[2]);
                st = sin(x[2]);
            }
            BestPair bp;
            if constexpr (THREAD)
                bp = thread_bracket<Ts, DIM>(P, V, o, vn, g, x, cs, uctl, ct, st);
            else
                bp = fast2 ? lane_bracket_2d<Ts>(P, V, g, x, cs, lane, uctl)
                           : lane_bracket<Ts, DIM>(P, V, o, vn, g, lane, uctl, ct, st);
            const int a = bp.arg;
            if (a < 0) break;        // every bracket NaN (a NaN in V): no control, unlabelled
            mm = fmin(mm, bp.second - bp.best);
            double f[3];
            traj_dynamics(P, x, cs, uctl[a], f, ct, st);
            bool out = false;
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
                g[d] = rn_add(g[d], __ddiv_rn(rn_mul(P.h, f[d]), P.dx[d]));
                if (P.periodic[d]) {
                    const double n = (double)P.n[d];
                    g[d] = __dsub_rn(g[d], rn_mul(n, floor(__ddiv_rn(g[d], n))));
                } else {
                    double hi = (double)(P.n[d] - 1);
                    mg = fmin(mg, fmin(fabs(g[d]), fabs(hi - g[d])));
                    if (g[d] < 0.0 || g[d] > hi) out = true;
                }
            }
            if (out) {
                ++s;
                break;
            }
        }
        // exit set (R9b): an unlabelled node whose value needs no target
        if (lab < 0 && Vexit && (double)V[t] >= (double)Vexit[t] - exit_tol) lab = -2;
        if (lane == 0) {
            label[t] = lab;
            if (margin_out) margin_out[t] = mm;
            if (geo_out) geo_out[t] = mg;
            if (steps_out) steps_out[t] = (int32_t)s;
        }
    }
}

struct ProlongArgs {
    int dim;
    int64_t nc[3], nf[3], R[3];
    int periodic[3];
    int64_t band;
    uint64_t all;       // every set: the m pieces (and the exit set when enabled)
    uint64_t pieces;    // the m pieces' sets
    uint64_t exit_bit;  // bit of the exit set (label -2), 0 when disabled
};

// the sets a coarse label stands for: piece k -> set k; -1 -> every piece's set (R9);
// -2 -> the exit set only (R9b)
__device__ __forceinline__ uint64_t label_bits(const ProlongArgs &A, int32_t l) {
    if (l >= 0) return l < 64 ? (1ull << l) : 0ull;
    return l == -2 ? A.exit_bit : A.pieces;
}

__device__ __forceinline__ int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    return (a % b != 0 && ((a < 0) != (b < 0))) ? q - 1 : q;
}

// MASK = false: coarse trajectory labels (k -> bit k, -1 -> every bit, R9);
// MASK = true: coarse membership bit masks (the RA sets)
template <bool MASK>
__global__ void k_prolong(const ProlongArgs A, const void *__restrict__ coarse,
                          const int8_t *__restrict__ fine_piece, int64_t Nf, uint64_t *mask) {
    const int32_t *lab = (const int32_t *)coarse;
    const uint64_t *cmask = (const uint64_t *)coarse;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < Nf;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t ii[3] = {t % A.nf[0], (t / A.nf[0]) % A.nf[1], t / (A.nf[0] * A.nf[1])};
        int64_t lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int d = 0; d < A.dim; ++d) {
            int64_t reach = A.R[d] + A.band;
            lo[d] = -floordiv(-(ii[d] - reach), A.R[d]);  // ceil
            hi[d] = floordiv(ii[d] + reach, A.R[d]);
        }
        uint64_t bits = 0;
        for (int64_t I2 = lo[2]; I2 <= hi[2]; ++I2)
            for (int64_t I1 = lo[1]; I1 <= hi[1]; ++I1)
                for (int64_t I0 = lo[0]; I0 <= hi[0]; ++I0) {
                    int64_t I[3] = {I0, I1, I2}, J[3] = {0, 0, 0};
                    bool ok = true;
                    for (int d = 0; d < A.dim; ++d) {
                        int64_t c = I[d];
                        if (A.periodic[d]) {
                            c %= A.nc[d];
                            if (c < 0) c += A.nc[d];
                        } else if (c < 0 || c > A.nc[d] - 1) {
                            ok = false;
                        }
                        J[d] = c;
                    }
                    if (!ok) continue;
                    const int64_t cidx = J[0] + A.nc[0] * (J[1] + A.nc[1] * J[2]);
                    if (MASK)
                        bits |= cmask[cidx];
                    else
                        bits |= label_bits(A, lab[cidx]);
                }
        int8_t p = fine_piece[t];
        if (p >= 0 && p < 64) bits |= 1ull << p;
        mask[t] = bits & A.all;
    }
}

// The same prolongation, one fine x-row (i1, i2) per CTA iteration: the y/z coarse
// intervals are uniform over the row, so the CTA first ORs, for every coarse x index J0,
// the coarse bits over the row's y-z box (ryz[J0], shared memory), then each fine node
// ORs ryz over its x interval — ~(cnt_y cnt_z + cnt_x) loads per node instead of
// cnt_x cnt_y cnt_z (125 for the Dubins grid).  OR is order-free: bit-identical.
__device__ __forceinline__ bool prolong_wrap(const ProlongArgs &A, int d, int64_t &c) {
    if (A.periodic[d]) {
        c %= A.nc[d];
        if (c < 0) c += A.nc[d];
        return true;
    }
    return c >= 0 && c <= A.nc[d] - 1;
}

template <bool MASK>
__global__ void __launch_bounds__(256)
    k_prolong_rows(const ProlongArgs A, const void *__restrict__ coarse,
                   const int8_t *__restrict__ fine_piece, uint64_t *mask) {
    extern __shared__ uint64_t ryz[];                 // [nc0]
    const int32_t *lab = (const int32_t *)coarse;
    const uint64_t *cmask = (const uint64_t *)coarse;
    const int64_t rows = A.nf[1] * A.nf[2];
    for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
        const int64_t i12[2] = {row % A.nf[1], row / A.nf[1]};
        int64_t lo[2] = {0, 0}, hi[2] = {0, 0};
        for (int e = 0; e < 2; ++e) {
            const int d = e + 1;
            if (d >= A.dim) continue;
            const int64_t reach = A.R[d] + A.band;
            lo[e] = -floordiv(-(i12[e] - reach), A.R[d]);   // ceil
            hi[e] = floordiv(i12[e] + reach, A.R[d]);
        }
        __syncthreads();                                   // the previous row's reads
        for (int64_t J0 = threadIdx.x; J0 < A.nc[0]; J0 += blockDim.x) {
            uint64_t b = 0;
            for (int64_t I2 = lo[1]; I2 <= hi[1]; ++I2) {
                int64_t J2 = I2;
                if (A.dim > 2 && !prolong_wrap(A, 2, J2)) continue;
                for (int64_t I1 = lo[0]; I1 <= hi[0]; ++I1) {
                    int64_t J1 = I1;
                    if (A.dim > 1 && !prolong_wrap(A, 1, J1)) continue;
                    const int64_t cidx = J0 + A.nc[0] * (J1 + A.nc[1] * J2);
                    if (MASK)
                        b |= cmask[cidx];
                    else
                        b |= label_bits(A, lab[cidx]);
                }
            }
            ryz[J0] = b;
        }
        __syncthreads();
        const int64_t reach0 = A.R[0] + A.band;
        for (int64_t i0 = threadIdx.x; i0 < A.nf[0]; i0 += blockDim.x) {
            const int64_t lo0 = -floordiv(-(i0 - reach0), A.R[0]), hi0 = floordiv(i0 + reach0, A.R[0]);
            uint64_t bits = 0;
            for (int64_t I0 = lo0; I0 <= hi0; ++I0) {
                int64_t J0 = I0;
                if (!prolong_wrap(A, 0, J0)) continue;
                bits |= ryz[J0];
            }
            const int64_t t = i0 + A.nf[0] * (i12[0] + A.nf[1] * i12[1]);
            const int8_t p = fine_piece[t];
            if (p >= 0 && p < 64) bits |= 1ull << p;
            mask[t] = bits & A.all;
        }
    }
}

// ISA step 2 (R9) from labels or masks of the coarse grid cg onto the nested fine grid fg
hj_status prolong_launch(const hj_grid &cg, const hj_grid &fg, const int32_t ratio[3],
                         int32_t band, int32_t m, const void *coarse, bool is_mask,
                         const int8_t *fine_piece, uint64_t *fine_mask, cudaStream_t s,
                         bool exit_set) {
    ProlongArgs A;
    memset(&A, 0, sizeof(A));
    A.dim = fg.dim;
    for (int d = 0; d < 3; ++d) {
        A.nc[d] = d < cg.dim ? cg.n[d] : 1;
        A.nf[d] = d < fg.dim ? fg.n[d] : 1;
        A.R[d] = d < fg.dim ? ratio[d] : 1;
        A.periodic[d] = d < fg.dim ? fg.periodic[d] : 0;
    }
    A.band = band;
    const int sets = m + (exit_set ? 1 : 0);
    A.all = sets >= 64 ? ~0ull : ((1ull << sets) - 1ull);
    A.exit_bit = exit_set ? (1ull << m) : 0ull;
    A.pieces = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
    const int64_t Nf = grid_nodes(fg);
    if (A.nc[0] <= 4096) {                  // row scheme (ryz fits in shared memory)
        const int64_t rows = A.nf[1] * A.nf[2];
        const int rb = (int)std::min<int64_t>(rows, 148 * 8);
        const size_t sm = (size_t)A.nc[0] * sizeof(uint64_t);
        if (is_mask)
            k_prolong_rows<true><<<rb, 256, sm, s>>>(A, coarse, fine_piece, fine_mask);
        else
            k_prolong_rows<false><<<rb, 256, sm, s>>>(A, coarse, fine_piece, fine_mask);
        HJ_CUDA(cudaGetLastError());
        return HJ_OK;
    }
    const int blocks = (int)std::min<int64_t>((Nf + 255) / 256, 148 * 16);
    if (is_mask)
        k_prolong<true><<<blocks, 256, 0, s>>>(A, coarse, fine_piece, Nf, fine_mask);
    else
        k_prolong<false><<<blocks, 256, 0, s>>>(A, coarse, fine_piece, Nf, fine_mask);
    HJ_CUDA(cudaGetLastError());
    return HJ_OK;
}

template <typename Ts>
static hj_status feedback_impl(const hj_grid &g, const hj_problem &p, const hj_fields &f,
                               const Ts *V, int32_t *astar, double *margin, cudaStream_t s) {
    auto P = make_dev_problem<double, Ts>(g, p, f);
    int64_t N = grid_nodes(g);
    int blocks = (int)std::min<int64_t>((N + 127) / 128, 148 * 16);
    if (g.dim == 2)
        k_feedback<Ts, 2><<<blocks, 128, 0, s>>>(P, V, f.piece, N, astar, margin);
    else
        k_feedback<Ts, 3><<<blocks, 128, 0, s>>>(P, V, f.piece, N, astar, margin);
    HJ_CUDA(cudaGetLastError());
    return HJ_OK;
}

template <typename Ts>
static hj_status label_impl(const hj_grid &g, const hj_problem &p, const hj_fields &f,
                            const Ts *V, const Ts *Vexit, double exit_tol, int64_t n_max,
                            int32_t *label, double *margin, double *geo, int32_t *steps,
                            cudaStream_t s) {
    auto P = make_dev_problem<double, Ts>(g, p, f);
    int64_t N = grid_nodes(g);
    // one warp per coarse node; one thread per node for small control sets
    const bool thread = p.n_controls <= HJ_LABEL_THREAD_MAX_K;
    int blocks = thread ? (int)std::min<int64_t>((N + 255) / 256, 148 * 8)
                        : (int)std::min<int64_t>((N + 7) / 8, 148 * 64);
    if (g.dim == 2) {
        if (thread)
            k_label_warp<Ts, 2, true><<<blocks, 256, 0, s>>>(P, V, f.piece, N, n_max, label,
                                                             margin, geo, steps, Vexit, exit_tol);
        else
            k_label_warp<Ts, 2><<<blocks, 256, 0, s>>>(P, V, f.piece, N, n_max, label, margin,
                                                       geo, steps, Vexit, exit_tol);
    } else {
        if (thread)
            k_label_warp<Ts, 3, true><<<blocks, 256, 0, s>>>(P, V, f.piece, N, n_max, label,
                                                             margin, geo, steps, Vexit, exit_tol);
        else
            k_label_warp<Ts, 3><<<blocks, 256, 0, s>>>(P, V, f.piece, N, n_max, label, margin,
                                                       geo, steps, Vexit, exit_tol);
    }
    HJ_CUDA(cudaGetLastError());
    return HJ_OK;
}

}  // namespace hj

using namespace hj;

extern "C" {

hj_status hj_coarse_feedback(const hj_grid *grid, const hj_problem *prob,
                             const hj_fields *fields, int32_t dtype, const void *V,
                             int32_t *astar, double *margin, void *stream) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(grid)) != HJ_OK) return st;
    if ((st = validate_problem(grid, prob)) != HJ_OK) return st;
    HJ_CHECK(fields && fields->piece, "fields.piece is required");
    HJ_CHECK(V && astar, "V / astar is NULL");
    HJ_CHECK(dtype == HJ_F32 || dtype == HJ_F64, "dtype must be HJ_F32 or HJ_F64");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == HJ_F64)
        return feedback_impl<double>(*grid, *prob, *fields, (const double *)V, astar, margin, s);
    return feedback_impl<float>(*grid, *prob, *fields, (const float *)V, astar, margin, s);
}

hj_status hj_label_subdomains(const hj_grid *cg, const hj_problem *cp, const hj_fields *cf,
                              int32_t dtype, const void *Vc, const void *Vexit, double exit_tol,
                              int64_t n_max, const hj_grid *fg, const int32_t ratio[3],
                              int32_t band, int32_t m, const int8_t *fine_piece, int32_t *label,
                              double *margin, double *geo, int32_t *steps, uint64_t *fine_mask,
                              void *stream) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(cg)) != HJ_OK) return st;
    if ((st = validate_grid(fg)) != HJ_OK) return st;
    if ((st = validate_problem(cg, cp)) != HJ_OK) return st;
    HJ_CHECK(cf && cf->piece, "coarse fields.piece is required");
    HJ_CHECK(Vc && label && fine_mask && fine_piece && ratio, "NULL argument");
    HJ_CHECK(m >= 1 && m + (Vexit ? 1 : 0) <= HJ_MAX_SUBDOMAINS,
             "m must be in [1, %d] (one set fewer with the exit set)", HJ_MAX_SUBDOMAINS);
    HJ_CHECK(band >= 0 && n_max >= 0, "band and n_max must be >= 0");
    HJ_CHECK(exit_tol >= 0, "exit_tol must be >= 0");
    HJ_CHECK(cg->dim == fg->dim, "coarse and fine grids differ in dim");
    HJ_CHECK(dtype == HJ_F32 || dtype == HJ_F64, "dtype must be HJ_F32 or HJ_F64");
    for (int d = 0; d < cg->dim; ++d) {
        HJ_CHECK(ratio[d] >= 1, "ratio[%d] must be >= 1", d);
        HJ_CHECK(cg->periodic[d] == fg->periodic[d], "periodicity differs on axis %d", d);
        if (fg->periodic[d])
            HJ_CHECK(fg->n[d] == ratio[d] * cg->n[d], "periodic axis %d not nested", d);
        else
            HJ_CHECK(fg->n[d] - 1 == ratio[d] * (cg->n[d] - 1), "axis %d not nested", d);
    }
    cudaStream_t s = (cudaStream_t)stream;
    st = dtype == HJ_F64 ? label_impl<double>(*cg, *cp, *cf, (const double *)Vc,
                                              (const double *)Vexit, exit_tol, n_max, label,
                                              margin, geo, steps, s)
                         : label_impl<float>(*cg, *cp, *cf, (const float *)Vc,
                                             (const float *)Vexit, exit_tol, n_max, label,
                                             margin, geo, steps, s);
    if (st != HJ_OK) return st;
    return prolong_launch(*cg, *fg, ratio, band, m, label, false, fine_piece, fine_mask, s,
                          Vexit != nullptr);
}

}  // extern "C"
