// hj_common.cuh — device-side problem description and the per-point building
// blocks of the semi-Lagrangian operator (PAPER.md eq. (Tdef)).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>

#include "../../include/hj.h"

namespace hj {

// views one sweep launch (or one cooperative launch) iterates together: the cooperative
// kernel keeps one view per lane of a warp (stopping decisions, residual reads); larger
// sets of sub-domains are solved in groups of this size, one group after the other
#define HJ_GROUP_VIEWS 32

// Problem constants as the kernels see them: everything prescaled on the host
// (in fp64, then rounded to Tc) so the inner loop only multiplies and adds.
//   Tc = arithmetic type, Ts = storage type of the node fields (speed, g, V).
template <typename Tc, typename Ts>
struct DevProblem {
    int dim, dyn, cost, K;
    int64_t n[3];
    int periodic[3];
    Tc lo[3], dx[3], hdx[3];   // hdx = h / dx  (foot offset per unit of f, index units)
    Tc h, beta, kcost;         // beta = 1/(1+lambda h); kcost = 1 - beta (Kruzkov)
    Tc A[9], b[3];
    Tc dub_v, dub_w, vdp_mu;
    Tc l0, lq, ln, lr;
    Tc v_out;
    int monotone;              // V^0 is a supersolution: iterates decrease (see hj_host.cuh)
    Tc ctrl[HJ_MAX_CONTROLS][3];
    Tc csq[HJ_MAX_CONTROLS];   // |a_k|^2
    const Ts *speed;           // node field or nullptr
    const Ts *g;               // node field or nullptr
};

// A rectangular window ("view") of the global grid holding one iterate pair:
// the whole grid for hj_solve, the bounding box of S_k for a sub-domain solve.
template <typename T>
struct SweepView {
    int64_t o[3];      // origin (global node index)
    int64_t vn[3];     // extent
    int64_t nodes;     // vn0*vn1*vn2
    T *V[2];           // iterate buffers (dense over the view)
    const int8_t *cls; // >= 0 target piece, -1 interior, -2 ghost (outside S_k)
    double *res;       // res[n] = ||V^{n+1} - V^n||_inf (atomicMax on the bits)
    unsigned long long *work;  // interior nodes evaluated (summed over sweeps)
};

template <typename T>
__device__ __forceinline__ T lerp(T a, T b, T w) {
    return fma(w, b - a, a);
}

// Value of node (i,j,k) (global indices, already inside the global box) read
// from a view; nodes outside the view are ghosts (R10) and read v_out.
template <typename Ts, int DIM>
__device__ __forceinline__ Ts view_fetch(const Ts *__restrict__ V, const int64_t o[3],
                                         const int64_t vn[3], int64_t i, int64_t j, int64_t k,
                                         Ts v_out) {
    int64_t li = i - o[0], lj = j - o[1], lk = (DIM == 3) ? (k - o[2]) : 0;
    if (li < 0 || li >= vn[0] || lj < 0 || lj >= vn[1]) return v_out;
    if (DIM == 3 && (lk < 0 || lk >= vn[2])) return v_out;
    return V[li + vn[0] * (lj + vn[1] * lk)];
}

// Reading R3: feet more than BOX_EPS cells outside the closed box read v_out;
// feet within BOX_EPS are clamped onto it (offsets that are zero in exact
// arithmetic, e.g. cos(pi/2), then decide the same way in fp32 and fp64).
constexpr double BOX_EPS = 1e-6;

// Multilinear interpolation I[V] at the point base + delta (index space, R4).
// The foot is kept as (integer node, small offset) so that the cell weights keep
// full precision on large grids in fp32; v_out outside the box (R3).
template <typename Tc, typename Ts, int DIM>
__device__ __forceinline__ Tc interp(const Ts *__restrict__ V, const int64_t o[3],
                                     const int64_t vn[3], const int64_t n[3],
                                     const int periodic[3], const int64_t base[3],
                                     const Tc delta[3], Tc v_out) {
    int64_t c0[3] = {0, 0, 0}, c1[3] = {0, 0, 0};
    Tc w[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) {
        Tc x = delta[d];
        int64_t nd = n[d], b = base[d];
        if (periodic[d]) {
            Tc f = floor(x);
            w[d] = x - f;
            int64_t c = (b + (int64_t)f) % nd;
            if (c < 0) c += nd;
            c0[d] = c;
            c1[d] = (c + 1 == nd) ? 0 : c + 1;
        } else {
            const Tc lo = -(Tc)b, hi = (Tc)(nd - 1 - b);
            if (!(x >= lo - (Tc)BOX_EPS && x <= hi + (Tc)BOX_EPS)) return v_out;
            x = x < lo ? lo : (x > hi ? hi : x);
            Tc f = floor(x);
            int64_t c = b + (int64_t)f;
            Tc ww = x - f;
            if (c > nd - 2) {   // only when x == hi exactly: the last cell at weight 1
                c = nd - 2;
                ww = Tc(1);
            }
            w[d] = ww;
            c0[d] = c;
            c1[d] = c + 1;
        }
    }
    const Ts vo = (Ts)v_out;
    if (DIM == 2) {
        Tc a = lerp<Tc>((Tc)view_fetch<Ts, 2>(V, o, vn, c0[0], c0[1], 0, vo),
                        (Tc)view_fetch<Ts, 2>(V, o, vn, c1[0], c0[1], 0, vo), w[0]);
        Tc b = lerp<Tc>((Tc)view_fetch<Ts, 2>(V, o, vn, c0[0], c1[1], 0, vo),
                        (Tc)view_fetch<Ts, 2>(V, o, vn, c1[0], c1[1], 0, vo), w[0]);
        return lerp<Tc>(a, b, w[1]);
    } else {
        Tc r[2];
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            int64_t kk = s ? c1[2] : c0[2];
            Tc a = lerp<Tc>((Tc)view_fetch<Ts, 3>(V, o, vn, c0[0], c0[1], kk, vo),
                            (Tc)view_fetch<Ts, 3>(V, o, vn, c1[0], c0[1], kk, vo), w[0]);
            Tc b = lerp<Tc>((Tc)view_fetch<Ts, 3>(V, o, vn, c0[0], c1[1], kk, vo),
                            (Tc)view_fetch<Ts, 3>(V, o, vn, c1[0], c1[1], kk, vo), w[0]);
            r[s] = lerp<Tc>(a, b, w[1]);
        }
        return lerp<Tc>(r[0], r[1], w[2]);
    }
}

// f(x, a_k) for the three dynamics families (hj.h HJ_DYN_*).
template <typename Tc, typename Ts>
__device__ __forceinline__ void dynamics(const DevProblem<Tc, Ts> &P, const Tc x[3], Tc c, int k,
                                         Tc f[3]) {
    if (P.dyn == HJ_DYN_AFFINE) {
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (d >= P.dim) {
                f[d] = Tc(0);
                continue;
            }
            Tc s = fma(c, P.ctrl[k][d], P.b[d]);
            for (int e = 0; e < P.dim; ++e) s = fma(P.A[3 * d + e], x[e], s);
            f[d] = s;
        }
    } else if (P.dyn == HJ_DYN_DUBINS) {
        f[0] = P.dub_v * cos(x[2]);
        f[1] = P.dub_v * sin(x[2]);
        f[2] = P.dub_w * P.ctrl[k][0];
    } else {
        f[0] = x[1];
        f[1] = fma(P.vdp_mu * (Tc(1) - x[0] * x[0]), x[1], P.ctrl[k][0] - x[0]);
        f[2] = Tc(0);
    }
}

// State part of the running cost: l0 + lq |x|^2 + ln |x| (non-periodic axes).
template <typename Tc, typename Ts>
__device__ __forceinline__ Tc cost_state(const DevProblem<Tc, Ts> &P, const Tc x[3]) {
    Tc x2 = Tc(0);
    for (int d = 0; d < P.dim; ++d)
        if (!P.periodic[d]) x2 = fma(x[d], x[d], x2);
    return P.l0 + P.lq * x2 + P.ln * sqrt(x2);
}

// cost_state of a 2-D non-periodic problem (the same operations, no loop over the axes)
template <typename Tc, typename Ts>
__device__ __forceinline__ Tc cost_state_2d(const DevProblem<Tc, Ts> &P, Tc x0, Tc x1) {
    Tc x2 = fma(x0, x0, Tc(0));
    x2 = fma(x1, x1, x2);
    return P.l0 + P.lq * x2 + P.ln * sqrt(x2);
}

__device__ __forceinline__ void atomic_max_nonneg(double *addr, double v) {
    atomicMax(reinterpret_cast<unsigned long long *>(addr),
              (unsigned long long)__double_as_longlong(v));
}

}  // namespace hj
