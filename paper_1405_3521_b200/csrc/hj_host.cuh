// hj_host.cuh — host-side helpers shared by the entry points: error reporting,
// validation, workspace carving and the fp64 -> Tc prescaling of the problem.
#pragma once

#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include <cmath>
#include <string>

#include "hj_common.cuh"

namespace hj {

void set_error(const char *fmt, ...);
void clear_error();

#define HJ_CUDA(call)                                                                    \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            ::hj::set_error("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_),     \
                            __FILE__, __LINE__);                                         \
            return HJ_ERR_CUDA;                                                          \
        }                                                                                \
    } while (0)

#define HJ_CHECK(cond, ...)               \
    do {                                  \
        if (!(cond)) {                    \
            ::hj::set_error(__VA_ARGS__); \
            return HJ_ERR_INVALID;        \
        }                                 \
    } while (0)

inline int64_t grid_nodes(const hj_grid &g) {
    int64_t s = 1;
    for (int d = 0; d < g.dim; ++d) s *= g.n[d];
    return s;
}

inline double grid_spacing(const hj_grid &g, int d) {
    double span = g.hi[d] - g.lo[d];
    return g.periodic[d] ? span / (double)g.n[d] : span / (double)(g.n[d] - 1);
}

hj_status validate_grid(const hj_grid *g);
hj_status validate_problem(const hj_grid *g, const hj_problem *p);

// V^0 (g on targets, v_out elsewhere) is a supersolution, T(V^0) <= V^0, when v_out
// bounds every bracket: Kruzkov with v_out >= 1 (brackets are beta I + 1 - beta <= 1
// for I <= 1), or discounted with lambda > 0 and v_out >= h l_max / (1 - beta) over
// the box.  T is monotone, so then V^{n+1} = T(V^n) <= V^n for every n in exact
// arithmetic and the sweep may clamp V^{n+1} = min(T(V^n), V^n): the identity on
// exact iterates, it removes upward rounding noise (no fp32 limit cycles; the
// stopping rule is always reached).  Off when a g field is given (g <= v_out unknown).
inline bool supersolution_start(const hj_grid &g, const hj_problem &p, const hj_fields &f) {
    if (f.g) return false;
    if (p.cost == HJ_COST_KRUZKOV) return p.v_out >= 1.0 && p.lambda > 0;
    if (p.lambda <= 0) return false;
    double x2 = 0, amax2 = 0;
    for (int d = 0; d < g.dim; ++d)
        if (!g.periodic[d]) {
            double m = std::max(std::fabs(g.lo[d]), std::fabs(g.hi[d]));
            x2 += m * m;
        }
    for (int k = 0; k < p.n_controls; ++k) {
        double a2 = 0;
        for (int c = 0; c < 3; ++c) a2 += p.controls[k][c] * p.controls[k][c];
        amax2 = std::max(amax2, a2);
    }
    double lmax = std::fabs(p.l0) + std::fabs(p.lq) * x2 + std::fabs(p.ln) * std::sqrt(x2) +
                  std::fabs(p.lr) * amax2;
    if (p.l0 < 0 || p.lq < 0 || p.ln < 0 || p.lr < 0) return false;
    double beta = 1.0 / (1.0 + p.lambda * p.h);
    return p.v_out >= p.h * lmax / (1.0 - beta) * (1.0 - 1e-12);
}

template <typename Tc, typename Ts>
DevProblem<Tc, Ts> make_dev_problem(const hj_grid &g, const hj_problem &p, const hj_fields &f) {
    DevProblem<Tc, Ts> P;
    memset(&P, 0, sizeof(P));
    P.dim = g.dim;
    P.dyn = p.dynamics;
    P.cost = p.cost;
    P.K = p.n_controls;
    for (int d = 0; d < 3; ++d) {
        P.n[d] = d < g.dim ? g.n[d] : 1;
        P.periodic[d] = d < g.dim ? g.periodic[d] : 0;
        double dx = d < g.dim ? grid_spacing(g, d) : 1.0;
        P.lo[d] = (Tc)(d < g.dim ? g.lo[d] : 0.0);
        P.dx[d] = (Tc)dx;
        P.hdx[d] = (Tc)(p.h / dx);
        P.b[d] = (Tc)p.b[d];
        for (int e = 0; e < 3; ++e) P.A[3 * d + e] = (Tc)p.A[d][e];
    }
    double beta = 1.0 / (1.0 + p.lambda * p.h);
    P.h = (Tc)p.h;
    P.beta = (Tc)beta;
    P.kcost = (Tc)(1.0 - beta);
    P.dub_v = (Tc)p.dubins_v;
    P.dub_w = (Tc)p.dubins_w;
    P.vdp_mu = (Tc)p.vdp_mu;
    P.l0 = (Tc)p.l0;
    P.lq = (Tc)p.lq;
    P.ln = (Tc)p.ln;
    P.lr = (Tc)p.lr;
    P.v_out = (Tc)p.v_out;
    for (int k = 0; k < p.n_controls; ++k) {
        double s = 0;
        for (int c = 0; c < 3; ++c) {
            P.ctrl[k][c] = (Tc)p.controls[k][c];
            s += p.controls[k][c] * p.controls[k][c];
        }
        P.csq[k] = (Tc)s;
    }
    P.speed = (const Ts *)f.speed;
    P.g = (const Ts *)f.g;
    P.monotone = supersolution_start(g, p, f) ? 1 : 0;
    return P;
}

// Bump allocator over a caller-owned device workspace (256-byte aligned).
struct Carver {
    char *base;
    size_t cap, off;
    Carver(void *b, size_t c) : base((char *)b), cap(c), off(0) {}
    static size_t align(size_t x) { return (x + 255) & ~(size_t)255; }
    void *take(size_t bytes) {
        void *p = base ? base + off : nullptr;
        off += align(bytes);
        return p;
    }
    bool ok() const { return off <= cap; }
};

// Thread-local pinned host staging buffer (residual read-back).
double *pinned_scratch(size_t count);

// ISA step 2 (R9): coarse labels (is_mask = false) or membership masks onto the fine grid
hj_status prolong_launch(const hj_grid &cg, const hj_grid &fg, const int32_t ratio[3],
                         int32_t band, int32_t m, const void *coarse, bool is_mask,
                         const int8_t *fine_piece, uint64_t *fine_mask, cudaStream_t s,
                         bool exit_set = false);

}  // namespace hj
