// hj_sweep.cuh — Jacobi sweeps V^{n+1} = T(V^n) over a set of views
// (PAPER.md eq. (SL), operator (Tdef) line 238-245, readings R1-R4).
//
// A view is the whole grid (hj_solve) or the bounding box of one sub-domain
// (hj_solve_partitioned); all views of a call iterate in the same launches and stop
// independently.  Exact short-cuts, all bit-identical to the plain Jacobi sweep:
//   * stopped views: work of a view that met the stopping rule (res[n-1] < tol) is
//     skipped, so the stop is exactly the first n with ||V^{n+1}-V^n|| < tol (R6);
//   * quiet tiles / nodes: T(V) on a tile depends only on V over its dependency
//     neighbourhood; if nothing there changed (bitwise) in sweep n-1 then
//     V^{n+1} = V^n on the tile, which the other buffer already holds — device work
//     lists (one-sweep kernels), per-tile flags (blocked kernel) or node-level dirty
//     masks (cooperative kernel) visit only what can change.
//
// Kernels: k_sweep_local2d_coop (hj_sweep_coop.cuh; the whole iteration
// in one cooperative launch: local, field-within-one-cell and Dubins classes),
// k_sweep_local2d_tb (hj_sweep_tb.cuh; 8 sweeps per launch), k_sweep_local2d_x2 /
// k_sweep_local2d (one sweep per launch, local class), k_sweep_field2d (any 2-D affine /
// Van der Pol), k_sweep_dubins (3-D Dubins), k_sweep_generic (anything).
#pragma once

#include <algorithm>
#include <type_traits>
#include <vector>

#include "hj_host.cuh"

namespace hj {

// ---------------------------------------------------------------------------
// shared pieces
// ---------------------------------------------------------------------------
template <typename T>
struct TileView {          // per-view tiling, filled by sweep_prepare
    int32_t nt[3];         // tiles per axis
    int64_t tiles;         // nt0*nt1*nt2
    int64_t tile_base;     // first global tile index of this view
    uint8_t *chg;          // [2][tiles] changed flags (parity of the sweep / block)
    int32_t rerun;         // temporally blocked kernel: sub-sweeps of the stop re-run
};

// Device work list of the tiles a sweep (or a block of sweeps) must visit: a tile is
// listed for sweep n+1 iff a tile within the dependency radius changed in sweep n
// (the exact "quiet tile" rule, see above), so launches are persistent grids that
// walk the list instead of one CTA per tile.  Two parities of (items, mark bitmap)
// and a ring of three counters: launch n reads count[n%3], appends to count[(n+1)%3]
// and zeroes count[(n+2)%3]; every visited tile clears its own mark bit.
struct WorkList {
    int32_t *items[2];
    int32_t *count;       // [4]: the ring [0..2] and the live-tile count [3]
    uint32_t *mark[2];    // bitmaps over global tile ids
    int32_t *live;        // tiles holding at least one interior node (the only ones that
                          // can ever change: targets keep g, ghosts keep v_out)
};

template <typename T>
struct SweepGroup {        // device-resident description of one launch
    SweepView<T> v[HJ_GROUP_VIEWS];
    TileView<T> t[HJ_GROUP_VIEWS];
    WorkList wl;
    int total_tiles;
    int dense;             // 1: visit every tile every sweep, one CTA per tile, no list
                           //    (discounted problems change everywhere until they stop)
    int n_views;
    int tile_dim[3];       // TX, TY, TZ (nodes)
    int radius[3];         // dependency radius in tiles
    int halo[3];           // foot bound in cells, ceil(max |delta_d|) (fast-path test)
    int periodic[3];       // periodic axes (views span them fully)
};

// Locate (view, tile) of this CTA; false if the view has stopped.
template <typename T>
__device__ __forceinline__ int find_view(const SweepGroup<T> *__restrict__ G, int64_t b) {
    int v = 0;
    while (v + 1 < G->n_views && G->t[v + 1].tile_base <= b) ++v;
    return v;
}

// the same for a warp-uniform tile id: lane v tests view v+1 (one load and a ballot)
template <typename T>
__device__ __forceinline__ int find_view_warp(const SweepGroup<T> *__restrict__ G, int64_t b) {
    const int lane = threadIdx.x & 31;
    return __popc(__ballot_sync(0xffffffffu,
                                lane + 1 < G->n_views && G->t[lane + 1].tile_base <= b));
}

// (tile ids are int: SweepGroup::total_tiles — 32-bit divisions)
template <typename T>
__device__ __forceinline__ void tile_coords(const TileView<T> &tv, int64_t tile, int tc[3]) {
    const int t = (int)tile, n0 = tv.nt[0], n1 = tv.nt[1];
    const int q = t / n0;
    tc[0] = t - q * n0;
    tc[1] = q % n1;
    tc[2] = q / n1;
}

__device__ __forceinline__ void wl_push(const WorkList &wl, int64_t nit, int gid) {
    const uint32_t bit = 1u << (gid & 31);
    uint32_t *w = &wl.mark[nit & 1][gid >> 5];
    // already listed (the common case when the active set is dense): no atomic
    if (*(volatile uint32_t *)w & bit) return;
    const uint32_t old = atomicOr(w, bit);
    if (!(old & bit)) wl.items[nit & 1][atomicAdd(&wl.count[nit % 3], 1)] = gid;
}

// list every tile within (rx, ry, rz) tiles of tile tc of view v for launch nit
template <typename T>
__device__ __forceinline__ void push_neighbours(const SweepGroup<T> *__restrict__ G, int v,
                                                const int tc[3], int rx, int ry, int rz,
                                                int64_t nit) {
    const TileView<T> &tv = G->t[v];
    const int wx = 2 * rx + 1, wy = 2 * ry + 1, wz = 2 * rz + 1;
    const int count = wx * wy * wz;
    for (int e = threadIdx.x; e < count; e += blockDim.x) {
        int c[3] = {tc[0] + e % wx - rx, tc[1] + (e / wx) % wy - ry, tc[2] + e / (wx * wy) - rz};
        bool ok = true;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            if (c[d] >= 0 && c[d] < tv.nt[d]) continue;
            if (G->periodic[d])
                c[d] = ((c[d] % tv.nt[d]) + tv.nt[d]) % tv.nt[d];
            else
                ok = false;
        }
        if (ok)
            wl_push(G->wl, nit,
                    (int)(tv.tile_base + c[0] + tv.nt[0] * ((int64_t)c[1] + (int64_t)tv.nt[1] * c[2])));
    }
}

// Persistent walk over the work list of sweep `it` (one-sweep kernels).  Inside the
// body: v, vw, tv, tile, tc[3]; the body sets changed_ (block-uniform).
#define HJ_LIST_BEGIN(G, it, tol)                                                          \
    const WorkList &wl_ = (G)->wl;                                                         \
    const bool dense_ = (G)->dense != 0;                                                   \
    const int cnt_ = *(volatile const int *)&wl_.count[dense_ ? 3 : (it) % 3];              \
    for (int idx_ = blockIdx.x; idx_ < cnt_; idx_ += gridDim.x) {                          \
        const int gid_ = dense_ ? wl_.live[idx_] : wl_.items[(it) & 1][idx_];              \
        const int v = find_view_warp(G, gid_);                                             \
        if (!dense_ && threadIdx.x == 0)                                                   \
            atomicAnd(&wl_.mark[(it) & 1][gid_ >> 5], ~(1u << (gid_ & 31)));                \
        const SweepView<T> &vw = (G)->v[v];                                                \
        if ((it) > 0 && *(volatile const double *)&vw.res[(it) - 1] < (tol)) continue;     \
        const TileView<T> &tv = (G)->t[v];                                                 \
        const int64_t tile = gid_ - tv.tile_base;                                          \
        int tc[3];                                                                         \
        tile_coords(tv, tile, tc);                                                         \
        int changed_ = 0;

#define HJ_LIST_END(G, it)                                                                 \
        if (changed_ && !dense_)                                                           \
            push_neighbours(G, v, tc, (G)->radius[0], (G)->radius[1], (G)->radius[2],     \
                            (it) + 1);                                                     \
        __syncthreads();                                                                   \
    }                                                                                      \
    if (!dense_ && blockIdx.x == 0 && threadIdx.x == 0) wl_.count[((it) + 2) % 3] = 0;

template <typename T>
__device__ __forceinline__ int tile_finish(const SweepGroup<T> *__restrict__ G, int v,
                                           int64_t tile, int64_t it, T rmax, int changed,
                                           int evaluated) {
    evaluated = __reduce_add_sync(0xffffffffu, evaluated);
    if ((threadIdx.x & 31) == 0 && evaluated)
        atomicAdd(G->v[v].work, (unsigned long long)evaluated);
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        T other = __shfl_down_sync(0xffffffffu, rmax, s);
        rmax = other > rmax ? other : rmax;
    }
    __shared__ T red[32];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rmax;
    int any = __syncthreads_or(changed);
    if (threadIdx.x == 0) {
        T m = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = red[w] > m ? red[w] : m;
        if (m > T(0)) atomic_max_nonneg(&G->v[v].res[it], (double)m);
    }
    return any;
}

template <typename T>
__device__ __forceinline__ bool same_bits(T a, T b);
template <>
__device__ __forceinline__ bool same_bits<float>(float a, float b) {
    return __float_as_uint(a) == __float_as_uint(b);
}
template <>
__device__ __forceinline__ bool same_bits<double>(double a, double b) {
    return __double_as_longlong(a) == __double_as_longlong(b);
}

// generic per-node bracket-min (global-memory corners)
template <typename T, int DIM>
__device__ __forceinline__ T node_update_generic(const DevProblem<T, T> &P, const T *__restrict__ Vi,
                                                 const int64_t o[3], const int64_t vn[3],
                                                 const int64_t gi[3], int64_t gidx) {
    T x[3] = {0, 0, 0};
#pragma unroll
    for (int d = 0; d < DIM; ++d) x[d] = fma((T)gi[d], P.dx[d], P.lo[d]);
    T cs = (P.speed && P.dyn == HJ_DYN_AFFINE) ? P.speed[gidx] : T(1);
    T base = (P.cost == HJ_COST_KRUZKOV) ? P.kcost : P.h * cost_state(P, x);
    T best = (T)INFINITY;
    for (int k = 0; k < P.K; ++k) {
        T f[3];
        dynamics(P, x, cs, k, f);
        T delta[3] = {0, 0, 0};
#pragma unroll
        for (int d = 0; d < DIM; ++d) delta[d] = P.hdx[d] * f[d];
        T I = interp<T, T, DIM>(Vi, o, vn, P.n, P.periodic, gi, delta, P.v_out);
        T ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(P.h * P.lr, P.csq[k], base);
        T cand = fma(P.beta, I, ck);
        best = cand < best ? cand : best;
    }
    return best;
}

// ---------------------------------------------------------------------------
// generic tiled kernel: tile 32 x 8 x 1, one node per thread
// ---------------------------------------------------------------------------
template <typename T, int DIM>
__global__ void __launch_bounds__(256)
    k_sweep_generic(const DevProblem<T, T> P, const SweepGroup<T> *__restrict__ G, int64_t it,
                    double tol) {
    HJ_LIST_BEGIN(G, it, tol)
    const int64_t o[3] = {vw.o[0], vw.o[1], vw.o[2]};
    const int64_t vn[3] = {vw.vn[0], vw.vn[1], vw.vn[2]};
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int64_t li = (int64_t)tc[0] * 32 + (threadIdx.x & 31);
    const int64_t lj = (int64_t)tc[1] * 8 + (threadIdx.x >> 5);
    const int64_t lk = tc[2];
    T rmax = T(0);
    int changed = 0, evaluated = 0;
    if (li < vn[0] && lj < vn[1] && lk < vn[2]) {
        const int64_t t = li + vn[0] * (lj + vn[1] * lk);
        const int64_t gi[3] = {li + o[0], lj + o[1], lk + o[2]};
        const int64_t gidx = gi[0] + P.n[0] * (gi[1] + P.n[1] * gi[2]);
        const int8_t c = vw.cls[t];
        const T vin = Vi[t];
        T vnew;
        if (c == -2)
            vnew = P.v_out;
        else if (c >= 0)
            vnew = P.g ? P.g[gidx] : T(0);
        else {
            vnew = node_update_generic<T, DIM>(P, Vi, o, vn, gi, gidx);
            if (P.monotone) vnew = fmin(vnew, vin);
            evaluated = 1;
        }
        Vo[t] = vnew;
        rmax = vnew > vin ? vnew - vin : vin - vnew;
        changed = !same_bits(vnew, vin);
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// local 2-D kernel: tile 32 x 32, 256 threads, 4 rows per thread
// ---------------------------------------------------------------------------
template <typename T>
struct LocalCtrl {
    // quadrant q: bit0 -> foot x offset <= 0, bit1 -> foot y offset <= 0.
    // ax = |u_x| h/dx, ay = |u_y| h/dy of the controls of that quadrant (padded to KQ
    // by repeating a control: repeats do not change a min); ck = per-control cost.
    T ax[4][32], ay[4][32], ck[4][32];
    // box of each quadrant's weights, [0, xmax] x [0, ymax] (exact pruning bound of
    // the temporally blocked kernel) and whether pruning is valid
    T xmax[4], ymax[4];
    int prune_ok;         // every ck >= 0
};

template <typename T, int KQ, bool PC>
__global__ void __launch_bounds__(256, 2)
    k_sweep_local2d(const DevProblem<T, T> P, const LocalCtrl<T> C,
                    const SweepGroup<T> *__restrict__ G, int64_t it, double tol) {
    constexpr int TX = 32, TY = 32, RY = 4, SW = TX + 2;
    __shared__ T s[(TY + 2) * SW];
    HJ_LIST_BEGIN(G, it, tol)
    const int64_t vn0 = vw.vn[0], vn1 = vw.vn[1];
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int64_t x0 = (int64_t)tc[0] * TX, y0 = (int64_t)tc[1] * TY;
    const T v_out = P.v_out;
    // stage the tile + 1-node halo (outside the view: ghost = v_out)
    for (int e = threadIdx.x; e < (TY + 2) * SW; e += 256) {
        const int r = e / SW, c = e - r * SW;
        const int64_t li = x0 + c - 1, lj = y0 + r - 1;
        T val = v_out;
        if (li >= 0 && lj >= 0 && li < vn0 && lj < vn1) val = Vi[li + vn0 * lj];
        s[e] = val;
    }
    __syncthreads();
    const int lx = threadIdx.x & 31, ly0 = (threadIdx.x >> 5) * RY;
    const int64_t o0 = vw.o[0], o1 = vw.o[1];
    const int64_t n0 = P.n[0], n1 = P.n[1];
    T rmax = T(0);
    int changed = 0, evaluated = 0;
#pragma unroll 1
    for (int r = 0; r < RY; ++r) {
        const int ly = ly0 + r;
        const int64_t li = x0 + lx, lj = y0 + ly;
        if (li >= vn0 || lj >= vn1) continue;
        const int64_t t = li + vn0 * lj;
        const int64_t gi[3] = {li + o0, lj + o1, 0};
        const int64_t gidx = gi[0] + n0 * gi[1];
        const int8_t c = vw.cls[t];
        const T *sp = s + (ly + 1) * SW + (lx + 1);
        const T V00 = sp[0];
        T vnew;
        if (c == -2) {
            vnew = v_out;
        } else if (c >= 0) {
            vnew = P.g ? P.g[gidx] : T(0);
        } else {
            const T Vm0 = sp[-1], Vp0 = sp[1], V0m = sp[-SW], V0p = sp[SW];
            const T Vmm = sp[-SW - 1], Vpm = sp[-SW + 1], Vmp = sp[SW - 1], Vpp = sp[SW + 1];
            const T sc = P.speed ? P.speed[gidx] : T(1);
            T base;
            if (P.cost == HJ_COST_KRUZKOV) {
                base = P.kcost;
            } else {
                const T x[3] = {fma((T)gi[0], P.dx[0], P.lo[0]), fma((T)gi[1], P.dx[1], P.lo[1]),
                                T(0)};
                base = P.h * cost_state(P, x);
            }
            const T C0 = fma(P.beta, V00, base);
            const T bs = P.beta * sc, bss = bs * sc;
            const bool lo_x = gi[0] == 0, hi_x = gi[0] == n0 - 1;
            const bool lo_y = gi[1] == 0, hi_y = gi[1] == n1 - 1;
            T best = (T)INFINITY;
            if (!(lo_x | hi_x | lo_y | hi_y)) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const T Vx = (q & 1) ? Vm0 : Vp0;
                    const T Vy = (q & 2) ? V0m : V0p;
                    const T Vxy = (q == 0) ? Vpp : (q == 1) ? Vmp : (q == 2) ? Vpm : Vmm;
                    const T Dx = Vx - V00, Dy = Vy - V00, Dxy = (Vxy - Vx) - Dy;
                    const T A1 = bs * Dx, A2 = bs * Dy, A3 = bss * Dxy;
#pragma unroll
                    for (int k = 0; k < KQ; ++k) {
                        const T ax = C.ax[q][k], ay = C.ay[q][k];
                        const T u = fma(ax, A1, PC ? C0 + C.ck[q][k] : C0);
                        const T cand = fma(ay, fma(ax, A3, A2), u);
                        best = fmin(best, cand);
                    }
                }
            } else {
                // box-edge node (R3): a foot moving out by more than BOX_EPS cells reads
                // v_out; within BOX_EPS it is clamped onto the edge (weight 0)
                const T c_out = fma(P.beta, v_out, base);
                const T eps = (T)BOX_EPS;
#pragma unroll 1
                for (int q = 0; q < 4; ++q) {
                    const bool ex = (q & 1) ? lo_x : hi_x, ey = (q & 2) ? lo_y : hi_y;
                    const T Vx = (q & 1) ? Vm0 : Vp0;
                    const T Vy = (q & 2) ? V0m : V0p;
                    const T Vxy = (q == 0) ? Vpp : (q == 1) ? Vmp : (q == 2) ? Vpm : Vmm;
                    const T Dx = P.beta * (Vx - V00), Dy = P.beta * (Vy - V00);
                    const T Dxy = P.beta * ((Vxy - Vx) - (Vy - V00));
#pragma unroll 1
                    for (int k = 0; k < KQ; ++k) {
                        T wx = sc * C.ax[q][k], wy = sc * C.ay[q][k];
                        const T ck = PC ? C.ck[q][k] : T(0);
                        const bool out = (ex && wx > eps) || (ey && wy > eps);
                        if (ex) wx = T(0);
                        if (ey) wy = T(0);
                        const T in = fma(wy, fma(wx, Dxy, Dy), fma(wx, Dx, C0)) + ck;
                        best = fmin(best, out ? c_out + ck : in);
                    }
                }
            }
            vnew = best;
            ++evaluated;
        }
        if (c == -1 && P.monotone) vnew = fmin(vnew, V00);
        Vo[t] = vnew;
        const T dv = vnew > V00 ? vnew - V00 : V00 - vnew;
        rmax = dv > rmax ? dv : rmax;
        changed |= !same_bits(vnew, V00);
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// local 2-D kernel, fp32, packed: two nodes per FFMA2 (sm_100a fma.rn.f32x2).
// Same tile, staging and per-node arithmetic as k_sweep_local2d<float> — each
// node's candidate is fma(ay, fma(ax, A3, A2), fma(ax, A1, C0)) in the same
// rounding order, so the result is bit-identical — but the rows (ly, ly+1) of a
// thread share every instruction: lane .x = row ly, lane .y = row ly+1, the
// control constants broadcast from uniform registers.  Per node x control update:
// 1.5 FFMA2 + 0.5 FMNMX3 issue slots (vs 3 FFMA + 0.5 FMNMX3 scalar).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ void sincos_t(float a, float *s, float *c) { sincosf(a, s, c); }
__device__ __forceinline__ void sincos_t(double a, double *s, double *c) { sincos(a, s, c); }

template <bool PC>
__device__ __forceinline__ float local_edge_node(const DevProblem<float, float> &P,
                                                 const LocalCtrl<float> &C, int KQ,
                                                 const float *sp, float C0, float sc,
                                                 float base, bool lo_x, bool hi_x, bool lo_y,
                                                 bool hi_y) {
    constexpr int SW = 34;
    const float V00 = sp[0], Vm0 = sp[-1], Vp0 = sp[1], V0m = sp[-SW], V0p = sp[SW];
    const float Vmm = sp[-SW - 1], Vpm = sp[-SW + 1], Vmp = sp[SW - 1], Vpp = sp[SW + 1];
    const float c_out = fmaf(P.beta, P.v_out, base);
    const float eps = (float)BOX_EPS;
    float best = INFINITY;
#pragma unroll 1
    for (int q = 0; q < 4; ++q) {
        const bool ex = (q & 1) ? lo_x : hi_x, ey = (q & 2) ? lo_y : hi_y;
        const float Vx = (q & 1) ? Vm0 : Vp0;
        const float Vy = (q & 2) ? V0m : V0p;
        const float Vxy = (q == 0) ? Vpp : (q == 1) ? Vmp : (q == 2) ? Vpm : Vmm;
        const float Dx = P.beta * (Vx - V00), Dy = P.beta * (Vy - V00);
        const float Dxy = P.beta * ((Vxy - Vx) - (Vy - V00));
#pragma unroll 1
        for (int k = 0; k < KQ; ++k) {
            float wx = sc * C.ax[q][k], wy = sc * C.ay[q][k];
            const float ck = PC ? C.ck[q][k] : 0.f;
            const bool out = (ex && wx > eps) || (ey && wy > eps);
            if (ex) wx = 0.f;
            if (ey) wy = 0.f;
            const float in = fmaf(wy, fmaf(wx, Dxy, Dy), fmaf(wx, Dx, C0)) + ck;
            best = fminf(best, out ? c_out + ck : in);
        }
    }
    return best;
}

template <int KQ, bool PC>
__global__ void __launch_bounds__(256, 2)
    k_sweep_local2d_x2(const DevProblem<float, float> P, const LocalCtrl<float> C,
                       const SweepGroup<float> *__restrict__ G, int64_t it, double tol) {
    using T = float;
    constexpr int TX = 32, TY = 32, RY = 4, SW = TX + 2;
    __shared__ float s[(TY + 2) * SW];
    HJ_LIST_BEGIN(G, it, tol)
    const int64_t vn0 = vw.vn[0], vn1 = vw.vn[1];
    const float *__restrict__ Vi = vw.V[it & 1];
    float *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int64_t x0 = (int64_t)tc[0] * TX, y0 = (int64_t)tc[1] * TY;
    const float v_out = P.v_out;
    for (int e = threadIdx.x; e < (TY + 2) * SW; e += 256) {
        const int r = e / SW, c = e - r * SW;
        const int64_t li = x0 + c - 1, lj = y0 + r - 1;
        float val = v_out;
        if (li >= 0 && lj >= 0 && li < vn0 && lj < vn1) val = Vi[li + vn0 * lj];
        s[e] = val;
    }
    __syncthreads();
    const int lx = threadIdx.x & 31, ly0 = (threadIdx.x >> 5) * RY;
    const int64_t o0 = vw.o[0], o1 = vw.o[1];
    const int64_t n0 = P.n[0], n1 = P.n[1];
    float rmax = 0.f;
    int changed = 0, evaluated = 0;
#pragma unroll 1
    for (int r = 0; r < RY; r += 2) {
        // per node of the pair: class, staged neighbourhood, speed, base cost
        bool valid[2], fast[2], edge[2][4];
        int8_t c[2];
        int64_t t[2], gidx[2];
        float C0[2], A1[4][2], A2[4][2], A3[4][2], sc[2], base[2];
        const float *sp[2];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const int ly = ly0 + r + p;
            const int64_t li = x0 + lx, lj = y0 + ly;
            valid[p] = li < vn0 && lj < vn1;
            t[p] = li + vn0 * lj;
            const int64_t gi0 = li + o0, gi1 = lj + o1;
            gidx[p] = gi0 + n0 * gi1;
            c[p] = valid[p] ? vw.cls[t[p]] : (int8_t)-2;
            sp[p] = s + (ly + 1) * SW + (lx + 1);
            edge[p][0] = gi0 == 0;
            edge[p][1] = gi0 == n0 - 1;
            edge[p][2] = gi1 == 0;
            edge[p][3] = gi1 == n1 - 1;
            const bool interior = valid[p] && c[p] == -1;
            fast[p] = interior && !(edge[p][0] | edge[p][1] | edge[p][2] | edge[p][3]);
            sc[p] = (interior && P.speed) ? P.speed[gidx[p]] : 1.f;
            if (P.cost == HJ_COST_KRUZKOV) {
                base[p] = P.kcost;
            } else {
                const float x[3] = {fmaf((float)gi0, P.dx[0], P.lo[0]),
                                    fmaf((float)gi1, P.dx[1], P.lo[1]), 0.f};
                base[p] = P.h * cost_state(P, x);
            }
            const float *q0 = sp[p];
            const float V00 = q0[0];
            C0[p] = fmaf(P.beta, V00, base[p]);
            const float bs = P.beta * sc[p], bss = bs * sc[p];
            const float Vm0 = q0[-1], Vp0 = q0[1], V0m = q0[-SW], V0p = q0[SW];
            const float Vmm = q0[-SW - 1], Vpm = q0[-SW + 1], Vmp = q0[SW - 1], Vpp = q0[SW + 1];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float Vx = (q & 1) ? Vm0 : Vp0;
                const float Vy = (q & 2) ? V0m : V0p;
                const float Vxy = (q == 0) ? Vpp : (q == 1) ? Vmp : (q == 2) ? Vpm : Vmm;
                const float Dx = Vx - V00, Dy = Vy - V00, Dxy = (Vxy - Vx) - Dy;
                A1[q][p] = bs * Dx;
                A2[q][p] = bs * Dy;
                A3[q][p] = bss * Dxy;
            }
        }
        float best[2] = {INFINITY, INFINITY};
        if (fast[0] || fast[1]) {
            const float2 c0 = f2(C0[0], C0[1]);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const float2 a1 = f2(A1[q][0], A1[q][1]), a2 = f2(A2[q][0], A2[q][1]);
                const float2 a3 = f2(A3[q][0], A3[q][1]);
#pragma unroll
                for (int k = 0; k < KQ; k += 2) {
                    const float ax0 = C.ax[q][k], ay0 = C.ay[q][k];
                    const float ax1 = C.ax[q][k + 1], ay1 = C.ay[q][k + 1];
                    const float2 u0 = __ffma2_rn(
                        f2(ax0, ax0), a1, PC ? __fadd2_rn(c0, f2(C.ck[q][k], C.ck[q][k])) : c0);
                    const float2 u1 = __ffma2_rn(
                        f2(ax1, ax1), a1,
                        PC ? __fadd2_rn(c0, f2(C.ck[q][k + 1], C.ck[q][k + 1])) : c0);
                    const float2 w0 = __ffma2_rn(f2(ax0, ax0), a3, a2);
                    const float2 w1 = __ffma2_rn(f2(ax1, ax1), a3, a2);
                    const float2 k0 = __ffma2_rn(f2(ay0, ay0), w0, u0);
                    const float2 k1 = __ffma2_rn(f2(ay1, ay1), w1, u1);
                    best[0] = fminf(best[0], fminf(k0.x, k1.x));
                    best[1] = fminf(best[1], fminf(k0.y, k1.y));
                }
            }
        }
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            if (!valid[p]) continue;
            const float V00 = sp[p][0];
            float vnew;
            if (c[p] == -2) {
                vnew = v_out;
            } else if (c[p] >= 0) {
                vnew = P.g ? P.g[gidx[p]] : 0.f;
            } else {
                vnew = fast[p] ? best[p]
                               : local_edge_node<PC>(P, C, KQ, sp[p], C0[p], sc[p], base[p],
                                                     edge[p][0], edge[p][1], edge[p][2],
                                                     edge[p][3]);
                if (P.monotone) vnew = fminf(vnew, V00);
                ++evaluated;
            }
            Vo[t[p]] = vnew;
            const float dv = vnew > V00 ? vnew - V00 : V00 - vnew;
            rmax = dv > rmax ? dv : rmax;
            changed |= !same_bits(vnew, V00);
        }
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// lean 2-D kernel for feet of the form  delta_k(x) = D(x) + S(x) * U_k  (index
// units), which covers every 2-D family of hj.h:
//   affine      D = (h/dx) (A x + b),             S = (h/dx) c(x),   U_k = u_k
//   Van der Pol D = (h/dx) (x1, mu(1-x0^2)x1-x0), S = (0, h/dx1),    U_k = (0, a_k)
// Any foot distance.  Corners are read through L1 (__ldg: the buffer read is never
// written in the same launch).  Tiles whose whole footprint (tile +- the host's
// foot bound) lies inside the view take the fast path: no box/view tests, 32-bit
// corner offsets; the other tiles use the full R3/R10 rule of interp().
// Tile 32 x 8, one node per thread.
// ---------------------------------------------------------------------------
// floor(d) and d - floor(d) without the conversion (XU) pipe, |d| < 2^22:
// t = RM(d + 1.5 2^23) (rounded toward -inf: the sum's ulp is 1, so t = 1.5 2^23 +
// floor(d) exactly) carries floor(d) in its mantissa.  Same values as floor() /
// d - floor(d) (fp64 keeps floor(): the double pipes are not the limit there).
__device__ __forceinline__ int floor_split(float d, float &w) {
    const float t = __fadd_rd(d, 12582912.0f);
    const float fl = __fsub_rn(t, 12582912.0f);
    w = d - fl;
    return __float_as_int(t) - 0x4B400000;
}
__device__ __forceinline__ int floor_split(double d, double &w) {
    const double fl = floor(d);
    w = d - fl;
    return (int)fl;
}

template <typename T, int DYN, bool KRUZ, int RY>
__global__ void __launch_bounds__(256, 4)
    k_sweep_field2d(const DevProblem<T, T> P, const SweepGroup<T> *__restrict__ G, int64_t it,
                    double tol) {
    HJ_LIST_BEGIN(G, it, tol)
    const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1];
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    // tile 32 x 8RY: lane -> column, warp -> rows warp, warp + 8, ...
    constexpr int TY = 8 * RY;
    const int li = tc[0] * 32 + (threadIdx.x & 31);
    // tile-uniform fast-path test: every corner of every foot inside the view
    const int hx = G->halo[0], hy = G->halo[1];
    const bool fast = tc[0] * 32 - hx >= 0 && tc[0] * 32 + 31 + hx + 1 <= vn0 - 1 &&
                      tc[1] * TY - hy >= 0 && tc[1] * TY + TY - 1 + hy + 1 <= vn1 - 1;
    T rmax = T(0);
    int changed = 0, evaluated = 0;
#pragma unroll 1
    for (int rr = 0; rr < RY; ++rr) {
    const int lj = tc[1] * TY + (threadIdx.x >> 5) + 8 * rr;
    if (li < vn0 && lj < vn1) {
        const int64_t t = li + (int64_t)vn0 * lj;
        const int64_t gi[3] = {li + vw.o[0], lj + vw.o[1], 0};
        const int64_t gidx = gi[0] + P.n[0] * gi[1];
        const int8_t c = vw.cls[t];
        const T vin = Vi[t];
        T vnew;
        if (c == -2) {
            vnew = P.v_out;
        } else if (c >= 0) {
            vnew = P.g ? P.g[gidx] : T(0);
        } else {
            const T x0 = fma((T)gi[0], P.dx[0], P.lo[0]), x1 = fma((T)gi[1], P.dx[1], P.lo[1]);
            T D0, D1, S0, S1;
            if (DYN == HJ_DYN_AFFINE) {
                const T cs = P.speed ? P.speed[gidx] : T(1);
                D0 = P.hdx[0] * fma(P.A[0], x0, fma(P.A[1], x1, P.b[0]));
                D1 = P.hdx[1] * fma(P.A[3], x0, fma(P.A[4], x1, P.b[1]));
                S0 = P.hdx[0] * cs;
                S1 = P.hdx[1] * cs;
            } else {   // Van der Pol
                D0 = P.hdx[0] * x1;
                D1 = P.hdx[1] * fma(P.vdp_mu * (T(1) - x0 * x0), x1, -x0);
                S0 = T(0);
                S1 = P.hdx[1];
            }
            T base;
            if (KRUZ) {
                base = P.kcost;
            } else {
                const T x[3] = {x0, x1, T(0)};
                base = P.h * cost_state(P, x);
            }
            const T hlr = P.h * P.lr;
            T best = (T)INFINITY;
            if (fast) {
                const T *__restrict__ Vn = Vi + t;
#pragma unroll 4
                for (int k = 0; k < P.K; ++k) {
                    // affine: u_k = controls[k][0..1]; Van der Pol: a_k = controls[k][0]
                    const T d0 = DYN == HJ_DYN_AFFINE ? fma(S0, P.ctrl[k][0], D0) : D0;
                    const T d1 = fma(S1, P.ctrl[k][DYN == HJ_DYN_AFFINE ? 1 : 0], D1);
                    T w0, w1;
                    const int i0 = floor_split(d0, w0), i1 = floor_split(d1, w1);
                    const T *__restrict__ p = Vn + (i0 + vn0 * i1);
                    const T a00 = __ldg(p), a10 = __ldg(p + 1);
                    const T a01 = __ldg(p + vn0), a11 = __ldg(p + vn0 + 1);
                    const T I = lerp<T>(lerp<T>(a00, a10, w0), lerp<T>(a01, a11, w0), w1);
                    const T ck = KRUZ ? base : fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(P.beta, I, ck));
                }
            } else {
                const int64_t o[3] = {vw.o[0], vw.o[1], 0};
                const int64_t vn[3] = {vn0, vn1, 1};
#pragma unroll 1
                for (int k = 0; k < P.K; ++k) {
                    const T delta[3] = {
                        DYN == HJ_DYN_AFFINE ? fma(S0, P.ctrl[k][0], D0) : D0,
                        fma(S1, P.ctrl[k][DYN == HJ_DYN_AFFINE ? 1 : 0], D1), T(0)};
                    const T I = interp<T, T, 2>(Vi, o, vn, P.n, P.periodic, gi, delta, P.v_out);
                    const T ck = KRUZ ? base : fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(P.beta, I, ck));
                }
            }
            vnew = best;
            if (P.monotone) vnew = fmin(vnew, vin);
            ++evaluated;
        }
        Vo[t] = vnew;
        const T dv = vnew > vin ? vnew - vin : vin - vnew;
        rmax = dv > rmax ? dv : rmax;
        changed |= !same_bits(vnew, vin);
    }
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// k_sweep_field2d for the affine problems whose controls all move the foot by the same
// amount along axis 0 (u_k = (u0, u1_k), no speed field: config 5's f = (x2, a - x1/2)).
// Then d0 = D0 + S0 u0, its cell i0 and weight w0 are the node's, not the control's, and
// the bilinear interpolant of control k is  lerp(X(i1_k), X(i1_k + 1), w1_k)  with
// X(j) = lerp(V(i0, j), V(i0 + 1, j), w0) the x-interpolated column at the node's foot
// abscissa — exactly the two inner lerps k_sweep_field2d forms.  With the controls sorted
// by u1 (host; the min over controls is order-free) the rows the controls touch are
// [i1_first, i1_last + 1]: the node forms that column once (two loads and one lerp per
// row, into its own column of shared memory — lane = bank, conflict-free) and then each
// control costs one floor, two shared loads and the y-lerp instead of four gathers and
// three lerps.  Every value is the one k_sweep_field2d forms: bit-identical iterates
// (asserted in the parity suite).  Tiles whose footprint leaves the view take
// k_sweep_field2d's general path.
// ---------------------------------------------------------------------------
template <typename T>
struct ColCtrl {
    T u0;                              // the shared axis-0 control component
    T u1[HJ_MAX_CONTROLS];             // axis-1 components, ascending
    T csq[HJ_MAX_CONTROLS];            // |a_k|^2 in the same order
    int rows;                          // column rows per node the shared buffer holds
};

// KC > 0: the control count, known at compile time (the loop unrolls and the control
// table becomes immediate constant-bank operands); 0: any count
template <typename T, bool KRUZ, int RY, int KC>
__global__ void __launch_bounds__(256, 4)
    k_sweep_field2d_col(const DevProblem<T, T> P, const ColCtrl<T> C,
                        const SweepGroup<T> *__restrict__ G, int64_t it, double tol) {
    extern __shared__ __align__(16) unsigned char col_dyn[];
    T *__restrict__ const colbuf = reinterpret_cast<T *>(col_dyn);     // [rows][256]
    const int K = KC > 0 ? KC : P.K;
    HJ_LIST_BEGIN(G, it, tol)
    const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1];
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    constexpr int TY = 8 * RY;
    const int li = tc[0] * 32 + (threadIdx.x & 31);
    const int hx = G->halo[0], hy = G->halo[1];
    const bool fast = tc[0] * 32 - hx >= 0 && tc[0] * 32 + 31 + hx + 1 <= vn0 - 1 &&
                      tc[1] * TY - hy >= 0 && tc[1] * TY + TY - 1 + hy + 1 <= vn1 - 1;
    T rmax = T(0);
    int changed = 0, evaluated = 0;
#pragma unroll 1
    for (int rr = 0; rr < RY; ++rr) {
    const int lj = tc[1] * TY + (threadIdx.x >> 5) + 8 * rr;
    if (li < vn0 && lj < vn1) {
        const int64_t t = li + (int64_t)vn0 * lj;
        const int64_t gi[3] = {li + vw.o[0], lj + vw.o[1], 0};
        const int64_t gidx = gi[0] + P.n[0] * gi[1];
        const int8_t c = vw.cls[t];
        const T vin = Vi[t];
        T vnew;
        if (c == -2) {
            vnew = P.v_out;
        } else if (c >= 0) {
            vnew = P.g ? P.g[gidx] : T(0);
        } else {
            const T x0 = fma((T)gi[0], P.dx[0], P.lo[0]), x1 = fma((T)gi[1], P.dx[1], P.lo[1]);
            const T D0 = P.hdx[0] * fma(P.A[0], x0, fma(P.A[1], x1, P.b[0]));
            const T D1 = P.hdx[1] * fma(P.A[3], x0, fma(P.A[4], x1, P.b[1]));
            const T S0 = P.hdx[0], S1 = P.hdx[1];       // (no speed field: c = 1)
            T base;
            if (KRUZ) {
                base = P.kcost;
            } else {
                const T x[3] = {x0, x1, T(0)};
                base = P.h * cost_state(P, x);
            }
            const T hlr = P.h * P.lr;
            T best = (T)INFINITY;
            T w0, wl, wh;
            const int i0 = floor_split(fma(S0, C.u0, D0), w0);
            const int jlo = floor_split(fma(S1, C.u1[0], D1), wl);
            const int nrows = floor_split(fma(S1, C.u1[K - 1], D1), wh) + 2 - jlo;
            if (fast && nrows <= C.rows) {
                // the column X(jlo .. jlo + nrows - 1) at the foot abscissa, row r of this
                // thread at colbuf[256 r + threadIdx.x]
                const T *__restrict__ p = Vi + t + i0 + (int64_t)vn0 * jlo;
                T *__restrict__ xw = colbuf + threadIdx.x;
#pragma unroll 4
                for (int r = 0; r < nrows; ++r) {
                    xw[256 * r] = lerp<T>(__ldg(p), __ldg(p + 1), w0);
                    p += vn0;
                }
                const int xoff = (int)threadIdx.x - 256 * jlo;   // row j at colbuf[xoff + 256 j]
#pragma unroll
                for (int k = 0; k < (KC > 0 ? KC : 1); ++k) {
                    if (KC == 0) break;
                    T w1;
                    const int q = xoff + 256 * floor_split(fma(S1, C.u1[k], D1), w1);
                    const T I = lerp<T>(colbuf[q], colbuf[q + 256], w1);
                    const T ck = KRUZ ? base : fma(hlr, C.csq[k], base);
                    best = fmin(best, fma(P.beta, I, ck));
                }
                if (KC == 0) {
#pragma unroll 4
                    for (int k = 0; k < K; ++k) {
                        T w1;
                        const int q = xoff + 256 * floor_split(fma(S1, C.u1[k], D1), w1);
                        const T I = lerp<T>(colbuf[q], colbuf[q + 256], w1);
                        const T ck = KRUZ ? base : fma(hlr, C.csq[k], base);
                        best = fmin(best, fma(P.beta, I, ck));
                    }
                }
            } else {
                const int64_t o[3] = {vw.o[0], vw.o[1], 0};
                const int64_t vn[3] = {vn0, vn1, 1};
#pragma unroll 1
                for (int k = 0; k < P.K; ++k) {
                    const T delta[3] = {fma(S0, P.ctrl[k][0], D0), fma(S1, P.ctrl[k][1], D1),
                                        T(0)};
                    const T I = interp<T, T, 2>(Vi, o, vn, P.n, P.periodic, gi, delta, P.v_out);
                    const T ck = KRUZ ? base : fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(P.beta, I, ck));
                }
            }
            vnew = best;
            if (P.monotone) vnew = fmin(vnew, vin);
            ++evaluated;
        }
        Vo[t] = vnew;
        const T dv = vnew > vin ? vnew - vin : vin - vnew;
        rmax = dv > rmax ? dv : rmax;
        changed |= !same_bits(vnew, vin);
    }
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// k_sweep_field2d_col for lattice-aligned controls: the axis-1 foot offsets of consecutive
// (sorted) controls are exactly one cell apart, S1 (u1[k] - u1[0]) = k (config 5:
// h/dy = 16, a_k = -1 + k/16 — the control step moves the foot by one row), and the
// axis-1 drift does not depend on x1 (A[1][1] = 0).  Then every control of a node shares
// the foot's axis-1 weight w1 and control k reads rows j0 + k, j0 + k + 1 of the node's
// x-interpolated column X:
//     bracket_k = beta lerp(X(j0 + k), X(j0 + k + 1), w1) + c_k,
//     (j0, w1) = floor split of fma(S1, u1[0], D1),  X(j) = lerp(V(i0, j), V(i0 + 1, j), w0).
// One thread takes R = 8 nodes of one column (consecutive rows): they share j0 and w1,
// and node n's rows are node 0's shifted by n, so the thread streams the K + R rows once
// (two loads each) and feeds every row to the nodes whose window holds it — per node and
// control one y-lerp, the cost FMA, beta I + c and the min; per node and row one x-lerp.
// The arithmetic is k_sweep_field2d's (same lerps, same fma for c_k, order-free min) with
// control k's foot split as (j0 + k, w1) instead of splitting fma(S1, u1[k], D1): equal
// whenever that fma is exactly fma(S1, u1[0], D1) + k (config 5: every operand is a
// dyadic rational of few bits — bit-identical iterates, asserted), else equal up to the
// rounding of the foot.  A thread whose nodes straddle an axis-0 cell boundary (i0 not
// the same for its 8 rows) or whose tile's footprint leaves the view takes
// k_sweep_field2d's per-control loop.
// ---------------------------------------------------------------------------
template <typename T, bool KRUZ, int KC>
__global__ void __launch_bounds__(256, 2)
    k_sweep_field2d_lat(const DevProblem<T, T> P, const ColCtrl<T> C,
                        const SweepGroup<T> *__restrict__ G, int64_t it, double tol) {
    constexpr int R = 8;                         // nodes per thread (rows), tile 32 x 64
    constexpr int TY = 8 * R;
    HJ_LIST_BEGIN(G, it, tol)
    const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1];
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int li = tc[0] * 32 + lane;
    const int lj0 = tc[1] * TY + R * warp;
    const int hx = G->halo[0], hy = G->halo[1];
    const bool fast = tc[0] * 32 - hx >= 0 && tc[0] * 32 + 31 + hx + 1 <= vn0 - 1 &&
                      tc[1] * TY - hy >= 0 && tc[1] * TY + TY - 1 + hy + 1 <= vn1 - 1;
    T rmax = T(0);
    int changed = 0, evaluated = 0;
    if (li < vn0) {
        const int64_t gi0 = li + vw.o[0];
        const T x0 = fma((T)gi0, P.dx[0], P.lo[0]);
        const T S0 = P.hdx[0], S1 = P.hdx[1];
        const T hlr = P.h * P.lr;
        // (view nodes < 2^31: host-checked — 32-bit node offsets)
        const int tb = li + vn0 * lj0;
        const int8_t *__restrict__ cp = vw.cls + tb;
        const T *__restrict__ vp = Vi + tb;
        int8_t cls[R];
        T vin[R], w0[R], base[R], best[R];
        int i0[R];
        bool anyint = false, uni = true;
#pragma unroll
        for (int n = 0; n < R; ++n) {
            const int lj = lj0 + n;
            const bool in = lj < vn1;
            cls[n] = in ? cp[n * vn0] : (int8_t)-3;
            vin[n] = in ? vp[n * vn0] : T(0);
            anyint |= cls[n] == -1;
            const T x1 = fma((T)(lj + (int)vw.o[1]), P.dx[1], P.lo[1]);
            const T D0 = P.hdx[0] * fma(P.A[0], x0, fma(P.A[1], x1, P.b[0]));
            i0[n] = floor_split(fma(S0, C.u0, D0), w0[n]);
            uni &= i0[n] == i0[0];
            base[n] = KRUZ ? P.kcost : P.h * cost_state_2d(P, x0, x1);
            best[n] = (T)INFINITY;
        }
        if (anyint) {
            // D1 does not depend on x1 (A[1][1] = 0): the row of node 0 stands for all
            const T x1r = fma((T)(lj0 + vw.o[1]), P.dx[1], P.lo[1]);
            const T D1 = P.hdx[1] * fma(P.A[3], x0, fma(P.A[4], x1r, P.b[1]));
            T w1;
            const int j0 = floor_split(fma(S1, C.u1[0], D1), w1);
            // the 8 rows' foot cells on axis 0: one cell (uni) or two adjacent cells (a
            // row of the column crosses a cell boundary: three values per row, each node
            // takes its pair — the same lerp operands)
            int i0lo = i0[0], i0hi = i0[0];
#pragma unroll
            for (int n = 1; n < R; ++n) {
                i0lo = min(i0lo, i0[n]);
                i0hi = max(i0hi, i0[n]);
            }
            // rows lj0 + j0 + r, r = 0 .. KC + R - 1; node n uses r = n .. n + KC
            auto stream_rows = [&](auto two_tag) {
                constexpr bool TWO = decltype(two_tag)::value;
                const T *__restrict__ p = Vi + (li + i0lo) + (int64_t)vn0 * (lj0 + j0);
                bool up[R];
#pragma unroll
                for (int n = 0; n < R; ++n) up[n] = TWO && i0[n] != i0lo;
                T xprev[R];
#pragma unroll
                for (int r = 0; r < KC + R; ++r) {
                    const T a = __ldg(p), b = __ldg(p + 1);
                    const T c = TWO ? __ldg(p + 2) : b;
                    p += vn0;
#pragma unroll
                    for (int n = 0; n < R; ++n) {
                        const int m = r - n;             // X index of node n
                        if (m < 0 || m > KC) continue;
                        const T X = TWO ? lerp<T>(up[n] ? b : a, up[n] ? c : b, w0[n])
                                        : lerp<T>(a, b, w0[n]);
                        if (m >= 1) {
                            const int k = m - 1;
                            const T I = lerp<T>(xprev[n], X, w1);
                            const T ck = KRUZ ? base[n] : fma(hlr, C.csq[k], base[n]);
                            best[n] = fmin(best[n], fma(P.beta, I, ck));
                        }
                        xprev[n] = X;
                    }
                }
            };
            // every value the streamed rows touch inside the view (this thread's footprint,
            // not the tile's: edge tiles keep most threads on this path); then every foot
            // is inside the box and the view, where interp() reads exactly these corners
            const bool tfast = li + i0lo >= 0 && li + i0hi + 1 <= vn0 - 1 && lj0 + j0 >= 0 &&
                               lj0 + j0 + KC + R - 1 <= vn1 - 1 && i0hi <= i0lo + 1;
            if (tfast && uni) {
                stream_rows(std::integral_constant<bool, false>());
            } else if (tfast) {
                stream_rows(std::integral_constant<bool, true>());
            } else {
                // k_sweep_field2d's per-control loop, node by node (unrolled: the
                // per-node arrays stay in registers)
                const int64_t o[3] = {vw.o[0], vw.o[1], 0};
                const int64_t vn[3] = {vn0, vn1, 1};
#pragma unroll
                for (int n = 0; n < R; ++n) {
                    if (cls[n] != -1) continue;
                    const int lj = lj0 + n;
                    const int64_t gi[3] = {gi0, lj + vw.o[1], 0};
                    const T x1 = fma((T)gi[1], P.dx[1], P.lo[1]);
                    const T D0 = P.hdx[0] * fma(P.A[0], x0, fma(P.A[1], x1, P.b[0]));
                    const T D1n = P.hdx[1] * fma(P.A[3], x0, fma(P.A[4], x1, P.b[1]));
                    T bn = (T)INFINITY;
                    if (fast) {
                        const T *__restrict__ Vn = Vi + li + (int64_t)vn0 * lj;
#pragma unroll 1
                        for (int k = 0; k < KC; ++k) {
                            T wa, wb;
                            const int ia = floor_split(fma(S0, C.u0, D0), wa);
                            const int ib = floor_split(fma(S1, C.u1[k], D1n), wb);
                            const T *__restrict__ q = Vn + (ia + (int64_t)vn0 * ib);
                            const T I = lerp<T>(lerp<T>(__ldg(q), __ldg(q + 1), wa),
                                                lerp<T>(__ldg(q + vn0), __ldg(q + vn0 + 1), wa),
                                                wb);
                            const T ck = KRUZ ? base[n] : fma(hlr, C.csq[k], base[n]);
                            bn = fmin(bn, fma(P.beta, I, ck));
                        }
                    } else {
#pragma unroll 1
                        for (int k = 0; k < KC; ++k) {
                            const T delta[3] = {fma(S0, C.u0, D0), fma(S1, C.u1[k], D1n), T(0)};
                            const T I = interp<T, T, 2>(Vi, o, vn, P.n, P.periodic, gi, delta,
                                                        P.v_out);
                            const T ck = KRUZ ? base[n] : fma(hlr, C.csq[k], base[n]);
                            bn = fmin(bn, fma(P.beta, I, ck));
                        }
                    }
                    best[n] = bn;
                }
            }
        }
#pragma unroll
        for (int n = 0; n < R; ++n) {
            if (cls[n] == -3) continue;
            const int lj = lj0 + n;
            T vnew;
            if (cls[n] == -2) {
                vnew = P.v_out;
            } else if (cls[n] >= 0) {
                vnew = P.g ? P.g[(gi0) + P.n[0] * (lj + vw.o[1])] : T(0);
            } else {
                vnew = best[n];
                if (P.monotone) vnew = fmin(vnew, vin[n]);
                ++evaluated;
            }
            Vo[tb + n * vn0] = vnew;
            const T dv = vnew > vin[n] ? vnew - vin[n] : vin[n] - vnew;
            rmax = dv > rmax ? dv : rmax;
            changed |= !same_bits(vnew, vin[n]);
        }
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

// ---------------------------------------------------------------------------
// Dubins car (§2 dynamics family; BASELINE config 4): the (x,y) part of
// every foot, h v (cos th, sin th), is the same for all controls of a node and
// only the heading moves with the control (h w a_k).  When |h w a_k| <= 1 heading
// cell, the trilinear interpolant at the foot is exactly
//     I_k = I0 + |d_k| (I_{+-1} - I0),   d_k = h w a_k / dth,
// with I_{-1}, I0, I_{+1} the bilinear (x,y) interpolants at the foot on the heading
// planes th-1, th, th+1 (periodic) — so per node 3 bilinear interpolants, then per
// control 1 select + 2 FMA + 1 min.  Tile 32 x 8 (x, y) on one heading plane.
// ---------------------------------------------------------------------------
template <typename T>
__global__ void __launch_bounds__(256)
    k_sweep_dubins(const DevProblem<T, T> P, const SweepGroup<T> *__restrict__ G, int64_t it,
                   double tol) {
    HJ_LIST_BEGIN(G, it, tol)
    const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1], vn2 = (int)vw.vn[2];
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int li = tc[0] * 32 + (threadIdx.x & 31);
    const int lj = tc[1] * 8 + (threadIdx.x >> 5);
    const int lk = tc[2];
    T rmax = T(0);
    int changed = 0, evaluated = 0;
    if (li < vn0 && lj < vn1) {
        const int64_t plane = (int64_t)vn0 * vn1;
        const int64_t t = li + (int64_t)vn0 * lj + plane * lk;
        const int64_t gi0 = li + vw.o[0], gi1 = lj + vw.o[1], gi2 = lk + vw.o[2];
        const int64_t gidx = gi0 + P.n[0] * (gi1 + P.n[1] * gi2);
        const int8_t c = vw.cls[t];
        const T vin = Vi[t];
        T vnew;
        if (c == -2) {
            vnew = P.v_out;
        } else if (c >= 0) {
            vnew = P.g ? P.g[gidx] : T(0);
        } else {
            const T th = fma((T)gi2, P.dx[2], P.lo[2]);
            T sn, cn;
            sincos_t(th, &sn, &cn);
            const T d0 = P.hdx[0] * (P.dub_v * cn), d1 = P.hdx[1] * (P.dub_v * sn);
            const T kc = P.kcost;
            T best = (T)INFINITY;
            // (x, y) part of the foot: box rule R3 on the global grid
            const T lo0 = -(T)gi0, hi0 = (T)(P.n[0] - 1 - gi0);
            const T lo1 = -(T)gi1, hi1 = (T)(P.n[1] - 1 - gi1);
            const T eps = (T)BOX_EPS;
            const bool inside = d0 >= lo0 - eps && d0 <= hi0 + eps && d1 >= lo1 - eps &&
                                d1 <= hi1 + eps;
            T base = kc;
            if (P.cost != HJ_COST_KRUZKOV) {
                const T x[3] = {fma((T)gi0, P.dx[0], P.lo[0]), fma((T)gi1, P.dx[1], P.lo[1]), th};
                base = P.h * cost_state(P, x);
            }
            const T hlr = P.h * P.lr;
            if (!inside) {
                for (int k = 0; k < P.K; ++k) {
                    const T ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(P.beta, P.v_out, ck));
                }
            } else {
                T x = d0 < lo0 ? lo0 : (d0 > hi0 ? hi0 : d0);
                T y = d1 < lo1 ? lo1 : (d1 > hi1 ? hi1 : d1);
                T fx = floor(x), fy = floor(y);
                int64_t cx = gi0 + (int64_t)fx, cy = gi1 + (int64_t)fy;
                T wx = x - fx, wy = y - fy;
                if (cx > P.n[0] - 2) { cx = P.n[0] - 2; wx = T(1); }
                if (cy > P.n[1] - 2) { cy = P.n[1] - 2; wy = T(1); }
                // view-local corners; outside the view: ghost v_out (R10)
                const int64_t ax = cx - vw.o[0], ay = cy - vw.o[1];
                const T vo = P.v_out;
                T I3[3];
#pragma unroll
                for (int s = 0; s < 3; ++s) {
                    int64_t kk = lk + s - 1;        // views span the periodic heading axis
                    if (kk < 0) kk += vn2;
                    if (kk >= vn2) kk -= vn2;
                    const T *pl = Vi + plane * kk;
                    auto at = [&](int64_t i, int64_t j) -> T {
                        return (i >= 0 && j >= 0 && i < vn0 && j < vn1) ? __ldg(pl + i + vn0 * j)
                                                                        : vo;
                    };
                    const T a = lerp<T>(at(ax, ay), at(ax + 1, ay), wx);
                    const T bb = lerp<T>(at(ax, ay + 1), at(ax + 1, ay + 1), wx);
                    I3[s] = lerp<T>(a, bb, wy);
                }
                const T dM = I3[0] - I3[1], dP = I3[2] - I3[1];
                const T hw = P.hdx[2] * P.dub_w;
#pragma unroll 4
                for (int k = 0; k < P.K; ++k) {
                    const T dk = hw * P.ctrl[k][0];
                    const T I = fma(fabs(dk), dk < T(0) ? dM : dP, I3[1]);
                    const T ck = (P.cost == HJ_COST_KRUZKOV) ? base : fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(P.beta, I, ck));
                }
            }
            vnew = best;
            if (P.monotone) vnew = fmin(vnew, vin);
            evaluated = 1;
        }
        Vo[t] = vnew;
        rmax = vnew > vin ? vnew - vin : vin - vnew;
        changed = !same_bits(vnew, vin);
    }
    changed_ = tile_finish(G, v, tile, it, rmax, changed, evaluated);
    HJ_LIST_END(G, it)
}

}  // namespace hj
#include "hj_sweep_tb.cuh"
#include "hj_sweep_coop.cuh"
namespace hj {

// ---------------------------------------------------------------------------
// host side: choose the kernel, tile the views, launch
// ---------------------------------------------------------------------------
enum SweepKind { SWEEP_GENERIC = 0, SWEEP_LOCAL2D = 1, SWEEP_FIELD2D = 2, SWEEP_DUBINS = 3 };

template <typename T>
struct SweepLaunch {
    int kind = SWEEP_GENERIC;
    int dim = 2;
    int dyn = HJ_DYN_AFFINE;
    int kq = 0;
    bool per_ctrl_cost = false;
    bool packed = false;                // fp32 local kernel on FFMA2 (k_sweep_local2d_x2)
    int tb = 1;                         // sweeps per launch (> 1: k_sweep_local2d_tb)
    bool coop = false;                  // whole iteration in k_sweep_local2d_coop
    void *wl_mem = nullptr;             // work-list / cooperative-state region
    std::vector<int64_t> vn0, vn1, vn2; // view extents (cooperative mini-tiling)
    int64_t gn0 = 0, gn1 = 0;           // grid extents
    bool dense = false;                 // SweepGroup::dense
    int64_t total_tiles = 0;
    SweepGroup<T> *d_group = nullptr;   // device copy (inside the caller's workspace)
    LocalCtrl<T> ctrl;
    int evals = 0;                      // brackets evaluated per interior node and sweep
                                        // (the control count unless a kernel prunes)
    bool col = false;                   // FIELD2D via k_sweep_field2d_col (shared u0)
    bool lat = false;                   // ... via k_sweep_field2d_lat (controls one row apart)
    ColCtrl<T> colctrl;
    int seg = 0, seg_nup = 0;           // FIELD_COOP segmented control order (CoopState)
    int16_t seg_order[HJ_MAX_CONTROLS];
};

// bytes of change flags a view needs under the smallest tiling (32 x 8 x 1)
// bytes of per-tile flags a view needs: [2][tiles] uint8 under the 32 x 8 tiling or
// [2][tiles] int32 (block-tagged) under the 32 x 32 tiling of the blocked kernel
inline int64_t chg_bytes_for(const int64_t vn[3]) {
    int64_t t8 = ((vn[0] + 31) / 32) * ((vn[1] + 7) / 8) * vn[2];
    int64_t t32 = ((vn[0] + 31) / 32) * ((vn[1] + 31) / 32) * vn[2];
    return std::max(2 * t8, 8 * t32);
}

// tiles of a view under the finest tiling any sweep kernel uses (32 x 8 x 1)
inline int64_t tiles_finest(const int64_t vn[3]) {
    return ((vn[0] + 31) / 32) * ((vn[1] + 7) / 8) * vn[2];
}

// bytes of the work list over views whose tiles (under the finest tiling) sum to T;
// the cooperative kernel's mini-tile state (8 x 8: <= 4 per 32 x 8 tile, 40 B each)
// shares the same region, so the larger of the two is reserved
inline int64_t wl_bytes_for(int64_t T) {
    const int64_t lists = 3 * 4 * T + 2 * 4 * ((T + 31) / 32) + 64 + 4 * 256;
    const int64_t coop = 4 * T * (4 * 8 + 2 * 4) + 16 * 256 + 8 * HJ_GROUP_VIEWS;
    return std::max(lists, coop);
}

hj_status speed_max(const void *speed, int dtype, int64_t N, cudaStream_t s, double *out);

// Largest |foot offset| per axis in cells over the whole box (a safe bound).
inline void foot_bound(const hj_grid &g, const hj_problem &p, double cmax, double H[3]) {
    double xmax[3] = {0, 0, 0};
    for (int d = 0; d < g.dim; ++d) xmax[d] = std::max(std::fabs(g.lo[d]), std::fabs(g.hi[d]));
    for (int d = 0; d < 3; ++d) H[d] = 0;
    double umax[3] = {0, 0, 0}, amax = 0;
    for (int k = 0; k < p.n_controls; ++k) {
        for (int d = 0; d < 3; ++d) umax[d] = std::max(umax[d], std::fabs(p.controls[k][d]));
        amax = std::max(amax, std::fabs(p.controls[k][0]));
    }
    for (int d = 0; d < g.dim; ++d) {
        double f = 0;
        if (p.dynamics == HJ_DYN_AFFINE) {
            f = cmax * umax[d] + std::fabs(p.b[d]);
            for (int e = 0; e < g.dim; ++e) f += std::fabs(p.A[d][e]) * xmax[e];
        } else if (p.dynamics == HJ_DYN_DUBINS) {
            f = d < 2 ? std::fabs(p.dubins_v) : std::fabs(p.dubins_w) * amax;
        } else {
            f = d == 0 ? xmax[1]
                       : std::fabs(p.vdp_mu) * (1 + xmax[0] * xmax[0]) * xmax[1] + xmax[0] + amax;
        }
        H[d] = p.h * f / grid_spacing(g, d);
    }
}

// Initial work list: every tile with an interior node (class -1) — one CTA per tile.
// The first launch visits exactly these; dense mode visits them at every sweep.
template <typename T>
__global__ void k_wl_live(const SweepGroup<T> *__restrict__ G) {
    const int gid = blockIdx.x;
    const int v = find_view(G, gid);
    const SweepView<T> &vw = G->v[v];
    const TileView<T> &tv = G->t[v];
    int tc[3];
    tile_coords(tv, gid - tv.tile_base, tc);
    const int TX = G->tile_dim[0], TY = G->tile_dim[1], TZ = G->tile_dim[2];
    int any = 0;
    for (int e = threadIdx.x; e < TX * TY * TZ && !any; e += blockDim.x) {
        const int64_t i = (int64_t)tc[0] * TX + e % TX, j = (int64_t)tc[1] * TY + (e / TX) % TY;
        const int64_t k = (int64_t)tc[2] * TZ + e / (TX * TY);
        if (i < vw.vn[0] && j < vw.vn[1] && k < vw.vn[2])
            any = vw.cls[i + vw.vn[0] * (j + vw.vn[1] * k)] == -1;
    }
    if (__syncthreads_or(any) && threadIdx.x == 0) {
        const WorkList &wl = G->wl;
        const int pos = atomicAdd(&wl.count[3], 1);
        wl.live[pos] = gid;
        wl.items[0][atomicAdd(&wl.count[0], 1)] = gid;
        atomicOr(&wl.mark[0][gid >> 5], 1u << (gid & 31));
    }
}

// Persistent grid of a work-list kernel: resident CTAs (occupancy x SMs), capped by
// the number of tiles.
// the current device and its SM count (per-device caches: a process may drive several)
static inline int current_device() {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) dev = 0;
    return dev;
}
static inline int device_sms() {
    static int sms[64] = {0};
    const int dev = current_device();
    if (!sms[dev] &&
        cudaDeviceGetAttribute(&sms[dev], cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
        sms[dev] = 148;
    return sms[dev];
}

template <typename K>
static unsigned grid_for(K kernel, int threads, size_t smem, int64_t total, bool dense = false) {
    (void)dense;   // dense mode walks the live list too (persistent grid)
    const int sms = device_sms();
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem) !=
            cudaSuccess ||
        per_sm < 1)
        per_sm = 1;
    return (unsigned)std::max<int64_t>(1, std::min<int64_t>(total, (int64_t)sms * per_sm));
}

template <typename T>
hj_status sweep_prepare(const hj_grid &g, const hj_problem &p, const hj_fields &f,
                        std::vector<SweepView<T>> &views, const std::vector<uint8_t *> &chg,
                        void *d_group_mem, void *wl_mem, cudaStream_t s, SweepLaunch<T> &L) {
    const int dtype = sizeof(T) == 8 ? HJ_F64 : HJ_F32;
    double cmax = 1.0;
    if (f.speed && p.dynamics == HJ_DYN_AFFINE) {
        hj_status st = speed_max(f.speed, dtype, grid_nodes(g), s, &cmax);
        if (st != HJ_OK) return st;
    }
    double H[3];
    foot_bound(g, p, cmax, H);
    L.dim = g.dim;
    bool iso = p.dynamics == HJ_DYN_AFFINE && g.dim == 2;
    for (int d = 0; d < 3 && iso; ++d) {
        if (p.b[d] != 0) iso = false;
        for (int e = 0; e < 3; ++e)
            if (p.A[d][e] != 0) iso = false;
    }
    const int want = p.sweep_kernel;
    if (want < HJ_SWEEP_AUTO || want > HJ_SWEEP_FIELD_LAT) {
        set_error("unknown sweep_kernel %d", want);
        return HJ_ERR_INVALID;
    }
    if (want == HJ_SWEEP_LOCAL_PACKED && sizeof(T) != 4) {
        set_error("HJ_SWEEP_LOCAL_PACKED is an fp32 kernel");
        return HJ_ERR_UNSUPPORTED;
    }
    const bool local = iso && H[0] <= 1 + 1e-6 && H[1] <= 1 + 1e-6 && !g.periodic[0] &&
                       !g.periodic[1] &&
                       (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_LOCAL_SCALAR ||
                        want == HJ_SWEEP_LOCAL_PACKED || want == HJ_SWEEP_LOCAL_TB ||
                        want == HJ_SWEEP_LOCAL_COOP);
    L.kind = SWEEP_GENERIC;
    int tile_dim[3] = {32, 8, 1};
    if (local) {
        // sort the controls by quadrant; balance controls on an axis (|u| < 1e-9)
        std::vector<int> quad[4];
        double dx = grid_spacing(g, 0), dy = grid_spacing(g, 1);
        std::vector<int> axis_ctrl;
        for (int k = 0; k < p.n_controls; ++k) {
            double ux = p.controls[k][0], uy = p.controls[k][1];
            if (std::fabs(ux) < 1e-9 || std::fabs(uy) < 1e-9) {
                axis_ctrl.push_back(k);
                continue;
            }
            quad[(ux < 0 ? 1 : 0) | (uy < 0 ? 2 : 0)].push_back(k);
        }
        for (int k : axis_ctrl) {
            double ux = p.controls[k][0], uy = p.controls[k][1];
            int best = -1;
            for (int q = 0; q < 4; ++q) {
                bool okx = std::fabs(ux) < 1e-9 || ((q & 1) ? ux < 0 : ux > 0);
                bool oky = std::fabs(uy) < 1e-9 || ((q & 2) ? uy < 0 : uy > 0);
                if (okx && oky && (best < 0 || quad[q].size() < quad[best].size())) best = q;
            }
            quad[best].push_back(k);
        }
        size_t mx = 1;
        for (auto &q : quad) mx = std::max(mx, q.size());
        const int choices[] = {4, 8, 12, 16, 24, 32};
        int kq = 0;
        for (int c : choices)
            if ((size_t)c >= mx) {
                kq = c;
                break;
            }
        if (kq) {
            L.kind = SWEEP_LOCAL2D;
            L.kq = kq;
            L.packed = sizeof(T) == 4 && want != HJ_SWEEP_LOCAL_SCALAR;
            if (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_LOCAL_COOP) {
                L.coop = true;
            } else if (want == HJ_SWEEP_LOCAL_TB) {
                // sweeps per launch: TB_SMAX, or HJ_TB_SWEEPS (2..TB_SMAX) for tuning
                static const int env_s = [] {
                    const char *e = getenv("HJ_TB_SWEEPS");
                    const int v = e ? atoi(e) : 0;
                    return v >= 2 && v <= TB_SMAX ? v : TB_SMAX;
                }();
                L.tb = env_s;
                tile_dim[0] = tile_dim[1] = TB_T;
            }
            L.per_ctrl_cost = p.cost == HJ_COST_DISCOUNTED && p.lr != 0;
            memset(&L.ctrl, 0, sizeof(L.ctrl));
            for (int q = 0; q < 4; ++q) {
                // an empty quadrant repeats some control of another quadrant's... any
                // control works as padding only inside its own quadrant: use a
                // weight-0 "stay" entry (ax = ay = 0 gives beta V00 + cost, which is
                // a valid bracket only if that control exists) -> repeat a real one.
                std::vector<int> &lst = quad[q];
                for (int j = 0; j < kq; ++j) {
                    int k = lst.empty() ? -1 : lst[std::min<size_t>(j, lst.size() - 1)];
                    if (k < 0) {
                        L.ctrl.ax[q][j] = L.ctrl.ay[q][j] = 0;
                        L.ctrl.ck[q][j] = (T)INFINITY;   // never the min
                        continue;
                    }
                    L.ctrl.ax[q][j] = (T)(std::fabs(p.controls[k][0]) * p.h / dx);
                    L.ctrl.ay[q][j] = (T)(std::fabs(p.controls[k][1]) * p.h / dy);
                    double a2 = 0;
                    for (int c = 0; c < 3; ++c) a2 += p.controls[k][c] * p.controls[k][c];
                    L.ctrl.ck[q][j] = (T)(p.h * p.lr * a2);
                }
                if (lst.empty()) L.per_ctrl_cost = true;   // the +inf padding needs ck
            }
            L.ctrl.prune_ok = 1;
            for (int q = 0; q < 4; ++q) {
                double xm = 0, ym = 0;
                for (int j = 0; j < kq; ++j) {
                    xm = std::max(xm, (double)L.ctrl.ax[q][j]);
                    ym = std::max(ym, (double)L.ctrl.ay[q][j]);
                    if (!(L.ctrl.ck[q][j] >= 0)) L.ctrl.prune_ok = 0;
                }
                L.ctrl.xmax[q] = (T)xm;
                L.ctrl.ymax[q] = (T)ym;
            }
            tile_dim[0] = 32;
            tile_dim[1] = 32;
        }
    }
    if (L.kind == SWEEP_GENERIC && want != HJ_SWEEP_GENERIC && want != HJ_SWEEP_LOCAL_SCALAR &&
        want != HJ_SWEEP_LOCAL_PACKED && want != HJ_SWEEP_LOCAL_TB &&
        want != HJ_SWEEP_LOCAL_COOP) {   // (FIELD_COOP: decided with FIELD2D)
        if (g.dim == 2 && (p.dynamics == HJ_DYN_AFFINE || p.dynamics == HJ_DYN_VANDERPOL) &&
            !g.periodic[0] && !g.periodic[1] &&
            (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_FIELD2D || want == HJ_SWEEP_FIELD_COOP ||
             want == HJ_SWEEP_FIELD_COL || want == HJ_SWEEP_FIELD_LAT))
            L.kind = SWEEP_FIELD2D;
        else if (p.dynamics == HJ_DYN_DUBINS && H[2] <= 1.0 && !g.periodic[0] && !g.periodic[1] &&
                 (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_DUBINS ||
                  want == HJ_SWEEP_DUBINS_COOP))
            L.kind = SWEEP_DUBINS;
    }
    L.dyn = p.dynamics;
    if (L.kind == SWEEP_FIELD2D && H[0] <= 1.0 && H[1] <= 1.0 &&
        (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_FIELD_COOP))
        L.coop = true;         // every foot within one cell: the cooperative kernel
    if (L.kind == SWEEP_DUBINS && H[0] <= 1.0 && H[1] <= 1.0 &&
        (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_DUBINS_COOP))
        L.coop = true;         // (x, y) feet within one cell: the cooperative kernel
    L.evals = p.n_controls;
    // the cooperative field class counts the brackets it computes itself (its segment
    // pruning skips some): the work counter is already node x control
    if (L.kind == SWEEP_FIELD2D && L.coop) L.evals = 1;
    if (L.kind == SWEEP_DUBINS && L.coop && p.cost == HJ_COST_KRUZKOV) {
        // coop_eval_dubins evaluates only each heading-sign group's extreme |d_k|
        double e[4] = {INFINITY, -INFINITY, INFINITY, -INFINITY};
        for (int k = 0; k < p.n_controls; ++k) {
            const double dk = p.controls[k][0], w = std::fabs(dk);
            const int o = dk < 0 ? 2 : 0;
            e[o] = std::min(e[o], w);
            e[o + 1] = std::max(e[o + 1], w);
        }
        L.evals = 0;
        for (int o = 0; o < 4; o += 2)
            if (e[o] <= e[o + 1]) L.evals += e[o] == e[o + 1] ? 1 : 2;
    }
    if (want == HJ_SWEEP_DUBINS_COOP && !(L.kind == SWEEP_DUBINS && L.coop)) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for it "
                  "(Dubins, feet within one cell)", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if (want == HJ_SWEEP_FIELD_COOP && !(L.kind == SWEEP_FIELD2D && L.coop)) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for it "
                  "(2-D affine / Van der Pol, feet within one cell)", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if (L.kind == SWEEP_FIELD2D && p.cost == HJ_COST_DISCOUNTED) {
        tile_dim[0] = 32;      // dense problems: 32 x 32 tiles (k_sweep_field2d<.., 4>)
        tile_dim[1] = 32;
    }
    if (L.kind == SWEEP_FIELD2D && !L.coop && p.dynamics == HJ_DYN_AFFINE && !f.speed &&
        (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_FIELD_COL || want == HJ_SWEEP_FIELD_LAT)) {
        // every control moves the foot by the same amount along axis 0: one x-lerped
        // column per node (k_sweep_field2d_col)
        bool shared = true;
        for (int k = 1; k < p.n_controls; ++k)
            if (p.controls[k][0] != p.controls[0][0]) shared = false;
        // column rows per node: the feet's axis-1 span plus the cell's upper row and a
        // floor's worth of slack; the shared column buffer is rows x 256 values
        double u1min = INFINITY, u1max = -INFINITY;
        for (int k = 0; k < p.n_controls; ++k) {
            u1min = std::min(u1min, p.controls[k][1]);
            u1max = std::max(u1max, p.controls[k][1]);
        }
        const int rows = (int)std::ceil(p.h / grid_spacing(g, 1) * (u1max - u1min)) + 3;
        if (rows * 256 * (int)sizeof(T) > 160 * 1024) shared = false;
        if (shared) {
            std::vector<int> ord(p.n_controls);
            for (int k = 0; k < p.n_controls; ++k) ord[k] = k;
            std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
                return p.controls[a][1] < p.controls[b][1];
            });
            L.col = true;
            memset(&L.colctrl, 0, sizeof(L.colctrl));
            L.colctrl.rows = rows;
            L.colctrl.u0 = (T)p.controls[0][0];
            for (int k = 0; k < p.n_controls; ++k) {
                const int q = ord[k];
                L.colctrl.u1[k] = (T)p.controls[q][1];
                double a2 = 0;
                for (int c = 0; c < 3; ++c) a2 += p.controls[q][c] * p.controls[q][c];
                L.colctrl.csq[k] = (T)a2;
            }
        }
    }
    if (L.kind == SWEEP_FIELD2D && L.coop && p.dynamics == HJ_DYN_AFFINE && !f.speed &&
        p.A[1][0] == 0 && p.A[1][1] == 0 && p.A[1][2] == 0 && p.b[1] == 0 && p.A[0][0] == 0 &&
        !getenv("HJ_NO_SEG")) {
        // drift along axis 0 only, independent of x0: d1 = h/dy u1 has the control's sign —
        // two groups (u1 >= 0, u1 < 0 in the kernel's arithmetic), each sorted by u0, and
        // d0 depends on the row only (coop_eval_field: one split search per row)
        std::vector<int> up, lo;
        for (int k = 0; k < p.n_controls; ++k)
            ((T)p.controls[k][1] < T(0) ? lo : up).push_back(k);
        auto by_u0 = [&](int a, int b) { return (T)p.controls[a][0] < (T)p.controls[b][0]; };
        std::stable_sort(up.begin(), up.end(), by_u0);
        std::stable_sort(lo.begin(), lo.end(), by_u0);
        L.seg = 1;
        L.seg_nup = (int)up.size();
        int i = 0;
        for (int k : up) L.seg_order[i++] = (int16_t)k;
        for (int k : lo) L.seg_order[i++] = (int16_t)k;
    }
    // (dense column kernel: 32 x 64 tiles, k_sweep_field2d_col<.., 8>.  Two adjacent nodes
    // per thread sharing their column rows — 16 % fewer instructions — measured no faster:
    // the row loads' latency, not issue, then bounds it; profiles/r2/README.)
    if (L.col && p.cost == HJ_COST_DISCOUNTED) tile_dim[1] = 64;
    if (L.col && sizeof(T) == 4 && p.cost == HJ_COST_DISCOUNTED && p.A[1][1] == 0.0 &&
        (want == HJ_SWEEP_AUTO || want == HJ_SWEEP_FIELD_LAT) && !getenv("HJ_NO_LAT") &&
        (p.n_controls == 17 || p.n_controls == 33 || p.n_controls == 65)) {
        // lattice-aligned controls (k_sweep_field2d_lat): in the kernel's own arithmetic
        // S1 (u1[k] - u1[0]) = k exactly for the sorted controls (S1 = h/dy as the kernel
        // holds it); the products and differences are of few-bit dyadic values, so the
        // check is done exactly in double
        const T S1 = (T)(p.h / grid_spacing(g, 1));
        bool unit = true;
        for (int k = 0; k < p.n_controls; ++k) {
            const double d = (double)S1 * ((double)L.colctrl.u1[k] - (double)L.colctrl.u1[0]);
            if (d != (double)k) unit = false;
        }
        L.lat = unit && g.n[0] * g.n[1] < ((int64_t)1 << 31);   // (32-bit node offsets)
    }
    if (want == HJ_SWEEP_FIELD_LAT && !L.lat) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for it "
                  "(2-D affine, discounted, no speed field, a shared axis-0 control "
                  "component, 17/33/65 controls whose axis-1 feet are exactly one row "
                  "apart, axis-1 drift independent of x1, fp32)", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if (want == HJ_SWEEP_FIELD_COL && !L.col) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for it "
                  "(2-D affine, no speed field, every control with the same axis-0 "
                  "component, feet beyond one cell)", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if ((want == HJ_SWEEP_FIELD2D && L.kind != SWEEP_FIELD2D) ||
        (want == HJ_SWEEP_DUBINS && L.kind != SWEEP_DUBINS)) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for it", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if ((want == HJ_SWEEP_LOCAL_SCALAR || want == HJ_SWEEP_LOCAL_PACKED ||
         want == HJ_SWEEP_LOCAL_TB || want == HJ_SWEEP_LOCAL_COOP) && L.kind != SWEEP_LOCAL2D) {
        set_error("sweep_kernel %d requested, but the problem does not qualify for the local "
                  "kernel (2-D, f = c(x) u_a, foot within one cell, no periodic axis)", want);
        return HJ_ERR_UNSUPPORTED;
    }
    if (views.empty() || views.size() > HJ_GROUP_VIEWS) {
        set_error("internal: a sweep group holds 1..%d views (got %zu)", HJ_GROUP_VIEWS,
                  views.size());
        return HJ_ERR_INVALID;
    }
    SweepGroup<T> hg;
    memset(&hg, 0, sizeof(hg));
    hg.n_views = (int)views.size();
    int64_t base = 0;
    for (int d = 0; d < 3; ++d) {
        hg.tile_dim[d] = tile_dim[d];
        hg.periodic[d] = d < g.dim ? g.periodic[d] : 0;
    }
    for (int d = 0; d < 3; ++d) {
        hg.radius[d] = d < g.dim ? (int)std::ceil((H[d] + 1.0) / tile_dim[d]) : 0;
        hg.halo[d] = d < g.dim ? (int)std::ceil(H[d] * (1.0 + 1e-6) + 1e-6) : 0;
        if (L.kind == SWEEP_LOCAL2D) hg.radius[d] = d < 2 ? 1 : 0;
    }
    for (size_t q = 0; q < views.size(); ++q) {
        hg.v[q] = views[q];
        TileView<T> &tv = hg.t[q];
        for (int d = 0; d < 3; ++d)
            tv.nt[d] = (int32_t)((views[q].vn[d] + tile_dim[d] - 1) / tile_dim[d]);
        tv.tiles = (int64_t)tv.nt[0] * tv.nt[1] * tv.nt[2];
        tv.tile_base = base;
        tv.chg = chg[q];
        base += tv.tiles;
    }
    L.total_tiles = base;
    hg.total_tiles = (int)base;
    // discounted problems change at every node until they stop: no list (one CTA per
    // tile); front-like (Kruzkov) problems and the blocked kernel walk the list
    L.dense = p.cost == HJ_COST_DISCOUNTED && L.tb <= 1;
    hg.dense = L.dense ? 1 : 0;
    {   // work lists (filled by k_wl_live after the group upload below)
        int32_t *items = (int32_t *)wl_mem;
        const int64_t W = (base + 31) / 32;
        hg.wl.items[0] = items;
        hg.wl.items[1] = items + base;
        hg.wl.live = items + 2 * base;
        hg.wl.mark[0] = (uint32_t *)(items + 3 * base);
        hg.wl.mark[1] = hg.wl.mark[0] + W;
        hg.wl.count = (int32_t *)(hg.wl.mark[1] + W);
        L.wl_mem = wl_mem;
        for (size_t q = 0; q < views.size(); ++q) {
            L.vn0.push_back(views[q].vn[0]);
            L.vn1.push_back(views[q].vn[1]);
            L.vn2.push_back(views[q].vn[2]);
        }
        L.gn0 = g.n[0];
        L.gn1 = g.dim > 1 ? g.n[1] : 1;
        cudaError_t e1 = L.coop ? cudaSuccess
                                : cudaMemsetAsync(hg.wl.mark[0], 0, (2 * W + 4) * sizeof(uint32_t), s);
        if (e1 != cudaSuccess) {
            set_error("sweep_prepare list: %s", cudaGetErrorString(e1));
            return HJ_ERR_CUDA;
        }
        for (size_t q = 0; q < views.size(); ++q) {
            cudaError_t e0 = cudaMemsetAsync(chg[q], 0, chg_bytes_for(views[q].vn), s);
            if (e0 != cudaSuccess) {
                set_error("sweep_prepare flags: %s", cudaGetErrorString(e0));
                return HJ_ERR_CUDA;
            }
        }
    }
    L.d_group = (SweepGroup<T> *)d_group_mem;
    cudaError_t e = cudaMemcpyAsync(L.d_group, &hg, sizeof(hg), cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) {
        set_error("sweep_prepare upload: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    if (base > 0 && !L.coop) k_wl_live<T><<<(unsigned)base, 128, 0, s>>>(L.d_group);
    // the host struct must outlive the async copy
    e = cudaStreamSynchronize(s);
    if (e != cudaSuccess) {
        set_error("sweep_prepare sync: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    return HJ_OK;
}

template <bool PC>
static void launch_local_x2(const DevProblem<float, float> &P, const SweepLaunch<float> &L,
                            int64_t it, double tol, cudaStream_t s) {
    dim3 grid(grid_for(k_sweep_local2d_x2<4, PC>, 256, 0, L.total_tiles, L.dense));
    switch (L.kq) {
        case 4: k_sweep_local2d_x2<4, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 8: k_sweep_local2d_x2<8, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 12: k_sweep_local2d_x2<12, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 16: k_sweep_local2d_x2<16, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 24: k_sweep_local2d_x2<24, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        default: k_sweep_local2d_x2<32, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
    }
}

template <typename T, bool PC>
static void launch_local(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it,
                         double tol, cudaStream_t s) {
    if constexpr (sizeof(T) == 4) {
        if (L.packed) return launch_local_x2<PC>(P, L, it, tol, s);
    }
    dim3 grid(grid_for(k_sweep_local2d<T, 4, PC>, 256, 0, L.total_tiles, L.dense));
    switch (L.kq) {
        case 4: k_sweep_local2d<T, 4, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 8: k_sweep_local2d<T, 8, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 12: k_sweep_local2d<T, 12, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 16: k_sweep_local2d<T, 16, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        case 24: k_sweep_local2d<T, 24, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
        default: k_sweep_local2d<T, 32, PC><<<grid, 256, 0, s>>>(P, L.ctrl, L.d_group, it, tol); break;
    }
}

template <typename T, int KQ, bool PC>
static void launch_tb_kq(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t n0, int S_run,
                         int rerun, double tol, cudaStream_t s) {
    static bool attr[64] = {false};   // opt in to > 48 KB dynamic shared memory, per device
    const size_t smem = sizeof(TBSmem<T>);
    const int dev = current_device();
    if (!attr[dev]) {
        cudaFuncSetAttribute(k_sweep_local2d_tb<T, KQ, PC>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = true;
    }
    k_sweep_local2d_tb<T, KQ, PC><<<grid_for(k_sweep_local2d_tb<T, KQ, PC>, 256, smem,
                                             L.total_tiles),
                                    256, smem, s>>>(
        P, L.ctrl, L.d_group, n0, L.tb, S_run, rerun, tol);
}

template <typename T, bool PC>
static void launch_tb(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t n0, int S_run,
                      int rerun, double tol, cudaStream_t s) {
    switch (L.kq) {
        case 4: launch_tb_kq<T, 4, PC>(P, L, n0, S_run, rerun, tol, s); break;
        case 8: launch_tb_kq<T, 8, PC>(P, L, n0, S_run, rerun, tol, s); break;
        case 12: launch_tb_kq<T, 12, PC>(P, L, n0, S_run, rerun, tol, s); break;
        case 16: launch_tb_kq<T, 16, PC>(P, L, n0, S_run, rerun, tol, s); break;
        case 24: launch_tb_kq<T, 24, PC>(P, L, n0, S_run, rerun, tol, s); break;
        default: launch_tb_kq<T, 32, PC>(P, L, n0, S_run, rerun, tol, s); break;
    }
}

// Re-run of the block holding the stop (temporally blocked kernel only): every view
// whose TileView::rerun > 0 recomputes that many sub-sweeps of block n0 / L.tb.
template <typename T>
hj_status sweep_launch_rerun(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t n0,
                             double tol, cudaStream_t s) {
    if (L.total_tiles == 0) return HJ_OK;
    if (L.per_ctrl_cost)
        launch_tb<T, true>(P, L, n0, 0, 1, tol, s);
    else
        launch_tb<T, false>(P, L, n0, 0, 1, tol, s);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("sweep re-run launch failed: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    return HJ_OK;
}

// The whole iteration of the local class in one cooperative launch (hj_sweep_coop.cuh).
// stop[v] (host, out) = iterations performed by view v.
// Cluster mode (views solved by one thread-block cluster each): the cluster size and
// how many such clusters are resident at once, or {0, 0} if no cluster of 8+ fits.
template <typename T, int KQ, bool PC, int EV>
static void coop_cluster_shape(size_t dyn, int &cs, int &maxc) {
    static int c_cs = -1, c_maxc = 0;
    if (c_cs < 0) {
        auto kern = k_sweep_local2d_coop<T, KQ, PC, EV, true>;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        c_cs = 0;
        for (int want : {16, 8}) {
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = want;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(want);
            cfg.blockDim = dim3(CoopNW<T>::nw * 32);
            cfg.dynamicSmemBytes = dyn;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            int m = 0;
            if (cudaOccupancyMaxActiveClusters(&m, (void *)kern, &cfg) == cudaSuccess && m >= 1) {
                c_cs = want;
                c_maxc = m;
                break;
            }
            cudaGetLastError();
        }
    }
    cs = c_cs;
    maxc = c_maxc;
}

template <typename T, int KQ, bool PC, int EV = 0>
static hj_status launch_coop_kq(const DevProblem<T, T> &P, const SweepLaunch<T> &L,
                                const CoopState &S, int64_t max_iter, double tol,
                                cudaStream_t s) {
    constexpr int BLK = EV == 3 ? 300 : 100;
    // the staged blocks, then (segmented field class) the per-row split table
    const size_t dyn = (size_t)CoopNW<T>::nw * 2 * BLK * sizeof(T) +
                       (S.seg_tab ? (size_t)4 * P.n[1] : 0);
    if (S.cluster) {        // one cluster per view (at most maxc resident at a time)
        int cs = 0, maxc = 0;
        coop_cluster_shape<T, KQ, PC, EV>(dyn, cs, maxc);
        if (cs > 0) {
            auto kern = k_sweep_local2d_coop<T, KQ, PC, EV, true>;
            const int ncl = std::max(1, std::min(S.n_views, maxc));
            cudaLaunchConfig_t cfg = {};
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.gridDim = dim3(ncl * cs);
            cfg.blockDim = dim3(CoopNW<T>::nw * 32);
            cfg.dynamicSmemBytes = dyn;
            cfg.stream = s;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            const SweepGroup<T> *g = L.d_group;
            cudaError_t e = cudaLaunchKernelEx(&cfg, kern, P, L.ctrl, g, S, max_iter, tol);
            if (e != cudaSuccess) {
                set_error("cluster sweep launch failed: %s", cudaGetErrorString(e));
                return HJ_ERR_CUDA;
            }
            return HJ_OK;
        }
    }
    static int grids[64] = {0};        // resident grid, per device
    static size_t dyn_set[64] = {0};   // dynamic shared memory opted in, per device
    const int dev = current_device();
    int &grid = grids[dev];
    if (dyn > dyn_set[dev]) {          // (more shared memory: re-check the occupancy)
        cudaFuncSetAttribute(k_sweep_local2d_coop<T, KQ, PC, EV>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
        dyn_set[dev] = dyn;
        grid = 0;
    }
    if (!grid) {
        const int sms = device_sms();
        int per_sm = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sweep_local2d_coop<T, KQ, PC, EV>,
                                                          CoopNW<T>::nw * 32, dyn) != cudaSuccess ||
            per_sm < 1)
            per_sm = 1;
        grid = sms * per_sm;
    }
    const SweepGroup<T> *g = L.d_group;
    void *args[] = {(void *)&P, (void *)&L.ctrl, (void *)&g, (void *)&S, (void *)&max_iter,
                    (void *)&tol};
    cudaError_t e = cudaLaunchCooperativeKernel((void *)k_sweep_local2d_coop<T, KQ, PC, EV>,
                                                dim3(grid), dim3(CoopNW<T>::nw * 32), args, dyn, s);
    if (e != cudaSuccess) {
        set_error("cooperative sweep launch failed: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    return HJ_OK;
}

template <typename T>
hj_status sweep_coop(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t max_iter,
                     double tol, cudaStream_t s, std::vector<int64_t> &stop) {
    const int nv = (int)L.vn0.size();
    CoopState S;
    memset(&S, 0, sizeof(S));
    S.n_views = nv;
    int64_t tot = 0;
    S.dubins = L.kind == SWEEP_DUBINS ? 1 : 0;
    S.seg = L.seg;
    S.seg_nup = L.seg_nup;
    // the split table (2 x n1 int16 behind the staged blocks) up to 16384 rows
    S.seg_tab = L.seg && L.gn1 <= 16384 && !getenv("HJ_NO_SEGTAB") ? 1 : 0;
    memcpy(S.seg_order, L.seg_order, sizeof(S.seg_order));
    for (int v = 0; v < nv; ++v) {
        S.mt_base[v] = tot;
        S.mt0[v] = (int32_t)((L.vn0[v] + 7) / 8);
        S.mt1[v] = (int32_t)((L.vn1[v] + 7) / 8);
        S.mt2[v] = (int32_t)L.vn2[v];
        tot += (int64_t)S.mt0[v] * S.mt1[v] * S.mt2[v];
    }
    S.mt_base[nv] = tot;
    S.total = tot;
    // scan every mask each sweep while that is a few loads per thread of the grid;
    // beyond, keep a list of the mini-tiles with a nonzero mask
    S.use_list = tot > (int64_t)148 * 512 * 2 ? 1 : 0;
    if (const char *e = getenv("HJ_COOP_LIST")) S.use_list = atoi(e) != 0;   // tests / tuning
    // cluster mode (each view on one 16-CTA cluster, hardware cluster barrier): measured
    // slower on every config (config 2 ISA fine 28 ms vs 11.6 ms; coarse 1.38 vs
    // 1.25 ms: a view's work on 16 SMs outweighs the cheaper barrier), so opt-in only
    S.cluster = 0;
    if (const char *e = getenv("HJ_COOP_CLUSTER")) S.cluster = atoi(e) != 0;
    if (S.cluster) S.seg_tab = 0;      // (cluster mode sizes its shared memory once)
    S.seg_prune = L.seg && !getenv("HJ_NO_SEGPRUNE") ? 1 : 0;
    if (S.cluster) S.use_list = 0;    // (the list ring is shared by all views)
    // load balance inside a CTA (CoopState::qsingle / heavy): the last 32 items of a CTA's
    // queue are claimed one at a time, and mini-tiles with more than 24 listed nodes are
    // queued in front of the lighter ones (longest first).  Measured on config 3's
    // whole-grid solve: 503 -> 481 ms (single claims) -> 476.5 ms (both); config 2 -2 %
    // (profiles/r2v/balance_ab.txt).  The Dubins class, whose items stage three planes,
    // lost 2 % with single claims and 0.4 % with the order: pairs only, list order.
    S.qsingle = L.kind == SWEEP_DUBINS ? 0 : 32;
    S.heavy = L.kind == SWEEP_DUBINS ? -1 : 24;
    if (const char *e = getenv("HJ_COOP_HEAVY")) S.heavy = std::max(-1, std::min(64, atoi(e)));
    if (const char *e = getenv("HJ_COOP_QSINGLE")) S.qsingle = std::max(0, atoi(e));
    {
        std::vector<int> ord(nv);
        for (int v = 0; v < nv; ++v) ord[v] = v;
        std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
            return S.mt_base[a + 1] - S.mt_base[a] > S.mt_base[b + 1] - S.mt_base[b];
        });
        for (int v = 0; v < nv; ++v) S.vorder[v] = ord[v];
    }
    Carver c(L.wl_mem, (size_t)1 << 62);
    S.imask = (unsigned long long *)c.take(8 * tot);
    S.emask = (unsigned long long *)c.take(8 * tot);
    S.dmask[0] = (unsigned long long *)c.take(8 * tot);
    S.dmask[1] = (unsigned long long *)c.take(8 * tot);
    S.items[0] = (int32_t *)c.take(4 * tot);
    S.items[1] = (int32_t *)c.take(4 * tot);
    S.count = (int32_t *)c.take(32);
    S.stop = (int64_t *)c.take(8 * HJ_GROUP_VIEWS);
    HJ_CUDA(cudaMemsetAsync(S.count, 0, 32, s));
    if (tot > 0) {
        const int blocks = (int)std::min<int64_t>((tot + 255) / 256, 148 * 8);
        k_coop_masks<T><<<blocks, 256, 0, s>>>(L.d_group, S, L.gn0, L.gn1);
        HJ_CUDA(cudaGetLastError());
    }
    hj_status st = HJ_OK;
    if (L.kind == SWEEP_DUBINS) {
        st = launch_coop_kq<T, 4, false, 3>(P, L, S, max_iter, tol, s);
    } else if (L.kind == SWEEP_FIELD2D) {
        st = L.dyn == HJ_DYN_AFFINE
                 ? launch_coop_kq<T, 4, false, HJ_DYN_AFFINE + 1>(P, L, S, max_iter, tol, s)
                 : launch_coop_kq<T, 4, false, HJ_DYN_VANDERPOL + 1>(P, L, S, max_iter, tol, s);
    } else switch (L.kq) {
        case 4: st = L.per_ctrl_cost ? launch_coop_kq<T, 4, true>(P, L, S, max_iter, tol, s)
                                     : launch_coop_kq<T, 4, false>(P, L, S, max_iter, tol, s); break;
        case 8: st = L.per_ctrl_cost ? launch_coop_kq<T, 8, true>(P, L, S, max_iter, tol, s)
                                     : launch_coop_kq<T, 8, false>(P, L, S, max_iter, tol, s); break;
        case 12: st = L.per_ctrl_cost ? launch_coop_kq<T, 12, true>(P, L, S, max_iter, tol, s)
                                      : launch_coop_kq<T, 12, false>(P, L, S, max_iter, tol, s); break;
        case 16: st = L.per_ctrl_cost ? launch_coop_kq<T, 16, true>(P, L, S, max_iter, tol, s)
                                      : launch_coop_kq<T, 16, false>(P, L, S, max_iter, tol, s); break;
        case 24: st = L.per_ctrl_cost ? launch_coop_kq<T, 24, true>(P, L, S, max_iter, tol, s)
                                      : launch_coop_kq<T, 24, false>(P, L, S, max_iter, tol, s); break;
        default: st = L.per_ctrl_cost ? launch_coop_kq<T, 32, true>(P, L, S, max_iter, tol, s)
                                      : launch_coop_kq<T, 32, false>(P, L, S, max_iter, tol, s); break;
    }
    if (st != HJ_OK) return st;
    stop.assign(nv, max_iter);
    HJ_CUDA(cudaMemcpyAsync(stop.data(), S.stop, nv * sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    return HJ_OK;
}

template <typename T, bool KRUZ, int RY, int KC>
static void launch_col_kc(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it,
                          double tol, cudaStream_t s) {
    auto kern = k_sweep_field2d_col<T, KRUZ, RY, KC>;
    const size_t smem = (size_t)L.colctrl.rows * 256 * sizeof(T);
    static size_t attr[64] = {0};      // dynamic shared memory opted in, per device
    const int dev = current_device();
    if (smem > attr[dev]) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr[dev] = smem;
    }
    kern<<<grid_for(kern, 256, smem, L.total_tiles, L.dense), 256, smem, s>>>(P, L.colctrl,
                                                                              L.d_group, it, tol);
}

// control counts with an unrolled instantiation: the 2^n + 1 point sets of a linspace
template <typename T, bool KRUZ, int RY>
static void launch_col(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it, double tol,
                       cudaStream_t s) {
    switch (P.K) {
        case 17: return launch_col_kc<T, KRUZ, RY, 17>(P, L, it, tol, s);
        case 33: return launch_col_kc<T, KRUZ, RY, 33>(P, L, it, tol, s);
        case 65: return launch_col_kc<T, KRUZ, RY, 65>(P, L, it, tol, s);
        default: return launch_col_kc<T, KRUZ, RY, 0>(P, L, it, tol, s);
    }
}

template <typename T, bool KRUZ>
static void launch_lat(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it, double tol,
                       cudaStream_t s) {
    switch (P.K) {
        case 17:
            k_sweep_field2d_lat<T, KRUZ, 17>
                <<<grid_for(k_sweep_field2d_lat<T, KRUZ, 17>, 256, 0, L.total_tiles, L.dense), 256,
                   0, s>>>(P, L.colctrl, L.d_group, it, tol);
            return;
        case 33:
            k_sweep_field2d_lat<T, KRUZ, 33>
                <<<grid_for(k_sweep_field2d_lat<T, KRUZ, 33>, 256, 0, L.total_tiles, L.dense), 256,
                   0, s>>>(P, L.colctrl, L.d_group, it, tol);
            return;
        default:
            k_sweep_field2d_lat<T, KRUZ, 65>
                <<<grid_for(k_sweep_field2d_lat<T, KRUZ, 65>, 256, 0, L.total_tiles, L.dense), 256,
                   0, s>>>(P, L.colctrl, L.d_group, it, tol);
            return;
    }
}

template <typename T, int DYN, bool KRUZ>
static void launch_field(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it,
                         double tol, cudaStream_t s) {
    if constexpr (DYN == HJ_DYN_AFFINE) {
        if constexpr (!KRUZ && sizeof(T) == 4) {   // (lattice kernel: fp32, discounted)
            if (L.lat && L.dense) {
                launch_lat<T, KRUZ>(P, L, it, tol, s);
                return;
            }
        }
        if (L.col) {
            if (L.dense)
                launch_col<T, KRUZ, 8>(P, L, it, tol, s);
            else
                launch_col<T, KRUZ, 1>(P, L, it, tol, s);
            return;
        }
    }
    if (L.dense)   // 32 x 32 tiles
        k_sweep_field2d<T, DYN, KRUZ, 4>
            <<<grid_for(k_sweep_field2d<T, DYN, KRUZ, 4>, 256, 0, L.total_tiles, true), 256, 0,
               s>>>(P, L.d_group, it, tol);
    else           // 32 x 8 tiles, work list
        k_sweep_field2d<T, DYN, KRUZ, 1>
            <<<grid_for(k_sweep_field2d<T, DYN, KRUZ, 1>, 256, 0, L.total_tiles), 256, 0, s>>>(
                P, L.d_group, it, tol);
}

// One launch: sweep `it` (L.tb == 1) or the block of L.tb sweeps starting at `it`.
template <typename T>
hj_status sweep_launch(const DevProblem<T, T> &P, const SweepLaunch<T> &L, int64_t it, double tol,
                       cudaStream_t s, int S_run = 0) {
    if (L.total_tiles == 0) return HJ_OK;
    if (L.kind == SWEEP_LOCAL2D && L.tb > 1) {
        if (S_run <= 0) S_run = L.tb;
        if (L.per_ctrl_cost)
            launch_tb<T, true>(P, L, it, S_run, 0, tol, s);
        else
            launch_tb<T, false>(P, L, it, S_run, 0, tol, s);
    } else if (L.kind == SWEEP_LOCAL2D) {
        if (L.per_ctrl_cost)
            launch_local<T, true>(P, L, it, tol, s);
        else
            launch_local<T, false>(P, L, it, tol, s);
    } else if (L.kind == SWEEP_FIELD2D) {
        const bool kz = P.cost == HJ_COST_KRUZKOV;
        if (L.dyn == HJ_DYN_AFFINE && kz)
            launch_field<T, HJ_DYN_AFFINE, true>(P, L, it, tol, s);
        else if (L.dyn == HJ_DYN_AFFINE)
            launch_field<T, HJ_DYN_AFFINE, false>(P, L, it, tol, s);
        else if (kz)
            launch_field<T, HJ_DYN_VANDERPOL, true>(P, L, it, tol, s);
        else
            launch_field<T, HJ_DYN_VANDERPOL, false>(P, L, it, tol, s);
    } else if (L.kind == SWEEP_DUBINS) {
        k_sweep_dubins<T><<<grid_for(k_sweep_dubins<T>, 256, 0, L.total_tiles, L.dense), 256, 0, s>>>(P, L.d_group, it, tol);
    } else if (L.dim == 2) {
        k_sweep_generic<T, 2><<<grid_for(k_sweep_generic<T, 2>, 256, 0, L.total_tiles, L.dense), 256, 0, s>>>(P, L.d_group, it, tol);
    } else {
        k_sweep_generic<T, 3><<<grid_for(k_sweep_generic<T, 3>, 256, 0, L.total_tiles, L.dense), 256, 0, s>>>(P, L.d_group, it, tol);
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("sweep launch failed: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    return HJ_OK;
}

}  // namespace hj
