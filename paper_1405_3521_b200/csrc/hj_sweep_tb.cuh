// hj_sweep_tb.cuh — temporally blocked local 2-D sweep: S Jacobi sweeps per launch
// (PAPER.md eq. (SL) line 235 / (Tdef) line 238-245, the north_star's "optional
// in-tile temporal blocking").
//
// Problem class: the one k_sweep_local2d handles (2-D, f = c(x) u_a, every foot
// within one cell, so T(V) at a node reads only its 3x3 neighbourhood).  A CTA owns
// a 32 x 32 tile and stages the tile plus an S-cell halo (<= 48 x 48) of V^n, the
// classes and the speed in shared memory; sub-sweep j = 1..S recomputes the region
// shrunk by j cells (overlapped tiling: the halo is recomputed redundantly, never
// exchanged), so after S sub-sweeps the owned 32 x 32 nodes hold exactly V^{n+S}.
// Every node update is the same arithmetic, in the same order, as k_sweep_local2d —
// the iterates are bit-identical to S launches of the one-sweep kernels.
//
// Per sub-sweep each CTA folds max |V^{n+j} - V^{n+j-1}| over its OWNED nodes into
// res[n+j-1] (per-warp atomicMax), so the host still sees every sweep's residual
// and the stopping rule (R6) stays exact: if the first n* with res < tol falls
// inside a block, that block is re-run from its (intact) input with S' = n* - n0
// sub-sweeps (tile flag `rerun`).
//
// Exact skipping at block granularity.  Flags per tile and block: bit0 = an owned
// node changed in the LAST sub-sweep, bit1 = changed in ANY sub-sweep.  If no tile
// within one tile (>= S cells) changed in the last sweep of block b-1, then
// V^{n0+S} = V^{n0} on the tile; the output buffer already holds it unless the tile
// itself changed during block b-1 (bit1), in which case the tile is copied.
//
// Box edges (R3) need a per-control out-of-box test; those nodes are few, so a warp
// evaluates each of its edge nodes cooperatively (controls spread over the lanes,
// then a warp min) instead of diverging through a 4 KQ-iteration loop.
#pragma once

namespace hj {

constexpr int TB_T = 32;      // owned tile edge
constexpr int TB_SMAX = 8;    // sub-sweeps per launch (max)
constexpr int TB_P = TB_T + 2 * TB_SMAX;   // staged pitch (48)
constexpr int TB_WSEG = 6 * (TB_P - 2);    // rows per warp (<= 6) x columns (<= 46)

// Optional per-CTA trace (profiling aid, off unless hj_debug_set_trace was called):
// [blockIdx] = {smid, start ns, end ns, computed nodes}.
struct TBTrace {
    unsigned long long *buf;
    long long cap;
    long long n0;          // record only the launch whose first sweep is n0
};
static __device__ TBTrace g_tb_trace = {nullptr, 0, 0};   // set by hj_debug_set_trace

template <typename T>
struct TBSmem {
    T V[2][TB_P * TB_P];
    T c[TB_P * TB_P];           // speed c(x) (1 if none)
    int16_t list[8][TB_WSEG];   // dirty interior nodes, one segment per warp (its rows)
    int16_t elist[8][128];      // dirty box-edge nodes (R3 path), one segment per warp
    int wcnt[2][8], wecnt[2][8];  // segment lengths (parity of the sub-sweep)
    int8_t cls[TB_P * TB_P];    // -2 ghost / outside the view, -1 interior, -3 interior
                                // on the box edge, >= 0 target
    // row bitmasks (bit c of word [r] = column c; the region is <= 48 < 64 wide)
    unsigned long long imask[TB_P];    // fast interior nodes (class -1)
    unsigned long long emask[TB_P];    // interior nodes on the box edge (class -3)
    unsigned int chm[2][TB_P][2];      // changed in the sub-sweep of that parity
};

template <typename T>
__device__ __forceinline__ T tb_edge_cand(const DevProblem<T, T> &P, const LocalCtrl<T> &C, int KQ,
                                          bool PC, const T *sp, int q, int k, T C0, T sc, T base,
                                          bool lo_x, bool hi_x, bool lo_y, bool hi_y) {
    constexpr int SW = TB_P;
    const T V00 = sp[0];
    const T Vx = (q & 1) ? sp[-1] : sp[1];
    const T Vy = (q & 2) ? sp[-SW] : sp[SW];
    const T Vxy = (q == 0) ? sp[SW + 1] : (q == 1) ? sp[SW - 1] : (q == 2) ? sp[-SW + 1] : sp[-SW - 1];
    const bool ex = (q & 1) ? lo_x : hi_x, ey = (q & 2) ? lo_y : hi_y;
    const T Dx = P.beta * (Vx - V00), Dy = P.beta * (Vy - V00);
    const T Dxy = P.beta * ((Vxy - Vx) - (Vy - V00));
    const T c_out = fma(P.beta, P.v_out, base);
    const T eps = (T)BOX_EPS;
    T wx = sc * C.ax[q][k], wy = sc * C.ay[q][k];
    const T ck = PC ? C.ck[q][k] : T(0);
    const bool out = (ex && wx > eps) || (ey && wy > eps);
    if (ex) wx = T(0);
    if (ey) wy = T(0);
    const T in = fma(wy, fma(wx, Dxy, Dy), fma(wx, Dx, C0)) + ck;
    return out ? c_out + ck : in;
}

// Interior bracket-min of a node pair (lanes .x/.y = nodes 0/1), quadrant by
// quadrant.  Same per-node arithmetic as k_sweep_local2d (bit-identical).
// Exact pruning (PRUNE): in quadrant q every candidate is
//   C0 + g(ax, ay),  g = ax A1 + ay A2 + ax ay A3 bilinear on [0, xmax_q] x [0, ymax_q],
// so it is >= C0 + min(g at the 4 box corners) = LB_q.  A quadrant is skipped when, for
// both nodes of every pair of the warp, LB_q exceeds the running best by more than the
// rounding error of a candidate (1e-6 (fp32) / 1e-14 (fp64) of the summed magnitudes):
// then no candidate of it can be below that best and the min is unchanged bit for bit.
// With the monotone clamp (V^{n+1} = min(T V^n, V^n)) the running best starts at V00.
template <typename T>
struct TBTraits;
template <>
struct TBTraits<float> {
    static constexpr float rel = 1e-6f;
};
template <>
struct TBTraits<double> {
    static constexpr double rel = 1e-14;
};

template <typename T, int KQ, bool PC>
__device__ __forceinline__ void tb_quadrant(const LocalCtrl<T> &C, int q, const T C0[2],
                                            const T A1[2], const T A2[2], const T A3[2],
                                            T best[2]);

template <int KQ, bool PC>
__device__ __forceinline__ void tb_quadrant_f(const LocalCtrl<float> &C, int q, const float C0[2],
                                              const float A1[2], const float A2[2],
                                              const float A3[2], float best[2]) {
    const float2 c0 = make_float2(C0[0], C0[1]);
    const float2 a1 = make_float2(A1[0], A1[1]), a2 = make_float2(A2[0], A2[1]);
    const float2 a3 = make_float2(A3[0], A3[1]);
#pragma unroll
    for (int k = 0; k < KQ; k += 2) {
        const float ax0 = C.ax[q][k], ay0 = C.ay[q][k];
        const float ax1 = C.ax[q][k + 1], ay1 = C.ay[q][k + 1];
        const float2 u0 = __ffma2_rn(make_float2(ax0, ax0), a1,
                                     PC ? __fadd2_rn(c0, make_float2(C.ck[q][k], C.ck[q][k])) : c0);
        const float2 u1 = __ffma2_rn(
            make_float2(ax1, ax1), a1,
            PC ? __fadd2_rn(c0, make_float2(C.ck[q][k + 1], C.ck[q][k + 1])) : c0);
        const float2 w0 = __ffma2_rn(make_float2(ax0, ax0), a3, a2);
        const float2 w1 = __ffma2_rn(make_float2(ax1, ax1), a3, a2);
        const float2 k0 = __ffma2_rn(make_float2(ay0, ay0), w0, u0);
        const float2 k1 = __ffma2_rn(make_float2(ay1, ay1), w1, u1);
        best[0] = fminf(best[0], fminf(k0.x, k1.x));
        best[1] = fminf(best[1], fminf(k0.y, k1.y));
    }
}

template <int KQ, bool PC>
__device__ __forceinline__ void tb_quadrant_d(const LocalCtrl<double> &C, int q, const double C0[2],
                                              const double A1[2], const double A2[2],
                                              const double A3[2], double best[2]) {
#pragma unroll
    for (int k = 0; k < KQ; ++k) {
        const double ax = C.ax[q][k], ay = C.ay[q][k];
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            const double u = fma(ax, A1[p], PC ? C0[p] + C.ck[q][k] : C0[p]);
            best[p] = fmin(best[p], fma(ay, fma(ax, A3[p], A2[p]), u));
        }
    }
}

template <typename T, int KQ, bool PC>
__device__ __forceinline__ void tb_quadrant(const LocalCtrl<T> &C, int q, const T C0[2],
                                            const T A1[2], const T A2[2], const T A3[2],
                                            T best[2]) {
    if constexpr (sizeof(T) == 4)
        tb_quadrant_f<KQ, PC>(C, q, C0, A1, A2, A3, best);
    else
        tb_quadrant_d<KQ, PC>(C, q, C0, A1, A2, A3, best);
}

// Pair arithmetic for the coefficient setup: two nodes per FADD2/FMUL2 in fp32
// (each lane rounds exactly like the scalar FADD/FMUL of k_sweep_local2d).
template <typename T>
struct Pr {
    T x, y;
};
__device__ __forceinline__ Pr<float> psub(Pr<float> a, Pr<float> b) {
    const float2 r = __fadd2_rn(make_float2(a.x, a.y), make_float2(-b.x, -b.y));
    return {r.x, r.y};
}
__device__ __forceinline__ Pr<float> pmul(Pr<float> a, Pr<float> b) {
    const float2 r = __fmul2_rn(make_float2(a.x, a.y), make_float2(b.x, b.y));
    return {r.x, r.y};
}
__device__ __forceinline__ Pr<double> psub(Pr<double> a, Pr<double> b) {
    return {a.x - b.x, a.y - b.y};
}
__device__ __forceinline__ Pr<double> pmul(Pr<double> a, Pr<double> b) {
    return {a.x * b.x, a.y * b.y};
}

// tb flags: bit0 changed in the last sub-sweep, bit1 changed in any sub-sweep.
// Staged classes: -3 marks an interior node ON the box edge (R3 slow path).
// One tile of one block of sweeps; returns 1 when an owned node changed in any
// sub-sweep (the caller then lists the 3 x 3 tiles around it for the next block).
template <typename T, int KQ, bool PC>
__device__ __forceinline__ int tb_tile(const DevProblem<T, T> &P, const LocalCtrl<T> &C,
                                       const SweepGroup<T> *__restrict__ G, TBSmem<T> &sm,
                                       const int64_t b, int64_t n0, int S_blk, int S_run,
                                       int rerun, double tol) {
    unsigned long long t_start = 0;
    long long ph_stage = 0, ph_scan = 0, ph_pairs = 0, ph_tail = 0, ph_t = 0;
    const bool tr = g_tb_trace.buf != nullptr;
    if (tr) {
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_start));
        ph_t = clock64();
    }
    const int v = find_view(G, b);
    const SweepView<T> &vw = G->v[v];
    const TileView<T> &tv = G->t[v];
    if (rerun) {                       // re-run of the block that contains the stop
        S_run = tv.rerun;
        if (S_run <= 0) return 0;
    }
    const int64_t blk = n0 / S_blk;
    // stopped view: some sweep of the previous block met the rule
    {
        int stop = 0;
        if (n0 > 0 && (int)threadIdx.x < S_blk)
            stop = *(volatile double *)&vw.res[n0 - S_blk + threadIdx.x] < tol;
        if (__syncthreads_or(stop)) return 0;
    }
    const int64_t tile = b - tv.tile_base;
    const int tcx = (int)(tile % tv.nt[0]), tcy = (int)(tile / tv.nt[0]);
    const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1];
    const T *__restrict__ Vi = vw.V[blk & 1];
    T *__restrict__ Vo = vw.V[(blk + 1) & 1];
    const int x0 = tcx * TB_T, y0 = tcy * TB_T;
    // per-tile flags of this block, tagged with the block index (a tile the list did
    // not visit keeps an older tag, which reads as "no change")
    int32_t *flags_out = reinterpret_cast<int32_t *>(tv.chg) + (blk & 1) * tv.tiles;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    // ---- exact skip (block granularity) ---------------------------------------
    if (n0 > 0) {
        const int32_t *prev = reinterpret_cast<const int32_t *>(tv.chg) + ((blk - 1) & 1) * tv.tiles;
        int act = 0, own = 0;
        if (threadIdx.x < 9) {
            const int cx = tcx + (int)threadIdx.x % 3 - 1, cy = tcy + (int)threadIdx.x / 3 - 1;
            if (cx >= 0 && cy >= 0 && cx < tv.nt[0] && cy < tv.nt[1]) {
                const int32_t tf = prev[cx + (int64_t)tv.nt[0] * cy];
                const int f = (tf >> 2) == (int32_t)(blk - 1) ? (tf & 3) : 0;
                act = f & 1;
                if (threadIdx.x == 4) own = (f >> 1) & 1;
            }
        }
        const int any_act = __syncthreads_or(act);
        if (!any_act) {
            const int any_own = __syncthreads_or(own);
            if (any_own) {             // V^{n0} -> output buffer (tile changed in block b-1)
                for (int r = warp; r < TB_T; r += 8) {
                    const int li = x0 + lane, lj = y0 + r;
                    if (li < vn0 && lj < vn1) {
                        const int64_t t = li + (int64_t)vn0 * lj;
                        Vo[t] = Vi[t];
                    }
                }
            }
            if (threadIdx.x == 0) flags_out[tile] = (int32_t)(blk << 2);
            return 0;
        }
    }
    // ---- stage tile + S-cell halo ---------------------------------------------
    const int S = S_run;
    const int R = TB_T + 2 * S;        // staged region edge (pitch TB_P)
    const int ox = x0 - S, oy = y0 - S;
    const int64_t n0g = vw.o[0] + ox, n1g = vw.o[1] + oy;   // global index of region (0,0)
    const int64_t gn0 = P.n[0], gn1 = P.n[1];
    const T v_out = P.v_out;
    for (int r = warp; r < R; r += 8) {
        for (int c = lane; c < R; c += 32) {
            const int li = ox + c, lj = oy + r;
            T val = v_out, sp = T(1);
            int8_t cl = -2;
            if (li >= 0 && lj >= 0 && li < vn0 && lj < vn1) {
                const int64_t t = li + (int64_t)vn0 * lj;
                val = Vi[t];
                cl = vw.cls[t];
                const int64_t g0 = n0g + c, g1 = n1g + r;
                if (P.speed) sp = P.speed[g0 + gn0 * g1];
                if (cl == -1 && (g0 == 0 || g1 == 0 || g0 == gn0 - 1 || g1 == gn1 - 1)) cl = -3;
            }
            const int si = r * TB_P + c;
            sm.V[0][si] = val;
            sm.V[1][si] = val;
            sm.cls[si] = cl;
            sm.c[si] = sp;
        }
    }
    __syncthreads();
    for (int r = warp; r < R; r += 8) {           // class masks; sub-sweep 1: all dirty
        const int8_t c0 = lane < R ? sm.cls[r * TB_P + lane] : (int8_t)-2;
        const int8_t c1 = lane + 32 < R ? sm.cls[r * TB_P + lane + 32] : (int8_t)-2;
        const unsigned i0 = __ballot_sync(0xffffffffu, c0 == -1),
                       i1 = __ballot_sync(0xffffffffu, c1 == -1);
        const unsigned e0 = __ballot_sync(0xffffffffu, c0 == -3),
                       e1 = __ballot_sync(0xffffffffu, c1 == -3);
        if (lane == 0) {
            sm.imask[r] = (unsigned long long)i0 | ((unsigned long long)i1 << 32);
            sm.emask[r] = (unsigned long long)e0 | ((unsigned long long)e1 << 32);
            sm.chm[0][r][0] = sm.chm[0][r][1] = 0xffffffffu;
            sm.chm[1][r][0] = sm.chm[1][r][1] = 0u;
        }
    }
    __syncthreads();
    if (tr) {
        const long long t = clock64();
        ph_stage += t - ph_t;
        ph_t = t;
    }
    const bool mono = P.monotone != 0;
    const T beta = P.beta;
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    int evaluated = 0, listed = 0, chg_any = 0;
    int cur = 0;
    for (int j = 1; j <= S; ++j) {
        const T *__restrict__ Vc = sm.V[cur];
        T *__restrict__ Vn = sm.V[cur ^ 1];
        const int lo = j, hi = R - 1 - j;           // compute region [j, R-1-j]^2
        // ---- 1. dirty interior nodes -> list.  A node's T(V) can change only if a node
        // of its 3x3 neighbourhood changed in sub-sweep j-1 (chg == j-1; all at j = 1).
        // Nodes not recomputed keep their value in BOTH buffers (they did not change in
        // j-1 either), so nothing is copied.
        {
            // warp w scans rows lo+w, lo+w+8, ... into its own segment: no atomics
            const unsigned (*pm)[2] = sm.chm[(j - 1) & 1];
            const unsigned clo = (lo >= 32 ? 0u : (~0u << lo)) &
                                 (hi >= 31 ? ~0u : ((1u << (hi + 1)) - 1u));
            const unsigned chi = (lo <= 32 ? ~0u : (~0u << (lo - 32))) &
                                 (hi >= 63 ? ~0u : (hi < 32 ? 0u : ((1u << (hi - 31)) - 1u)));
            const unsigned lt = (1u << lane) - 1u;
            int16_t *seg = sm.list[warp];
            int16_t *eseg = sm.elist[warp];
            int n = 0, ne = 0;
            for (int r = lo + warp; r <= hi; r += 8) {
                const unsigned mlo = pm[r - 1][0] | pm[r][0] | pm[r + 1][0];
                const unsigned mhi = pm[r - 1][1] | pm[r][1] | pm[r + 1][1];
                const unsigned dlo = (mlo | (mlo << 1) | (mlo >> 1) | (mhi << 31)) & clo;
                const unsigned dhi = (mhi | (mhi << 1) | (mhi >> 1) | (mlo >> 31)) & chi;
                const unsigned long long im = sm.imask[r], em = sm.emask[r];
                const unsigned ilo = dlo & (unsigned)im, ihi = dhi & (unsigned)(im >> 32);
                const unsigned elo = dlo & (unsigned)em, ehi = dhi & (unsigned)(em >> 32);
                const int pil = __popc(ilo), pel = __popc(elo);
                if ((ilo >> lane) & 1u) seg[n + __popc(ilo & lt)] = (int16_t)(r * TB_P + lane);
                if ((ihi >> lane) & 1u)
                    seg[n + pil + __popc(ihi & lt)] = (int16_t)(r * TB_P + 32 + lane);
                if ((elo >> lane) & 1u) eseg[ne + __popc(elo & lt)] = (int16_t)(r * TB_P + lane);
                if ((ehi >> lane) & 1u)
                    eseg[ne + pel + __popc(ehi & lt)] = (int16_t)(r * TB_P + 32 + lane);
                n += pil + __popc(ihi);
                ne += pel + __popc(ehi);
            }
            if (lane == 0) {
                sm.wcnt[j & 1][warp] = n;
                sm.wecnt[j & 1][warp] = ne;
            }
        }
        __syncthreads();
        // segment offsets of the interior list (every thread, 8 entries)
        int off[9];
        off[0] = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) off[w + 1] = off[w] + sm.wcnt[j & 1][w];
        int LE = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) LE += sm.wecnt[j & 1][w];
        const int L = off[8];
        listed += L + LE;
        if (tr) {
            const long long t = clock64();
            ph_scan += t - ph_t;
            ph_t = t;
        }
        // masks sub-sweep j+1 will set: that parity slot was last read by this scan
        // (before the barrier above) and is next written after the sub-sweep's end
        for (int r = threadIdx.x; r < TB_P; r += blockDim.x)
            sm.chm[(j + 1) & 1][r][0] = sm.chm[(j + 1) & 1][r][1] = 0u;
        // ---- 2. the bracket-min of the listed nodes, in pairs (i, i + 256) -----------
        T rmax = T(0);
        const int M = (L + 511) / 512;
        for (int m = 0; m < M; ++m) {
            const int iA = (int)threadIdx.x + 512 * m;
            int si[2];
            bool valid[2], owned[2];
            int8_t cl[2];
            T C0[2], V00[2], best[2];
            Pr<T> bs, bss, nb[9];     // nb: the 3 x 3 neighbourhood, row-major from (-1,-1)
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                valid[p] = iA + 256 * p < L;
                int sidx = (S + 1) * TB_P + S + 1;
                if (valid[p]) {
                    const int i = iA + 256 * p;
                    int w = 0;
#pragma unroll
                    for (int u = 1; u < 8; ++u) w += i >= off[u];
                    sidx = sm.list[w][i - off[w]];
                }
                si[p] = sidx;
                const int r = si[p] / TB_P, c = si[p] - (si[p] / TB_P) * TB_P;
                owned[p] = valid[p] && (unsigned)(r - S) < (unsigned)TB_T &&
                           (unsigned)(c - S) < (unsigned)TB_T;
                cl[p] = valid[p] ? sm.cls[si[p]] : (int8_t)-2;
                const T *q0 = Vc + si[p];
#pragma unroll
                for (int e = 0; e < 9; ++e) {
                    const T val = q0[(e / 3 - 1) * TB_P + (e % 3 - 1)];
                    if (p == 0) nb[e].x = val; else nb[e].y = val;
                }
                V00[p] = p == 0 ? nb[4].x : nb[4].y;
                T base = P.kcost;
                if (!kruz) {
                    const T x[3] = {fma((T)(n0g + c), P.dx[0], P.lo[0]),
                                    fma((T)(n1g + r), P.dx[1], P.lo[1]), T(0)};
                    base = P.h * cost_state(P, x);
                }
                C0[p] = fma(beta, V00[p], base);
                const T sc = sm.c[si[p]];
                const T b1 = beta * sc;
                if (p == 0) { bs.x = b1; bss.x = b1 * sc; } else { bs.y = b1; bss.y = b1 * sc; }
                // the clamp value V00 (monotone: V^{n+1} = min(T V^n, V^n)), else +inf
                best[p] = mono ? V00[p] : (T)INFINITY;
            }
            // all quadrant coefficients at once, both nodes per instruction:
            // quadrant q: x side (q&1 ? -1 : +1), y side (q&2 ? -1 : +1); same rounding
            // sequence as k_sweep_local2d: Dx = Vx - V00, Dy = Vy - V00,
            // Dxy = (Vxy - Vx) - Dy, A1 = bs Dx, A2 = bs Dy, A3 = bss Dxy
            {
                const Pr<T> c = nb[4];
                const Pr<T> Dxp = psub(nb[5], c), Dxm = psub(nb[3], c);
                const Pr<T> Dyp = psub(nb[7], c), Dym = psub(nb[1], c);
                const Pr<T> A1p = pmul(bs, Dxp), A1m = pmul(bs, Dxm);
                const Pr<T> A2p = pmul(bs, Dyp), A2m = pmul(bs, Dym);
                const Pr<T> A3q[4] = {pmul(bss, psub(psub(nb[8], nb[5]), Dyp)),
                                      pmul(bss, psub(psub(nb[6], nb[3]), Dyp)),
                                      pmul(bss, psub(psub(nb[2], nb[5]), Dym)),
                                      pmul(bss, psub(psub(nb[0], nb[3]), Dym))};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const Pr<T> a1 = (q & 1) ? A1m : A1p, a2 = (q & 2) ? A2m : A2p;
                    const T a1v[2] = {a1.x, a1.y}, a2v[2] = {a2.x, a2.y};
                    const T a3v[2] = {A3q[q].x, A3q[q].y};
                    tb_quadrant<T, KQ, PC>(C, q, C0, a1v, a2v, a3v, best);
                }
            }
#pragma unroll
            for (int p = 0; p < 2; ++p) {
                if (!valid[p]) continue;
                const T vnew = best[p];          // (monotone: already min(T V, V00))
                evaluated += owned[p];
                Vn[si[p]] = vnew;
                if (!same_bits(vnew, V00[p])) {
                    const int r = si[p] / TB_P, c = si[p] - r * TB_P;
                    atomicOr(&sm.chm[j & 1][r][c >> 5], 1u << (c & 31));
                    chg_any |= owned[p];
                    if (owned[p]) {
                        const T dv = vnew > V00[p] ? vnew - V00[p] : V00[p] - vnew;
                        rmax = dv > rmax ? dv : rmax;
                    }
                }
            }
        }
        if (tr) {
            const long long t = clock64();
            ph_pairs += t - ph_t;
            ph_t = t;
        }
        int eoff[9];
        eoff[0] = 0;
#pragma unroll
        for (int w = 0; w < 8; ++w) eoff[w + 1] = eoff[w] + sm.wecnt[j & 1][w];
        // ---- 3. box-edge nodes (R3), same edge formula as k_sweep_local2d: 4 nodes per
        // warp at a time, 8 lanes per node splitting the controls, then an 8-lane min
        {
            const int sg = lane >> 3, sl = lane & 7;
            for (int e0 = 4 * warp; e0 < LE; e0 += 32) {
                const int e = e0 + sg;
                const bool ok = e < LE;
                int esi = (S + 1) * TB_P + S + 1;
                if (ok) {
                    int w = 0;
#pragma unroll
                    for (int u = 1; u < 8; ++u) w += e >= eoff[u];
                    esi = sm.elist[w][e - eoff[w]];
                }
                const int sr = esi / TB_P, scol = esi - sr * TB_P;
                const int64_t g0 = n0g + scol, g1 = n1g + sr;
                T base = P.kcost;
                if (!kruz) {
                    const T x[3] = {fma((T)g0, P.dx[0], P.lo[0]), fma((T)g1, P.dx[1], P.lo[1]),
                                    T(0)};
                    base = P.h * cost_state(P, x);
                }
                const T eV00 = Vc[esi];
                const T eC0 = fma(beta, eV00, base);
                const T e_sc = sm.c[esi];
                const bool lx = g0 == 0, hx = g0 == gn0 - 1, ly = g1 == 0, hy = g1 == gn1 - 1;
                // lane sl: quadrant sl >> 1, controls k = (sl & 1), (sl & 1) + 2, ...
                T e_best = (T)INFINITY;
                {
                    const int q = sl >> 1;
                    const T *sp = Vc + esi;
                    const T eV = sp[0];
                    const T Vx = (q & 1) ? sp[-1] : sp[1];
                    const T Vy = (q & 2) ? sp[-TB_P] : sp[TB_P];
                    const T Vxy = (q == 0)   ? sp[TB_P + 1]
                                  : (q == 1) ? sp[TB_P - 1]
                                  : (q == 2) ? sp[-TB_P + 1]
                                             : sp[-TB_P - 1];
                    const bool ex = (q & 1) ? lx : hx, ey = (q & 2) ? ly : hy;
                    const T Dx = beta * (Vx - eV), Dy = beta * (Vy - eV);
                    const T Dxy = beta * ((Vxy - Vx) - (Vy - eV));
                    const T c_out = fma(beta, P.v_out, base);
                    const T eps = (T)BOX_EPS;
#pragma unroll 4
                    for (int k = sl & 1; k < KQ; k += 2) {
                        T wx = e_sc * C.ax[q][k], wy = e_sc * C.ay[q][k];
                        const T ck = PC ? C.ck[q][k] : T(0);
                        const bool out = (ex && wx > eps) || (ey && wy > eps);
                        if (ex) wx = T(0);
                        if (ey) wy = T(0);
                        const T in = fma(wy, fma(wx, Dxy, Dy), fma(wx, Dx, eC0)) + ck;
                        e_best = fmin(e_best, out ? c_out + ck : in);
                    }
                }
#pragma unroll
                for (int o = 4; o > 0; o >>= 1)
                    e_best = fmin(e_best, __shfl_xor_sync(0xffffffffu, e_best, o));
                if (ok && sl == 0) {
                    const T vnew = mono ? fmin(e_best, eV00) : e_best;
                    const bool own = (unsigned)(sr - S) < (unsigned)TB_T &&
                                     (unsigned)(scol - S) < (unsigned)TB_T;
                    evaluated += own;
                    Vn[esi] = vnew;
                    if (!same_bits(vnew, eV00)) {
                        atomicOr(&sm.chm[j & 1][sr][scol >> 5], 1u << (scol & 31));
                        chg_any |= own;
                        if (own) {
                            const T dv = vnew > eV00 ? vnew - eV00 : eV00 - vnew;
                            rmax = dv > rmax ? dv : rmax;
                        }
                    }
                }
            }
        }
        // residual of sweep n0+j-1 over the owned nodes (per-warp atomic)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const T other = __shfl_xor_sync(0xffffffffu, rmax, o);
            rmax = other > rmax ? other : rmax;
        }
        if (lane == 0 && rmax > T(0)) atomic_max_nonneg(&vw.res[n0 + j - 1], (double)rmax);
        cur ^= 1;
        __syncthreads();
        if (tr) {
            const long long t = clock64();
            ph_tail += t - ph_t;
            ph_t = t;
        }
    }
    int chg_last = 0;
    if (threadIdx.x < TB_T) {                       // owned rows S..S+31, cols S..S+31
        const int r = S + threadIdx.x;
        const unsigned long long m =
            (unsigned long long)sm.chm[S & 1][r][0] | ((unsigned long long)sm.chm[S & 1][r][1] << 32);
        chg_last = ((m >> S) & 0xffffffffull) != 0;
    }
    // ---- owned nodes of V^{n0+S} -> global -------------------------------------
    const T *__restrict__ Vf = sm.V[cur];
    for (int r = warp; r < TB_T; r += 8) {
        const int li = x0 + lane, lj = y0 + r;
        if (li < vn0 && lj < vn1) Vo[li + (int64_t)vn0 * lj] = Vf[(r + S) * TB_P + (lane + S)];
    }
    evaluated = __reduce_add_sync(0xffffffffu, evaluated);
    if (lane == 0 && evaluated) atomicAdd(vw.work, (unsigned long long)evaluated);
    const int any_last = __syncthreads_or(chg_last);
    const int any_any = __syncthreads_or(chg_any);
    if (threadIdx.x == 0)
        flags_out[tile] = (int32_t)(blk << 2) | (any_last ? 1 : 0) | (any_any ? 2 : 0);
    if (g_tb_trace.buf && threadIdx.x == 0 && b < g_tb_trace.cap && n0 == g_tb_trace.n0 &&
        !rerun) {
        unsigned long long t_end, smid;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_end));
        unsigned s32;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(s32));
        smid = s32;
        unsigned long long *o = g_tb_trace.buf + 8 * b;
        o[4] = (unsigned long long)ph_stage;
        o[5] = (unsigned long long)ph_scan;
        o[6] = (unsigned long long)ph_pairs;
        o[7] = (unsigned long long)ph_tail;
        o[0] = smid;
        o[1] = t_start;
        o[2] = t_end;
        o[3] = (unsigned long long)listed;
    }
    return any_any;
}

// Persistent walk over the block's work list (or, for the re-run of the stop block,
// over every tile: the per-tile flags then decide, exactly as in the list walk).
#ifndef HJ_TB_MINB
#define HJ_TB_MINB 3
#endif
template <typename T, int KQ, bool PC>
__global__ void __launch_bounds__(256, HJ_TB_MINB)
    k_sweep_local2d_tb(const DevProblem<T, T> P, const LocalCtrl<T> C,
                       const SweepGroup<T> *__restrict__ G, int64_t n0, int S_blk, int S_run,
                       int rerun, double tol) {
    extern __shared__ __align__(16) unsigned char tb_raw[];
    TBSmem<T> &sm = *reinterpret_cast<TBSmem<T> *>(tb_raw);
    const WorkList &wl_ = G->wl;
    const int64_t blk = n0 / S_blk;
    const int cnt_ = rerun ? G->total_tiles : *(volatile const int *)&wl_.count[blk % 3];
    for (int idx_ = blockIdx.x; idx_ < cnt_; idx_ += gridDim.x) {
        const int gid = rerun ? idx_ : wl_.items[blk & 1][idx_];
        if (!rerun && threadIdx.x == 0)
            atomicAnd(&wl_.mark[blk & 1][gid >> 5], ~(1u << (gid & 31)));
        const int any = tb_tile<T, KQ, PC>(P, C, G, sm, gid, n0, S_blk, S_run, rerun, tol);
        if (any && !rerun) {
            const int v = find_view(G, (int64_t)gid);
            int tc[3];
            tile_coords(G->t[v], gid - G->t[v].tile_base, tc);
            push_neighbours(G, v, tc, 1, 1, 0, blk + 1);
        }
        __syncthreads();
    }
    if (!rerun && blockIdx.x == 0 && threadIdx.x == 0) wl_.count[(blk + 2) % 3] = 0;
}

}  // namespace hj
