// hj_sweep_coop.cuh — the whole value iteration of the local 2-D class in ONE
// cooperative launch (PAPER.md eq. (SL), (Tdef) line 238-245, stopping rule
// line 341-345 / reading R6).
//
// Problem class: the one k_sweep_local2d handles (2-D, f = c(x) u_a, every foot within
// one cell).  Work unit: an 8 x 8 "mini-tile" of a view plus a 64-bit mask of its nodes
// whose T(V) can change in this sweep (a node of their 3 x 3 neighbourhood changed in
// the previous one).  Every sweep the resident grid walks the list of mini-tiles with a
// nonzero mask, a warp per mini-tile: it stages the 10 x 10 block of V^n around it in
// shared memory, evaluates the listed nodes two per lane (FFMA2, the same per-node
// arithmetic as k_sweep_local2d: bit-identical iterates), writes V^{n+1}, and ORs the
// 3 x 3 dilation of its changed nodes into the masks of the 9 surrounding mini-tiles
// for sweep n+1 — a mini-tile whose mask was empty is appended to the next list.  Then
// one grid-wide barrier (coop_grid_barrier: a monotone arrival counter); at the start of
// sweep n+1 every CTA reads the per-view residuals of sweep n together with its mask
// scan and applies the stopping rule itself before any evaluation (identical decisions
// everywhere), so the host never waits per sweep.  No halo is recomputed, no tile is
// visited whose nodes cannot change, and the node-level work is spread over all SMs
// every sweep.  (Opt-in cluster mode, HJ_COOP_CLUSTER=1: one thread-block cluster per
// view with the hardware cluster barrier — measured slower.)
//
// Nodes not recomputed hold the same value in both buffers (they did not change in the
// previous sweep either), so nothing is copied; the final iterate of view v is in
// V[stop_v & 1], stop_v = the first n with res[n-1] < tol (or max_iter).
#pragma once

#include <cooperative_groups.h>

#ifndef HJ_SEG_UNROLL
#define HJ_SEG_UNROLL 4      // the segmented control loop (2: +1.6 %, 8: +6 %; balance_ab.txt)
#endif

namespace hj {
constexpr int kSegUnroll = HJ_SEG_UNROLL;

// keep a value in a register as computed (stops the compiler from re-deriving it from
// its inputs inside a loop, which it otherwise does under register pressure)
__device__ __forceinline__ void opaque(float &x) { asm volatile("" : "+f"(x)); }
__device__ __forceinline__ void opaque(double &x) { asm volatile("" : "+d"(x)); }

struct CoopState {
    int64_t mt_base[HJ_GROUP_VIEWS + 1];   // first global mini-tile id of each view
    int32_t mt0[HJ_GROUP_VIEWS], mt1[HJ_GROUP_VIEWS], mt2[HJ_GROUP_VIEWS];
    unsigned long long *imask;      // [total] fast interior nodes (class -1)
    unsigned long long *emask;      // [total] interior nodes on the box edge (class -3)
    unsigned long long *dmask[2];   // [total] nodes to evaluate in sweep n (parity n)
    int32_t *items[2];              // [total] mini-tiles with a nonzero mask (parity n)
    int32_t *count;                 // [3] ring: sweep n reads count[n % 3]; [3] the grid
                                    // barrier
    int64_t *stop;                  // [n_views] iterations performed (output)
    int use_list;                   // 1: walk items/count (many mini-tiles); 0: scan all
    int dubins;                     // 3-D Dubins views: 8 x 8 mini-tiles per heading plane
    int n_views;
    int64_t total;
    int32_t vorder[HJ_GROUP_VIEWS];   // cluster mode: views by decreasing size
    int cluster;                    // 1: cluster mode (k_sweep_local2d_coop<..., CL>)
    // field class with a drift along axis 0 only and no speed field (config 3): the sign
    // of d1 is the control's, so the controls are kept as two groups (u1 >= 0, then
    // u1 < 0), each sorted by u0 — d0 < 0 on a prefix of each (coop_eval_field)
    int seg, seg_nup;
    int seg_prune;                  // 1: skip segments by their corner bound (exact)
    int seg_tab;                    // 1: the per-row split points are tabulated in dynamic
                                    // shared memory once per launch (2 x n1 int16)
    // load balance inside a CTA: the last qsingle items of its queue are claimed one at a
    // time instead of in pairs (a finer tail in front of the CTA barrier)
    int qsingle;
    int heavy;                      // queue order: items with more than `heavy` listed nodes
                                    // first (-1: every item, i.e. the list's own order)
    int16_t seg_order[HJ_MAX_CONTROLS];
};

// one entry of the segmented control table (shared memory)
#ifndef HJ_SEG_VEC
#define HJ_SEG_VEC 0       // (1: one 64-bit load per control — measured 1 % slower on config 3)
#endif
#if HJ_SEG_VEC
template <typename T>
struct __align__(2 * sizeof(T)) SegCtl {
    T u0, w1;                  // one 64-bit (fp32) shared load per control
};
#else
template <typename T>
struct SegCtl {
    T u0, w1;
};
#endif

__device__ __forceinline__ int coop_view(const CoopState &S, int64_t gid) {
    int v = 0;
    while (v + 1 < S.n_views && S.mt_base[v + 1] <= gid) ++v;
    return v;
}

// the same for a warp-uniform gid, from a shared copy of mt_base: lane v tests view v+1
// (one shared load and a ballot instead of a serial walk over the parameter bank)
__device__ __forceinline__ int coop_view_warp(const int32_t *__restrict__ smtb, int nv, int gid) {
    const int lane = threadIdx.x & 31;
    return __popc(__ballot_sync(0xffffffffu, lane + 1 < nv && smtb[lane + 1] <= gid));
}

// classes of the mini-tiles of every view: one thread per mini-tile
template <typename T>
__global__ void k_coop_masks(const SweepGroup<T> *__restrict__ G, CoopState S, int64_t gn0,
                             int64_t gn1) {
    for (int64_t gid = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gid < S.total;
         gid += (int64_t)gridDim.x * blockDim.x) {
        const int v = coop_view(S, gid);
        const SweepView<T> &vw = G->v[v];
        const int64_t mt = gid - S.mt_base[v];
        const int mx = (int)(mt % S.mt0[v]);
        const int my = (int)((mt / S.mt0[v]) % S.mt1[v]);
        const int mz = (int)(mt / ((int64_t)S.mt0[v] * S.mt1[v]));
        unsigned long long im = 0, em = 0;
        for (int b = 0; b < 64; ++b) {
            const int64_t li = (int64_t)mx * 8 + (b & 7), lj = (int64_t)my * 8 + (b >> 3);
            if (li >= vw.vn[0] || lj >= vw.vn[1]) continue;
            if (vw.cls[li + vw.vn[0] * (lj + vw.vn[1] * mz)] != -1) continue;
            const int64_t g0 = li + vw.o[0], g1 = lj + vw.o[1];
            if (!S.dubins && (g0 == 0 || g1 == 0 || g0 == gn0 - 1 || g1 == gn1 - 1))
                em |= 1ull << b;   // (Dubins nodes apply the box rule themselves)
            else
                im |= 1ull << b;
        }
        S.imask[gid] = im;
        S.emask[gid] = em;
        S.dmask[0][gid] = im | em;     // sweep 0 evaluates every interior node
        S.dmask[1][gid] = 0;
        if (S.use_list && (im | em)) S.items[0][atomicAdd(&S.count[0], 1)] = (int32_t)gid;
    }
}

// the 3 x 3 dilation of an 8 x 8 change mask (bit = 8 row + col), restricted to the
// mini-tile at offset (dx, dy) in {-1, 0, 1}^2
__device__ __forceinline__ unsigned long long coop_spread(unsigned long long cm, int dx, int dy) {
    const unsigned long long C0 = 0x0101010101010101ull, C7 = 0x8080808080808080ull;
    const unsigned long long h = cm | ((cm << 1) & ~C0) | ((cm >> 1) & ~C7);
    unsigned long long x;
    if (dx == 0) {
        x = h;                                       // columns stay
    } else if (dx == 1) {
        x = (cm & C7) >> 7;                          // our column 7 -> their column 0
    } else {
        x = (cm & C0) << 7;                          // our column 0 -> their column 7
    }
    const unsigned long long v = x | (x << 8) | (x >> 8);   // rows +-1
    if (dy == 0) return v;
    if (dy == 1) return (x >> 56) & 0xffull;                 // our row 7 -> their row 0
    return (x & 0xffull) << 56;                              // our row 0 -> their row 7
}

// Phase B of one mini-tile: the listed nodes of block b (10 x 10, V^n staged), speeds
// sp[64] (staged), classes masks di (interior) / de (box edge).  Writes V^{n+1} and
// returns, per lane, the changed-node bits, the residual and the evaluated count.
template <typename T, int KQ, bool PC>
__device__ __forceinline__ void coop_eval(const DevProblem<T, T> &P, const LocalCtrl<T> &C,
                                          const SweepView<T> &vw, const T *__restrict__ b,
                                          const T *__restrict__ spd, int8_t *lstw,
                                          const T *__restrict__ sctl,
                                          unsigned long long di, unsigned long long de,
                                          int64_t x0, int64_t y0, T *__restrict__ Vo,
                                          T &rmax_out, unsigned long long &cm_out,
                                          int &evald_out) {
    constexpr int BP = 10;
    const int lane = threadIdx.x & 31;
    const bool mono = P.monotone != 0;
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    const T beta = P.beta, v_out = P.v_out;
    const int64_t gn0 = P.n[0], gn1 = P.n[1];
    const int64_t vn0 = vw.vn[0];
    // compact the interior nodes: lane l takes bits l and l+32
    const unsigned lt = (1u << lane) - 1u;
    const unsigned dlo = (unsigned)di, dhi = (unsigned)(di >> 32);
    const int plo = __popc(dlo), nI = plo + __popc(dhi);
    if ((dlo >> lane) & 1u) lstw[__popc(dlo & lt)] = (int8_t)lane;
    if ((dhi >> lane) & 1u) lstw[plo + __popc(dhi & lt)] = (int8_t)(32 + lane);
    __syncwarp();
            T rmax = T(0);
    unsigned long long cm = 0;             // changed nodes (bit = local index)
    int evald = 0;
    if (nI > 0) {
    int loc[2];
    bool valid[2];
    T C0[2], V00[2], best[2];
    Pr<T> bs, bss, nb[9];
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        valid[p] = lane + 32 * p < nI;
        loc[p] = valid[p] ? (int)lstw[lane + 32 * p] : 0;
        const int r = loc[p] >> 3, c = loc[p] & 7;
        const T *q0 = b + (r + 1) * BP + (c + 1);
#pragma unroll
        for (int e = 0; e < 9; ++e) {
            const T val = q0[(e / 3 - 1) * BP + (e % 3 - 1)];
            if (p == 0) nb[e].x = val; else nb[e].y = val;
        }
        V00[p] = p == 0 ? nb[4].x : nb[4].y;
        const int64_t g0 = x0 + c + vw.o[0], g1 = y0 + r + vw.o[1];
        T base = P.kcost;
        if (!kruz) {
            const T x[3] = {fma((T)g0, P.dx[0], P.lo[0]), fma((T)g1, P.dx[1], P.lo[1]),
                            T(0)};
            base = P.h * cost_state(P, x);
        }
        C0[p] = fma(beta, V00[p], base);
        const T sc = spd[loc[p]];
        const T b1 = beta * sc;
        if (p == 0) { bs.x = b1; bss.x = b1 * sc; } else { bs.y = b1; bss.y = b1 * sc; }
        best[p] = mono ? V00[p] : (T)INFINITY;
    }
    {   // quadrant coefficients, both nodes per instruction (k_sweep_local2d order)
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
        const int r = loc[p] >> 3, c = loc[p] & 7;
        const T vnew = best[p];
        Vo[(x0 + c) + vn0 * (y0 + r)] = vnew;
        ++evald;
        if (!same_bits(vnew, V00[p])) {
            cm |= 1ull << loc[p];
            const T dv = vnew > V00[p] ? vnew - V00[p] : V00[p] - vnew;
            rmax = dv > rmax ? dv : rmax;
        }
    }
    }
    // box-edge nodes (R3): 8 at a time, 4 lanes per node (one per quadrant, all its
    // controls)
    const int nE = __popcll(de);
    if (nE > 0) {
    const int sg = lane >> 2, qd = lane & 3;
    const unsigned elo = (unsigned)de, ehi = (unsigned)(de >> 32);
    const int pel = __popc(elo);
    for (int e0 = 0; e0 < nE; e0 += 8) {
        // this group's node: the (e0 + sg)-th set bit of de
        const int gi = e0 + sg;
        const bool ok = gi < nE;
        const int loc = !ok ? 0 : gi < pel ? (int)__fns(elo, 0, gi + 1)
                                           : 32 + (int)__fns(ehi, 0, gi - pel + 1);
        const int r = loc >> 3, c = loc & 7;
        const T *sp = b + (r + 1) * BP + (c + 1);
        const int64_t g0 = x0 + c + vw.o[0], g1 = y0 + r + vw.o[1];
        T base = P.kcost;
        if (!kruz) {
            const T x[3] = {fma((T)g0, P.dx[0], P.lo[0]), fma((T)g1, P.dx[1], P.lo[1]),
                            T(0)};
            base = P.h * cost_state(P, x);
        }
        const T eV00 = sp[0];
        const T eC0 = fma(beta, eV00, base);
        const T e_sc = spd[loc];
        const bool lx = g0 == 0, hx = g0 == gn0 - 1, ly = g1 == 0, hy = g1 == gn1 - 1;
        T e_best = (T)INFINITY;
        {
            const T Vx = (qd & 1) ? sp[-1] : sp[1];
            const T Vy = (qd & 2) ? sp[-BP] : sp[BP];
            const T Vxy = sp[((qd & 2) ? -BP : BP) + ((qd & 1) ? -1 : 1)];
            const bool ex = (qd & 1) ? lx : hx, ey = (qd & 2) ? ly : hy;
            const T Dx = beta * (Vx - eV00), Dy = beta * (Vy - eV00);
            const T Dxy = beta * ((Vxy - Vx) - (Vy - eV00));
            const T c_out = fma(beta, v_out, base);
            const T eps = (T)BOX_EPS;
            // (the control tables from shared memory: qd differs across the lanes, a
            // lane-divergent constant-bank read would serialise)
            const T *__restrict__ tax = sctl + qd * KQ, *__restrict__ tay = sctl + (4 + qd) * KQ;
            const T *__restrict__ tck = sctl + (8 + qd) * KQ;
#pragma unroll 8
            for (int k = 0; k < KQ; ++k) {
                T wx = e_sc * tax[k], wy = e_sc * tay[k];
                const T ck = PC ? tck[k] : T(0);
                const bool out = (ex && wx > eps) || (ey && wy > eps);
                if (ex) wx = T(0);
                if (ey) wy = T(0);
                const T in = fma(wy, fma(wx, Dxy, Dy), fma(wx, Dx, eC0)) + ck;
                e_best = fmin(e_best, out ? c_out + ck : in);
            }
        }
        e_best = fmin(e_best, __shfl_xor_sync(0xffffffffu, e_best, 1));
        e_best = fmin(e_best, __shfl_xor_sync(0xffffffffu, e_best, 2));
        if (ok && qd == 0) {
            const T vnew = mono ? fmin(e_best, eV00) : e_best;
            Vo[(x0 + c) + vn0 * (y0 + r)] = vnew;
            ++evald;
            if (!same_bits(vnew, eV00)) {
                cm |= 1ull << loc;
                const T dv = vnew > eV00 ? vnew - eV00 : eV00 - vnew;
                rmax = dv > rmax ? dv : rmax;
            }
        }
    }
    }
    rmax_out = rmax;
    cm_out = cm;
    evald_out = evald;
}

// Phase B for the FIELD class with every foot within one cell (|delta_d| <= 1, e.g. the
// Zermelo drift of config 3): per control the foot's cell is the quadrant given by the
// signs of its offsets, so the bilinear interpolant is
//   V00 + |d0| D0(s0) + |d1| (D1(s1) + |d0| D01(s0,s1))
// with the node's 4 one-sided and 4 cross differences (prescaled by beta) selected by
// sign — no floor, no index arithmetic.  Box-edge nodes (class -3) take the general R3
// interpolation (interp()) on the global V^n, as k_sweep_field2d's slow path.
template <typename T, int DYN>
__device__ __forceinline__ void coop_eval_field(const DevProblem<T, T> &P, const SweepView<T> &vw,
                                                const T *__restrict__ Vi, const T *__restrict__ b,
                                                const T *__restrict__ spd, int8_t *lstw,
                                                unsigned long long di, unsigned long long de,
                                                int64_t x0, int64_t y0, T *__restrict__ Vo,
                                                T &rmax_out, unsigned long long &cm_out,
                                                int &evald_out, const SegCtl<T> *__restrict__ seg,
                                                const T *__restrict__ seg_csq, int seg_nup,
                                                int16_t *__restrict__ rsplit,
                                                const int16_t *__restrict__ seg_tab,
                                                T seg_w1max) {
    constexpr int BP = 10;
    const int lane = threadIdx.x & 31;
    const bool mono = P.monotone != 0;
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    const T beta = P.beta;
    const int64_t vn0 = vw.vn[0];
    const T hlr = P.h * P.lr;
    // every listed node (interior and box edge) is one lane-slot: lane l takes the l-th
    // and (l+32)-th set bit of di | de
    const unsigned long long dall = di | de;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned dlo = (unsigned)dall, dhi = (unsigned)(dall >> 32);
    const int plo = __popc(dlo), nN = plo + __popc(dhi);
    if ((dlo >> lane) & 1u) lstw[__popc(dlo & lt)] = (int8_t)lane;
    if ((dhi >> lane) & 1u) lstw[plo + __popc(dhi & lt)] = (int8_t)(32 + lane);
    if (DYN == HJ_DYN_AFFINE && seg && lane < 16) {
        // segmented mode (the drift moves along axis 0 only and does not depend on x0, no
        // speed field): d0 depends on the row only, so the two split points of each of the
        // mini-tile's 8 rows are found once (lanes 0-15: row lane & 7, group lane >> 3)
        const int rr = lane & 7, grp = lane >> 3;
        const T xx0 = fma((T)(x0 + vw.o[0]), P.dx[0], P.lo[0]);
        const T xx1 = fma((T)(y0 + rr + vw.o[1]), P.dx[1], P.lo[1]);
        const T D0r = P.hdx[0] * fma(P.A[0], xx0, fma(P.A[1], xx1, P.b[0]));
        const T S0r = P.hdx[0] * T(1);
        int lo = grp ? seg_nup : 0, hi = grp ? P.K : seg_nup;
        if (seg_tab) {
            // (a mini-tile row past the grid holds no node: clamp, the value is unused)
            lo = seg_tab[grp * (int)P.n[1] + min((int)(y0 + rr + vw.o[1]), (int)P.n[1] - 1)];
        } else {
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (fma(S0r, seg[mid].u0, D0r) < T(0)) lo = mid + 1; else hi = mid;
            }
        }
        rsplit[lane] = (int16_t)lo;
    }
    __syncwarp();
    T rmax = T(0);
    unsigned long long cm = 0;
    int evald = 0;
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {
        const int slot = lane + 32 * p;
        if (slot >= nN) continue;
        const int loc = lstw[slot];
        const int r = loc >> 3, c = loc & 7;
        const T *q0 = b + (r + 1) * BP + (c + 1);
        const T V00 = q0[0];
        const int64_t gi[3] = {x0 + c + vw.o[0], y0 + r + vw.o[1], 0};
        const T xx0 = fma((T)gi[0], P.dx[0], P.lo[0]), xx1 = fma((T)gi[1], P.dx[1], P.lo[1]);
        T D0, D1, S0, S1;
        if (DYN == HJ_DYN_AFFINE) {
            const T cs = spd[loc];
            D0 = P.hdx[0] * fma(P.A[0], xx0, fma(P.A[1], xx1, P.b[0]));
            D1 = P.hdx[1] * fma(P.A[3], xx0, fma(P.A[4], xx1, P.b[1]));
            S0 = P.hdx[0] * cs;
            S1 = P.hdx[1] * cs;
        } else {
            D0 = P.hdx[0] * xx1;
            D1 = P.hdx[1] * fma(P.vdp_mu * (T(1) - xx0 * xx0), xx1, -xx0);
            S0 = T(0);
            S1 = P.hdx[1];
        }
        T base = P.kcost;
        if (!kruz) {
            const T x[3] = {xx0, xx1, T(0)};
            base = P.h * cost_state(P, x);
        }
        T best = mono ? V00 : (T)INFINITY;
        int nb = P.K;            // brackets computed for this node (segment pruning: fewer)
        if ((di >> loc) & 1ull) {
            // one-sided and cross differences, prescaled by beta
            const T Vp0 = q0[1], Vm0 = q0[-1], V0p = q0[BP], V0m = q0[-BP];
            const T Dxp = beta * (Vp0 - V00), Dxm = beta * (Vm0 - V00);
            const T Dyp = beta * (V0p - V00), Dym = beta * (V0m - V00);
            const T X00 = beta * ((q0[BP + 1] - Vp0) - (V0p - V00));    // +x +y
            const T X10 = beta * ((q0[BP - 1] - Vm0) - (V0p - V00));    // -x +y
            const T X01 = beta * ((q0[-BP + 1] - Vp0) - (V0m - V00));   // +x -y
            const T X11 = beta * ((q0[-BP - 1] - Vm0) - (V0m - V00));   // -x -y
            const T C0 = fma(beta, V00, base);
            if (DYN == HJ_DYN_AFFINE && seg) {
                // segmented control loop (CoopState::seg): per group, the controls with
                // d0 = fma(S0, u0, D0) < 0 are a prefix of the u0-sorted order (fma is
                // monotone in u0 for S0 > 0); each of the four (group, side) segments has
                // fixed differences — the same bracket fma(w1, fma(w0, A3, A2),
                // fma(w0, A1, ck)) per control as the select loop below, no sign tests
                const int K = P.K;
                const int bnd[5] = {0, rsplit[r], seg_nup, rsplit[8 + r], K};
                // segment pruning (exact): on a segment the bracket is the bilinear form
                // ck + w0 A1 + w1 (A2 + w0 A3) of (w0, w1) in the box [w0 of its first and
                // last control] x [0, max w1] (w0 is monotone along the segment), so its
                // minimum over the segment is at least the smallest of the box's four
                // corners; with ck >= C0 (hlr >= 0) a segment whose corner bound, less
                // a rounding slack that covers both the corners' and the brackets' own
                // fp rounding, is not below the running best cannot change
                // the min — skipped.  With the monotone clamp the best starts at V00, so
                // the quadrants whose cell rises from V00 go first.
                const bool prune = seg_w1max >= T(0) && (kruz || hlr >= T(0));
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    // q = 0: -x +y, 1: +x +y, 2: -x -y, 3: +x -y
                    const T A1 = (q & 1) ? Dxp : Dxm;
                    const T A2 = (q & 2) ? Dym : Dyp;
                    const T A3 = q == 0 ? X10 : (q == 1 ? X00 : (q == 2 ? X11 : X01));
                    if (prune && bnd[q] < bnd[q + 1]) {
                        const T wa = fabs(fma(S0, seg[bnd[q]].u0, D0));
                        const T wb = fabs(fma(S0, seg[bnd[q + 1] - 1].u0, D0));
                        const T ca = fma(wa, A1, C0), cb = fma(wb, A1, C0);
                        const T da = fma(seg_w1max, fma(wa, A3, A2), ca);
                        const T db = fma(seg_w1max, fma(wb, A3, A2), cb);
                        const T lb = fmin(fmin(ca, cb), fmin(da, db));
                        const T slack = (fabs(C0) + fabs(A1) + fabs(A2) + fabs(A3)) *
                                        T(9.5367431640625e-07);        // 2^-20
                        if (lb - slack >= best) {
                            nb -= bnd[q + 1] - bnd[q];
                            continue;
                        }
                    }
#pragma unroll(kSegUnroll)
                    for (int k = bnd[q]; k < bnd[q + 1]; ++k) {
                        const T w0 = fabs(fma(S0, seg[k].u0, D0));
                        const T ck = kruz ? C0 : C0 + hlr * seg_csq[k];
                        best = fmin(best, fma(seg[k].w1, fma(w0, A3, A2), fma(w0, A1, ck)));
                    }
                }
            } else {
            T dx8[8] = {Dxp, Dxm, Dyp, Dym, X00, X10, X01, X11};
#pragma unroll
            for (int e = 0; e < 8; ++e) opaque(dx8[e]);
#pragma unroll 4
            for (int k = 0; k < P.K; ++k) {
                const T d0 = DYN == HJ_DYN_AFFINE ? fma(S0, P.ctrl[k][0], D0) : D0;
                const T d1 = fma(S1, P.ctrl[k][DYN == HJ_DYN_AFFINE ? 1 : 0], D1);
                const bool nx = d0 < T(0), ny = d1 < T(0);
                const T A1 = nx ? dx8[1] : dx8[0], A2 = ny ? dx8[3] : dx8[2];
                const T A3 = ny ? (nx ? dx8[7] : dx8[6]) : (nx ? dx8[5] : dx8[4]);
                const T w0 = fabs(d0), w1 = fabs(d1);
                const T ck = kruz ? C0 : C0 + hlr * P.csq[k];
                best = fmin(best, fma(w1, fma(w0, A3, A2), fma(w0, A1, ck)));
            }
            }
        } else {
            // box edge (R3): interp()'s arithmetic step for step (box test, clamp onto the
            // box, floor, weights, the last-cell rule, three lerps), the corners read from
            // the staged block — it holds V^n of the view and v_out outside it, exactly
            // what interp()'s view_fetch returns.  A corner one past the block only occurs
            // with weight 0 (foot offset exactly +1), where any finite value gives the same
            // lerp, so its index is clamped.  Offsets beyond one cell (not expected for the
            // class) take interp() on the global V^n.
            const int64_t o[3] = {vw.o[0], vw.o[1], 0};
            const int64_t vn[3] = {vw.vn[0], vw.vn[1], 1};
            const T eps = (T)BOX_EPS;
            const T lo0 = -(T)gi[0], hi0 = (T)(P.n[0] - 1 - gi[0]);
            const T lo1 = -(T)gi[1], hi1 = (T)(P.n[1] - 1 - gi[1]);
            T eb = (T)INFINITY;
#pragma unroll 1
            for (int k = 0; k < P.K; ++k) {
                const T e0 = DYN == HJ_DYN_AFFINE ? fma(S0, P.ctrl[k][0], D0) : D0;
                const T e1 = fma(S1, P.ctrl[k][DYN == HJ_DYN_AFFINE ? 1 : 0], D1);
                T I;
                if (!(e0 >= lo0 - eps && e0 <= hi0 + eps) || !(e1 >= lo1 - eps && e1 <= hi1 + eps)) {
                    I = P.v_out;
                } else {
                    const T xa = e0 < lo0 ? lo0 : (e0 > hi0 ? hi0 : e0);
                    const T xb = e1 < lo1 ? lo1 : (e1 > hi1 ? hi1 : e1);
                    const T fa = floor(xa), fb = floor(xb);
                    if (fa < T(-1) || fa > T(1) || fb < T(-1) || fb > T(1)) {
                        const T delta[3] = {e0, e1, T(0)};
                        I = interp<T, T, 2>(Vi, o, vn, P.n, P.periodic, gi, delta, P.v_out);
                    } else {
                        int ca = (int)fa, cb = (int)fb;
                        T wa = xa - fa, wb = xb - fb;
                        if (gi[0] + ca > P.n[0] - 2) {
                            ca = (int)(P.n[0] - 2 - gi[0]);
                            wa = T(1);
                        }
                        if (gi[1] + cb > P.n[1] - 2) {
                            cb = (int)(P.n[1] - 2 - gi[1]);
                            wb = T(1);
                        }
                        const int ba = c + 1 + ca, bb = r + 1 + cb;      // block col / row
                        const int ba1 = min(ba + 1, BP - 1), bb1 = min(bb + 1, BP - 1);
                        const T a = lerp<T>(b[bb * BP + ba], b[bb * BP + ba1], wa);
                        const T a2 = lerp<T>(b[bb1 * BP + ba], b[bb1 * BP + ba1], wa);
                        I = lerp<T>(a, a2, wb);
                    }
                }
                const T ck = kruz ? base : fma(hlr, P.csq[k], base);
                eb = fmin(eb, fma(beta, I, ck));
            }
            best = mono ? fmin(eb, V00) : eb;
        }
        Vo[(x0 + c) + vn0 * (y0 + r)] = best;
        evald += nb;
        if (!same_bits(best, V00)) {
            cm |= 1ull << loc;
            const T dv = best > V00 ? best - V00 : V00 - best;
            rmax = dv > rmax ? dv : rmax;
        }
    }
    rmax_out = rmax;
    cm_out = cm;
    evald_out = evald;
}

// Phase B for the Dubins car (config 4): the listed nodes of one 8 x 8 mini-tile of
// heading plane z, with the 10 x 10 blocks of planes z-1, z, z+1 staged (b[0..299]).
// Same arithmetic as k_sweep_dubins: the (x, y) foot h v (cos th, sin th) is the same
// for all controls (box rule R3 once per node), three bilinear interpolants, then per
// control I0 + |d_k| (I+-1 - I0).
template <typename T>
__device__ __forceinline__ void coop_eval_dubins(const DevProblem<T, T> &P, const SweepView<T> &vw,
                                                 const T *__restrict__ b, int8_t *lstw,
                                                 unsigned long long di, int64_t x0, int64_t y0,
                                                 int64_t z, T d0, T d1, T *__restrict__ Vo,
                                                 const T *__restrict__ wext,
                                                 T &rmax_out, unsigned long long &cm_out,
                                                 int &evald_out) {
    constexpr int BP = 10;
    const int lane = threadIdx.x & 31;
    const bool mono = P.monotone != 0;
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    const T beta = P.beta;
    const int64_t vn0 = vw.vn[0], vn1 = vw.vn[1];
    const T hlr = P.h * P.lr;
    const unsigned lt = (1u << lane) - 1u;
    const unsigned dlo = (unsigned)di, dhi = (unsigned)(di >> 32);
    const int plo = __popc(dlo), nN = plo + __popc(dhi);
    if ((dlo >> lane) & 1u) lstw[__popc(dlo & lt)] = (int8_t)lane;
    if ((dhi >> lane) & 1u) lstw[plo + __popc(dhi & lt)] = (int8_t)(32 + lane);
    __syncwarp();
    T rmax = T(0);
    unsigned long long cm = 0;
    int evald = 0;
    const T hw = P.hdx[2] * P.dub_w;
#pragma unroll 1
    for (int p = 0; p < 2; ++p) {
        const int slot = lane + 32 * p;
        if (slot >= nN) continue;
        const int loc = lstw[slot];
        const int r = loc >> 3, c = loc & 7;
        const int64_t gi0 = x0 + c + vw.o[0], gi1 = y0 + r + vw.o[1];
        const T *q0 = b + BP * BP + (r + 1) * BP + (c + 1);   // plane z, the node
        const T V00 = q0[0];
        T base = P.kcost;
        if (!kruz) {
            const T x[3] = {fma((T)gi0, P.dx[0], P.lo[0]), fma((T)gi1, P.dx[1], P.lo[1]),
                            fma((T)(z + vw.o[2]), P.dx[2], P.lo[2])};
            base = P.h * cost_state(P, x);
        }
        const T lo0 = -(T)gi0, hi0 = (T)(P.n[0] - 1 - gi0);
        const T lo1 = -(T)gi1, hi1 = (T)(P.n[1] - 1 - gi1);
        const T eps = (T)BOX_EPS;
        const bool inside = d0 >= lo0 - eps && d0 <= hi0 + eps && d1 >= lo1 - eps &&
                            d1 <= hi1 + eps;
        T best = (T)INFINITY;
        if (!inside) {
            for (int k = 0; k < P.K; ++k) {
                const T ck = kruz ? base : fma(hlr, P.csq[k], base);
                best = fmin(best, fma(beta, P.v_out, ck));
            }
        } else {
            T x = d0 < lo0 ? lo0 : (d0 > hi0 ? hi0 : d0);
            T y = d1 < lo1 ? lo1 : (d1 > hi1 ? hi1 : d1);
            T fx = floor(x), fy = floor(y);
            int64_t cx = gi0 + (int64_t)fx, cy = gi1 + (int64_t)fy;
            T wx = x - fx, wy = y - fy;
            if (cx > P.n[0] - 2) { cx = P.n[0] - 2; wx = T(1); }
            if (cy > P.n[1] - 2) { cy = P.n[1] - 2; wy = T(1); }
            // cell offsets in {-1, 0, 1}: +1 when the foot offset is exactly one cell (h =
            // dx / max|f| puts every foot of the th = 0 and th = pi/2 planes there); then
            // the cell's far corner lies one past the staged block and enters with weight
            // 0, where any finite value gives the same lerp — its index is clamped into
            // the block (reading past it took other warps' data and, at the end of the
            // shared window, faulted: the config-4 nondeterminism of round 2)
            const int rx = (int)(cx - gi0), ry = (int)(cy - gi1);
            const int bx0 = c + 1 + rx, by0 = r + 1 + ry;
            const int bx1 = min(bx0 + 1, BP - 1), by1 = min(by0 + 1, BP - 1);
            T I3[3];
#pragma unroll
            for (int s = 0; s < 3; ++s) {
                const T *pl = b + s * BP * BP;
                const T a = lerp<T>(pl[by0 * BP + bx0], pl[by0 * BP + bx1], wx);
                const T bb = lerp<T>(pl[by1 * BP + bx0], pl[by1 * BP + bx1], wx);
                I3[s] = lerp<T>(a, bb, wy);
            }
            const T dM = I3[0] - I3[1], dP = I3[2] - I3[1];
            if (kruz) {
                // Kruzkov (every control costs the same): within each sign group of
                // d_k = h w a_k / dth the computed bracket fl(beta fl(|d_k| D + I0) + c) is
                // monotone in |d_k| (D = I_{+-1} - I0 fixed, rounding is monotone), so
                // its minimum over the group is at the group's smallest or largest
                // |d_k| — the same min as the loop over all controls, bit for bit.
                // wext: {min, max} |d_k| over d_k >= 0, then over d_k < 0 (+inf / -inf
                // when a group is empty: those candidates never win).
                if (wext[0] <= wext[1]) {
                    best = fmin(best, fma(beta, fma(wext[0], dP, I3[1]), base));
                    best = fmin(best, fma(beta, fma(wext[1], dP, I3[1]), base));
                }
                if (wext[2] <= wext[3]) {
                    best = fmin(best, fma(beta, fma(wext[2], dM, I3[1]), base));
                    best = fmin(best, fma(beta, fma(wext[3], dM, I3[1]), base));
                }
            } else {
#pragma unroll 4
                for (int k = 0; k < P.K; ++k) {
                    const T dk = hw * P.ctrl[k][0];
                    const T I = fma(fabs(dk), dk < T(0) ? dM : dP, I3[1]);
                    const T ck = fma(hlr, P.csq[k], base);
                    best = fmin(best, fma(beta, I, ck));
                }
            }
        }
        if (mono) best = fmin(best, V00);
        Vo[(x0 + c) + vn0 * ((y0 + r) + vn1 * z)] = best;
        ++evald;
        if (!same_bits(best, V00)) {
            cm |= 1ull << loc;
            const T dv = best > V00 ? best - V00 : V00 - best;
            rmax = dv > rmax ? dv : rmax;
        }
    }
    rmax_out = rmax;
    cm_out = cm;
    evald_out = evald;
}

// Grid-wide barrier of the resident (cooperative) grid on a monotone arrival counter
// (zeroed before the launch): thread 0 of each CTA publishes the CTA's writes (fence),
// adds its arrival without waiting for a reply, and polls until all gridDim.x arrivals
// of barrier n+1 are in.  One round trip less than a generation-flip barrier whose
// arrival atomic returns.  The acquire load invalidates the SM's L1, so the CTA's reads
// after the barrier see the other CTAs' writes.
__device__ __forceinline__ void coop_grid_barrier(unsigned *ctr, unsigned target) {
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while ((int)(v - target) < 0);
    }
    __syncthreads();
}

template <typename T>
struct CoopBits;
template <>
struct CoopBits<float> {
    using U = unsigned;
    static __device__ __forceinline__ U bits(float x) { return __float_as_uint(x); }
    static __device__ __forceinline__ float value(U b) { return __uint_as_float(b); }
};
template <>
struct CoopBits<double> {
    using U = unsigned long long;
    static __device__ __forceinline__ U bits(double x) { return (U)__double_as_longlong(x); }
    static __device__ __forceinline__ double value(U b) { return __longlong_as_double((long long)b); }
};

#ifndef HJ_COOP_DUBINS_MINB
#define HJ_COOP_DUBINS_MINB 2   // resident 512-thread CTAs per SM asked of ptxas, Dubins class
#endif
#ifndef HJ_COOP_DUBINS_DYNQ
#define HJ_COOP_DUBINS_DYNQ 1   // the Dubins class claims pairs from the CTA queue too (0: the
                                // static split (w, w + NW), ...: config 4 99.8 vs 89.2 ms)
#endif
#ifndef HJ_COOP_TRACE
#define HJ_COOP_TRACE 0      // 1: per-sweep phase timestamps (tools/coop_trace.py, a variant build)
#endif

// warps per CTA: fp32 one 512-thread CTA per SM (fewer barrier arrivals); fp64 (its
// staged blocks are twice the size) two 256-thread CTAs per SM
#ifndef HJ_COOP_MINB32
#define HJ_COOP_MINB32 1     // resident 512-thread CTAs per SM asked of ptxas for fp32
#endif
#ifndef HJ_COOP_NP
#define HJ_COOP_NP 2           // items per claim at the front of a CTA's queue, field class
#endif
#ifndef HJ_COOP_NP_LOCAL
#define HJ_COOP_NP_LOCAL 1     // the same for the local class
#endif
#ifndef HJ_COOP_NW32
#define HJ_COOP_NW32 16      // warps per CTA for fp32
#endif
template <typename T>
struct CoopNW {
    static constexpr int nw = sizeof(T) == 4 ? HJ_COOP_NW32 : 8;
    static constexpr int minb = sizeof(T) == 4 ? HJ_COOP_MINB32 : 2;
};

// EV: 0 = local class (LocalCtrl, FFMA2 quadrants), HJ_DYN_AFFINE + 1 / HJ_DYN_VANDERPOL + 1
// = field class with feet within one cell, 3 = Dubins (3-D, heading planes)
// CL: cluster mode — each thread-block cluster solves whole views on its own (views
// are independent problems until the gather): view vorder[c], vorder[c + #clusters], ...
// for cluster c, with the hardware cluster barrier between sweeps instead of the
// grid-wide one.
template <typename T, int KQ, bool PC, int EV = 0, bool CL = false>
// (Dubins, EV 3: two 512-thread CTAs per SM at 64 registers measured 10 % faster on
// config 4; the 2-D classes spill and lose at 64 registers — profiles/r2/occupancy_r2j.txt)
__global__ void __launch_bounds__(CoopNW<T>::nw * 32,
                                  EV == 3 && CoopNW<T>::nw <= 16 ? HJ_COOP_DUBINS_MINB : CoopNW<T>::minb)
    k_sweep_local2d_coop(const DevProblem<T, T> P, const LocalCtrl<T> C,
                         const SweepGroup<T> *__restrict__ G, const CoopState S,
                         int64_t max_iter, double tol) {
    constexpr int COOP_NW = CoopNW<T>::nw;
    constexpr int BP = 10;                         // staged block pitch
    constexpr int BLK = EV == 3 ? 3 * BP * BP : BP * BP;   // Dubins: planes z-1, z, z+1
    constexpr int SPD = EV == 3 ? 1 : 64;
    // the staged blocks (the largest piece) live in dynamic shared memory
    extern __shared__ __align__(16) unsigned char coop_dyn[];
    T(*blk)[2][BLK] = reinterpret_cast<T(*)[2][BLK]>(coop_dyn);
    __shared__ T spd[COOP_NW][2][SPD];
    __shared__ int8_t lst[COOP_NW][2][64];
    __shared__ int32_t qgid[COOP_NW * 32];
    __shared__ unsigned long long qmask[COOP_NW * 32], qemask[COOP_NW * 32];
    __shared__ int wcnt[COOP_NW];
    __shared__ int qnext;          // the next unclaimed queue position (warps claim pairs)
    // per-CTA max of the sweep's |V^{n+1} - V^n| as the bits of a T >= 0 (monotone as
    // unsigned: native shared atomicMax, no CAS loop), evaluated-node count
    __shared__ typename CoopBits<T>::U cres[HJ_GROUP_VIEWS];
    __shared__ unsigned cwork[HJ_GROUP_VIEWS];
    // the views, copied once: the grid barrier invalidates L1, so reading G every sweep
    // would put a global round trip in front of every dependent load
    __shared__ SweepView<T> sview[HJ_GROUP_VIEWS];
    // local class: the quadrant control tables ax | ay | ck, [3][4][KQ]
    __shared__ T sctl[EV == 0 ? 12 * KQ : 1];
    // field class, drift along axis 0 only: the segmented control table (CoopState::seg)
    __shared__ SegCtl<T> sseg[EV == 1 ? HJ_MAX_CONTROLS : 1];
    __shared__ T sseg_csq[EV == 1 ? HJ_MAX_CONTROLS : 1];
    __shared__ int16_t srsplit[EV == 1 ? COOP_NW : 1][16];   // per warp: the row splits
    if (EV == 1 && S.seg)
        for (int i = threadIdx.x; i < P.K; i += blockDim.x) {
            const int k = S.seg_order[i];
            sseg[i].u0 = P.ctrl[k][0];
            sseg[i].w1 = fabs(fma(P.hdx[1] * T(1), P.ctrl[k][1], T(0)));
            sseg_csq[i] = P.csq[k];
        }
    // segment pruning (coop_eval_field): the largest axis-1 weight of any control
    __shared__ T sseg_w1max;
    if (EV == 1 && S.seg) {
        __syncthreads();                       // (sseg complete)
        if (threadIdx.x == 0) {
            T m = T(0);
            for (int i = 0; i < P.K; ++i) m = fmax(m, sseg[i].w1);
            sseg_w1max = m;
        }
    }
    // segmented mode: the two split points of every global row, tabulated once (behind the
    // blocks in dynamic shared memory).  d0 = fma(S0, u0, D0) with D0 a function of the row
    // alone (A[0][0] = 0: fma(0, x0, y) is y for every finite x0, so x0 = lo0 stands in)
    int16_t *const segtab = reinterpret_cast<int16_t *>(coop_dyn + sizeof(T) * COOP_NW * 2 * BLK);
    if (EV == 1 && S.seg && S.seg_tab) {
        __syncthreads();                       // (sseg complete)
        const int n1 = (int)P.n[1];
        for (int e = threadIdx.x; e < 2 * n1; e += blockDim.x) {
            const int grp = e >= n1, row = e - grp * n1;
            const T xx0 = P.lo[0];
            const T xx1 = fma((T)row, P.dx[1], P.lo[1]);
            const T D0r = P.hdx[0] * fma(P.A[0], xx0, fma(P.A[1], xx1, P.b[0]));
            const T S0r = P.hdx[0] * T(1);
            int lo = grp ? S.seg_nup : 0, hi = grp ? P.K : S.seg_nup;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (fma(S0r, sseg[mid].u0, D0r) < T(0)) lo = mid + 1; else hi = mid;
            }
            segtab[e] = (int16_t)lo;
        }
    }
    // the views' mini-tile numbering, in shared memory (warp-uniform lookups by ballot)
    __shared__ int32_t smtb[HJ_GROUP_VIEWS + 1], smt0[HJ_GROUP_VIEWS], smt1[HJ_GROUP_VIEWS],
        smt2[HJ_GROUP_VIEWS];
    if (threadIdx.x <= (unsigned)S.n_views) {
        smtb[threadIdx.x] = (int32_t)S.mt_base[threadIdx.x];
        if (threadIdx.x < (unsigned)S.n_views) {
            smt0[threadIdx.x] = S.mt0[threadIdx.x];
            smt1[threadIdx.x] = S.mt1[threadIdx.x];
            smt2[threadIdx.x] = S.mt2[threadIdx.x];
        }
    }
    // Dubins: extreme |h w a_k / dth| of each sign group (coop_eval_dubins)
    __shared__ T dub_wext[4];
    if (EV == 3 && threadIdx.x == 0) {
        const T hw = P.hdx[2] * P.dub_w;
        T e[4] = {(T)INFINITY, -(T)INFINITY, (T)INFINITY, -(T)INFINITY};
        for (int k = 0; k < P.K; ++k) {
            const T dk = hw * P.ctrl[k][0];
            const T w = fabs(dk);
            const int o = dk < T(0) ? 2 : 0;
            e[o] = fmin(e[o], w);
            e[o + 1] = fmax(e[o + 1], w);
        }
        for (int i = 0; i < 4; ++i) dub_wext[i] = e[i];
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < (unsigned)S.n_views) sview[threadIdx.x] = G->v[threadIdx.x];
    // (strided: 12 KQ entries can exceed the block — fp64 runs 256 threads, KQ up to 32)
    if (EV == 0)
        for (int i = threadIdx.x; i < 12 * KQ; i += blockDim.x) {
            const int w = i / (4 * KQ), q = (i / KQ) % 4, k = i % KQ;
            sctl[i] = w == 0 ? C.ax[q][k] : w == 1 ? C.ay[q][k] : C.ck[q][k];
        }
    const bool mono = P.monotone != 0;
    const bool kruz = P.cost == HJ_COST_KRUZKOV;
    const T beta = P.beta, v_out = P.v_out;
    const int64_t gn0 = P.n[0], gn1 = P.n[1];
    const unsigned all = S.n_views >= 32 ? 0xffffffffu : ((1u << S.n_views) - 1u);
    // the CTA group that sweeps together: the whole grid, or (CL) this CTA's cluster
    unsigned grank = blockIdx.x, gsize = gridDim.x, grp = 0, ngrp = 1;
    if constexpr (CL) {
        asm("mov.u32 %0, %%cluster_ctarank;" : "=r"(grank));
        asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(gsize));
        asm("mov.u32 %0, %%clusterid.x;" : "=r"(grp));
        asm("mov.u32 %0, %%nclusterid.x;" : "=r"(ngrp));
    }
    // (debug trace, tools/coop_trace.py: read once — after each barrier a global read
    // would cost an L2 round trip in front of the CTA's arrival)
    unsigned long long *const tr_buf = g_tb_trace.buf;
    const long long tr_cap = g_tb_trace.cap;
    // (compiled in only with -DHJ_COOP_TRACE=1: the timestamps would otherwise hold ~14
    // registers live across the sweep loop)
    const bool tr = HJ_COOP_TRACE && tr_buf != nullptr && blockIdx.x == 0 && threadIdx.x == 0;
    const bool tr_all = HJ_COOP_TRACE && tr_buf != nullptr && threadIdx.x == 0 && gridDim.x <= 256;
    unsigned long long t_a = 0, t_b = 0, t_s = 0, t_l = 0, t_e = 0, t_m = 0, t_q = 0;
    int qitems = 0;
    for (int vs = (int)grp; vs < (CL ? S.n_views : 1); vs += (int)ngrp) {
    const int vsel = CL ? S.vorder[vs] : -1;
    unsigned stopped = CL ? (all & ~(1u << vsel)) : 0u;   // bit v: view v met the rule
    const int64_t cbase = CL ? S.mt_base[vsel] : 0;
    const int64_t ctot = CL ? S.mt_base[vsel + 1] - cbase : S.total;
    int64_t n = 0;
    for (; n < max_iter; ++n) {
        // the stopping rule on res[n-1], applied identically by every warp of every CTA:
        // lane v reads view v's residual here, so that the round trip overlaps the
        // scan's loads; the ballot below (before any evaluation) spreads the decisions
        const bool chk = n > 0 && lane < S.n_views && !((stopped >> lane) & 1u);
        const double rprev = chk ? *(volatile const double *)&sview[lane].res[n - 1] : 0.0;
        bool decided = n == 0;
        if (tr) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_a));
            t_s = t_l = t_e = t_m = t_q = 0;
            qitems = 0;
        }
        if (threadIdx.x < HJ_GROUP_VIEWS) {
            cres[threadIdx.x] = 0;
            cwork[threadIdx.x] = 0u;
        }
        __syncthreads();
        unsigned long long *dcur = S.dmask[n & 1], *dnext = S.dmask[(n + 1) & 1];
        // CTA c owns the mini-tiles c, c + G, c + 2G, ... (strided: the active ones spread
        // over all CTAs).  Chunks of 256 candidates: load their masks, compact the nonzero
        // ones in shared memory, then the warps take two per iteration.
        // (list mode: the candidates are the listed mini-tiles of this sweep instead)
        const int64_t ncand =
            S.use_list ? (int64_t)*(volatile const int32_t *)&S.count[n % 3] : ctot;
        const int32_t *litems = S.items[n & 1];
        const int64_t per_cta = ncand > grank ? (ncand - grank + gsize - 1) / gsize : 0;
        for (int64_t ch = 0; ch < per_cta; ch += COOP_NW * 32) {
        int chunk_n;
        {
            const int64_t k = ch + threadIdx.x;
            const int64_t idx = grank + k * (int64_t)gsize;
            const int64_t g = k < per_cta ? (S.use_list ? (int64_t)litems[idx] : cbase + idx) : 0;
            const unsigned long long m = k < per_cta ? dcur[g] : 0ull;
            // the class masks ride along with the dirty mask (one round trip for all three)
            const unsigned long long cim = k < per_cta ? S.imask[g] : 0ull;
            const unsigned long long cem = k < per_cta ? S.emask[g] : 0ull;
            // the queue is filled from both ends: mini-tiles with more than `heavy` listed
            // nodes from the front (claimed first, in pairs), the lighter ones from the back
            // (they end up in the single-claim tail) — longest first in front of the barrier
            const bool hv = m != 0ull && __popcll(m & (cim | cem)) > S.heavy;
            const unsigned bal = __ballot_sync(0xffffffffu, hv);
            const unsigned ball = __ballot_sync(0xffffffffu, m != 0ull && !hv);
            if (lane == 0) wcnt[warp] = __popc(bal) | (__popc(ball) << 16);
            __syncthreads();
            // this warp's offsets and the chunk's totals: one shared load + two warp
            // reductions (lane w holds warp w's counts, heavy | light << 16)
            const int wc = lane < COOP_NW ? wcnt[lane] : 0;
            const int base_i = __reduce_add_sync(0xffffffffu, lane < warp ? wc : 0);
            const int tot_i = __reduce_add_sync(0xffffffffu, wc);
            chunk_n = (tot_i & 0xffff) + (tot_i >> 16);
            if (m) {
                const unsigned lt = (1u << lane) - 1u;
                const int pos = hv ? (base_i & 0xffff) + __popc(bal & lt)
                                   : chunk_n - 1 - ((base_i >> 16) + __popc(ball & lt));
#ifdef HJ_DEBUG_BOUNDS
                if (pos < 0 || pos >= chunk_n || chunk_n > COOP_NW * 32)
                    printf("HJ_DEBUG queue: n %lld pos %d chunk_n %d\n", (long long)n, pos, chunk_n),
                        __trap();
#endif
                qgid[pos] = (int32_t)g;
                qmask[pos] = m & cim;
                qemask[pos] = m & cem;
                dcur[g] = 0ull;                    // consumed
            }
            if (threadIdx.x == 0) qnext = 0;
            __syncthreads();                       // the queue is complete
        }
        const int cnt = chunk_n;
        if (!decided) {
            const unsigned now = __ballot_sync(0xffffffffu, chk && rprev < tol);
            if (now) {
                if (grank == 0 && threadIdx.x == 0)
                    for (unsigned m = now; m; m &= m - 1) S.stop[__ffs(m) - 1] = n;
                stopped |= now;
            }
            decided = true;
        }
        if (stopped == all) continue;              // (every CTA: the same decision)
        if (tr && t_s == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_s));
        if (tr) qitems += cnt;
        // two mini-tiles per warp iteration: every global load of both (masks, the
        // 10 x 10 blocks of V^n, the speeds) is issued before any is used, and the mask
        // updates of both go out together
        // the warps claim two queued mini-tiles at a time from a shared counter: a warp that
        // finishes early takes the next pair instead of waiting at the CTA barrier
        // (HJ_COOP_DUBINS_DYNQ=0: the Dubins class takes the static split (warp, warp + NW),
        // (warp + 2 NW, ...) instead)
        constexpr bool DYNQ = EV != 3 || HJ_COOP_DUBINS_DYNQ;
        // items per claim at the front of the queue (HJ_COOP_NP=1, a build switch: one item
        // per claim throughout — no pair state in registers; measured with two CTAs per SM)
        // The local class takes one item per claim throughout: its sweeps hold few items per
        // CTA, where the finer claims win (config 2 whole grid 8.28 -> 7.48 ms, ISA step
        // 11.96 -> 11.31 ms); the field class keeps pairs + a single tail (config 3: 478 vs
        // 514 ms singles only) — profiles/r2v/balance_ab.txt.
        constexpr int NP = EV == 3 ? 2 : (EV == 0 ? HJ_COOP_NP_LOCAL : HJ_COOP_NP);
        // (the queue's last qsingle items go one per claim: a finer tail for the CTA barrier)
        const int pz = DYNQ ? (NP == 1 ? 0 : cnt - min(cnt, S.qsingle)) : cnt;   // items claimed in pairs
        const int npair = (pz + 1) >> 1;
        for (int itw = warp;; itw += 2 * COOP_NW) {
            int it = itw, lim2 = cnt;
            if (DYNQ) {
                if (lane == 0) it = atomicAdd(&qnext, 1);
                it = __shfl_sync(0xffffffffu, it, 0);
                if (it < npair) {
                    it *= 2;
                    lim2 = pz;
                } else {
                    it = pz + (it - npair);
                    lim2 = 0;                                      // a single item
                }
            }
            if (it >= cnt) break;
            const int it2 = DYNQ ? it + 1 : it + COOP_NW;    // the pair's second item
            // 32-bit mini-tile arithmetic (ids are int32; a 2-D view's nodes < 2^31)
            int gid[2];
            gid[0] = qgid[it];
            gid[1] = it2 < lim2 ? qgid[it2] : -1;
            int vv[2] = {0, 0}, mx[2] = {0, 0}, my[2] = {0, 0}, mz[2] = {0, 0};
            unsigned long long dd[2] = {0ull, 0ull}, em[2] = {0ull, 0ull};
#ifdef HJ_DEBUG_BOUNDS
            if (it < 0 || it >= COOP_NW * 32 || gid[0] < 0 || gid[0] >= S.total ||
                gid[1] >= S.total)
                printf("HJ_DEBUG pair: n %lld it %d cnt %d gid %d %d total %lld\n", (long long)n,
                       it, cnt, gid[0], gid[1], (long long)S.total), __trap();
#endif
#pragma unroll
            for (int s2 = 0; s2 < NP; ++s2) {
                const int g = gid[s2] < 0 ? gid[0] : gid[s2];
                const int v = coop_view_warp(smtb, S.n_views, g);
                const int mt = g - smtb[v], m0 = smt0[v];

                vv[s2] = v;
                if (EV == 3) {
                    const int pl = m0 * smt1[v];
                    mz[s2] = mt / pl;
                    const int r = mt - mz[s2] * pl;
                    my[s2] = r / m0;
                    mx[s2] = r - my[s2] * m0;
                } else {
                    mz[s2] = 0;
                    my[s2] = mt / m0;
                    mx[s2] = mt - my[s2] * m0;
                }
                dd[s2] = gid[s2] >= 0 ? qmask[s2 ? it2 : it] : 0ull;
                em[s2] = gid[s2] >= 0 ? qemask[s2 ? it2 : it] : 0ull;
            }
            // staged V^n blocks and speeds, loads first.  A block inside its view (the
            // common case) reads rows of V^n at a fixed stride: no bounds tests.
            constexpr int NLD = (BLK + 31) / 32;
            T ld[2][NLD], lsp[2][2];
#pragma unroll
            for (int s2 = 0; s2 < NP; ++s2) {
                const SweepView<T> &vw = sview[vv[s2]];
                const int vn0 = (int)vw.vn[0], vn1 = (int)vw.vn[1], vn2 = (int)vw.vn[2];
                const T *__restrict__ Vi = vw.V[n & 1];
                const int x0 = mx[s2] * 8, y0 = my[s2] * 8;
                const bool inner = x0 >= 1 && y0 >= 1 && x0 + 9 <= vn0 && y0 + 9 <= vn1;
                if (inner) {
                    const T *__restrict__ src = Vi + ((int64_t)(y0 - 1) * vn0 + (x0 - 1));
                    // Dubins: planes z-1, z, z+1 (periodic in the view, as below)
                    int64_t poff[3] = {0, 0, 0};
                    if (EV == 3) {
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            int lk = mz[s2] - 1 + q;
                            if (lk < 0) lk += vn2;
                            if (lk >= vn2) lk -= vn2;
                            poff[q] = (int64_t)lk * vn0 * vn1;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < NLD; ++k) {
                        const int e = lane + 32 * k;
                        const int q = e / (BP * BP), ee = e - (BP * BP) * q;
                        const int64_t po = q == 0 ? poff[0] : (q == 1 ? poff[1] : poff[2]);
                        ld[s2][k] = e < BLK ? src[po + (ee / BP) * vn0 + ee % BP] : v_out;
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < NLD; ++k) {
                        const int e = lane + 32 * k;
                        const int ee = e % (BP * BP);
                        const int li = x0 - 1 + ee % BP, lj = y0 - 1 + ee / BP;
                        int lk = 0;
                        if (EV == 3) {               // heading plane z-1+e/100, periodic
                            lk = mz[s2] - 1 + e / (BP * BP);
                            if (lk < 0) lk += vn2;
                            if (lk >= vn2) lk -= vn2;
                        }
                        ld[s2][k] = (e < BLK && li >= 0 && lj >= 0 && li < vn0 && lj < vn1)
                                        ? Vi[li + (int64_t)vn0 * (lj + (int64_t)vn1 * lk)]
                                        : v_out;
                    }
                }
                if (EV != 3 && P.speed) {
                    const int o0 = (int)vw.o[0], o1 = (int)vw.o[1];
                    const T *__restrict__ sp = P.speed + ((int64_t)(y0 + o1) * gn0 + (x0 + o0));
#pragma unroll
                    for (int k = 0; k < 2; ++k) {
                        const int e = lane + 32 * k;
                        const int li = x0 + (e & 7), lj = y0 + (e >> 3);
                        lsp[s2][k] = (inner || (li < vn0 && lj < vn1)) ? sp[(e >> 3) * gn0 + (e & 7)]
                                                                       : T(1);
                    }
                } else {
                    lsp[s2][0] = lsp[s2][1] = T(1);
                }
            }
#pragma unroll
            for (int s2 = 0; s2 < NP; ++s2) {
#pragma unroll
                for (int k = 0; k < NLD; ++k)
                    if (lane + 32 * k < BLK) blk[warp][s2][lane + 32 * k] = ld[s2][k];
                if (EV != 3) {
                    spd[warp][s2][lane % SPD] = lsp[s2][0];
                    spd[warp][s2][(lane + 32) % SPD] = lsp[s2][1];
                }
            }
            __syncwarp();
            if (tr && t_l == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_l));
            unsigned long long cmv[2] = {0ull, 0ull};
#pragma unroll 1
            for (int s2 = 0; s2 < NP; ++s2) {
                // (selects, not indexing: a runtime index would put the arrays in local memory)
                const int v = s2 ? vv[1] : vv[0];
                if ((s2 ? gid[1] : gid[0]) < 0 || ((stopped >> v) & 1u)) continue;
                const SweepView<T> &vw = sview[v];
                const int64_t x0 = (int64_t)(s2 ? mx[1] : mx[0]) * 8;
                const int64_t y0 = (int64_t)(s2 ? my[1] : my[0]) * 8;
                const unsigned long long d_s = s2 ? dd[1] : dd[0], e_s = s2 ? em[1] : em[0];
                T rmax;
                unsigned long long cm;
                int evald;
                if constexpr (EV == 3) {
                    const int z = s2 ? mz[1] : mz[0];
                    const T th = fma((T)(z + vw.o[2]), P.dx[2], P.lo[2]);
                    T sn, cn;
                    sincos_t(th, &sn, &cn);
                    coop_eval_dubins<T>(P, vw, blk[warp][s2], lst[warp][s2], d_s | e_s,
                                        x0, y0, z, P.hdx[0] * (P.dub_v * cn),
                                        P.hdx[1] * (P.dub_v * sn), vw.V[(n + 1) & 1], dub_wext,
                                        rmax, cm, evald);
                } else if constexpr (EV == 0)
                    coop_eval<T, KQ, PC>(P, C, vw, blk[warp][s2], spd[warp][s2], lst[warp][s2],
                                         sctl, d_s, e_s, x0, y0, vw.V[(n + 1) & 1], rmax, cm,
                                         evald);
                else
                    coop_eval_field<T, EV - 1>(P, vw, vw.V[n & 1], blk[warp][s2], spd[warp][s2],
                                               lst[warp][s2], d_s, e_s, x0, y0,
                                               vw.V[(n + 1) & 1], rmax, cm, evald,
                                               EV == 1 && S.seg ? sseg : nullptr, sseg_csq,
                                               S.seg_nup, srsplit[EV == 1 ? warp : 0],
                                               EV == 1 && S.seg_tab ? segtab : nullptr,
                                               S.seg_prune ? sseg_w1max : T(-1));
                cm = ((unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)(cm >> 32)) << 32) |
                     (unsigned long long)__reduce_or_sync(0xffffffffu, (unsigned)cm);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const T other = __shfl_xor_sync(0xffffffffu, rmax, o);
                    rmax = other > rmax ? other : rmax;
                }
                evald = __reduce_add_sync(0xffffffffu, evald);
                if (lane == 0) {
                    if (rmax > T(0))
                        atomicMax(&cres[v], CoopBits<T>::bits(rmax));
                    atomicAdd(&cwork[v], (unsigned)evald);
                }
                if (s2) cmv[1] = cm; else cmv[0] = cm;
            }
            if (tr && t_e == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_e));
            // sweep n+1: the 3 x 3 dilation of the changed nodes into the 9 mini-tiles
            // around each item (lanes 0-8: item 0, lanes 16-24: item 1)
            // (Dubins: the same in-plane dilation into planes z-1, z, z+1: 27 mini-tiles,
            // two per lane)
#pragma unroll
            for (int rep = 0; rep < (EV == 3 ? 2 : 1); ++rep) {
                const int s2 = lane >> 4, l9 = (lane & 15) + 16 * rep;
                const unsigned long long cm = s2 ? cmv[1] : cmv[0];
                if (cm && l9 < (EV == 3 ? 27 : 9)) {
                    const int v = s2 ? vv[1] : vv[0];
                    const int dx = l9 % 3 - 1, dy = (l9 / 3) % 3 - 1, dz = l9 / 9 - 1;
                    const int nx = (s2 ? mx[1] : mx[0]) + dx, ny = (s2 ? my[1] : my[0]) + dy;
                    int nz = (s2 ? mz[1] : mz[0]) + (EV == 3 ? dz : 0);
                    if (EV == 3) {
                        if (nz < 0) nz += smt2[v];
                        if (nz >= smt2[v]) nz -= smt2[v];
                    }
                    if (nx >= 0 && ny >= 0 && nx < smt0[v] && ny < smt1[v]) {
                        const unsigned long long bits = coop_spread(cm, dx, dy);
                        if (bits) {
                            const int nid = smtb[v] + nx + smt0[v] * (ny + smt1[v] * nz);
                            if (S.use_list) {    // a mask that was empty: list the mini-tile
                                const unsigned long long old = atomicOr(&dnext[nid], bits);
                                if (old == 0ull)
                                    S.items[(n + 1) & 1][atomicAdd(&S.count[(n + 1) % 3], 1)] =
                                        (int32_t)nid;
                            } else {             // fire and forget: the scan finds it
                                atomicOr(&dnext[nid], bits);
                            }
                        }
                    }
                }
            }
            __syncwarp();
            if (tr && t_m == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_m));
        }
        __syncthreads();                           // the queue is reused by the next chunk
        if (tr && t_q == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_q));
        }
        if (!decided) {                            // (no candidates in this CTA)
            const unsigned now = __ballot_sync(0xffffffffu, chk && rprev < tol);
            if (now) {
                if (grank == 0 && threadIdx.x == 0)
                    for (unsigned m = now; m; m &= m - 1) S.stop[__ffs(m) - 1] = n;
                stopped |= now;
            }
        }
        if (stopped == all) break;
        // per-CTA residual / work of this sweep, one atomic per view (the chunk loop ended
        // on a CTA barrier, or never ran: cres/cwork are final)
        if (threadIdx.x < (unsigned)S.n_views) {
            const int v = threadIdx.x;
            const double m = (double)CoopBits<T>::value(cres[v]);
            const unsigned long long w = cwork[v];
            if (m > 0.0) atomic_max_nonneg(&sview[v].res[n], m);
            if (w) atomicAdd(sview[v].work, w);
        }
        if (S.use_list && blockIdx.x == 0 && threadIdx.x == 0) S.count[(n + 2) % 3] = 0;
        if (tr) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_b));
        if (tr_all && n < tr_cap) {
            unsigned long long t_arr;              // every CTA's arrival (load balance)
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_arr));
            tr_buf[8 * tr_cap + 256 * n + blockIdx.x] = t_arr;
        }
        if constexpr (CL) {
            // (acquire: the SM's L1 is invalidated, the cluster's writes are visible)
            asm volatile("barrier.cluster.arrive.release.aligned;\n\t"
                         "barrier.cluster.wait.acquire.aligned;" ::: "memory");
        } else {
            coop_grid_barrier(reinterpret_cast<unsigned *>(S.count + 3),
                              (unsigned)(n + 1) * gridDim.x);
        }
        if (tr && n < tr_cap) {
            unsigned long long t_c;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t_c));
            unsigned long long *o = tr_buf + 8 * n;
            o[0] = t_a;
            o[1] = t_b;
            o[2] = t_c;
            o[3] = ((t_s - t_a) << 16) | (unsigned long long)qitems;
            o[4] = t_l;
            o[5] = t_e;
            o[6] = t_m;
            o[7] = t_q;
        }
    }
    if (grank == 0 && threadIdx.x == 0)
        for (int v = 0; v < S.n_views; ++v)
            if (!((stopped >> v) & 1u)) S.stop[v] = max_iter;
    }
}

}  // namespace hj
