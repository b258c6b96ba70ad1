// hj_sweep.cuh — one Jacobi sweep V^{n+1} = T(V^n) over a set of views
// (PAPER.md eq. (SL), operator (Tdef) line 238-245, readings R1-R4).
//
// Kernel family:
//   k_sweep_generic<T, DIM>   any dynamics / cost / h: per node, per control, the
//                             foot, the multilinear interpolation and the min of the
//                             bracket, corners read through L1/L2.
// Every sweep kernel:
//   - exits at once if its view already stopped (res[n-1] < tol), so launching a
//     few sweeps past convergence is free and the stop is exactly the first n with
//     ||V^{n+1}-V^n|| < tol (R6);
//   - folds |V^{n+1}-V^n| into res[n] with one atomicMax per CTA.
#pragma once

#include <vector>

#include "hj_host.cuh"

namespace hj {

template <typename T, int DIM>
__global__ void __launch_bounds__(256)
    k_sweep_generic(const DevProblem<T, T> P, const SweepView<T> *__restrict__ views, int64_t it,
                    double tol) {
    const SweepView<T> &vw = views[blockIdx.y];
    if (it > 0 && *(volatile double *)&vw.res[it - 1] < tol) return;
    const int64_t o[3] = {vw.o[0], vw.o[1], vw.o[2]};
    const int64_t vn[3] = {vw.vn[0], vw.vn[1], vw.vn[2]};
    const T *__restrict__ Vi = vw.V[it & 1];
    T *__restrict__ Vo = vw.V[(it + 1) & 1];
    const int8_t *__restrict__ cls = vw.cls;
    const int64_t nodes = vw.nodes;
    T rmax = T(0);
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nodes;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t li = t % vn[0], r = t / vn[0];
        int64_t lj = r % vn[1], lk = r / vn[1];
        int64_t gi[3] = {li + o[0], lj + o[1], lk + o[2]};
        int64_t gidx = gi[0] + P.n[0] * (gi[1] + P.n[1] * gi[2]);
        int8_t c = cls[t];
        T vin = Vi[t];
        T v;
        if (c == -2) {
            v = P.v_out;
        } else if (c >= 0) {
            v = P.g ? P.g[gidx] : T(0);
        } else {
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
            v = best;
        }
        Vo[t] = v;
        T dv = v > vin ? v - vin : vin - v;
        rmax = dv > rmax ? dv : rmax;
    }
    // CTA max -> one atomic
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
        T other = __shfl_down_sync(0xffffffffu, rmax, s);
        rmax = other > rmax ? other : rmax;
    }
    __shared__ T red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = rmax;
    __syncthreads();
    if (threadIdx.x == 0) {
        T m = red[0];
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) m = red[w] > m ? red[w] : m;
        if (m > T(0)) atomic_max_nonneg(&vw.res[it], (double)m);
    }
}

template <typename T>
struct SweepLaunch {
    int dim;
    dim3 grid;
    int n_views;
};

template <typename T>
hj_status sweep_prepare(const hj_grid &g, const hj_problem &p,
                        const std::vector<SweepView<T>> &views, SweepLaunch<T> &L) {
    int64_t mx = 1;
    for (auto &v : views) mx = std::max<int64_t>(mx, v.nodes);
    L.dim = g.dim;
    L.n_views = (int)views.size();
    L.grid = dim3((unsigned)std::min<int64_t>((mx + 255) / 256, 148 * 8), L.n_views);
    return HJ_OK;
}

template <typename T>
hj_status sweep_launch(const DevProblem<T, T> &P, const SweepView<T> *d_views,
                       const SweepLaunch<T> &L, int64_t it, double tol, cudaStream_t s) {
    if (L.dim == 2)
        k_sweep_generic<T, 2><<<L.grid, 256, 0, s>>>(P, d_views, it, tol);
    else
        k_sweep_generic<T, 3><<<L.grid, 256, 0, s>>>(P, d_views, it, tol);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("sweep launch failed: %s", cudaGetErrorString(e));
        return HJ_ERR_CUDA;
    }
    return HJ_OK;
}

template <typename T>
void sweep_release(SweepLaunch<T> &) {}

}  // namespace hj
