// ubench_alu.cu — issue-rate microbenchmark of the sweep's inner loop variants on
// sm_100a (measure before choosing the kernel design).
//
// Each variant evaluates the bilinear bracket-min of the local 2-D sweep,
//   cand_k = fma(ay_k, fma(ax_k, A3, A2), fma(ax_k, A1, C0)),  best = min_k cand_k,
// over K = 64 controls held in constant memory, for NB nodes per thread, REPS times
// (a dependency through C0 keeps the compiler from hoisting).  Reported: node x
// control updates per SM clock (clock64 inside the kernel) and per second.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ub tools/ubench_alu.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int K = 64;
__constant__ float c_ax[K], c_ay[K];
__constant__ float2 c_ax2[K / 2], c_ay2[K / 2];

template <int NB>
__global__ void __launch_bounds__(256) v_scalar(float *out, long long *cyc, int reps) {
    float C0[NB], A1[NB], A2[NB], A3[NB], best[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        C0[n] = threadIdx.x * 1e-3f + n;
        A1[n] = 0.1f + n * 1e-3f;
        A2[n] = 0.2f - threadIdx.x * 1e-6f;
        A3[n] = 0.01f + threadIdx.x * 1e-7f;
        best[n] = 1e30f;
    }
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int n = 0; n < NB; ++n) best[n] = 1e30f;
#pragma unroll
        for (int k = 0; k < K; ++k) {
            const float ax = c_ax[k], ay = c_ay[k];
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                float u = fmaf(ax, A1[n], C0[n]);
                float c = fmaf(ay, fmaf(ax, A3[n], A2[n]), u);
                best[n] = fminf(best[n], c);
            }
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) C0[n] = fmaf(best[n], 1e-30f, C0[n]);
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int n = 0; n < NB; ++n) s += best[n];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// FFMA2 over control pairs
template <int NB>
__global__ void __launch_bounds__(256) v_pair(float *out, long long *cyc, int reps) {
    float2 C0[NB], A1[NB], A2[NB], A3[NB];
    float best[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        float c = threadIdx.x * 1e-3f + n;
        C0[n] = make_float2(c, c);
        A1[n] = make_float2(0.1f + n * 1e-3f, 0.1f + n * 1e-3f);
        float a2 = 0.2f - threadIdx.x * 1e-6f;
        A2[n] = make_float2(a2, a2);
        A3[n] = make_float2(0.01f + threadIdx.x * 1e-7f, 0.01f + threadIdx.x * 1e-7f);
        best[n] = 1e30f;
    }
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int n = 0; n < NB; ++n) best[n] = 1e30f;
#pragma unroll
        for (int k = 0; k < K / 2; ++k) {
            const float2 ax = c_ax2[k], ay = c_ay2[k];
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                float2 u = __ffma2_rn(ax, A1[n], C0[n]);
                float2 w = __ffma2_rn(ax, A3[n], A2[n]);
                float2 c = __ffma2_rn(ay, w, u);
                best[n] = fminf(best[n], fminf(c.x, c.y));
            }
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            float c = fmaf(best[n], 1e-30f, C0[n].x);
            C0[n] = make_float2(c, c);
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int n = 0; n < NB; ++n) s += best[n];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

// FFMA2 over node pairs (controls broadcast)
template <int NB>
__global__ void __launch_bounds__(256) v_nodepair(float *out, long long *cyc, int reps) {
    float2 C0[NB], A1[NB], A2[NB], A3[NB], best[NB];
#pragma unroll
    for (int n = 0; n < NB; ++n) {
        float c = threadIdx.x * 1e-3f + n;
        C0[n] = make_float2(c, c + 0.5f);
        A1[n] = make_float2(0.1f + n * 1e-3f, 0.11f);
        float a2 = 0.2f - threadIdx.x * 1e-6f;
        A2[n] = make_float2(a2, a2 * 0.5f);
        A3[n] = make_float2(0.01f + threadIdx.x * 1e-7f, 0.02f);
        best[n] = make_float2(1e30f, 1e30f);
    }
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
#pragma unroll
        for (int n = 0; n < NB; ++n) best[n] = make_float2(1e30f, 1e30f);
#pragma unroll
        for (int k = 0; k < K; k += 2) {
            const float2 ax = c_ax2[k / 2], ay = c_ay2[k / 2];
            const float2 axa = make_float2(ax.x, ax.x), aya = make_float2(ay.x, ay.x);
            const float2 axb = make_float2(ax.y, ax.y), ayb = make_float2(ay.y, ay.y);
#pragma unroll
            for (int n = 0; n < NB; ++n) {
                float2 u = __ffma2_rn(axa, A1[n], C0[n]);
                float2 w = __ffma2_rn(axa, A3[n], A2[n]);
                float2 c = __ffma2_rn(aya, w, u);
                float2 u2 = __ffma2_rn(axb, A1[n], C0[n]);
                float2 w2 = __ffma2_rn(axb, A3[n], A2[n]);
                float2 c2 = __ffma2_rn(ayb, w2, u2);
                best[n].x = fminf(best[n].x, fminf(c.x, c2.x));
                best[n].y = fminf(best[n].y, fminf(c.y, c2.y));
            }
        }
#pragma unroll
        for (int n = 0; n < NB; ++n) {
            C0[n].x = fmaf(best[n].x, 1e-30f, C0[n].x);
            C0[n].y = fmaf(best[n].y, 1e-30f, C0[n].y);
        }
    }
    long long t1 = clock64();
    float s = 0;
#pragma unroll
    for (int n = 0; n < NB; ++n) s += best[n].x + best[n].y;
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

template <typename F>
void run(const char *name, F kern, int nb, int blocks_per_sm) {
    const int sms = 148, threads = 256, reps = 2000;
    int blocks = sms * blocks_per_sm;
    float *out;
    long long *cyc;
    cudaMalloc(&out, blocks * threads * sizeof(float));
    cudaMalloc(&cyc, blocks * sizeof(long long));
    kern<<<blocks, threads>>>(out, cyc, 10);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, cyc, reps);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long *h = new long long[blocks];
    cudaMemcpy(h, cyc, blocks * sizeof(long long), cudaMemcpyDeviceToHost);
    double mean = 0;
    for (int i = 0; i < blocks; ++i) mean += h[i];
    mean /= blocks;
    double upd = (double)blocks * threads * reps * K * nb;
    double per_clk_sm = upd / sms / mean;   // all CTAs of an SM run concurrently
    printf("%-14s NB=%d occ=%d  %.2f updates/clk/SM  %.2f T updates/s  (%.3f ms)  err=%s\n", name,
           nb, blocks_per_sm, per_clk_sm, upd / (ms * 1e-3) / 1e12, ms,
           cudaGetErrorString(cudaGetLastError()));
    delete[] h;
    cudaFree(out);
    cudaFree(cyc);
}

int main() {
    float ax[K], ay[K];
    for (int k = 0; k < K; ++k) {
        ax[k] = 0.3f + 0.01f * k;
        ay[k] = 0.7f - 0.01f * k;
    }
    cudaMemcpyToSymbol(c_ax, ax, sizeof(ax));
    cudaMemcpyToSymbol(c_ay, ay, sizeof(ay));
    cudaMemcpyToSymbol(c_ax2, ax, sizeof(ax));
    cudaMemcpyToSymbol(c_ay2, ay, sizeof(ay));
    for (int occ : {2, 4}) {
        run("scalar", v_scalar<1>, 1, occ);
        run("scalar", v_scalar<2>, 2, occ);
        run("scalar", v_scalar<4>, 4, occ);
        run("ctrlpair", v_pair<1>, 1, occ);
        run("ctrlpair", v_pair<2>, 2, occ);
        run("ctrlpair", v_pair<4>, 4, occ);
        run("nodepair", v_nodepair<1>, 2, occ);
        run("nodepair", v_nodepair<2>, 4, occ);
    }
    return 0;
}
