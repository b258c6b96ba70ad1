// hj_solve.cu — the value-iteration sweep of the SL Bellman operator
// (PAPER.md eq. (SL), (Tdef) line 238-245), the device-side stopping
// rule (line 341-345, reading R6) and the ISA fine stage (steps 3-4, line 400-407).
#include <algorithm>
#include <deque>
#include <vector>

#include "hj_host.cuh"
#include "hj_sweep.cuh"

namespace hj {

// ---------------------------------------------------------------------------
// small kernels
// ---------------------------------------------------------------------------
template <typename T>
__global__ void k_init_view(const SweepView<T> *views, T v_out, const T *g, const int64_t n0,
                            const int64_t n1) {
    const SweepView<T> &vw = views[blockIdx.y];
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < vw.nodes;
         t += (int64_t)gridDim.x * blockDim.x) {
        int8_t c = vw.cls[t];
        T v = v_out;
        if (c >= 0) {
            if (g) {
                int64_t li = t % vw.vn[0], r = t / vw.vn[0];
                int64_t lj = r % vw.vn[1], lk = r / vw.vn[1];
                int64_t gi = (li + vw.o[0]) + n0 * ((lj + vw.o[1]) + n1 * (lk + vw.o[2]));
                v = g[gi];
            } else {
                v = T(0);
            }
        }
        vw.V[0][t] = v;
        vw.V[1][t] = v;
    }
}

template <typename T>
__global__ void k_count_interior(const SweepView<T> *views, unsigned long long *counts) {
    const SweepView<T> &vw = views[blockIdx.y];
    unsigned long long c = 0;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < vw.nodes;
         t += (int64_t)gridDim.x * blockDim.x)
        c += (vw.cls[t] == -1);
    for (int s = 16; s > 0; s >>= 1) c += __shfl_down_sync(0xffffffffu, c, s);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&counts[blockIdx.y], c);
}

// class array of sub-domain k over its box: piece inside S_k, -2 (ghost) outside
__global__ void k_subdomain_classes(const uint64_t *__restrict__ mask,
                                    const int8_t *__restrict__ piece, int k, int64_t o0,
                                    int64_t o1, int64_t o2, int64_t vn0, int64_t vn1,
                                    int64_t nodes, int64_t n0, int64_t n1, int8_t *cls) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nodes;
         t += (int64_t)gridDim.x * blockDim.x) {
        int64_t li = t % vn0, r = t / vn0;
        int64_t lj = r % vn1, lk = r / vn1;
        int64_t gi = (li + o0) + n0 * ((lj + o1) + n1 * (lk + o2));
        cls[t] = ((mask[gi] >> k) & 1ull) ? piece[gi] : (int8_t)-2;
    }
}

template <typename T>
struct AsmView {
    int64_t o[3], vn[3];
    const T *V;
    int32_t sub;
};

template <typename T>
__global__ void k_assemble(const AsmView<T> *__restrict__ av, int nv,
                           const uint64_t *__restrict__ mask, int64_t n0, int64_t n1,
                           int64_t N, T v_out, T *Vbar) {
    for (int64_t gi = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; gi < N;
         gi += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t bits = mask[gi];
        int64_t i = gi % n0, r = gi / n0;
        int64_t j = r % n1, k = r / n1;
        T v = v_out;
        for (int q = 0; q < nv; ++q) {
            const AsmView<T> &a = av[q];
            if (!((bits >> a.sub) & 1ull)) continue;
            int64_t li = i - a.o[0], lj = j - a.o[1], lk = k - a.o[2];
            if (li < 0 || lj < 0 || lk < 0 || li >= a.vn[0] || lj >= a.vn[1] || lk >= a.vn[2])
                continue;
            T x = a.V[li + a.vn[0] * (lj + a.vn[1] * lk)];
            v = x < v ? x : v;
        }
        Vbar[gi] = v;
    }
}

// Bounding box and node count of every sub-domain in the fine mask.  Warp-aggregated:
// for each sub-domain bit present in the warp's 32 nodes, one warp reduction per
// coordinate bound and one shared update per warp (a node of reading R9 carries every
// bit, so per-node shared atomics contended on the same m addresses).
__global__ void __launch_bounds__(256)
    k_plan(const uint64_t *__restrict__ mask, int64_t N, int64_t n0, int64_t n1, int m,
           int *bb /* [m][6]: lo0..2, hi0..2 */, unsigned long long *cnt) {
    __shared__ int s_lo[HJ_MAX_SUBDOMAINS][3], s_hi[HJ_MAX_SUBDOMAINS][3];
    __shared__ unsigned s_cnt[HJ_MAX_SUBDOMAINS];
    for (int t = threadIdx.x; t < HJ_MAX_SUBDOMAINS; t += blockDim.x) {
        for (int d = 0; d < 3; ++d) {
            s_lo[t][d] = 0x7fffffff;
            s_hi[t][d] = -1;
        }
        s_cnt[t] = 0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint64_t mm = m >= 64 ? ~0ull : ((1ull << m) - 1ull);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t w0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); w0 < N;
         w0 += stride) {
        const int64_t gi = w0 + lane;
        const uint64_t bits = gi < N ? (mask[gi] & mm) : 0ull;
        uint64_t any = ((uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)(bits >> 32)) << 32) |
                       (uint64_t)__reduce_or_sync(0xffffffffu, (unsigned)bits);
        if (!any) continue;
        int c[3];
        c[0] = (int)(gi % n0);
        const int64_t r = gi / n0;
        c[1] = (int)(r % n1);
        c[2] = (int)(r / n1);
        while (any) {
            const int k = __ffsll((long long)any) - 1;
            any &= any - 1;
            const bool has = (bits >> k) & 1ull;
            const unsigned cntk = __popc(__ballot_sync(0xffffffffu, has));
            int lo[3], hi[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                lo[d] = __reduce_min_sync(0xffffffffu, has ? c[d] : 0x7fffffff);
                hi[d] = __reduce_max_sync(0xffffffffu, has ? c[d] : -1);
            }
            if (lane == 0) {
#pragma unroll
                for (int d = 0; d < 3; ++d) {
                    atomicMin(&s_lo[k][d], lo[d]);
                    atomicMax(&s_hi[k][d], hi[d]);
                }
                atomicAdd(&s_cnt[k], cntk);
            }
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        if (!s_cnt[k]) continue;
        for (int d = 0; d < 3; ++d) {
            atomicMin(&bb[6 * k + d], s_lo[k][d]);
            atomicMax(&bb[6 * k + 3 + d], s_hi[k][d]);
        }
        atomicAdd(&cnt[k], (unsigned long long)s_cnt[k]);
    }
}

template <typename T>
__global__ void k_absmax(const T *__restrict__ x, int64_t N, unsigned long long *out) {
    double m = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N;
         i += (int64_t)gridDim.x * blockDim.x)
        m = fmax(m, fabs((double)x[i]));
    for (int s = 16; s > 0; s >>= 1) m = fmax(m, __shfl_down_sync(0xffffffffu, m, s));
    if ((threadIdx.x & 31) == 0) atomicMax(out, (unsigned long long)__double_as_longlong(m));
}

hj_status speed_max(const void *speed, int dtype, int64_t N, cudaStream_t s, double *out) {
    double *pin = pinned_scratch(1);
    HJ_CHECK(pin != nullptr, "cudaMallocHost failed");
    static thread_local unsigned long long *scratch[64] = {nullptr};   // per device, kept
    int dev = 0;
    HJ_CUDA(cudaGetDevice(&dev));
    HJ_CHECK(dev >= 0 && dev < 64, "device index out of range");
    if (!scratch[dev]) HJ_CUDA(cudaMalloc(&scratch[dev], sizeof(unsigned long long)));
    unsigned long long *d = scratch[dev];
    HJ_CUDA(cudaMemsetAsync(d, 0, sizeof(*d), s));
    int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 8);
    if (dtype == HJ_F64)
        k_absmax<double><<<blocks, 256, 0, s>>>((const double *)speed, N, d);
    else
        k_absmax<float><<<blocks, 256, 0, s>>>((const float *)speed, N, d);
    HJ_CUDA(cudaMemcpyAsync(pin, d, sizeof(double), cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    *out = pin[0];
    return HJ_OK;
}

__global__ void k_fill_int(int *p, int n, int v_lo, int v_hi) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) p[t] = ((t % 6) < 3) ? v_lo : v_hi;
}

// ---------------------------------------------------------------------------
// the iteration driver: sweeps in batches, residuals read back one batch
// behind so the device never waits for the host; every view stops at its own
// first n with res[n] < tol (the sweep kernel itself skips converged views).
// ---------------------------------------------------------------------------
struct IterResult {
    std::vector<int64_t> iters;
    std::vector<double> resid;
    std::vector<int> converged;
    std::vector<int> buf;          // V[buf] holds the final iterate of each view
    float ms = 0.f;
    int64_t launches = 0;
};

// Sweeps are launched in batches (L.tb sweeps per launch for the temporally blocked
// kernel, 1 otherwise) and the residuals read back one batch behind; each view
// stops at its own first n with res[n-1] < tol.  With L.tb > 1 a view whose stop
// falls inside a block re-runs that block from its intact input with the exact
// number of sub-sweeps, so the final iterate is V^{n*} bit for bit.
template <typename T>
static hj_status iterate(const DevProblem<T, T> &P, SweepLaunch<T> &L, int nv,
                         double *res_base, int64_t res_stride, double tol, int64_t max_iter,
                         cudaStream_t s, IterResult &out) {
    if (L.coop) {   // the whole iteration in one cooperative launch
        out.iters.assign(nv, max_iter);
        out.resid.assign(nv, INFINITY);
        out.converged.assign(nv, 0);
        out.buf.assign(nv, 0);
        cudaEvent_t c0, c1;
        HJ_CUDA(cudaEventCreate(&c0));
        HJ_CUDA(cudaEventCreate(&c1));
        HJ_CUDA(cudaEventRecord(c0, s));
        std::vector<int64_t> stop;
        hj_status st = sweep_coop(P, L, max_iter, tol, s, stop);
        if (st != HJ_OK) return st;
        HJ_CUDA(cudaEventRecord(c1, s));
        std::vector<double> last(nv, INFINITY);
        for (int v = 0; v < nv; ++v)
            if (stop[v] >= 1)
                HJ_CUDA(cudaMemcpyAsync(&last[v], res_base + v * res_stride + stop[v] - 1,
                                        sizeof(double), cudaMemcpyDeviceToHost, s));
        HJ_CUDA(cudaStreamSynchronize(s));
        HJ_CUDA(cudaEventElapsedTime(&out.ms, c0, c1));
        cudaEventDestroy(c0);
        cudaEventDestroy(c1);
        for (int v = 0; v < nv; ++v) {
            out.iters[v] = stop[v];
            out.resid[v] = last[v];
            out.converged[v] = last[v] < tol;
            out.buf[v] = (int)(stop[v] & 1);
        }
        out.launches = 2;
        return HJ_OK;
    }
    const int S = std::max(1, L.tb);
    const int64_t B = S > 1 ? 4 * S : 16;          // sweeps per read-back batch
    double *pin = pinned_scratch((size_t)2 * nv * B);
    HJ_CHECK(pin != nullptr, "cudaMallocHost failed for the residual staging buffer");
    cudaEvent_t ev[2], t0, t1;
    for (auto &e : ev) HJ_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    HJ_CUDA(cudaEventCreate(&t0));
    HJ_CUDA(cudaEventCreate(&t1));
    out.iters.assign(nv, max_iter);
    out.resid.assign(nv, INFINITY);
    out.converged.assign(nv, 0);
    out.buf.assign(nv, 0);
    int n_done = 0;

    struct Batch {
        int64_t start, count;
        int slot;
    };
    std::deque<Batch> inflight;
    int64_t next = 0;
    int slot = 0;
    HJ_CUDA(cudaEventRecord(t0, s));
    while (true) {
        while (inflight.size() < 2 && next < max_iter && n_done < nv) {
            int64_t cnt = std::min<int64_t>(B, max_iter - next);
            for (int64_t it = next; it < next + cnt; it += S) {
                hj_status st =
                    sweep_launch(P, L, it, tol, s, (int)std::min<int64_t>(S, next + cnt - it));
                if (st != HJ_OK) return st;
                ++out.launches;
            }
            for (int v = 0; v < nv; ++v)
                HJ_CUDA(cudaMemcpyAsync(pin + ((size_t)slot * nv + v) * B,
                                        res_base + v * res_stride + next, cnt * sizeof(double),
                                        cudaMemcpyDeviceToHost, s));
            HJ_CUDA(cudaEventRecord(ev[slot], s));
            inflight.push_back({next, cnt, slot});
            next += cnt;
            slot ^= 1;
        }
        if (inflight.empty()) break;
        Batch b = inflight.front();
        inflight.pop_front();
        HJ_CUDA(cudaEventSynchronize(ev[b.slot]));
        for (int v = 0; v < nv; ++v) {
            if (out.converged[v]) continue;
            for (int64_t i = 0; i < b.count; ++i) {
                double r = pin[((size_t)b.slot * nv + v) * B + i];
                out.resid[v] = r;
                if (r < tol) {
                    out.converged[v] = 1;
                    out.iters[v] = b.start + i + 1;
                    ++n_done;
                    break;
                }
            }
        }
        if (n_done == nv) break;
    }
    // drain: batches still in flight only contain launches that exit at once
    for (int v = 0; v < nv; ++v) {
        const int64_t n = out.iters[v];
        const int64_t blk = (n - 1) / S;
        out.buf[v] = (int)((blk + 1) & 1);
    }
    if (S > 1) {
        // re-run the blocks that contain a stop (grouped by block)
        std::vector<int64_t> blocks;
        for (int v = 0; v < nv; ++v) {
            const int64_t n = out.iters[v], blk = (n - 1) / S;
            if (out.converged[v] && n - blk * S < S) blocks.push_back(blk);
        }
        std::sort(blocks.begin(), blocks.end());
        blocks.erase(std::unique(blocks.begin(), blocks.end()), blocks.end());
        for (int64_t blk : blocks) {
            std::vector<int32_t> rr(nv, 0);
            for (int v = 0; v < nv; ++v) {
                const int64_t n = out.iters[v];
                if (out.converged[v] && (n - 1) / S == blk && n - blk * S < S)
                    rr[v] = (int32_t)(n - blk * S);
            }
            for (int v = 0; v < nv; ++v)
                HJ_CUDA(cudaMemcpyAsync(&L.d_group->t[v].rerun, &rr[v], sizeof(int32_t),
                                        cudaMemcpyHostToDevice, s));
            hj_status st = sweep_launch_rerun(P, L, blk * S, tol, s);
            if (st != HJ_OK) return st;
            ++out.launches;
            HJ_CUDA(cudaStreamSynchronize(s));      // rr must outlive the copies
        }
    }
    HJ_CUDA(cudaEventRecord(t1, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    HJ_CUDA(cudaGetLastError());
    HJ_CUDA(cudaEventElapsedTime(&out.ms, t0, t1));
    for (auto &e : ev) cudaEventDestroy(e);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    return HJ_OK;
}

static hj_status validate_fields(const hj_fields *f) {
    HJ_CHECK(f != nullptr, "fields is NULL");
    HJ_CHECK(f->piece != nullptr, "fields.piece is required");
    return HJ_OK;
}

// ---------------------------------------------------------------------------
// hj_solve
// ---------------------------------------------------------------------------
template <typename T>
static size_t solve_ws(const hj_grid &g, int64_t max_iter) {
    int64_t N = grid_nodes(g);
    int64_t vn[3] = {g.n[0], g.dim > 1 ? g.n[1] : 1, g.dim > 2 ? g.n[2] : 1};
    Carver c(nullptr, 0);
    c.take(N * sizeof(T));
    c.take(max_iter * sizeof(double));
    c.take(chg_bytes_for(vn));
    c.take(sizeof(SweepGroup<T>));
    c.take(64);
    c.take(wl_bytes_for(tiles_finest(vn)));
    return c.off;
}

template <typename T>
static hj_status solve_impl(const hj_grid &grid, const hj_problem &prob, const hj_fields &f,
                            T *V, double tol, int64_t max_iter, void *ws, size_t ws_bytes,
                            cudaStream_t s, hj_report *rep) {
    int64_t N = grid_nodes(grid);
    SweepView<T> hv;
    memset(&hv, 0, sizeof(hv));
    for (int d = 0; d < 3; ++d) {
        hv.o[d] = 0;
        hv.vn[d] = d < grid.dim ? grid.n[d] : 1;
    }
    Carver c(ws, ws_bytes);
    T *V1 = (T *)c.take(N * sizeof(T));
    double *res = (double *)c.take(max_iter * sizeof(double));
    uint8_t *chg = (uint8_t *)c.take(chg_bytes_for(hv.vn));
    void *group = c.take(sizeof(SweepGroup<T>));
    unsigned long long *cnt = (unsigned long long *)c.take(64);
    void *wl = c.take(wl_bytes_for(tiles_finest(hv.vn)));
    if (!c.ok()) {
        set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
        return HJ_ERR_WORKSPACE;
    }
    hv.nodes = N;
    hv.V[0] = V;
    hv.V[1] = V1;
    hv.cls = f.piece;
    hv.res = res;
    hv.work = cnt + 1;
    auto P = make_dev_problem<T, T>(grid, prob, f);
    HJ_CUDA(cudaMemsetAsync(res, 0, max_iter * sizeof(double), s));
    HJ_CUDA(cudaMemsetAsync(cnt, 0, 64, s));
    std::vector<SweepView<T>> hvs{hv};
    std::vector<uint8_t *> chgs{chg};
    SweepLaunch<T> L;
    hj_status st = sweep_prepare(grid, prob, f, hvs, chgs, group, wl, s, L);
    if (st != HJ_OK) return st;
    const SweepView<T> *d_view = &L.d_group->v[0];
    int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 16);
    k_init_view<T><<<dim3(blocks, 1), 256, 0, s>>>(d_view, (T)prob.v_out, (const T *)f.g,
                                                   hv.vn[0], hv.vn[1]);
    k_count_interior<T><<<dim3(blocks, 1), 256, 0, s>>>(d_view, cnt);
    HJ_CUDA(cudaGetLastError());
    IterResult r;
    st = iterate<T>(P, L, 1, res, 0, tol, max_iter, s, r);
    if (st != HJ_OK) return st;
    int64_t it = r.iters[0];
    if (r.buf[0]) HJ_CUDA(cudaMemcpyAsync(V, V1, N * sizeof(T), cudaMemcpyDeviceToDevice, s));
    unsigned long long counts[2] = {0, 0};
    HJ_CUDA(cudaMemcpyAsync(counts, cnt, sizeof(counts), cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    const unsigned long long interior = counts[0];
    if (rep) {
        rep->evaluated_updates = (int64_t)counts[1] * L.evals;
        rep->iterations = it;
        rep->residual = r.resid[0];
        rep->converged = r.converged[0];
        rep->node_updates = (int64_t)interior * prob.n_controls * it;
        rep->device_ms = r.ms;
        rep->launches = r.launches + 3 + (f.speed ? 1 : 0);
    }
    if (!r.converged[0]) {
        set_error("not converged after %lld iterations (residual %g)", (long long)it, r.resid[0]);
        return HJ_ERR_NOT_CONVERGED;
    }
    return HJ_OK;
}

// ---------------------------------------------------------------------------
// partitioned solve (ISA steps 3-4)
// ---------------------------------------------------------------------------
struct PartLayout {
    std::vector<size_t> off_v0, off_v1, off_cls, off_chg;
    size_t off_res, off_views, off_asm, off_cnt, off_wl, total;
};

template <typename T>
static PartLayout part_layout(int m, const hj_subdomain *plan, int64_t max_iter) {
    PartLayout L;
    Carver c(nullptr, 0);
    for (int k = 0; k < m; ++k) {
        int64_t bn = plan[k].n_nodes > 0 ? plan[k].box_nodes : 0;
        L.off_v0.push_back(c.off);
        c.take(bn * sizeof(T));
        L.off_v1.push_back(c.off);
        c.take(bn * sizeof(T));
        L.off_cls.push_back(c.off);
        c.take(bn);
        int64_t vn[3] = {1, 1, 1};
        for (int d = 0; d < 3; ++d)
            if (plan[k].n_nodes > 0) vn[d] = plan[k].hi[d] - plan[k].lo[d] + 1;
        L.off_chg.push_back(c.off);
        c.take(plan[k].n_nodes > 0 ? chg_bytes_for(vn) : 0);
    }
    int64_t tiles = 0;
    for (int k = 0; k < m; ++k) {
        if (plan[k].n_nodes <= 0) continue;
        int64_t vn[3];
        for (int d = 0; d < 3; ++d) vn[d] = plan[k].hi[d] - plan[k].lo[d] + 1;
        tiles += tiles_finest(vn);
    }
    L.off_wl = c.off;
    c.take(wl_bytes_for(tiles));
    L.off_res = c.off;
    c.take((size_t)m * max_iter * sizeof(double));
    L.off_views = c.off;
    c.take(sizeof(SweepGroup<T>));
    L.off_asm = c.off;
    c.take((size_t)m * sizeof(AsmView<T>));
    L.off_cnt = c.off;
    c.take((size_t)2 * m * sizeof(unsigned long long));
    L.total = c.off;
    return L;
}

template <typename T>
static hj_status partitioned_impl(const hj_grid &grid, const hj_problem &prob,
                                  const hj_fields &f, const uint64_t *mask, int m,
                                  const hj_subdomain *plan, uint64_t solve_set, double tol,
                                  int64_t max_iter, T *Vbar, void *ws, size_t ws_bytes,
                                  cudaStream_t s, hj_report *reps) {
    PartLayout L = part_layout<T>(m, plan, max_iter);
    if (ws_bytes < L.total) {
        set_error("workspace too small: need %zu bytes, got %zu", L.total, ws_bytes);
        return HJ_ERR_WORKSPACE;
    }
    char *base = (char *)ws;
    int64_t n0 = grid.n[0], n1 = grid.dim > 1 ? grid.n[1] : 1;
    int64_t N = grid_nodes(grid);
    double *res = (double *)(base + L.off_res);
    void *group = base + L.off_views;
    AsmView<T> *d_asm = (AsmView<T> *)(base + L.off_asm);
    unsigned long long *cnt = (unsigned long long *)(base + L.off_cnt);

    std::vector<SweepView<T>> hv;
    std::vector<uint8_t *> chgs;
    std::vector<int> subs;
    for (int k = 0; k < m; ++k) {
        if (!((solve_set >> k) & 1ull) || plan[k].n_nodes == 0) continue;
        SweepView<T> v;
        memset(&v, 0, sizeof(v));
        v.nodes = 1;
        for (int d = 0; d < 3; ++d) {
            v.o[d] = d < grid.dim ? plan[k].lo[d] : 0;
            v.vn[d] = d < grid.dim ? plan[k].hi[d] - plan[k].lo[d] + 1 : 1;
            v.nodes *= v.vn[d];
        }
        if (v.nodes != plan[k].box_nodes) {
            set_error("plan[%d] inconsistent: box_nodes %lld vs box %lld", k,
                      (long long)plan[k].box_nodes, (long long)v.nodes);
            return HJ_ERR_INVALID;
        }
        v.V[0] = (T *)(base + L.off_v0[k]);
        v.V[1] = (T *)(base + L.off_v1[k]);
        v.cls = (const int8_t *)(base + L.off_cls[k]);
        v.res = res + (size_t)hv.size() * max_iter;
        v.work = cnt + m + hv.size();
        int blocks = (int)std::min<int64_t>((v.nodes + 255) / 256, 148 * 16);
        k_subdomain_classes<<<blocks, 256, 0, s>>>(mask, f.piece, k, v.o[0], v.o[1], v.o[2],
                                                   v.vn[0], v.vn[1], v.nodes, n0, n1,
                                                   (int8_t *)v.cls);
        hv.push_back(v);
        chgs.push_back((uint8_t *)(base + L.off_chg[k]));
        subs.push_back(k);
    }
    int nv = (int)hv.size();
    int gblocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 16);
    if (nv == 0) {
        std::vector<AsmView<T>> none;
        k_assemble<T><<<gblocks, 256, 0, s>>>(d_asm, 0, mask, n0, n1, N, (T)prob.v_out, Vbar);
        HJ_CUDA(cudaGetLastError());
        HJ_CUDA(cudaStreamSynchronize(s));
        return HJ_OK;
    }
    HJ_CUDA(cudaMemsetAsync(res, 0, (size_t)nv * max_iter * sizeof(double), s));
    HJ_CUDA(cudaMemsetAsync(cnt, 0, (size_t)2 * m * sizeof(unsigned long long), s));
    auto P = make_dev_problem<T, T>(grid, prob, f);
    // the views iterate together in groups of up to HJ_GROUP_VIEWS (one sweep launch, or
    // one cooperative launch, per group); the groups run one after the other
    IterResult r;
    r.buf.assign(nv, 0);
    r.iters.assign(nv, 0);
    r.converged.assign(nv, 0);
    r.resid.assign(nv, 0.0);
    r.ms = 0;
    r.launches = 0;
    int evals = prob.n_controls;
    for (int c0 = 0; c0 < nv; c0 += HJ_GROUP_VIEWS) {
        const int cn = std::min(nv - c0, HJ_GROUP_VIEWS);
        std::vector<SweepView<T>> hvc(hv.begin() + c0, hv.begin() + c0 + cn);
        std::vector<uint8_t *> chc(chgs.begin() + c0, chgs.begin() + c0 + cn);
        int64_t mx = 1;
        for (auto &v : hvc) mx = std::max(mx, v.nodes);
        SweepLaunch<T> SL;
        hj_status st = sweep_prepare(grid, prob, f, hvc, chc, group, base + L.off_wl, s, SL);
        if (st != HJ_OK) return st;
        evals = SL.evals;
        const SweepView<T> *d_views = &SL.d_group->v[0];
        int blocks = (int)std::min<int64_t>((mx + 255) / 256, 148 * 16);
        k_init_view<T><<<dim3(blocks, cn), 256, 0, s>>>(d_views, (T)prob.v_out, (const T *)f.g,
                                                        n0, n1);
        k_count_interior<T><<<dim3(blocks, cn), 256, 0, s>>>(d_views, cnt + c0);
        HJ_CUDA(cudaGetLastError());
        IterResult rc;
        st = iterate<T>(P, SL, cn, res + (size_t)c0 * max_iter, max_iter, tol, max_iter, s, rc);
        if (st != HJ_OK) return st;
        for (int q = 0; q < cn; ++q) {
            r.buf[c0 + q] = rc.buf[q];
            r.iters[c0 + q] = rc.iters[q];
            r.converged[c0 + q] = rc.converged[q];
            r.resid[c0 + q] = rc.resid[q];
        }
        r.ms += rc.ms;
        r.launches += rc.launches;
    }
    std::vector<AsmView<T>> ha(nv);
    for (int q = 0; q < nv; ++q) {
        for (int d = 0; d < 3; ++d) {
            ha[q].o[d] = hv[q].o[d];
            ha[q].vn[d] = hv[q].vn[d];
        }
        ha[q].V = hv[q].V[r.buf[q]];
        ha[q].sub = subs[q];
    }
    HJ_CUDA(cudaMemcpyAsync(d_asm, ha.data(), nv * sizeof(AsmView<T>), cudaMemcpyHostToDevice, s));
    k_assemble<T><<<gblocks, 256, 0, s>>>(d_asm, nv, mask, n0, n1, N, (T)prob.v_out, Vbar);
    HJ_CUDA(cudaGetLastError());
    std::vector<unsigned long long> interior(2 * m, 0);
    HJ_CUDA(cudaMemcpyAsync(interior.data(), cnt, 2 * m * sizeof(unsigned long long),
                            cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    bool all = true;
    for (int q = 0; q < nv; ++q) {
        all = all && r.converged[q];
        if (reps) {
            hj_report &rp = reps[subs[q]];
            rp.iterations = r.iters[q];
            rp.residual = r.resid[q];
            rp.converged = r.converged[q];
            rp.node_updates = (int64_t)interior[q] * prob.n_controls * r.iters[q];
            rp.evaluated_updates = (int64_t)interior[m + q] * evals;
            rp.device_ms = r.ms;
            rp.launches = q == 0 ? r.launches + nv + 3 + (f.speed ? 1 : 0) : 0;  // counted once
        }
    }
    if (!all) {
        set_error("a sub-domain did not converge within %lld iterations", (long long)max_iter);
        return HJ_ERR_NOT_CONVERGED;
    }
    return HJ_OK;
}

// ---------------------------------------------------------------------------
// RA: the paper's reconstruction of the independent sub-domains (PAPER.md line
// 310-331): m auxiliary solves with only piece i as the target, V = min_i V_i, and
// Sigma_i = X_i + {j : |V_i(j) - V(j)| <= 2 (C dx^q + M dx)}.
// ---------------------------------------------------------------------------
__global__ void k_piece_only(const int8_t *__restrict__ piece, int i, int64_t N, int8_t *out) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x)
        out[j] = piece[j] == i ? (int8_t)i : (int8_t)-1;
}

template <typename T>
__global__ void k_ra_masks(const T *__restrict__ Vaux, int m, int64_t N,
                           const int8_t *__restrict__ piece, double thr, T *Vmin,
                           uint64_t *mask) {
    for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
         j += (int64_t)gridDim.x * blockDim.x) {
        T v = Vaux[j];
        for (int i = 1; i < m; ++i) v = fmin(v, Vaux[(int64_t)i * N + j]);
        uint64_t bits = 0;
        for (int i = 0; i < m; ++i) {
            const double d = fabs((double)Vaux[(int64_t)i * N + j] - (double)v);
            if (piece[j] == i || d <= thr) bits |= 1ull << i;
        }
        Vmin[j] = v;
        mask[j] = bits;
    }
}

template <typename T>
static size_t ra_ws(const hj_grid &g, int64_t max_iter) {
    return Carver::align(grid_nodes(g)) + solve_ws<T>(g, max_iter);
}

template <typename T>
static hj_status ra_impl(const hj_grid &cg, const hj_problem &cp, const hj_fields &cf, int m,
                         double C, double M, double q, double tol, int64_t max_iter,
                         const hj_grid &fg, const int32_t ratio[3], int32_t band,
                         const int8_t *fine_piece, T *Vaux, T *Vmin, uint64_t *cmask,
                         uint64_t *fmask, void *ws, size_t ws_bytes, cudaStream_t s,
                         hj_report *reps) {
    const int64_t N = grid_nodes(cg);
    if (ws_bytes < ra_ws<T>(cg, max_iter)) {
        set_error("workspace too small: need %zu bytes, got %zu", ra_ws<T>(cg, max_iter), ws_bytes);
        return HJ_ERR_WORKSPACE;
    }
    int8_t *pi = (int8_t *)ws;
    char *sws = (char *)ws + Carver::align(N);
    const size_t sws_bytes = ws_bytes - Carver::align(N);
    const int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 16);
    for (int i = 0; i < m; ++i) {          // 1) the auxiliary problems (dG := X_i)
        k_piece_only<<<blocks, 256, 0, s>>>(cf.piece, i, N, pi);
        HJ_CUDA(cudaGetLastError());
        hj_fields fi = cf;
        fi.piece = pi;
        hj_report r;
        memset(&r, 0, sizeof(r));
        hj_status st = solve_impl<T>(cg, cp, fi, Vaux + (int64_t)i * N, tol, max_iter, sws,
                                     sws_bytes, s, &r);
        if (reps) reps[i] = r;
        if (st != HJ_OK) return st;
    }
    double dx = 0;                         // 2-3) V = min_i V_i, the sets Sigma_i
    for (int d = 0; d < cg.dim; ++d) dx = std::max(dx, grid_spacing(cg, d));
    const double thr = 2.0 * (C * std::pow(dx, q) + M * dx);
    k_ra_masks<T><<<blocks, 256, 0, s>>>(Vaux, m, N, cf.piece, thr, Vmin, cmask);
    HJ_CUDA(cudaGetLastError());
    if (fmask) {                           // ISA step 2 with the band (R9)
        hj_status st = prolong_launch(cg, fg, ratio, band, m, cmask, true, fine_piece, fmask, s);
        if (st != HJ_OK) return st;
    }
    HJ_CUDA(cudaStreamSynchronize(s));
    return HJ_OK;
}

}  // namespace hj

using namespace hj;

extern "C" {

/* Profiling aid (not part of the documented ABI surface): per-CTA trace of the
 * temporally blocked sweep into a device buffer of 4 * cap uint64; NULL disables. */
int hj_debug_set_trace(void *dev_buf, long long cap, long long n0) {
    TBTrace t{(unsigned long long *)dev_buf, dev_buf ? cap : 0, n0};
    return cudaMemcpyToSymbol(g_tb_trace, &t, sizeof(t)) == cudaSuccess ? 0 : 1;
}

size_t hj_solve_workspace_bytes(const hj_grid *grid, int32_t dtype, int64_t max_iter) {
    if (!grid || validate_grid(grid) != HJ_OK || max_iter < 1) return 0;
    int64_t N = grid_nodes(*grid);
    return dtype == HJ_F64 ? solve_ws<double>(*grid, max_iter) : solve_ws<float>(*grid, max_iter);
}

hj_status hj_solve(const hj_grid *grid, const hj_problem *prob, const hj_fields *fields,
                   int32_t dtype, void *V, double tol, int64_t max_iter, void *workspace,
                   size_t ws_bytes, void *stream, hj_report *report) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(grid)) != HJ_OK) return st;
    if ((st = validate_problem(grid, prob)) != HJ_OK) return st;
    if ((st = validate_fields(fields)) != HJ_OK) return st;
    HJ_CHECK(V != nullptr && workspace != nullptr, "V / workspace is NULL");
    HJ_CHECK(max_iter >= 1, "max_iter must be >= 1");
    HJ_CHECK(tol > 0, "tol must be > 0");
    HJ_CHECK(dtype == HJ_F32 || dtype == HJ_F64, "dtype must be HJ_F32 or HJ_F64");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == HJ_F64)
        return solve_impl<double>(*grid, *prob, *fields, (double *)V, tol, max_iter, workspace,
                                  ws_bytes, s, report);
    return solve_impl<float>(*grid, *prob, *fields, (float *)V, tol, max_iter, workspace,
                             ws_bytes, s, report);
}

size_t hj_ra_workspace_bytes(const hj_grid *coarse_grid, int32_t dtype, int64_t max_iter) {
    if (!coarse_grid || validate_grid(coarse_grid) != HJ_OK || max_iter < 1) return 0;
    return dtype == HJ_F64 ? ra_ws<double>(*coarse_grid, max_iter)
                           : ra_ws<float>(*coarse_grid, max_iter);
}

hj_status hj_ra_subdomains(const hj_grid *cg, const hj_problem *cp, const hj_fields *cf,
                           int32_t dtype, int32_t m, double C, double M, double q, double tol,
                           int64_t max_iter, const hj_grid *fg, const int32_t ratio[3],
                           int32_t band, const int8_t *fine_piece, void *Vaux, void *Vmin,
                           uint64_t *coarse_mask, uint64_t *fine_mask, void *workspace,
                           size_t ws_bytes, void *stream, hj_report *reports) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(cg)) != HJ_OK) return st;
    if ((st = validate_problem(cg, cp)) != HJ_OK) return st;
    if ((st = validate_fields(cf)) != HJ_OK) return st;
    HJ_CHECK(m >= 1 && m <= HJ_MAX_SUBDOMAINS, "m must be in [1, %d]", HJ_MAX_SUBDOMAINS);
    HJ_CHECK(Vaux && Vmin && coarse_mask && workspace, "NULL argument");
    HJ_CHECK(C >= 0 && M >= 0 && q > 0, "need C >= 0, M >= 0, q > 0");
    HJ_CHECK(max_iter >= 1 && tol > 0, "need max_iter >= 1 and tol > 0");
    HJ_CHECK(dtype == HJ_F32 || dtype == HJ_F64, "dtype must be HJ_F32 or HJ_F64");
    if (fine_mask) {
        HJ_CHECK(fg && ratio && fine_piece, "fine_mask needs fine_grid, ratio and fine_piece");
        if ((st = validate_grid(fg)) != HJ_OK) return st;
        HJ_CHECK(band >= 0 && cg->dim == fg->dim, "band >= 0 and equal dims required");
        for (int d = 0; d < cg->dim; ++d) {
            HJ_CHECK(ratio[d] >= 1, "ratio[%d] must be >= 1", d);
            if (fg->periodic[d])
                HJ_CHECK(fg->n[d] == ratio[d] * cg->n[d], "periodic axis %d not nested", d);
            else
                HJ_CHECK(fg->n[d] - 1 == ratio[d] * (cg->n[d] - 1), "axis %d not nested", d);
        }
    }
    cudaStream_t s = (cudaStream_t)stream;
    const hj_grid &fgr = fine_mask ? *fg : *cg;
    if (dtype == HJ_F64)
        return ra_impl<double>(*cg, *cp, *cf, m, C, M, q, tol, max_iter, fgr, ratio, band,
                               fine_piece, (double *)Vaux, (double *)Vmin, coarse_mask, fine_mask,
                               workspace, ws_bytes, s, reports);
    return ra_impl<float>(*cg, *cp, *cf, m, C, M, q, tol, max_iter, fgr, ratio, band, fine_piece,
                          (float *)Vaux, (float *)Vmin, coarse_mask, fine_mask, workspace,
                          ws_bytes, s, reports);
}

hj_status hj_partition_plan(const hj_grid *grid, const uint64_t *fine_mask, int32_t m,
                            int32_t dtype, int64_t max_iter, hj_subdomain *plan,
                            size_t *ws_bytes, void *stream) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(grid)) != HJ_OK) return st;
    HJ_CHECK(m >= 1 && m <= HJ_MAX_SUBDOMAINS, "m must be in [1, %d]", HJ_MAX_SUBDOMAINS);
    HJ_CHECK(fine_mask && plan && ws_bytes, "NULL argument");
    HJ_CHECK(max_iter >= 1, "max_iter must be >= 1");
    cudaStream_t s = (cudaStream_t)stream;
    int64_t N = grid_nodes(*grid);
    // a small device scratch kept for the process (one per device), not a per-call malloc
    static thread_local void *scratch[64] = {nullptr};
    int dev = 0;
    HJ_CUDA(cudaGetDevice(&dev));
    HJ_CHECK(dev >= 0 && dev < 64, "device index out of range");
    if (!scratch[dev])
        HJ_CUDA(cudaMalloc(&scratch[dev], sizeof(int) * 6 * HJ_MAX_SUBDOMAINS +
                                              sizeof(unsigned long long) * HJ_MAX_SUBDOMAINS));
    int *d_bb = (int *)scratch[dev];
    unsigned long long *d_cnt = (unsigned long long *)(d_bb + 6 * HJ_MAX_SUBDOMAINS);
    k_fill_int<<<1, 6 * HJ_MAX_SUBDOMAINS, 0, s>>>(d_bb, 6 * HJ_MAX_SUBDOMAINS, 0x7fffffff, -1);
    HJ_CUDA(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long) * HJ_MAX_SUBDOMAINS, s));
    int blocks = (int)std::min<int64_t>((N + 255) / 256, 148 * 8);
    int64_t n0 = grid->n[0], n1 = grid->dim > 1 ? grid->n[1] : 1;
    k_plan<<<blocks, 256, 0, s>>>(fine_mask, N, n0, n1, m, d_bb, d_cnt);
    int hbb[6 * HJ_MAX_SUBDOMAINS];
    unsigned long long hcnt[HJ_MAX_SUBDOMAINS];
    HJ_CUDA(cudaMemcpyAsync(hbb, d_bb, sizeof(hbb), cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaMemcpyAsync(hcnt, d_cnt, sizeof(hcnt), cudaMemcpyDeviceToHost, s));
    HJ_CUDA(cudaStreamSynchronize(s));
    HJ_CUDA(cudaGetLastError());
    for (int k = 0; k < m; ++k) {
        hj_subdomain &p = plan[k];
        memset(&p, 0, sizeof(p));
        p.n_nodes = (int64_t)hcnt[k];
        if (!p.n_nodes) continue;
        p.box_nodes = 1;
        int64_t extent = 1;
        for (int d = 0; d < 3; ++d) {
            if (d >= grid->dim) {
                p.lo[d] = p.hi[d] = 0;
                continue;
            }
            if (grid->periodic[d]) {
                p.lo[d] = 0;
                p.hi[d] = grid->n[d] - 1;
            } else {
                p.lo[d] = hbb[6 * k + d];
                p.hi[d] = hbb[6 * k + 3 + d];
            }
            p.box_nodes *= p.hi[d] - p.lo[d] + 1;
            extent = std::max<int64_t>(extent, p.hi[d] - p.lo[d] + 1);
        }
        // sweeps scale with the extent, work per sweep with the nodes
        p.work = (double)p.n_nodes * (double)extent;
    }
    *ws_bytes = dtype == HJ_F64 ? part_layout<double>(m, plan, max_iter).total
                                : part_layout<float>(m, plan, max_iter).total;
    return HJ_OK;
}

hj_status hj_solve_partitioned(const hj_grid *grid, const hj_problem *prob,
                               const hj_fields *fields, int32_t dtype, const uint64_t *fine_mask,
                               int32_t m, const hj_subdomain *plan, uint64_t solve_set, double tol,
                               int64_t max_iter, void *Vbar, void *workspace, size_t ws_bytes,
                               void *stream, hj_report *reports) {
    clear_error();
    hj_status st;
    if ((st = validate_grid(grid)) != HJ_OK) return st;
    if ((st = validate_problem(grid, prob)) != HJ_OK) return st;
    if ((st = validate_fields(fields)) != HJ_OK) return st;
    HJ_CHECK(m >= 1 && m <= HJ_MAX_SUBDOMAINS, "m must be in [1, %d]", HJ_MAX_SUBDOMAINS);
    HJ_CHECK(fine_mask && plan && Vbar && workspace, "NULL argument");
    HJ_CHECK(max_iter >= 1 && tol > 0, "need max_iter >= 1 and tol > 0");
    HJ_CHECK(dtype == HJ_F32 || dtype == HJ_F64, "dtype must be HJ_F32 or HJ_F64");
    cudaStream_t s = (cudaStream_t)stream;
    if (dtype == HJ_F64)
        return partitioned_impl<double>(*grid, *prob, *fields, fine_mask, m, plan, solve_set,
                                        tol, max_iter, (double *)Vbar, workspace, ws_bytes, s,
                                        reports);
    return partitioned_impl<float>(*grid, *prob, *fields, fine_mask, m, plan, solve_set, tol,
                                   max_iter, (float *)Vbar, workspace, ws_bytes, s, reports);
}

}  // extern "C"
