// hj_host.cu — error state, validation and the host-side partitioner.
#include <algorithm>
#include <numeric>
#include <vector>

#include "hj_host.cuh"

namespace hj {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

void clear_error() { g_err[0] = 0; }

hj_status validate_grid(const hj_grid *g) {
    HJ_CHECK(g != nullptr, "grid is NULL");
    HJ_CHECK(g->dim == 2 || g->dim == 3, "grid.dim must be 2 or 3 (got %d)", g->dim);
    for (int d = 0; d < g->dim; ++d) {
        HJ_CHECK(g->n[d] >= 2, "grid.n[%d] must be >= 2 (got %lld)", d, (long long)g->n[d]);
        HJ_CHECK(g->hi[d] > g->lo[d], "grid.hi[%d] must exceed grid.lo[%d]", d, d);
    }
    HJ_CHECK(grid_nodes(*g) < ((int64_t)1 << 40), "grid too large");
    return HJ_OK;
}

hj_status validate_problem(const hj_grid *g, const hj_problem *p) {
    HJ_CHECK(p != nullptr, "problem is NULL");
    HJ_CHECK(p->n_controls >= 1 && p->n_controls <= HJ_MAX_CONTROLS,
             "n_controls must be in [1, %d] (got %d)", HJ_MAX_CONTROLS, p->n_controls);
    HJ_CHECK(p->dynamics >= 0 && p->dynamics <= 2, "unknown dynamics %d", p->dynamics);
    HJ_CHECK(p->cost == HJ_COST_KRUZKOV || p->cost == HJ_COST_DISCOUNTED, "unknown cost %d",
             p->cost);
    HJ_CHECK(p->dynamics != HJ_DYN_DUBINS || g->dim == 3, "Dubins dynamics needs dim 3");
    HJ_CHECK(p->dynamics != HJ_DYN_DUBINS || g->periodic[2], "Dubins heading axis must be periodic");
    HJ_CHECK(p->dynamics != HJ_DYN_VANDERPOL || g->dim == 2, "Van der Pol dynamics needs dim 2");
    HJ_CHECK(p->h > 0 && std::isfinite(p->h), "h must be > 0");
    HJ_CHECK(p->lambda >= 0 && std::isfinite(p->lambda), "lambda must be >= 0");
    HJ_CHECK(std::isfinite(p->v_out), "v_out must be finite");
    return HJ_OK;
}

double *pinned_scratch(size_t count) {
    static thread_local double *buf = nullptr;
    static thread_local size_t cap = 0;
    if (count > cap) {
        if (buf) cudaFreeHost(buf);
        size_t want = std::max<size_t>(count, 4096);
        if (cudaMallocHost(&buf, want * sizeof(double)) != cudaSuccess) {
            buf = nullptr;
            cap = 0;
            return nullptr;
        }
        cap = want;
    }
    return buf;
}

}  // namespace hj

extern "C" {

const char *hj_last_error(void) { return hj::g_err; }

const char *hj_version(void) { return "hj-b200 0.1 sm_100a"; }

// Longest-processing-time-first: sort sub-domains by decreasing work, give each
// to the currently least-loaded rank (ties: lowest rank / lowest index).
hj_status hj_assign_subdomains(int32_t m, const hj_subdomain *plan, int32_t n_ranks,
                               int32_t *owner) {
    hj::clear_error();
    HJ_CHECK(m >= 1 && m <= HJ_MAX_SUBDOMAINS, "m must be in [1, %d]", HJ_MAX_SUBDOMAINS);
    HJ_CHECK(n_ranks >= 1, "n_ranks must be >= 1");
    HJ_CHECK(plan != nullptr && owner != nullptr, "plan/owner is NULL");
    std::vector<int> order(m);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(),
                     [&](int a, int b) { return plan[a].work > plan[b].work; });
    std::vector<double> load(n_ranks, 0.0);
    for (int k : order) {
        int best = 0;
        for (int r = 1; r < n_ranks; ++r)
            if (load[r] < load[best]) best = r;
        owner[k] = best;
        load[best] += plan[k].work;
    }
    return HJ_OK;
}

}  // extern "C"
