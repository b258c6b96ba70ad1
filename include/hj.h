/*
 * hj.h — C ABI of the B200 semi-Lagrangian Hamilton-Jacobi-Bellman hot path.
 *
 * Implements, on sm_100a, the data-parallel hot path of
 *   A. Festa, "Reconstruction of independent sub-domains for a class of
 *   Hamilton-Jacobi equations and application to parallel computing"
 *   (arxiv 1405.3521; /root/reference/PAPER.md, cited as "PAPER.md line N").
 *
 * The four operations the north_star names, plus the two host helpers the
 * partitioned solve needs:
 *
 *   hj_solve              value iteration V^{n+1} = T(V^n) of the SL scheme
 *                         (PAPER.md eq. (SL); operator (Tdef), line 238-245)
 *   hj_coarse_feedback    discrete optimal feedback a*(x_i) = argmin of the Tdef
 *                         bracket at every node of a (coarse) grid
 *   hj_label_subdomains   label every coarse node by the target piece its discrete
 *                         optimal feedback trajectory reaches; prolong the labels to
 *                         the fine grid with an overlap band (ISA steps 1-2,
 *                         PAPER.md line 396-418)
 *   hj_ra_subdomains      the paper's RA reconstruction (auxiliary solves + threshold,
 *                         PAPER.md line 310-331), prolonged the same way
 *   hj_partition_plan     bounding boxes / sizes of the fine sub-domains
 *   hj_assign_subdomains  host partitioner: sub-domains -> ranks (GPUs)
 *   hj_solve_partitioned  independent fine solves on the sub-domains and the
 *                         min-assembly Vbar(j) = min{V_i(j) | x_j in S_i}
 *                         (ISA steps 3-4)
 *
 * CONVENTIONS (all entry points)
 *  - Grid: node (i0,i1,i2) at x_d = lo[d] + i_d*dx_d, dx_d = (hi-lo)/(n-1), or
 *    (hi-lo)/n on a periodic axis.  Node fields are dense, axis 0 fastest:
 *    flat index = i0 + n0*(i1 + n1*i2).  dim is 2 or 3.
 *  - "device" pointers must be CUDA device (or managed) memory on the current
 *    device; "host" pointers are ordinary host memory.  Callers pass workspaces
 *    sized by the *_bytes / plan queries and own every buffer; the library's only
 *    own allocations are a < 2 KB device scratch per device and thread (kept for the
 *    process, allocated on first use) and a small pinned host staging buffer per thread.  All device work is enqueued on
 *    `stream` (a cudaStream_t, NULL = legacy default stream).
 *  - Value dtype: HJ_F32 or HJ_F64 selects the storage and arithmetic type of V
 *    and of the node fields speed/g.  Feedback and labelling decisions are
 *    always taken in fp64 (on V converted to fp64).
 *  - Errors: every function returns hj_status; on failure nothing is written to
 *    host outputs except what is documented, and hj_last_error() returns a
 *    one-line message (thread-local).  No function aborts the process.
 *  - Readings of the paper (R1..R13) are listed in DESIGN.md §3.
 */
#ifndef HJ_H_
#define HJ_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HJ_MAX_DIM 3
#define HJ_MAX_CONTROLS 128
#define HJ_MAX_SUBDOMAINS 64    /* sets of a membership mask (its uint64 bits): the
                                   target pieces plus, optionally, the exit set */

typedef enum {
    HJ_OK = 0,
    HJ_ERR_INVALID = 1,        /* bad argument (message says which)            */
    HJ_ERR_CUDA = 2,           /* a CUDA runtime call failed                    */
    HJ_ERR_NOT_CONVERGED = 3,  /* max_iter reached; outputs are valid iterates */
    HJ_ERR_UNSUPPORTED = 4,    /* valid but not implemented combination        */
    HJ_ERR_WORKSPACE = 5       /* workspace too small                           */
} hj_status;

enum { HJ_F32 = 0, HJ_F64 = 1 };

/* Dynamics families f(x,a) (§2 line 33-37, "y' = f(y,a)"). */
enum {
    HJ_DYN_AFFINE = 0,     /* f = c(x) u_a + A x + b   (u_a = controls[k][0..dim-1])   */
    HJ_DYN_DUBINS = 1,     /* dim 3: f = (v cos x2, v sin x2, w a), a = controls[k][0] */
    HJ_DYN_VANDERPOL = 2   /* dim 2: f = (x1, mu (1 - x0^2) x1 - x0 + a), PAPER.md
                              line 536;   a = controls[k][0]                         */
};

/* Cost families: the Tdef bracket (R1) is  beta I[V](x + h f(x,a)) + c(x,a)  with
 * beta = 1/(1 + lambda h) and
 *   HJ_COST_KRUZKOV:     c = 1 - beta   (Kruzkov-transformed minimum time, v = 1-exp(-lambda T))
 *   HJ_COST_DISCOUNTED:  c = h l(x,a),  l = l0 + lq |x|^2 + ln |x| + lr |a|^2
 *                        (|x| over the non-periodic axes, |a| over controls[k][0..2]). */
enum { HJ_COST_KRUZKOV = 0, HJ_COST_DISCOUNTED = 1 };

/* Sweep kernels (all compute the same Jacobi sweep).  AUTO picks, in
 * order: LOCAL_COOP when the problem qualifies for the local kernels (2-D, f = c(x) u_a,
 * every foot within one cell, no periodic axis): the whole iteration in one cooperative
 * launch over node-level dirty 8x8 mini-tiles (LOCAL_TB: 8 sweeps per launch, temporally
 * blocked in shared memory) — FFMA2-packed for fp32, bit-identical iterates to the
 * one-sweep LOCAL_PACKED (fp32 only) / LOCAL_SCALAR kernels; FIELD_COOP for any other 2-D
 * affine / Van der Pol problem whose feet stay within one cell (the same cooperative
 * scheme, the foot's cell picked by the signs of its offsets); FIELD_COL for the other 2-D
 * affine problems without a speed field whose controls share their axis-0 component
 * (config 5: one x-interpolated column per node, walked once over the controls sorted by
 * their axis-1 component — bit-identical iterates to FIELD2D), and among those FIELD_LAT
 * for discounted problems with 17/33/65 controls whose axis-1 feet are exactly one row
 * apart and whose axis-1 drift does not depend on x1 (config 5: eight nodes of a column
 * per thread stream the rows once; every control shares the foot's axis-1 weight —
 * bit-identical to FIELD2D when the per-control foot sums are exact, as on config 5);
 * FIELD2D for the other 2-D
 * affine / Van der Pol problems without periodic axes; DUBINS_COOP (the cooperative
 * scheme on 8x8 mini-tiles of each heading plane) for Dubins problems whose (x, y) and
 * heading steps stay within one cell; DUBINS for Dubins dynamics whose heading step is <= 1 cell; GENERIC
 * otherwise.  The two LOCAL kernels give bit-identical iterates; the others evaluate
 * the same bracket in other operation orders (equal up to rounding). */
enum { HJ_SWEEP_AUTO = 0, HJ_SWEEP_GENERIC = 1, HJ_SWEEP_LOCAL_SCALAR = 2,
       HJ_SWEEP_LOCAL_PACKED = 3, HJ_SWEEP_FIELD2D = 4, HJ_SWEEP_DUBINS = 5,
       HJ_SWEEP_LOCAL_TB = 6, HJ_SWEEP_LOCAL_COOP = 7, HJ_SWEEP_FIELD_COOP = 8,
       HJ_SWEEP_DUBINS_COOP = 9, HJ_SWEEP_FIELD_COL = 10, HJ_SWEEP_FIELD_LAT = 11 };

typedef struct {
    int32_t dim;            /* 2 or 3                                          */
    int32_t periodic[3];    /* 1 = periodic axis (e.g. Dubins heading)         */
    int64_t n[3];           /* nodes per axis, >= 2 (unused axes: 1)           */
    double lo[3], hi[3];    /* box [lo, hi] (periodic: [lo, hi) )              */
} hj_grid;

typedef struct {
    int32_t dynamics;                        /* HJ_DYN_*                      */
    int32_t cost;                            /* HJ_COST_*                     */
    int32_t n_controls;                      /* 1 .. HJ_MAX_CONTROLS          */
    int32_t sweep_kernel;                    /* HJ_SWEEP_*: 0 = automatic choice;
                                                an explicit kernel the problem does
                                                not qualify for -> HJ_ERR_UNSUPPORTED */
    double controls[HJ_MAX_CONTROLS][3];     /* discrete control set A (PAPER.md
                                                line 248), meaning per dynamics */
    double A[3][3], b[3];                    /* affine drift                  */
    double dubins_v, dubins_w, vdp_mu;
    double lambda;                           /* discount, >= 0                */
    double h;                                /* fictitious time step, > 0     */
    double l0, lq, ln, lr;                   /* running cost coefficients     */
    double v_out;                            /* value of a foot outside the box
                                                and of ghost nodes (R3): 1 for
                                                Kruzkov ("T = +inf")           */
} hj_problem;

/* Node fields describing the problem on one grid (device pointers). */
typedef struct {
    const void *speed;      /* c(x) in the value dtype, or NULL (c == 1); only
                               HJ_DYN_AFFINE reads it.  Off-grid (trajectory) points
                               use its multilinear interpolation.                */
    const int8_t *piece;    /* REQUIRED: target piece of each node (the vectors X_i,
                               PAPER.md line 314), -1 = not a target node.  Target
                               nodes are the boundary nodes dG of Tdef.          */
    const void *g;          /* g(x_i) on target nodes in the value dtype, or NULL
                               (g == 0)                                          */
} hj_fields;

typedef struct {
    int64_t iterations;     /* applications of T performed until the stop       */
    double residual;        /* ||V^{n} - V^{n-1}||_inf of the last one          */
    int32_t converged;      /* residual < tol                                   */
    int32_t reserved;
    int64_t node_updates;   /* Jacobi work: interior nodes x controls x iterations */
    double device_ms;       /* device time of the iteration (CUDA events)       */
    int64_t launches;       /* kernels this call launched (sweeps + helpers)    */
    int64_t evaluated_updates; /* interior nodes x controls actually evaluated: the
                               sweeps skip tiles whose inputs did not change (their
                               T(V) is known exactly), so this is <= node_updates  */
} hj_report;

typedef struct {            /* one fine sub-domain S_k (hj_partition_plan)       */
    int64_t lo[3], hi[3];   /* inclusive node bounding box (full extent on
                               periodic axes); empty if n_nodes == 0            */
    int64_t n_nodes;        /* nodes with bit k set in the fine mask            */
    int64_t box_nodes;      /* nodes of the bounding box                        */
    double work;            /* work estimate used by hj_assign_subdomains       */
} hj_subdomain;

/* Thread-local message of the last failure ("" if none). */
const char *hj_last_error(void);

/* Library version string and the compiled device architecture ("sm_100a"). */
const char *hj_version(void);

/* ---------------------------------------------------------------------------
 * hj_solve — value iteration of the semi-Lagrangian scheme on the whole grid.
 *
 * Operation (PAPER.md eq. (SL), (Tdef) line 238-245, reading R1):
 *   [T(V)]_i = min_{a in A} { beta I[V](x_i + h f(x_i,a)) + c(x_i,a) }  (interior)
 *   [T(V)]_i = g(x_i)                                                    (target)
 * I = multilinear interpolation (line 247, R4); feet outside the box read
 * v_out (R3).  V^0 = g on target nodes, v_out elsewhere; iterate V^{n+1} = T(V^n)
 * (Jacobi, line 248) and stop at the first n with ||V^{n+1}-V^n||_inf < tol
 * (stopping remark, line 341-345; R6) or after max_iter applications.
 *
 * Arguments
 *   grid, prob, fields  problem statement (host structs; fields hold device ptrs)
 *   dtype               HJ_F32 / HJ_F64
 *   V                   device, N = prod(n) values: OUTPUT, the final iterate
 *   tol, max_iter       stopping rule; max_iter >= 1
 *   workspace, ws_bytes device scratch of at least hj_solve_workspace_bytes()
 *   stream              cudaStream_t
 *   report              host, may be NULL
 * Returns HJ_OK, HJ_ERR_NOT_CONVERGED (V holds iterate max_iter), or an error.
 * Synchronises the stream before returning.
 * ------------------------------------------------------------------------- */
size_t hj_solve_workspace_bytes(const hj_grid *grid, int32_t dtype, int64_t max_iter);

hj_status hj_solve(const hj_grid *grid, const hj_problem *prob, const hj_fields *fields,
                   int32_t dtype, void *V, double tol, int64_t max_iter, void *workspace,
                   size_t ws_bytes, void *stream, hj_report *report);

/* ---------------------------------------------------------------------------
 * hj_coarse_feedback — the discrete optimal feedback at every node:
 *   astar[i]  = lowest index k minimising the Tdef bracket at x_i (R7),
 *               -1 on target nodes;
 *   margin[i] = second smallest bracket - smallest (+inf if one control,
 *               +inf on target nodes).
 * V: device, N values of dtype (normally the converged hj_solve output).
 * astar: device int32[N]; margin: device double[N] (may be NULL).
 * Decisions are taken in fp64.  Asynchronous on `stream`.
 * ------------------------------------------------------------------------- */
hj_status hj_coarse_feedback(const hj_grid *grid, const hj_problem *prob,
                             const hj_fields *fields, int32_t dtype, const void *V,
                             int32_t *astar, double *margin, void *stream);

/* ---------------------------------------------------------------------------
 * hj_label_subdomains — reconstruction of the independent sub-domains.
 *
 * (a) For every coarse node z (R8): y_0 = z, y_{s+1} = y_s + h f(y_s, a*(y_s)) with
 *     a*(y) the lowest-index argmin of the Tdef bracket evaluated AT y (V
 *     interpolated); the label is the piece of the first y_s whose nearest node
 *     (floor(g + 1/2) in index space) is a target node; -1 if y leaves the box or
 *     n_max steps pass.  (Independent sub-domain: PAPER.md Definition 2.2 line
 *     150-152, Proposition 2.3 line 156-163 — optimal trajectories stay in it.)
 *     Exit set (reading R9b): with Vexit given, an unlabelled node whose value needs no
 *     target, Vc(z) >= Vexit(z) - exit_tol, is labelled -2: it belongs to the
 *     sub-domain of the box-boundary piece of Gamma (exit cost v_out), set m.
 * (b) Prolongation with overlap band (R9; ISA step 2, line 398-418): fine node i
 *     is in S_k iff a coarse node I labelled k has |i_d - R_d I_d| <= R_d + band on
 *     every axis; a node labelled -1 counts for every piece's set (0..m-1), a node
 *     labelled -2 for the exit set m only; fine target nodes of piece k are always in S_k.
 *
 * coarse_grid/prob/coarse_fields/dtype/Vc  the coarse problem and its solution
 *     (device Vc); the trajectory uses coarse_prob.h.
 * Vexit          device, N_c values of dtype: the coarse solution with NO target node
 *                (the exit is the only way the cost ends), or NULL (no exit set: -1
 *                labels join every piece's set, R9)
 * exit_tol       >= 0, the exit test's threshold (ignored without Vexit)
 * n_max          step budget per trajectory (>= 0)
 * fine_grid      nested fine grid: (n_f - 1) = R (n_c - 1), or n_f = R n_c periodic
 * ratio[3]       R per axis (1 for unused axes); band >= 0 in fine cells
 * m              number of target pieces, 1..64 (1..63 with Vexit: the exit set is bit m)
 * fine_piece     device int8[N_f] target pieces on the fine grid; piece values must
 *                lie in [-1, m): a piece >= m (not checked on the device) belongs to
 *                no sub-domain bit
 * The trajectory's own arithmetic (x(y_s), the speed at y_s, f, y_s + h f / dx) is
 * evaluated with every operation rounded separately in the recursion's left-to-right
 * order, so the positions depend only on the controls taken (R8/R11); an
 * all-NaN bracket set (a NaN in Vc) ends the trajectory unlabelled (-1).
 * Outputs (device): label int32[N_c]; margin double[N_c] = min control margin
 *     along the trajectory; geo double[N_c] = min distance (index units) of a
 *     rounding / box decision to its threshold; steps int32[N_c];
 *     fine_mask uint64[N_f] bit k = node in S_k (k = m: the exit set).
 *     margin/geo/steps may be NULL.
 * Asynchronous on `stream`.
 * ------------------------------------------------------------------------- */
hj_status hj_label_subdomains(const hj_grid *coarse_grid, const hj_problem *coarse_prob,
                              const hj_fields *coarse_fields, int32_t dtype, const void *Vc,
                              const void *Vexit, double exit_tol, int64_t n_max,
                              const hj_grid *fine_grid, const int32_t ratio[3], int32_t band,
                              int32_t m, const int8_t *fine_piece, int32_t *label,
                              double *margin, double *geo, int32_t *steps,
                              uint64_t *fine_mask, void *stream);

/* ---------------------------------------------------------------------------
 * hj_ra_subdomains — the paper's own reconstruction algorithm RA (PAPER.md
 * line 310-331), an alternative to hj_label_subdomains' trajectory labels:
 *   1) for i = 0..m-1 solve V_i = T_i(V_i) on the (coarse) grid with only piece i as
 *      the target (dG := X_i; the other pieces' nodes are ordinary nodes), as hj_solve;
 *   2) V = min_i V_i;
 *   3) Sigma_i = X_i + {x_j : |V_i(j) - V(j)| <= 2 (C dx^q + M dx)}, dx = the largest
 *      spacing of the grid (C, M, q: the constants of condition (C), line 290-300);
 * then, if fine_mask != NULL, ISA step 2: the sets are prolonged to the nested fine grid
 * with the overlap band exactly as hj_label_subdomains does with labels (R9).
 * Vaux: device, m * N_c values of dtype (V_i of piece i at [i * N_c]); Vmin: device
 * N_c values; coarse_mask: device uint64[N_c], bit i = node in Sigma_i; fine_mask:
 * device uint64[N_f] or NULL.  workspace: device, >= hj_ra_workspace_bytes().
 * reports: host hj_report[m] (one per auxiliary solve), may be NULL.
 * Returns HJ_ERR_NOT_CONVERGED if an auxiliary solve hit max_iter.  Synchronises.
 * ------------------------------------------------------------------------- */
size_t hj_ra_workspace_bytes(const hj_grid *coarse_grid, int32_t dtype, int64_t max_iter);

hj_status hj_ra_subdomains(const hj_grid *coarse_grid, const hj_problem *coarse_prob,
                           const hj_fields *coarse_fields, int32_t dtype, int32_t m, double C,
                           double M, double q, double tol, int64_t max_iter,
                           const hj_grid *fine_grid, const int32_t ratio[3], int32_t band,
                           const int8_t *fine_piece, void *Vaux, void *Vmin,
                           uint64_t *coarse_mask, uint64_t *fine_mask, void *workspace,
                           size_t ws_bytes, void *stream, hj_report *reports);

/* ---------------------------------------------------------------------------
 * hj_partition_plan — sizes of the fine sub-domains S_0..S_{m-1} from the mask
 * (m = the number of sets: the pieces, plus one for the exit set when labelled with it).
 * fine_mask: device uint64[N]; plan: host hj_subdomain[m] (output).
 * *ws_bytes (output) = workspace hj_solve_partitioned needs to solve ALL m
 * sub-domains with this dtype/max_iter (a subset needs no more).
 * Synchronises the stream.
 * ------------------------------------------------------------------------- */
hj_status hj_partition_plan(const hj_grid *fine_grid, const uint64_t *fine_mask, int32_t m,
                            int32_t dtype, int64_t max_iter, hj_subdomain *plan,
                            size_t *ws_bytes, void *stream);

/* ---------------------------------------------------------------------------
 * hj_assign_subdomains — host-only partitioner of the independent sub-domains
 * over n_ranks GPUs: longest-processing-time-first on plan[k].work.
 * owner: host int32[m] (output), owner[k] in [0, n_ranks).  Deterministic.
 * ------------------------------------------------------------------------- */
hj_status hj_assign_subdomains(int32_t m, const hj_subdomain *plan, int32_t n_ranks,
                               int32_t *owner);

/* ---------------------------------------------------------------------------
 * hj_solve_partitioned — ISA steps 3-4 for the sub-domains in `solve_set`.
 *
 * For every k with bit k of solve_set: value iteration (as hj_solve) on S_k, with
 * nodes outside S_k acting as ghost nodes holding v_out (R10) and every target
 * node inside S_k holding g; all selected sub-domains iterate concurrently and
 * stop independently (in groups of up to 32 at a time).  Then
 *     Vbar[j] = min { V_k[j] : k in solve_set, bit k of fine_mask[j] }   (v_out if none).
 * Multi-GPU: each rank passes its own solve_set; the element-wise MIN of the
 * ranks' Vbar over NCCL is the ISA result (no exchange during the solves).
 *
 * Vbar: device, N_f values (output).  workspace: device, >= plan ws_bytes.
 * reports: host hj_report[m] (entries of unsolved k untouched), may be NULL.
 * Returns HJ_ERR_NOT_CONVERGED if any selected sub-domain hit max_iter.
 * Synchronises the stream.
 * ------------------------------------------------------------------------- */
hj_status hj_solve_partitioned(const hj_grid *fine_grid, const hj_problem *prob,
                               const hj_fields *fine_fields, int32_t dtype,
                               const uint64_t *fine_mask, int32_t m, const hj_subdomain *plan,
                               uint64_t solve_set, double tol, int64_t max_iter, void *Vbar,
                               void *workspace, size_t ws_bytes, void *stream,
                               hj_report *reports);

#ifdef __cplusplus
}
#endif
#endif /* HJ_H_ */
