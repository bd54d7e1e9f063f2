/*
 * mmf.h — C ABI of the B200 (sm_100a) Sinkhorn-sweep library for entropy-regularised dynamic
 * multi-commodity min-cost flow (Haasler, Ringh, Chen, Karlsson, arXiv:2106.14485).
 *
 * The library runs the hot path of the paper's Algorithm 2 (alg:multi_commodity, PAPER.md
 * P:1085-1107) in the node form of SURVEY.md §8.0: per sweep
 *   a2  U0 = mu0 ./ beta_0                                   (eq:sinkhorn_graph_E P:859)
 *   a3  for t = 0..T-1:  F_t[a] = K_t[a] W_t[a] sum_l alpha_t[i_a,l] beta_{t+1}[j_a,l]   (cor:proj P:1078)
 *                        W_t[a] <- min(W_t[a] d_t[a] / F_t[a], 1)                  (eq:sinkhorn_graph_Vineq P:861)
 *                        alpha_{t+1}[j,:] = sum_{a->j} alpha_t[i_a,:] K_t[a] W_t[a] (eq:psi_hat P:1031-1036)
 *   a4  UT = muT ./ alpha_T
 *   a5  for t = T-1..0:  beta_t[i,:] = sum_{a: i_a=i} K_t[a] W_t[a] beta_{t+1}[j_a,:] (eq:psi P:1038-1043)
 * with K_t = exp(-C_t/eps) (eq:K_multicommodity P:1010-1013).  Arcs are the directed edges plus any
 * self-loops ("stay" arcs) the caller includes.
 *
 * Conventions: d = +INFINITY leaves an arc
 * uncapacitated (W = 1 always); d = 0 closes it (W = 0); F = 0 with d > 0 gives W = 1; at the
 * boundary scalings 0/0 := 0 and x/0 with x > 0 raises the sticky MMF_EINFEASIBLE.
 *
 * Numerics: messages are stored as (significand, integer binary exponent) pairs — "extended range"
 * (SURVEY D3): fp32 significand + int16 exponent in MMF_FP32, fp64 significand + int32 exponent in
 * MMF_FP64 — so that horizons whose log-message span exceeds the native exponent range
 * (thousands of nats) neither underflow nor lose relative precision.  Flows are linear M-typed.
 *
 * Threading and ownership: one host thread per context.  All host input arrays are borrowed for the
 * duration of the call only (copied / converted).  The CUDA stream and the workspace are borrowed
 * for the context's lifetime.  Every call returns a status; nothing throws across the ABI.
 * mmf_last_error() returns a context-owned string valid until the next call on that context.
 */
#ifndef MMF_H_
#define MMF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct mmf_ctx mmf_ctx; /* opaque */

typedef enum {
  MMF_OK = 0,
  MMF_EVERIFY = 1,     /* reserved (mirrors SPEC S:625 exit code 1) */
  MMF_EINVAL = 2,      /* invalid argument / validation failure at setup */
  MMF_ENOTCONV = 3,    /* reserved for solve-to-tolerance */
  MMF_EINFEASIBLE = 4, /* sticky: x/0 with x > 0 at a boundary scaling (a2/a4) */
  MMF_ENOMEM = 5,      /* workspace too small / allocation failure */
  MMF_ECUDA = 6,       /* CUDA runtime error */
  MMF_ENCCL = 7,       /* NCCL error */
  MMF_ESTATE = 8,      /* call out of order */
  MMF_ERANGE = 9       /* sticky: extended exponent overflow, or NaN in a flow */
} mmf_status;

typedef enum { MMF_FP64 = 0, MMF_FP32 = 1 } mmf_prec;

typedef struct {
  int64_t sweeps;        /* sweeps run since mmf_init */
  double mass;           /* <K, U> of the end-of-sweep tensor = sum_{l,j} alpha_T beta_T (all ranks) */
  double src_mismatch;   /* sum_{l,i} |U0 beta_0 - mu0|   (end-of-sweep source marginal error, L1) */
  double sink_mismatch;  /* sum_{l,j} |alpha_T UT - muT| (≈ 0 right after a4) */
  double cap_violation;  /* max_{t,a} (F_t[a] - d_t[a])_+ over capacitated arcs */
  double dual;           /* thm:solution dual objective: eps*(-mass + <mu0,log U0> + <muT,log UT> + <d,log W>
                            + <d_node, log u_node>) */
  double primal;         /* sum_{t,a} C_t[a] F_t[a] */
} mmf_stats;

/* Create a context on CUDA device `device` with message precision `prec`.  `cuda_stream` is a
 * borrowed cudaStream_t (NULL = legacy default stream); all device work is ordered on it. */
mmf_status mmf_create(mmf_ctx** out, int device, mmf_prec prec, void* cuda_stream);

/* Graph: N nodes, n_arcs arcs (tail[a] -> head[a]), node ids in [0, N).  Self-loops allowed (one
 * per node at most); duplicate (tail, head) pairs are rejected.  Arc a's position in
 * these arrays is the "user arc order" of every [T][A] input and output below. */
mmf_status mmf_set_graph(mmf_ctx* ctx, int32_t N, int64_t n_arcs, const int32_t* tail, const int32_t* head);

/* Costs C_t[a] (finite, any sign) and eps > 0.  time_varying = 0: cost is [n_arcs] for every step;
 * 1: cost is [T][n_arcs] (per-step topology/cost).  K = exp(-C/eps) is formed in fp64. */
mmf_status mmf_set_costs(mmf_ctx* ctx, int32_t T, double eps, const double* cost, int time_varying);

/* Capacities d_t[a] >= 0 of the bimarginal inequality constraints sum_l P_{t,t+1}(M^l) <= d_t (eq:omt_multi_graph_reg
 * P:763-770 with V_<=; eq:multicommodity P:659-661): +INFINITY = uncapacitated (W = 1), 0 = closed (W = 0);
 * layout as for costs.  NaN or negative -> MMF_EINVAL; before mmf_set_costs -> MMF_ESTATE. */
mmf_status mmf_set_capacity(mmf_ctx* ctx, const double* cap, int time_varying);

/* Dense source / sink distributions R^(0,1), R^(0,T) of commodities [l_begin, l_begin + l_count) of L_global
 * (the commodity-mode marginals of eq:multicommodity P:609-612, node form SURVEY 8.0): mu0, muT are [l_count][N]
 * row-major, finite, >= 0, with equal per-commodity masses (rel. 1e-12); else MMF_EINVAL.  A rank of
 * a sharded run passes only its own slice (rem:multi_tensor_scheme P:1139-1147). */
mmf_status mmf_set_marginals(mmf_ctx* ctx, int32_t L_global, int32_t l_begin, int32_t l_count,
                             const double* mu0, const double* muT);

/* Point-mass commodities (the OD pairs of P:1168-1173): commodity l moves mass[l] > 0 (finite) from
 * node src[l] to node dst[l] (ids in [0, N), else MMF_EINVAL); same slicing as mmf_set_marginals. */
mmf_status mmf_set_point_marginals(mmf_ctx* ctx, int32_t L_global, int32_t l_begin, int32_t l_count,
                                   const int32_t* src, const int32_t* dst, const double* mass);

/* Commodity-dependent node costs (the commodity-dependent kernel K_L = exp(-C_L/eps) of
 * eq:K_multicommodity P:1010-1013, restricted to costs that depend on the arc's head node): c is [l_count][N]
 * row-major for this rank's commodities (call after the marginals and mmf_set_costs, before mmf_init); commodity l
 * pays c[l][j] for each intermediate layer t = 1..T-1 it spends at node j, i.e. its arc costs are
 * C_t[a] + c[l][head(a)] for t = 0..T-2 (reading R-N; the boundary layers 0 and T carry the marginals
 * alone).  Values must be finite with |c / eps| log2(e) <= 8000, else MMF_EINVAL; NULL clears.  The factors
 * D = exp(-c/eps) are formed in fp64 and stored like K; stats' "primal" stays the arc-cost term. */
mmf_status mmf_set_node_costs(mmf_ctx* ctx, const double* c);

/* Node (state) capacities: the paper's inequality constraints on the state marginals,
 * P_t(M) <= d_t for the intermediate layers (eq:multicommodity P:676-683, Algorithm 2's u_t update P:1093; with the
 * arc-state and traffic-routing state spaces of P:612, P:704-720 the states are the nodes of this library's graph):
 * sum_l alpha_t[j,l] beta_t[j,l] <= d_t[j] for t = 1..T-1, with a shared dual u_t[j] in [0, 1] updated in the
 * forward pass right after alpha_t.  cap is [N] (every layer) or [T+1][N] (time_varying; layers 0 and T ignored), user
 * node order, +INFINITY free, 0 closed; NaN / negative -> MMF_EINVAL; call after mmf_set_costs, before the layout.
 * Supported on the pipelined fp32 path (L >= 256) and kernels = 1, Gauss-Seidel and symmetric schedules, one rank
 * (else MMF_EINVAL at mmf_init); checkpoints do not cover them.  NULL clears. */
mmf_status mmf_set_node_capacity(mmf_ctx* ctx, const double* cap, int time_varying);

/* The node-capacity duals u_t[j] (fp64, [T+1][N] user node order; 1 at free nodes and at layers 0, T).  Synchronises. */
mmf_status mmf_read_node_duals(mmf_ctx* ctx, double* out_T1xN);

/* Per-commodity entry / exit times (rem:multi_tensor_scheme P:1139-1149 and P:692-693:
 * commodities that enter and leave the network at different times, each with its own transport tensor): commodity l
 * of this context's slice is in the network on layers t_in[l] .. t_out[l] (0 <= t_in < t_out <= T): its source mass
 * sits at layer t_in, its sink mass at layer t_out, and it uses no arc outside steps t_in .. t_out - 1.  Point-mass
 * commodities and a single rank only (else MMF_EINVAL); call after the marginals, before mmf_workspace_bytes /
 * mmf_init (then the problem is fixed: further set_* calls return MMF_ESTATE).  Realised inside the library by
 * holding nodes (a source holding node whose release arc exists only at step t_in - 1, a sink holding node whose
 * absorb arc exists only at step t_out; zero cost, K = 0 at the other steps), which every readout hides: outputs keep the user's [T][n_arcs]
 * shape and arc order.  NULL clears. */
mmf_status mmf_set_commodity_times(mmf_ctx* ctx, const int32_t* t_in, const int32_t* t_out);

/* Device bytes needed once graph, costs, capacities and marginals are set. */
mmf_status mmf_workspace_bytes(const mmf_ctx* ctx, size_t* bytes);

/* Borrowed device workspace (>= mmf_workspace_bytes, 256-byte aligned).  If never called,
 * mmf_init allocates an owned workspace with cudaMalloc. */
mmf_status mmf_set_workspace(mmf_ctx* ctx, void* dptr, size_t bytes);

/* Multi-GPU commodity sharding (rem:multi_tensor_scheme P:1139-1147: the commodities couple only through the
 * shared capacity duals, i.e. through the aggregate flows F_t = sum_l F^l_t): join an NCCL communicator of `nranks` ranks from a 128-byte
 * ncclUniqueId (bootstrapped by the caller, e.g. torch.distributed).  Every rank must then make the
 * same calls with identical graph / cost / capacity arrays and its own commodity slice; the
 * per-step edge flows F_t are all-reduced (sum) over NVLink before the capacity-dual update.
 * The communicator is owned by the context.  Returns MMF_ENCCL if NCCL is unavailable. */
mmf_status mmf_attach_nccl(mmf_ctx* ctx, const void* unique_id128, int nranks, int rank);

/* Fill out128 with a fresh ncclUniqueId (call on one rank, then broadcast the 128 bytes). */
mmf_status mmf_nccl_unique_id(void* out128);

/* Options (call before mmf_init unless noted; unknown key or out-of-range value -> MMF_EINVAL, a
 * pre-init key after mmf_init -> MMF_ESTATE).  All kernel selections compute the same sweep (parity
 * tested); they differ only in speed.
 *   "graph"    1 = capture one sweep as a CUDA graph (default 1; may be changed any time)
 *   "profile"  1 = per-kernel CUDA-event timing for mmf_read_kernel_stats (any time)
 *   "prefetch" 1 = L2 prefetch hints in the wide-lane kernels (any time; recaptures the graph)
 *   "reorder"  1 = locality node reordering (default 1)
 *   "kernels"  kernel family 1, 3..6 (default 6 = TMA-pipelined forward (2 pipelines / CTA) and
 *              backward (3 pipelines / CTA), node-tile backward on high-degree graphs ("tbwd"); 5 single-pipeline;
 *              4 register head-flow; 3 wide-lane; 1 per-node reference kernels; 2 (the round-1 node tiles) was
 *              removed -> MMF_EINVAL)
 *   "bwd"      backward kernel with kernels >= 5: 0 auto, 1 three-pipeline, 2 sliding window, 3 single
 *   "schedule" 0 = Gauss-Seidel (Algorithm 2, default), 1 = damped Jacobi (every W_t from
 *              one alpha/beta pair, W <- W^(1-theta) min(W d / F, 1)^theta; one all-reduce of the T x n_arcs
 *              flows per sweep on the multi-GPU path)
 *              2 = symmetric Gauss-Seidel (Algorithm 2's forward pass, then a backward pass that
 *              updates every W_t again before forming beta_t; keeps all T + 1 alpha layers, one extra flow pass)
 *   "theta_milli"  Jacobi damping theta in 1/1000 (0 .. 1000, default 500)
 *   "fgw", "fng", "fnp"  pipelined forward: warps per consumer group (8, 4, 2), groups per pipeline,
 *              pipelines per CTA (0 = default; the compiled combinations are listed in pipefwd.cuh)
 *   "wintma"   window backward row blocks by 2-D tensor TMA (1) or cp.async (0)
 *   "order"    node order: kernels 3..5: 0 input, 1 reverse Cuthill-McKee, 2 BFS tiles (default); kernels 6:
 *              1 RCM, 3 the window kernel's cost model, 4 most neighbour overlap between consecutive nodes even where
 *              the pipelined kernels do not apply; default (other values): most neighbour overlap for fp32 with
 *              L >= 256 (the pipelined kernels), the window cost model otherwise (fp64, L < 256) and with bwd=2
 *   "cpt"      commodities per thread 0 (auto), 1, 2, 4, 8
 *   "tile", "halo", "cpc"  tile sizes of the kernels = 2 family
 *   "wrap"     three-pipeline backward: -1 auto, 0 items never wrap around the ring, 1 items may wrap
 *   "stripw"   (experiments) strip width of the neighbour-overlap node order (0 = chosen by its score)
 *   "dry", "copy"  profiling / diagnostic modes of the pipelined kernels (dry 1: producers only, 2: no flows,
 *              3: no dual update; results invalid; never in production)
 *   "l2hint"   pipelined kernels: L2 evict_last policy on the gathered message rows (measured no gain; default 0)
 *   "pexch"    multi-GPU / virtual-rank Gauss-Seidel exchange (rem:multi_tensor_scheme P:1139-1147) on the pipelined
 *              forward split around the all-reduce (flows-only launch, dual update, alpha-only launch): 1 on, 0 off
 *              (wide-lane two-pass kernels), -1 auto (default: on for 1024-commodity slices)
 *   "tbwd"     backward on node tiles (BFS blobs of "tile" nodes whose out-halo stays within "halo" rows; the halo
 *              rows of a (tile, commodity chunk) staged once by TMA, the tile's nodes computed from shared memory):
 *              1 on, 0 off, -1 auto (default: fp32, L >= 256 and mean degree >= 7, e.g. BJ [3] and [5]); it sets
 *              the node order to the tile order
 *   "wcp"      wide-lane kernels: commodity chunks per CTA (0 auto: 1 for fp32 rows of >= 16 chunks, else 8; the CTA's
 *              8 / wcp warps-per-chunk take neighbouring nodes)
 *   "tfwd"     forward on the same node tiles (alpha_t and the flow partials of step t per (tile, 128-commodity chunk)
 *              from staged in- and out-halo rows, then a fixed-order chunk sum and the dual update): 1 on, 0 off
 *              (default; measured slower than the wide-lane forward on [5]), -1 where the pipelined forward does not
 *              apply; single rank, no node capacities */
mmf_status mmf_set_option(mmf_ctx* ctx, const char* key, int64_t value);

/* W = 1, UT = 1 on supp(muT), one backward pass (Alg. 2 "Initialize").  Async. */
mmf_status mmf_init(mmf_ctx* ctx);

/* Enqueue n full sweeps (a2..a5) on the stream.  Async; errors surface at mmf_sync / read_*. */
mmf_status mmf_sweep(mmf_ctx* ctx, int32_t n);

/* Virtual ranks (the coupling of rem:multi_tensor_scheme P:1139-1147 on one device): ctxs[0..G-1]
 * (1 <= G <= 8) are initialised contexts of the same problem on the same device and stream, each holding one
 * commodity slice (mmf_set_*_marginals with l_begin / l_count), no NCCL, option kernels >= 3, Gauss-Seidel.  Runs n
 * sweeps of all of them together with the multi-GPU exchange path's kernels: per forward step every shard's partial
 * flows F_t -> a device-side sum in fixed shard order (in place of ncclAllReduce) -> every shard's dual update.  The
 * capacity duals stay identical across the contexts; each context's edge-flow readout covers its own commodities.
 * Async, no CUDA graph; errors surface at mmf_sync.  MMF_EINVAL on mismatched contexts, MMF_ESTATE if one is not
 * initialised. */
mmf_status mmf_sweep_group(mmf_ctx* const* ctxs, int32_t G, int32_t n);

/* Wait for the stream; report sticky device errors (MMF_EINFEASIBLE / MMF_ERANGE, with the first
 * (commodity, node) in mmf_last_error) and NCCL async errors. */
mmf_status mmf_sync(mmf_ctx* ctx);

/* Solve to tolerance (SPEC solve): run sweeps until the error of the end-of-sweep state
 *   err = ( sum_{l,i} |U0 beta_0 - mu0| + sum_{l,j} |alpha_T UT - muT| + sum_{t,a} (F_t[a] - d_t[a])_+ ) / mass
 * (marginal L1 mismatches plus the total capacity excess, relative to the tensor mass; reduced on the device,
 * all ranks) is below tol, evaluated every check_every sweeps, at most max_sweeps sweeps.  err_hist
 * (nullable) receives the error of every check (ceil(max_sweeps / check_every) entries at most).
 * Returns MMF_OK when converged, MMF_ENOTCONV when the sweep cap was reached first (the state is valid;
 * max_sweeps = 0 returns the initial state, err = +inf).  Synchronises. */
mmf_status mmf_solve(mmf_ctx* ctx, double tol, int32_t max_sweeps, int32_t check_every, int32_t* sweeps_done,
                     double* err_out, double* err_hist);

/* Per-commodity arc flows of step t (0 <= t < T) of the end-of-sweep state, F^l_t[a] = alpha_t[i_a,l] K_t[a]
 * W_t[a] beta_{t+1}[j_a,l] (cor:proj P:1078 in node form), fp64, [n_arcs][l_count] in user
 * arc order, this rank's commodities.  Recomputes the forward messages up to t.  Synchronises. */
mmf_status mmf_read_commodity_flows(mmf_ctx* ctx, int32_t t, double* out_AxL);

/* Checkpoint / resume.  The iteration state is the capacity duals W [T][n_arcs], the sink
 * scaling UT and the last source scaling U0 (this rank's commodities) of the end-of-sweep state, plus the sweep
 * count; records and beta_t are recomputed on load (the next sweep's a2 recomputes U0 from them), so a restored
 * context reads out and continues exactly like the saved one (bitwise, with the same options).  The buffer is
 * opaque and versioned ("MMFSTAT2"): W in user arc order, UT and U0 in user node order, a header with the problem
 * shape, a hash of the graph and a hash of T, eps, costs and capacities, checked by mmf_load_state (MMF_EINVAL on
 * mismatch or a corrupt header).  mmf_save_state / mmf_load_state synchronise; call them after mmf_init.
 * Before the first sweep U0 = 0 (Alg. 2 computes U0 first), so readouts then return zero flows. */
mmf_status mmf_state_bytes(const mmf_ctx* ctx, size_t* bytes);
mmf_status mmf_save_state(mmf_ctx* ctx, void* host_buf, size_t bytes);
mmf_status mmf_load_state(mmf_ctx* ctx, const void* host_buf, size_t bytes);

/* End-of-sweep edge flows F_t[a] = sum over ALL commodities (all ranks), fp64, [T][n_arcs] in user
 * arc order: one extra forward pass without updates (cor:proj P:1078-1079).  Synchronises. */
mmf_status mmf_read_edge_flows(mmf_ctx* ctx, double* out_TxA);

/* Capacity duals W_t[a] = u_t = exp(-lambda_t/eps) in [0, 1] (thm:solution P:777-788, the V_<= scalings updated by
 * eq:sinkhorn_graph_Vineq P:861), fp64, [T][n_arcs] user arc order (values below 2^-1074 read 0).  Synchronises. */
mmf_status mmf_read_cap_duals(mmf_ctx* ctx, double* out_TxA);

/* Statistics of the end-of-sweep state (see mmf_stats).  Synchronises. */
mmf_status mmf_read_stats(mmf_ctx* ctx, mmf_stats* out);

/* Kernel accounting: launches (cumulative) and, with option "profile", device milliseconds per
 * kernel kind.  kinds: 0 bwd_step, 1 fwd_flow, 2 fwd_reduce, 3 fwd_update, 4 boundary, 5 other,
 * 6 fwd_fused.  n = array length (<= 8). */
mmf_status mmf_read_kernel_stats(mmf_ctx* ctx, int64_t* launches, double* ms, int n);

/* Algorithmic bytes moved by one sweep (SURVEY §8(d) byte model, with this build's element size). */
mmf_status mmf_sweep_bytes(const mmf_ctx* ctx, double* bytes_total, double* bytes_per_kind, int n);

/* Free owned resources (not the borrowed stream / workspace).  Safe on NULL. */
mmf_status mmf_destroy(mmf_ctx* ctx);

/* Last error message of this context (or of the last failed mmf_create if ctx is NULL). */
const char* mmf_last_error(const mmf_ctx* ctx);

/* Library version string. */
const char* mmf_version(void);

#ifdef __cplusplus
}
#endif
#endif /* MMF_H_ */
