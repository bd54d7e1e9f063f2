// mmf.cu — host engine and C ABI (include/mmf.h) of the B200 Sinkhorn-sweep library.
//
// Host side: validation (SURVEY §8(b) error conventions), locality node reordering, CSR build,
// fp64 -> extended-range conversion of K = exp(-C/eps) and the marginals, workspace layout, the
// sweep launch sequence (a2, T x forward step, a4, T x backward step) optionally
// captured once as a CUDA graph, readouts and statistics, and the NCCL per-step all-reduce of the
// edge flows for commodity sharding.
#include "../../include/mmf.h"
#include "kernels.cuh"
#include "tiled.cuh"
#include "win.cuh"
#include "tilebwd.cuh"

#include <dlfcn.h>
#include <future>
#include <thread>
#include <nvtx3/nvToolsExt.h>  // (header-only NVTX3: ranges go to a profiler when one is attached, else no-ops)
#include <cstdlib>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

using namespace mmf;

// ------------------------------------------------------------------------------------------------
// NCCL, resolved at run time from the process (torch loads libnccl.so.2) so the library itself has
// no link-time NCCL dependency.
namespace {
typedef int ncclResult_t_;
typedef void* ncclComm_t_;
struct NcclUid {
  char internal[128];
};
struct NcclApi {
  bool ok = false;
  ncclResult_t_ (*CommInitRank)(ncclComm_t_*, int, NcclUid, int) = nullptr;
  ncclResult_t_ (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t_, cudaStream_t) = nullptr;
  ncclResult_t_ (*CommDestroy)(ncclComm_t_) = nullptr;
  ncclResult_t_ (*CommGetAsyncError)(ncclComm_t_, ncclResult_t_*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t_) = nullptr;
  ncclResult_t_ (*GetUniqueId)(NcclUid*) = nullptr;
};
// ncclDataType_t / ncclRedOp_t values (stable NCCL ABI)
constexpr int NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8, NCCL_SUM = 0;

NcclApi& nccl_api() {
  static NcclApi api;
  static bool tried = false;
  if (tried) return api;
  tried = true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) return api;
  api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
  api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
  api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
  api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
  api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
  api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
  api.ok = api.CommInitRank && api.AllReduce && api.CommDestroy && api.CommGetAsyncError;
  return api;
}

std::string g_create_error;

enum Kind { K_BWD = 0, K_FLOW = 1, K_REDUCE = 2, K_UPDATE = 3, K_BOUNDARY = 4, K_OTHER = 5, K_FUSED = 6, K_NKINDS = 8 };

}  // namespace

struct mmf_ctx {
  int device = 0;
  mmf_prec prec = MMF_FP64;
  cudaStream_t stream = nullptr;  // borrowed
  cudaStream_t priv = nullptr;    // owned (graph capture / launch)
  std::string err;

  // ---- host problem, user order
  int N = 0;
  int64_t A = 0;
  std::vector<int> tail, head;
  int T = 0;
  double eps = 0;
  std::vector<double> cost;
  bool cost_tv = false, have_cost = false;
  std::vector<double> cap;
  bool cap_tv = false, have_cap = false;
  int Lg = 0, l_begin = 0, L = 0;
  bool point = false, have_marg = false;
  std::vector<double> mu0, muT, mass;
  std::vector<int> src, dst;
  std::vector<double> node_cost;  // [L][N] this rank's commodities (NEXT-2), empty = none
  // NEXT-4 entry / exit times (point-mass commodities): t_in / t_out per commodity, empty = 0 / T.  Realised by
  // augmenting the graph before the first layout (augment_times): per commodity a source holding node (its loop and
  // a release arc to the source that exists only at step t_in - 1) and a sink holding node (an absorb arc from the sink that exists
  // only at step t_out, and its loop); user arcs keep their positions, readouts cover them only.
  std::vector<int> t_in, t_out;
  std::vector<double> node_cap;  // NEXT-3 node (state) capacities [N] or [T+1][N] (user node order), empty = none
  bool node_cap_tv = false;
  bool augmented = false;
  int N_user = 0;
  int64_t A_user = 0;
  std::vector<double> cost_user, cap_user;  // (the user's arrays: primal / violation in mmf_read_stats)

  // ---- options
  bool opt_graph = true, opt_reorder = true, opt_profile = false;
  int opt_kernels = 6;  // 6 = sliding-window backward + pipelined forward (production), 5 = TMA-pipelined backward
                        // + head-flow forward, 4 = register-gather head-flow
                        // kernels, 3 = wide-lane kernels, 2 = smem-staged tile kernels, 1 = per-node reference kernels
  int opt_tile = 32;    // max nodes per tile
  int opt_cpt = 0;      // commodities per lane (0 = auto: 2 for fp32, 1 for fp64)
  int opt_halo = 0;     // max in-/out-halo nodes per tile (0 = auto: 2 * tile)
  int opt_cpc = 0;      // commodity chunks per CTA (0 = auto)
  int opt_order = 2;    // node order: kernels 2-5: 0 input order, 1 reverse Cuthill-McKee, 2 BFS tiles; kernels 6:
                        // 1 RCM, 3 window cost model, else most neighbour overlap (choose_reuse_order)
  int opt_prefetch = 0; // wide kernels: L1 prefetch of significand rows in pass 1
  int opt_dry = 0;      // diagnostics: pipelined backward consumers skip the arithmetic
  int opt_copy = 0;     // pipelined kernels' row staging: 0 = TMA bulk copies, 1 = per-lane cp.async
  int opt_wintma = 1;   // window kernels: 1 = 2-D TMA row-block loads, 0 = per-thread cp.async
  int opt_schedule = 0;      // 0 Gauss-Seidel (Algorithm 2), 1 damped Jacobi
  int opt_theta_milli = 500;  // Jacobi damping theta in 1/1000
  int opt_l2hint = 0;         // pipelined kernels: L2 evict_last policy on the gathered rows
  int opt_stripw = 0;   // (experiments) restrict the neighbour-overlap order's strip candidates to this width
  int opt_wrap = -1;    // k_bwd_pipe2 ring wrap: -1 auto, 0 items never wrap, 1 items may wrap
  int opt_fgw = 0;      // pipelined forward: warps per consumer group (0 auto, 8, 4, 2)
  int opt_fng = 0;      // pipelined forward: consumer groups per pipeline (0 auto, 1 .. 6)
  int opt_fnp = 0;
  int opt_tbwd = -1;    // backward: 1 = node tiles with staged out-halos (tilebwd.cuh; nodes ordered into tiles), 0 off,
                        // -1 auto: fp32, L >= 256 and mean degree >= 7 (measured: [5] 34.4 vs 40.0 ms/sweep, [3] 5.4 vs
                        // 7.7; [4], degree 4.8, 71 vs 31)
  bool tile_bwd = false;
  TileCfg tbc{};
  int opt_wcp = 0;      // wide-lane kernels: commodity chunks per CTA (0 auto = 8; 8 / wcp neighbouring nodes per CTA)
  int opt_tfwd = 0;     // forward on node tiles (k_fwd_tile2 + k_tile_dual, with the tile backward's tiles): 1 on, 0 off
                        // (default: measured slower than the wide-lane forward on [5], 77.5 vs 67.2 ms/sweep), -1 where
                        // the tile backward runs and the pipelined forward does not apply
  bool tile_fwd = false;
  TileCfgF tfc{};
  std::vector<int> h_tf_desc, h_tf_meta;
  const int* d_tf_desc = nullptr;
  const int* d_tf_meta = nullptr;
  float* d_tf_part = nullptr;
  int tb_cpt = 4;
  int opt_pexch = -1;   // multi-GPU / virtual-rank Gauss-Seidel exchange on the pipelined kernels: 1 on, 0 off (wide-lane
                        // two-pass), -1 auto = 1024-commodity slices (measured on [4]: 92 vs 115 ms/sweep at L = 1024, but
                        // 74 vs 66 at 512 and 64 vs 57 at 256)      // pipelined forward: pipelines per CTA (0 auto, 1, 2)
  int opt_bwd = 0;      // backward kernel: 0 = auto (two-pipeline TMA kernel where it applies, else the window
                        // kernel), 1 = two-pipeline TMA kernel, 2 = window kernel, 3 = pipe (1 pipeline)
  PipeCfg5 pb2{};       // two-pipeline backward configuration
  bool pipe2_bwd = false;

  // ---- derived
  int Lp = 0, G = 0, block = 0, maxdeg_in = 0;
  int CPT = 1, LC = 32, nch = 1;
  std::vector<int> newid;       // user node -> internal
  std::vector<int> int_of_arc;  // user arc -> internal arc
  bool prepared = false;        // host graph structures below are valid
  std::vector<int> h_tail, h_head, h_inptr, h_outptr, h_outarc, h_outhead;
  std::vector<int> h_fpos;  // internal arc -> position in the exchange buffer (capacitated at some step), else -1
  int64_t Ecap = 0;
  bool fpos_ok = false;
  int ntiles = 0, tileB = 0, max_hin = 0, max_hout = 0, max_ia = 0, max_oa = 0;
  std::vector<int> h_tb_desc, h_tb_meta;  // tile backward: per-tile descriptors (8 ints) and 16-B aligned static metadata
  const int* d_tb_desc = nullptr;
  const int* d_tb_meta = nullptr;
  std::vector<int> h_tile_ptr, h_hin_ptr, h_hin_node, h_hout_ptr, h_hout_node, h_in_hidx, h_out_hidx;
  TileMeta tm{};
  PipeCfg pc{1, 1};
  WideCfg wc{};
  HeadCfg hc{};
  PipeCfg5 pb{};      // pipelined backward kernel (opt_kernels == 5)
  PipeCfg5 pf{};      // pipelined forward kernel
  int pf_gw = 8, pf_ng = 1, pf_np = 2;  // its consumer groups: GW warps each, NG per pipeline, NP pipelines
  bool pipe_bwd = false, pipe_fwd = false;
  // sliding-window kernels (opt_kernels == 6)
  bool win_bwd = false;
  int win_cpt = 2, win_Wb = 0;  // chosen with the node order in prepare()
  WinCfg wcb{};                 // backward window configuration
  WinDir wdo{};                 // out-direction tables (device pointers)
  WinTmaps tmb{};               // TMA views of the beta store (backward gathers)
  bool win_tma = false;
  std::vector<int> h_wsrc_out, h_wfptr_out, h_wfnode_out;
  int ell_din = 0;
  int sms = 148;

  // ---- device
  void* ws = nullptr;
  size_t ws_bytes = 0;
  bool ws_owned = false;
  DevPtrs dp{};
  bool inited = false;
  int64_t sweeps = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  int64_t graph_launch_tally[K_NKINDS] = {};
  cudaEvent_t ev_user = nullptr, ev_priv = nullptr;

  // ---- NCCL
  ncclComm_t_ comm = nullptr;
  int nranks = 1, rank = 0;

  // ---- accounting
  int64_t launches[K_NKINDS] = {};
  double ms[K_NKINDS] = {};
  bool capturing = false;
  struct Prof {
    int kind;
    cudaEvent_t a, b;
  };
  std::vector<Prof> prof;
  std::vector<cudaEvent_t> ev_pool;

  size_t sm() const { return prec == MMF_FP32 ? sizeof(float) : sizeof(double); }
  int* d_int_of_arc = nullptr;  // (readouts: user arc -> internal arc, uploaded on first use)
  double* d_export = nullptr;    // (readouts: [T][A] fp64 staging, allocated on first use)
  void* pinned = nullptr;        // (readouts: pinned bounce buffer of d2h_staged, allocated on first use)
  cudaEvent_t ev_d2h[2] = {nullptr, nullptr};
  size_t se() const { return prec == MMF_FP32 ? sizeof(int16_t) : sizeof(int32_t); }
};

namespace {

mmf_status fail(mmf_ctx* c, mmf_status s, const std::string& msg) {
  if (c) c->err = msg;
  return s;
}

// host-side phase timer (MMF_VERBOSE: printed to stderr)
struct HostTimer {
  const char* name;
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  explicit HostTimer(const char* n) : name(n) {}
  ~HostTimer() {
    if (getenv("MMF_VERBOSE"))
      fprintf(stderr, "[mmf] host %s %.1f ms\n", name,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
};

// NVTX range of a host-side scope (sweep, pass, step, readout); under CUDA-graph capture the ranges mark the capture
struct Nvtx {
  explicit Nvtx(const char* name) { nvtxRangePushA(name); }
  ~Nvtx() { nvtxRangePop(); }
};

#define CU2(c, call)                                                                               \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(c, MMF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));               \
  } while (0)

#define CU(call)                                                                                   \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess)                                                                         \
      return fail(ctx, MMF_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e_));             \
  } while (0)

// ------------------------------------------------------------------------------------------------
// reverse Cuthill-McKee over the undirected support of the arcs: nodes adjacent in the graph get
// nearby internal ids, so a step's gathers of alpha/beta rows hit L2 (and the same DRAM pages).
std::vector<int> rcm_newid(int N, const std::vector<int>& tail, const std::vector<int>& head) {
  std::vector<int> deg(N, 0);
  for (size_t a = 0; a < tail.size(); ++a)
    if (tail[a] != head[a]) {
      deg[tail[a]]++;
      deg[head[a]]++;
    }
  std::vector<int64_t> ptr(N + 1, 0);
  for (int v = 0; v < N; ++v) ptr[v + 1] = ptr[v] + deg[v];
  std::vector<int> adj(ptr[N]);
  std::vector<int64_t> fill(ptr.begin(), ptr.end() - 1);
  for (size_t a = 0; a < tail.size(); ++a)
    if (tail[a] != head[a]) {
      adj[fill[tail[a]]++] = head[a];
      adj[fill[head[a]]++] = tail[a];
    }
  std::vector<int> byDeg(N);
  std::iota(byDeg.begin(), byDeg.end(), 0);
  std::stable_sort(byDeg.begin(), byDeg.end(), [&](int a, int b) { return deg[a] < deg[b]; });
  std::vector<char> seen(N, 0);
  std::vector<int> order;
  order.reserve(N);
  std::vector<int> nb;
  for (int s : byDeg) {
    if (seen[s]) continue;
    seen[s] = 1;
    size_t head_q = order.size();
    order.push_back(s);
    while (head_q < order.size()) {
      int v = order[head_q++];
      nb.clear();
      for (int64_t k = ptr[v]; k < ptr[v + 1]; ++k)
        if (!seen[adj[k]]) {
          seen[adj[k]] = 1;
          nb.push_back(adj[k]);
        }
      std::stable_sort(nb.begin(), nb.end(), [&](int a, int b) { return deg[a] < deg[b]; });
      order.insert(order.end(), nb.begin(), nb.end());
    }
  }
  std::vector<int> newid(N);
  for (int k = 0; k < N; ++k) newid[order[N - 1 - k]] = k;
  return newid;
}

// fp64 -> (significand, binary exponent) with significand in [1, 2); 0 -> (0, EZERO)
inline void to_xf(double x, double& m, int& e) {
  if (!(x > 0)) {
    m = 0;
    e = EZERO;
    return;
  }
  int ex;
  double fr = std::frexp(x, &ex);  // x = fr 2^ex, fr in [0.5, 1)
  m = fr * 2.0;
  e = ex - 1;
}

// K = exp(lk) with lk = -C/eps formed in fp64 (Q20): x = lk log2(e) split into floor + fraction
inline void k_to_xf(double lk, double& m, int& e) {
  long double x = (long double)lk * 1.4426950408889634073599246810018921L;
  long double fl = std::floor(x);
  m = (double)std::exp2(x - fl);
  e = (int)fl;
  if (m >= 2.0) {
    m *= 0.5;
    e += 1;
  }
}

struct Layout {
  size_t off = 0;
  size_t take(size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  }
};

// Node tiles: BFS-grown blobs (seeds in reverse Cuthill-McKee order) of at most B nodes whose in-halo
// and out-halo (tails of the tile's in-arcs, heads of its out-arcs) stay within `cap` nodes, so the
// shared-memory footprint of a tile is bounded and uniform.  On grids and geometric graphs the blobs
// are compact (halo / tile ~ 2 instead of the mean degree).
void make_tiles(int N, const std::vector<int>& tail, const std::vector<int>& head, int B, int cap, bool reorder,
                std::vector<int>& order, std::vector<int>& tile_ptr) {
  order.clear();
  tile_ptr.assign(1, 0);
  if (!reorder) {
    for (int v = 0; v < N; ++v) order.push_back(v);
    for (int v = B; v < N; v += B) tile_ptr.push_back(v);
    tile_ptr.push_back(N);
    return;
  }
  const size_t A = tail.size();
  auto csr = [&](const std::vector<int>& key, const std::vector<int>& val, std::vector<int64_t>& ptr,
                 std::vector<int>& out, bool skip_loops) {
    ptr.assign(N + 1, 0);
    for (size_t a = 0; a < A; ++a)
      if (!(skip_loops && tail[a] == head[a])) ptr[key[a] + 1]++;
    for (int v = 0; v < N; ++v) ptr[v + 1] += ptr[v];
    out.resize(ptr[N]);
    std::vector<int64_t> f(ptr.begin(), ptr.end() - 1);
    for (size_t a = 0; a < A; ++a)
      if (!(skip_loops && tail[a] == head[a])) out[f[key[a]]++] = val[a];
  };
  std::vector<int64_t> pin, pout, pu1, pu2;
  std::vector<int> nin, nout, u1, u2;
  csr(head, tail, pin, nin, false);   // in-neighbours (tails of in-arcs), loops included
  csr(tail, head, pout, nout, false); // out-neighbours
  csr(tail, head, pu1, u1, true);     // undirected support for the BFS: out ...
  csr(head, tail, pu2, u2, true);     // ... and in
  std::vector<int> rid = rcm_newid(N, tail, head);
  std::vector<int> seeds(N);
  for (int v = 0; v < N; ++v) seeds[rid[v]] = v;
  std::vector<int> mark_in(N, -1), mark_out(N, -1);
  std::vector<char> done(N, 0);
  int tid = 0, n_in = 0, n_out = 0;
  auto cost = [&](int u, int& di, int& dout) {
    di = dout = 0;
    for (int64_t k = pin[u]; k < pin[u + 1]; ++k) di += mark_in[nin[k]] != tid;
    for (int64_t k = pout[u]; k < pout[u + 1]; ++k) dout += mark_out[nout[k]] != tid;
  };
  auto add = [&](int u) {
    done[u] = 1;
    order.push_back(u);
    for (int64_t k = pin[u]; k < pin[u + 1]; ++k)
      if (mark_in[nin[k]] != tid) {
        mark_in[nin[k]] = tid;
        n_in++;
      }
    for (int64_t k = pout[u]; k < pout[u + 1]; ++k)
      if (mark_out[nout[k]] != tid) {
        mark_out[nout[k]] = tid;
        n_out++;
      }
  };
  for (int s : seeds) {
    if (done[s]) continue;
    n_in = n_out = 0;
    const size_t q0 = order.size();
    add(s);
    for (size_t qi = q0; qi < order.size() && (int)(order.size() - q0) < B; ++qi) {
      const int v = order[qi];
      for (int pass = 0; pass < 2; ++pass) {
        const std::vector<int64_t>& pp = pass ? pu2 : pu1;
        const std::vector<int>& nn = pass ? u2 : u1;
        for (int64_t k = pp[v]; k < pp[v + 1] && (int)(order.size() - q0) < B; ++k) {
          const int u = nn[k];
          if (done[u]) continue;
          int di, dout;
          cost(u, di, dout);
          if (n_in + di <= cap && n_out + dout <= cap) add(u);
        }
      }
    }
    tile_ptr.push_back((int)order.size());
    ++tid;
  }
}

void build_window_tables(mmf_ctx* c);
bool tbwd_wanted(const mmf_ctx* c);

void derive_shapes(mmf_ctx* c) {
  HostTimer ht("derive_shapes");
  int cpt_auto = c->prec == MMF_FP32 ? 2 : 1;
  if (c->opt_kernels == 4) {  // register-gather path: 4 fp32 commodities per lane keep 6 rows in registers
    if (c->prec == MMF_FP32)
      cpt_auto = c->L >= 128 ? 4 : 2;
    else
      cpt_auto = c->L >= 64 ? 2 : 1;
  } else if (c->opt_kernels == 3 || c->opt_kernels >= 5) {
    if (c->prec == MMF_FP32)
      cpt_auto = c->L >= 512 ? 8 : (c->L >= 128 ? 4 : 2);
    else
      cpt_auto = c->L >= 64 ? 2 : 1;
  }
  c->CPT = c->opt_cpt ? c->opt_cpt : cpt_auto;
  if (c->prec == MMF_FP64) c->CPT = std::min(c->CPT, 2);   // fp64 lanes: at most 2 (16-byte loads)
  c->LC = 32 * c->CPT;
  c->Lp = ((c->L + c->LC - 1) / c->LC) * c->LC;
  // pipelined backward (fp32, ELL width <= 32): slice width SW = 256 * cp commodities, S stages of
  // Dout rows x SW x 6 B in shared memory; the message row length Lp is padded to a multiple of SW
  c->pipe_bwd = false;
  if (c->opt_kernels >= 5 && c->prec == MMF_FP32 && c->pb.D > 0 && c->pb.D <= 32 && c->L >= 256) {
    // slice width SW = 256 * cp; the row ring holds R rows of SW (6 B each); want >= ~6 average items
    // in flight (A / N rows each) plus one worst-case item
    const size_t budget = 220 * 1024;
    const int L256 = (c->L + 255) / 256 * 256;
    const double avg = (double)c->A / std::max(c->N, 1);
    const int SD = PIPE_SD;
    auto rows_fit = [&](int SW) {
      int R = 0;
      while (pipe_smem(R + 1, SD, c->pb.D, SW).total <= budget) ++R;
      return R;
    };
    int cp = 4;
    while (cp > 1 && (256 * cp > L256 || rows_fit(256 * cp) < c->pb.D + (int)(4 * avg))) cp >>= 1;
    const int SW = 256 * cp;
    const int R = rows_fit(SW);
    if (R >= 2 * c->pb.D) {  // contiguous items: any item fits once the older ones are released
      c->pipe_bwd = true;
      c->pb.SW = SW;
      c->pb.R = R;
      c->pb.SD = SD;
      c->pb.dry = c->opt_dry;
      c->pb.copy = c->opt_copy;
      const int q = std::max(SW, c->LC);
      c->Lp = (c->L + q - 1) / q * q;
      c->pb.ns = c->Lp / SW;
      c->pb.nitems = c->N * c->pb.ns;
    }
  }
  // sliding-window backward (kernels == 6): tables depend on the order chosen in prepare()
  c->win_bwd = false;
  if (c->opt_kernels == 6 && c->prec == MMF_FP32 && c->L >= 32 && !c->h_outptr.empty()) {
    build_window_tables(c);
    const int SW = 32 * c->win_cpt;
    const int q = std::max(SW, c->LC);
    const int Lp = std::max(c->Lp, (c->L + q - 1) / q * q);
    WinCfg& w = c->wcb;
    w.ns = Lp / SW;
    w.dry = c->opt_dry;
    w.nseg = std::max(1, c->sms / w.ns);
    w.segB = (w.nblk + w.nseg - 1) / w.nseg;
    w.nseg = (w.nblk + w.segB - 1) / w.segB;
    const size_t sm = c->win_cpt == 4 ? win_smem<4>(w).total : c->win_cpt == 2 ? win_smem<2>(w).total : win_smem<1>(w).total;
    // (many narrow slices re-stream the window and records once per slice: the pipelined kernel wins there)
    if (sm <= 227 * 1024 && Lp % SW == 0 && w.ns <= 64) {
      c->win_bwd = true;
      c->Lp = Lp;
      if (c->pipe_bwd) {
        c->pb.ns = c->Lp / c->pb.SW;
        c->pb.nitems = c->N * c->pb.ns;
      }
    }
  }
  // two-pipeline backward (same slices as the pipelined backward; rings of >= D rows per pipeline)
  c->pipe2_bwd = false;
  if (c->pipe_bwd && (c->opt_bwd == 1 || c->opt_bwd == 0)) {  // (auto: measured fastest on [3], [4], [5])
    const size_t budget = 220 * 1024 / BWD_NP;
    int R = 0;
    while (pipe_smem(R + 1, FWD_SD, c->pb.D, c->pb.SW).total <= budget) ++R;
    if (R >= c->pb.D) {
      c->pipe2_bwd = true;
      c->pb2 = c->pb;
      c->pb2.R = R;
      c->pb2.ns = c->Lp / c->pb.SW;
      c->pb2.nitems = c->N * c->pb2.ns;
      c->win_bwd = c->win_bwd && c->opt_bwd == 2;
      // items that never wrap save per-row offset arithmetic but waste ring slots: worth it when items are
      // long or the ring holds many of them (measured: [5], [3] gain; [4] loses)
      const double avg = (double)c->A / std::max(c->N, 1);
      c->pb2.wrap = c->opt_wrap >= 0 ? c->opt_wrap : !(avg >= 8.0 || R >= 3.0 * avg);
    }
  }
  if (c->opt_bwd == 3) c->win_bwd = false;
  // pipelined forward: one item per node (all Lp commodities in one slice of the backward's width), NG
  // consumer groups of GW warps per pipeline (a warp owns 32 CPT = SW / GW commodities)
  c->pipe_fwd = false;
  if (c->pipe_bwd && c->pb.ns == 1 && c->ell_din > 0 && c->ell_din <= 32) {
    const int SW = c->pb.SW;
    int gw = 8, ng = 1, np = 2;  // (the first compiled combination of this SW, unless options choose)
    bool first = true;
#define MMF_FWD_FIRST(sw, cpt, g, n, q)                                                         \
  if (SW == sw && first && (!c->opt_fgw || c->opt_fgw == g) && (!c->opt_fng || c->opt_fng == n) && \
      (!c->opt_fnp || c->opt_fnp == q)) {                                                       \
    gw = g;                                                                                     \
    ng = n;                                                                                     \
    np = q;                                                                                     \
    first = false;                                                                              \
  }
    MMF_FWD_COMBOS(MMF_FWD_FIRST)
#undef MMF_FWD_FIRST
    const size_t budget = 226 * 1024 / np;
    int R = 0;
    while (pfwd_smem(R + 1, c->ell_din, SW, ng).total <= budget) ++R;
    const int rmin = c->ell_din + (MMF_FWD_OWNG ? 0 : 1);  // rows of the largest item
    if (!first && R >= rmin) {  // (an item's rows may wrap around its pipeline's ring)
      c->pipe_fwd = true;
      c->pf = c->pb;
      c->pf.D = c->ell_din;
      c->pf.R = R;
      c->pf_gw = gw;
      c->pf_ng = ng;
      c->pf_np = np;
    }
  }
  // tile backward (option tbwd): stages of the largest out-halo x SW commodities; SW = 256 when two stages fit
  c->tile_bwd = false;
  if (tbwd_wanted(c) && c->max_hout > 0) {
    const size_t budget = 226 * 1024;
    const int MA = c->max_oa;
    int MB = 0;  // (largest static metadata block, ints)
    for (int k = 0; k < c->ntiles; ++k) MB = std::max(MB, c->h_tb_desc[(size_t)k * 8 + 7]);
    int cpt = (c->Lp % 256 == 0 && tb_smem(2, c->max_hout, 256, MA, MB) <= budget) ? 8 : 4;
    const int SW = 32 * cpt;
    int nst = 1;
    while (nst < 6 && tb_smem(nst + 1, c->max_hout, SW, MA, MB) <= budget) ++nst;
    if (c->Lp % SW == 0 && nst >= 2) {
      c->tile_bwd = true;
      c->tb_cpt = cpt;
      c->tbc.nst = nst;
      c->tbc.H = c->max_hout;
      c->tbc.MA = MA;
      c->tbc.MB = MB;
      c->tbc.nch = c->Lp / SW;
      c->tbc.nitems = c->ntiles * c->tbc.nch;
    }
  }
  // tile forward (option tfwd): stages of the in- and out-halo rows x 128 commodities + records + metadata
  c->tile_fwd = false;
  if (c->tile_bwd && c->opt_tfwd != 0 && (c->opt_tfwd > 0 || !c->pipe_fwd) && c->node_cap.empty() && c->Lp % 128 == 0) {
    const size_t budget = 226 * 1024;
    int MM = 0, MAi = 0;
    for (int k = 0; k < c->ntiles; ++k) {
      MM = std::max(MM, c->h_tf_desc[(size_t)k * 16 + 11]);
      MAi = std::max(MAi, c->h_tf_desc[(size_t)k * 16 + 3]);
    }
    int nst = 1;
    while (nst < 4 && tf_smem(nst + 1, c->max_hin, c->max_hout, 128, MAi, c->max_oa, MM) <= budget) ++nst;
    if (nst >= 2) {
      c->tile_fwd = true;
      c->tfc.nst = nst;
      c->tfc.Hin = c->max_hin;
      c->tfc.Hout = c->max_hout;
      c->tfc.MAi = MAi;
      c->tfc.MAo = c->max_oa;
      c->tfc.MM = MM;
      c->tfc.nch = c->Lp / 128;
      c->tfc.nitems = c->ntiles * c->tfc.nch;
    }
  }
  c->nch = c->Lp / c->LC;
  // wide path: warps = (nodes per CTA) x (chunks per CTA) = 8
  {
    // (auto: 8 chunks of one node per CTA; 1 chunk of 8 neighbouring nodes when the rows are sliced into >= 16 chunks:
    // their shared neighbour rows hit in L1, measured [5] forward 67.3 -> 62.5 ms per sweep)
    int cp = c->opt_wcp > 0 ? c->opt_wcp : (c->prec == MMF_FP32 && c->nch >= 16 ? 1 : 8);
    while (cp > 1 && cp > c->nch) cp >>= 1;
    c->wc.cpcta = cp;
    c->wc.npc = (WIDE_THREADS / 32) / cp;
    c->wc.ngroup = (c->nch + cp - 1) / cp;
    c->wc.nch = c->nch;
    c->wc.prefetch = c->opt_prefetch;
    int mo = 0;
    if (!c->h_outptr.empty())
      for (int j0 = 0; j0 < c->N; j0 += c->wc.npc)
        mo = std::max(mo, c->h_outptr[std::min(j0 + c->wc.npc, c->N)] - c->h_outptr[j0]);
    c->wc.max_oa = mo;
  }
  // head-flow path: all chunks of a node in one CTA
  {
    HeadCfg& h = c->hc;
    h.nch = c->nch;
    h.wpn = c->nch <= HF_WARPS ? c->nch : HF_WARPS;
    h.npc = c->nch <= HF_WARPS ? std::max(1, HF_WARPS / c->nch) : 1;
    int mi = 0;
    if (!c->h_inptr.empty())
      for (int j0 = 0; j0 < c->N; j0 += h.npc)
        mi = std::max(mi, c->h_inptr[std::min(j0 + h.npc, c->N)] - c->h_inptr[j0]);
    h.max_ia = std::max(mi, 1);
  }
  // chunk groups per tile: enough CTAs for ~4 per SM, each CTA pipelining cpc chunks
  {
    const int target = 4 * 148;
    int ng = c->opt_cpc > 0 ? (c->nch + c->opt_cpc - 1) / c->opt_cpc
                            : std::max(1, std::min(c->nch, (target + std::max(c->ntiles, 1) - 1) / std::max(c->ntiles, 1)));
    c->pc.cpc = (c->nch + ng - 1) / ng;
    c->pc.ngroup = (c->nch + c->pc.cpc - 1) / c->pc.cpc;
  }
  int chunks = c->Lp / 32;
  int w = 8;
  while (chunks % w) w >>= 1;
  c->block = 32 * w;
  c->G = c->Lp / c->block;
}

// host-side graph structures: node order (tiles), internal arc order (in-CSR by head), out-CSR,
// tile halos and halo-local indices.  Depends on the graph and options only.
// ---- sliding-window node order (opt_kernels == 6) -------------------------------------------------
// Candidates: the input order, reverse Cuthill-McKee, and "strip" versions of both (the order cut into rows
// of its 90th-percentile bandwidth, then strips of w columns visited strip by strip, row by row: on a
// row-major grid this is the classic strip order, bandwidth w instead of the row length).  For each
// candidate and window half-width Wb (in 32-node blocks) the fraction f of moving arcs whose endpoints
// lie more than Wb blocks apart is measured; cost = (|A|/N) f + 2 Wb / (blocks per segment) (+ a small
// penalty for 32-commodity slices), subject to the window fitting in shared memory.
std::vector<int> strip_newid(const std::vector<int>& rank, int b, int w) {
  const int N = (int)rank.size();
  std::vector<int> ord(N);
  std::iota(ord.begin(), ord.end(), 0);
  b = std::max(b, 1);
  std::sort(ord.begin(), ord.end(), [&](int x, int y) {
    const int rx = rank[x] / b, cx = rank[x] % b, ry = rank[y] / b, cy = rank[y] % b;
    const int sx = cx / w, sy = cy / w;
    if (sx != sy) return sx < sy;
    if (rx != ry) return rx < ry;
    return cx < cy;
  });
  std::vector<int> nid(N);
  for (int k = 0; k < N; ++k) nid[ord[k]] = k;
  return nid;
}

// ---- row-reuse node order (the pipelined kernels' default) ------------------------------------------
// A pipeline walks consecutive nodes; a row gathered for one of the last few items is still resident in its
// ring.  Score of an order = the fraction of gathered rows (in-lists: forward; out-lists: backward) whose
// node was gathered within the previous RU_WIN items.  Candidates: input, reverse Cuthill-McKee, and strip
// versions of both (strip_newid) of widths 2 .. 32.
constexpr int RU_WIN = 3;
double reuse_frac(const mmf_ctx* c, const std::vector<int>& nid, bool in_lists) {
  const int N = c->N;
  const size_t A = c->tail.size();
  std::vector<int> ptr(N + 1, 0), lst(A);
  for (size_t a = 0; a < A; ++a) ptr[nid[in_lists ? c->head[a] : c->tail[a]] + 1]++;
  for (int v = 0; v < N; ++v) ptr[v + 1] += ptr[v];
  std::vector<int> fill(ptr.begin(), ptr.end() - 1);
  for (size_t a = 0; a < A; ++a) {
    const int item = nid[in_lists ? c->head[a] : c->tail[a]];
    lst[fill[item]++] = nid[in_lists ? c->tail[a] : c->head[a]];
  }
  std::vector<int> last(N, -(1 << 30));
  size_t hit = 0;
  for (int j = 0; j < N; ++j)
    for (int q = ptr[j]; q < ptr[j + 1]; ++q) {
      const int r = lst[q];
      hit += j - last[r] <= RU_WIN;
      last[r] = j;
    }
  return A ? (double)hit / (double)A : 0.0;
}
void choose_reuse_order(mmf_ctx* c) {
  HostTimer ht("choose_reuse_order");
  const int N = c->N;
  const size_t A = c->tail.size();
  std::vector<int> id(N);
  std::iota(id.begin(), id.end(), 0);
  std::vector<int> rcm = rcm_newid(N, c->tail, c->head);
  // candidates: input, RCM, and strip versions of both; built and scored on host threads (one per candidate)
  struct Cand {
    int base, w;
  };
  std::vector<Cand> spec = {{0, 0}, {1, 0}};
  const std::vector<int>* bases[2] = {&id, &rcm};
  for (int base = 0; base < 2; ++base) {
    std::vector<int> d;
    const std::vector<int>& b = *bases[base];
    for (size_t a = 0; a < A; ++a)
      if (c->tail[a] != c->head[a]) d.push_back(std::abs(b[c->tail[a]] - b[c->head[a]]));
    if (d.empty()) continue;
    std::nth_element(d.begin(), d.begin() + (size_t)(0.90 * (d.size() - 1)), d.end());
    const int b90 = d[(size_t)(0.90 * (d.size() - 1))];
    for (int w : {2, 4, 8, 16, 32})
      if (b90 > 2 * w && (!c->opt_stripw || c->opt_stripw == w)) spec.push_back({base, w * 1000000 + b90});
  }
  const size_t first = (c->opt_stripw && spec.size() > 2) ? 2 : 0;
  std::vector<std::vector<int>> cands(spec.size());
  std::vector<double> score(spec.size(), -1.0);
  std::vector<std::future<void>> jobs;
  for (size_t ci = first; ci < spec.size(); ++ci)
    jobs.push_back(std::async(std::launch::async, [&, ci]() {
      const Cand& k = spec[ci];
      cands[ci] = k.w == 0 ? *bases[k.base] : strip_newid(*bases[k.base], k.w % 1000000, k.w / 1000000);
      score[ci] = reuse_frac(c, cands[ci], true) + reuse_frac(c, cands[ci], false);
    }));
  for (auto& j : jobs) j.get();
  double best = -1.0;
  size_t bi = first;
  for (size_t ci = first; ci < spec.size(); ++ci) {  // (same choice as a serial scan: first of the best)
    if (getenv("MMF_VERBOSE")) fprintf(stderr, "[mmf] reuse order cand %zu: %.3f\n", ci, 0.5 * score[ci]);
    if (score[ci] > best + 1e-9) {
      best = score[ci];
      bi = ci;
    }
  }
  c->newid = cands[bi];
  c->win_Wb = 0;
  c->win_cpt = 4;
}

size_t win_bwd_smem(int cpt, int Wb, int farmax, int maxrec, int segB) {
  WinCfg wc{};
  wc.RBa = 2 * Wb + 1 + WIN_PD;
  wc.farmax = std::max(farmax, 1);
  wc.maxrec = maxrec;
  wc.segB = segB;
  return cpt == 4 ? win_smem<4>(wc).total : cpt == 2 ? win_smem<2>(wc).total : win_smem<1>(wc).total;
}

void choose_window_order(mmf_ctx* c) {
  const int N = c->N;
  const size_t A = c->tail.size();
  std::vector<std::vector<int>> cands;
  cands.emplace_back(N);
  std::iota(cands[0].begin(), cands[0].end(), 0);
  cands.push_back(rcm_newid(N, c->tail, c->head));
  for (int base = 0; base < 2; ++base) {
    std::vector<int> d;
    for (size_t a = 0; a < A; ++a)
      if (c->tail[a] != c->head[a]) d.push_back(std::abs(cands[base][c->tail[a]] - cands[base][c->head[a]]));
    if (d.empty()) continue;
    // the "row length" of the order: the 90th percentile of |i - j| over moving arcs (robust to a few
    // percent of long-range arcs such as highways)
    std::nth_element(d.begin(), d.begin() + (size_t)(0.90 * (d.size() - 1)), d.end());
    const int b90 = d[(size_t)(0.90 * (d.size() - 1))];
    for (int w : {32, 64})
      if (b90 > 2 * w) cands.push_back(strip_newid(cands[base], b90, w));
  }
  const double deg = (double)A / std::max(N, 1);
  const int nblk = (N + WIN_BR - 1) / WIN_BR;
  const size_t budget = 225 * 1024;
  double best = 1e30;
  int bi = 0, bW = 0, bc = 2;
  std::vector<int> mark(N, -1), nfar(nblk);
  for (size_t ci = 0; ci < cands.size(); ++ci) {
    const std::vector<int>& nid = cands[ci];
    // records of each block (out-direction: grouped by tail)
    std::vector<int> recs(nblk, 0);
    int moving = 0;
    for (size_t a = 0; a < A; ++a) {
      recs[nid[c->tail[a]] / WIN_BR]++;
      moving += c->tail[a] != c->head[a];
    }
    const int maxrec = *std::max_element(recs.begin(), recs.end());
    for (int Wb = 0; Wb <= 12; ++Wb) {
      // far fraction and the largest per-block count of distinct far rows at this half-width
      std::fill(nfar.begin(), nfar.end(), 0);
      std::fill(mark.begin(), mark.end(), -1);
      int far = 0;
      for (size_t a = 0; a < A; ++a) {
        const int bt = nid[c->tail[a]] / WIN_BR, k = nid[c->head[a]];
        if (std::abs(k / WIN_BR - bt) <= Wb) continue;
        ++far;
        if (mark[k] != bt) {
          mark[k] = bt;
          nfar[bt]++;
        }
      }
      const int farmax = *std::max_element(nfar.begin(), nfar.end());
      const double f = moving ? (double)far / moving : 0.0;
      for (int cpt : {4, 2, 1}) {
        const int SW = 32 * cpt;
        if (SW > 2 * c->L && cpt > 1) continue;  // (slices wider than the commodity count waste lanes)
        const int ns = (c->L + SW - 1) / SW;
        const int nseg = std::max(1, c->sms / std::max(ns, 1));
        const int segB = (nblk + nseg - 1) / nseg;
        const size_t sm = win_bwd_smem(cpt, Wb, farmax, maxrec, segB);
        if (sm > budget) continue;
        const double cost = deg * f + 2.0 * Wb / std::max(segB, 1) + (cpt == 4 ? 0.0 : cpt == 2 ? 0.08 : 0.3);
        if (getenv("MMF_VERBOSE") && Wb <= 4)
          fprintf(stderr, "[mmf] order cand %zu cpt %d Wb %d far %.4f farmax %d cost %.3f smem %zu\n", ci, cpt, Wb, f,
                  farmax, cost, sm);
        if (cost < best) {
          best = cost;
          bi = (int)ci;
          bW = Wb;
          bc = cpt;
        }
      }
    }
  }
  c->newid = cands[bi];
  c->win_Wb = bW;
  c->win_cpt = bc;
}

// window tables of the out-direction (backward gathers): per out-CSR record the window slot or far index
void build_window_tables(mmf_ctx* c) {
  HostTimer ht("build_window_tables");
  const int N = c->N, Wb = c->win_Wb, RBa = 2 * Wb + 1 + WIN_PD;
  const int nblk = (N + WIN_BR - 1) / WIN_BR;
  const int64_t A = c->A;
  c->h_wsrc_out.assign(A, 0);
  c->h_wfptr_out.assign(nblk + 1, 0);
  c->h_wfnode_out.clear();
  int farmax = 0, maxrec = 0;
  std::vector<int> seen(N, -1);
  for (int b = 0; b < nblk; ++b) {
    const int v0 = b * WIN_BR, v1 = std::min(N, v0 + WIN_BR);
    maxrec = std::max(maxrec, c->h_outptr[v1] - c->h_outptr[v0]);
    int nf = 0;
    for (int v = v0; v < v1; ++v)
      for (int q = c->h_outptr[v]; q < c->h_outptr[v + 1]; ++q) {
        const int k = c->h_outhead[q];
        const int rb = k / WIN_BR;
        if (std::abs(rb - b) <= Wb) {
          c->h_wsrc_out[q] = (rb % RBa) * WIN_BR + k % WIN_BR;
        } else {
          if (seen[k] != b) {
            seen[k] = b;
            c->h_wfnode_out.push_back(k);
            ++nf;
          }
          int idx = 0;
          for (int f = c->h_wfptr_out[b]; f < (int)c->h_wfnode_out.size(); ++f)
            if (c->h_wfnode_out[f] == k) {
              idx = f - c->h_wfptr_out[b];
              break;
            }
          c->h_wsrc_out[q] = RBa * WIN_BR + idx;
        }
      }
    c->h_wfptr_out[b + 1] = (int)c->h_wfnode_out.size();
    farmax = std::max(farmax, nf);
  }
  c->wcb.Wb = Wb;
  c->wcb.RBa = RBa;
  c->wcb.farmax = std::max(farmax, 1);
  c->wcb.maxrec = std::max(maxrec, 1);
  c->wcb.nblk = nblk;
}

// 2-D TMA tensor maps of a message store (slots x N rows of Lp commodities): box = 32 rows x SW
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
bool make_tmaps(mmf_ctx* c, void* msig, void* mexp, int slots, int SW, WinTmaps& out) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess || !f) return false;
    fn = (EncodeTiledFn)f;
  }
  const cuuint64_t rows = (cuuint64_t)slots * c->N;
  const cuuint32_t box[2] = {(cuuint32_t)SW, (cuuint32_t)WIN_BR};
  const cuuint32_t es[2] = {1, 1};
  cuuint64_t dim[2] = {(cuuint64_t)c->Lp, rows};
  cuuint64_t st_s[1] = {(cuuint64_t)c->Lp * 4};
  cuuint64_t st_e[1] = {(cuuint64_t)c->Lp * 2};
  if (fn(&out.sig, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, msig, dim, st_s, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (fn(&out.exp, CU_TENSOR_MAP_DATA_TYPE_UINT16, 2, mexp, dim, st_e, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  return true;
}

void augment_times(mmf_ctx* c) {
  if (c->augmented) return;
  c->N_user = c->N;
  c->A_user = c->A;
  c->cost_user = c->cost;
  c->cap_user = c->cap;
  if (c->t_in.empty()) return;
  const int T = c->T;
  const int64_t A0 = c->A;
  std::vector<int> ta, ha;                 // appended arcs
  std::vector<std::vector<double>> costa;  // their per-step costs: 0 when open, +inf (absent, K = 0) otherwise
  auto arc = [&](int u, int v, int open_step) {  // open_step < 0: always open
    ta.push_back(u);
    ha.push_back(v);
    std::vector<double> cp(T, INFINITY);
    for (int t = 0; t < T; ++t)
      if (open_step < 0 || t == open_step) cp[t] = 0.0;
    costa.push_back(cp);
  };
  int N = c->N;
  for (int l = 0; l < c->L; ++l) {
    if (c->t_in[l] > 0) {
      const int h = N++;
      arc(h, h, -1);
      arc(h, c->src[l], c->t_in[l] - 1);
      c->src[l] = h;
    }
    if (c->t_out[l] < T) {
      const int g = N++;
      arc(c->dst[l], g, c->t_out[l]);
      arc(g, g, -1);
      c->dst[l] = g;
    }
  }
  const int64_t A1 = A0 + (int64_t)ta.size();
  c->tail.insert(c->tail.end(), ta.begin(), ta.end());
  c->head.insert(c->head.end(), ha.begin(), ha.end());
  // costs become per step (the appended arcs exist at their open steps only: cost +inf = absent from the graph,
  // P:691, so K = 0 there from the start, as in the native multi-tensor form); capacities: the appended arcs are free
  std::vector<double> cc((size_t)T * A1);
  for (int t = 0; t < T; ++t) {
    for (int64_t a = 0; a < A0; ++a) cc[(size_t)t * A1 + a] = c->cost[(c->cost_tv ? (size_t)t * A0 : 0) + a];
    for (size_t q = 0; q < ta.size(); ++q) cc[(size_t)t * A1 + A0 + q] = costa[q][t];
  }
  c->cost.swap(cc);
  c->cost_tv = true;
  if (c->cap_tv) {
    std::vector<double> kc((size_t)T * A1, INFINITY);
    for (int t = 0; t < T; ++t) std::copy(c->cap.begin() + (size_t)t * A0, c->cap.begin() + (size_t)(t + 1) * A0, kc.begin() + (size_t)t * A1);
    c->cap.swap(kc);
  } else {
    c->cap.resize(A1, INFINITY);
  }
  // node costs: 0 at the holding nodes
  if (!c->node_cost.empty()) {
    std::vector<double> nc((size_t)c->L * N, 0.0);
    for (int l = 0; l < c->L; ++l)
      std::copy(c->node_cost.begin() + (size_t)l * c->N, c->node_cost.begin() + (size_t)(l + 1) * c->N, nc.begin() + (size_t)l * N);
    c->node_cost.swap(nc);
  }
  if (!c->node_cap.empty()) {  // (holding nodes are free)
    const int TN = c->node_cap_tv ? T + 1 : 1;
    std::vector<double> dn((size_t)TN * N, INFINITY);
    for (int t = 0; t < TN; ++t)
      std::copy(c->node_cap.begin() + (size_t)t * c->N, c->node_cap.begin() + (size_t)(t + 1) * c->N, dn.begin() + (size_t)t * N);
    c->node_cap.swap(dn);
  }
  c->N = N;
  c->A = A1;
  c->augmented = true;
}

// the tile backward applies (option tbwd; decided before the node order, which it dictates)
bool tbwd_wanted(const mmf_ctx* c) {
  if (c->prec != MMF_FP32 || c->opt_kernels != 6 || c->opt_tbwd == 0) return false;
  if (c->opt_tbwd > 0) return true;
  return c->L >= 256 && c->A >= 7 * (int64_t)c->N && c->opt_bwd == 0;
}

void prepare(mmf_ctx* c) {
  if (c->prepared) return;
  HostTimer ht("prepare");
  c->fpos_ok = false;  // (int_of_arc follows the node order)
  augment_times(c);
  const int N = c->N;
  const int64_t A = c->A;
  std::vector<int> order;
  const int B = c->opt_kernels >= 2 ? c->opt_tile : std::max(N, 1);
  if (tbwd_wanted(c)) {
    // node tiles for the tile backward: BFS-grown blobs of at most `tile` nodes whose halos stay within `halo`
    const int Bt = c->opt_tile;
    make_tiles(N, c->tail, c->head, Bt, c->opt_halo > 0 ? c->opt_halo : 2 * Bt, c->opt_reorder, order, c->h_tile_ptr);
    c->newid.assign(N, 0);
    for (int k = 0; k < N; ++k) c->newid[order[k]] = k;
    c->win_Wb = 0;
    c->win_cpt = 4;
  } else if (c->opt_kernels == 6 && c->opt_reorder) {
    // node order: the window kernel's cost model for the window backward (bwd=2) and for the other kernel
    // families (measured better for them on [2]), plain RCM on request (order=1), else the order with the most
    // neighbour overlap between consecutive nodes (measured best for the pipelined kernels: [4] 85.4 vs 87.1
    // ms per sweep with the window order, 94.8 with RCM)
    const bool pipelined = c->prec == MMF_FP32 && c->L >= 256;  // (where the pipelined kernels apply)
    if (c->opt_bwd == 2 || c->opt_order == 3 || (!pipelined && c->opt_order != 4 && c->opt_order != 1)) {
      choose_window_order(c);
    } else if (c->opt_order == 1) {
      c->newid = rcm_newid(N, c->tail, c->head);
      c->win_Wb = 0;
      c->win_cpt = 4;
    } else {
      choose_reuse_order(c);
    }
    c->h_tile_ptr.assign(1, 0);
    for (int v = B; v < N; v += B) c->h_tile_ptr.push_back(v);
    c->h_tile_ptr.push_back(N);
  } else if (c->opt_kernels >= 2 && c->opt_order == 2) {
    make_tiles(N, c->tail, c->head, B, c->opt_halo > 0 ? c->opt_halo : 2 * B, c->opt_reorder, order, c->h_tile_ptr);
    c->newid.assign(N, 0);
    for (int k = 0; k < N; ++k) c->newid[order[k]] = k;
  } else if (c->opt_kernels >= 2) {
    if (c->opt_reorder && c->opt_order == 1) {
      c->newid = rcm_newid(N, c->tail, c->head);
    } else {
      c->newid.resize(N);
      std::iota(c->newid.begin(), c->newid.end(), 0);
    }
    c->h_tile_ptr.assign(1, 0);
    for (int v = B; v < N; v += B) c->h_tile_ptr.push_back(v);
    c->h_tile_ptr.push_back(N);
  } else {
    if (c->opt_reorder) {
      c->newid = rcm_newid(N, c->tail, c->head);
    } else {
      c->newid.resize(N);
      std::iota(c->newid.begin(), c->newid.end(), 0);
    }
    c->h_tile_ptr = {0, N};
  }
  c->ntiles = (int)c->h_tile_ptr.size() - 1;
  c->tileB = 0;
  for (int k = 0; k < c->ntiles; ++k) c->tileB = std::max(c->tileB, c->h_tile_ptr[k + 1] - c->h_tile_ptr[k]);

  HostTimer ht1("prepare: csr");
  std::vector<int> it(A), ih(A);
  for (int64_t a = 0; a < A; ++a) {
    it[a] = c->newid[c->tail[a]];
    ih[a] = c->newid[c->head[a]];
  }
  // arcs sorted by (head, tail): two stable counting sorts (by tail, then by head); the pairs are unique, so this is
  // the order of a lexicographic comparison sort
  auto counting_sort = [N](const std::vector<int64_t>& in, const std::vector<int>& key) {
    std::vector<int64_t> cnt(N + 1, 0), out(in.size());
    for (int64_t x : in) cnt[key[x] + 1]++;
    for (int v = 0; v < N; ++v) cnt[v + 1] += cnt[v];
    for (int64_t x : in) out[cnt[key[x]]++] = x;
    return out;
  };
  std::vector<int64_t> ord(A);
  std::iota(ord.begin(), ord.end(), 0);
  ord = counting_sort(counting_sort(ord, it), ih);
  c->int_of_arc.assign(A, 0);
  c->h_tail.assign(A, 0);
  c->h_head.assign(A, 0);
  c->h_inptr.assign(N + 1, 0);
  c->h_outptr.assign(N + 1, 0);
  c->h_outarc.assign(A, 0);
  c->h_outhead.assign(A, 0);
  for (int64_t k = 0; k < A; ++k) {
    c->int_of_arc[ord[k]] = (int)k;
    c->h_tail[k] = it[ord[k]];
    c->h_head[k] = ih[ord[k]];
    c->h_inptr[ih[ord[k]] + 1]++;
  }
  for (int v = 0; v < N; ++v) c->h_inptr[v + 1] += c->h_inptr[v];
  c->maxdeg_in = 0;
  for (int v = 0; v < N; ++v) c->maxdeg_in = std::max(c->maxdeg_in, c->h_inptr[v + 1] - c->h_inptr[v]);
  std::vector<int64_t> ordo(A);
  std::iota(ordo.begin(), ordo.end(), 0);  // (already sorted by head: one stable pass by tail gives (tail, head))
  ordo = counting_sort(ordo, c->h_tail);
  for (int64_t k = 0; k < A; ++k) {
    c->h_outarc[k] = (int)ordo[k];
    c->h_outhead[k] = c->h_head[ordo[k]];
    c->h_outptr[c->h_tail[ordo[k]] + 1]++;
  }
  for (int v = 0; v < N; ++v) c->h_outptr[v + 1] += c->h_outptr[v];
  c->pb.D = 0;
  int din = 0;
  for (int v = 0; v < N; ++v) {
    c->pb.D = std::max(c->pb.D, c->h_outptr[v + 1] - c->h_outptr[v]);
    din = std::max(din, c->h_inptr[v + 1] - c->h_inptr[v]);
  }
  c->ell_din = din;

  // halos (tile backward only; the other families get empty tables of the right sizes)
  if (!tbwd_wanted(c)) {
    const size_t nt = (size_t)c->ntiles;
    c->h_hin_ptr.assign(nt + 1, 0);
    c->h_hout_ptr.assign(nt + 1, 0);
    c->h_hin_node.clear();
    c->h_hout_node.clear();
    c->h_in_hidx.assign(A, 0);
    c->h_out_hidx.assign(A, 0);
    c->max_hin = c->max_hout = c->max_ia = c->max_oa = 0;
    c->h_tb_desc.clear();
    c->h_tb_meta.clear();
    c->h_tf_desc.clear();
    c->h_tf_meta.clear();
    c->prepared = true;
    return;
  }
  HostTimer ht2("prepare: halos");
  std::vector<int> tile_of(N);
  for (int k = 0; k < c->ntiles; ++k)
    for (int v = c->h_tile_ptr[k]; v < c->h_tile_ptr[k + 1]; ++v) tile_of[v] = k;
  c->h_hin_ptr.assign(1, 0);
  c->h_hout_ptr.assign(1, 0);
  c->h_hin_node.clear();
  c->h_hout_node.clear();
  c->h_in_hidx.assign(A, 0);
  c->h_out_hidx.assign(A, 0);
  c->max_hin = c->max_hout = c->max_ia = c->max_oa = 0;
  std::vector<int> tmp;
  for (int k = 0; k < c->ntiles; ++k) {
    const int v0 = c->h_tile_ptr[k], v1 = c->h_tile_ptr[k + 1];
    c->max_ia = std::max(c->max_ia, c->h_inptr[v1] - c->h_inptr[v0]);
    c->max_oa = std::max(c->max_oa, c->h_outptr[v1] - c->h_outptr[v0]);
    tmp.assign(c->h_tail.begin() + c->h_inptr[v0], c->h_tail.begin() + c->h_inptr[v1]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    const size_t base_in = c->h_hin_node.size();
    c->h_hin_node.insert(c->h_hin_node.end(), tmp.begin(), tmp.end());
    c->h_hin_ptr.push_back((int)c->h_hin_node.size());
    c->max_hin = std::max(c->max_hin, (int)tmp.size());
    for (int a = c->h_inptr[v0]; a < c->h_inptr[v1]; ++a)
      c->h_in_hidx[a] = (int)(std::lower_bound(c->h_hin_node.begin() + base_in, c->h_hin_node.end(), c->h_tail[a]) -
                              (c->h_hin_node.begin() + base_in));
    tmp.assign(c->h_outhead.begin() + c->h_outptr[v0], c->h_outhead.begin() + c->h_outptr[v1]);
    std::sort(tmp.begin(), tmp.end());
    tmp.erase(std::unique(tmp.begin(), tmp.end()), tmp.end());
    const size_t base_out = c->h_hout_node.size();
    c->h_hout_node.insert(c->h_hout_node.end(), tmp.begin(), tmp.end());
    c->h_hout_ptr.push_back((int)c->h_hout_node.size());
    c->max_hout = std::max(c->max_hout, (int)tmp.size());
    for (int q = c->h_outptr[v0]; q < c->h_outptr[v1]; ++q)
      c->h_out_hidx[q] = (int)(std::lower_bound(c->h_hout_node.begin() + base_out, c->h_hout_node.end(), c->h_outhead[q]) -
                               (c->h_hout_node.begin() + base_out));
  }
  // tile backward: per tile {v0, nv, q0, na, h0, nh, meta offset (ints, multiple of 4), meta ints (multiple of 4)} and
  // the static metadata [nv + 1 local out-CSR offsets | pad | na halo indices | pad] at 16-byte aligned offsets, so
  // that the producer stages a tile with one descriptor load and bulk copies only
  c->h_tb_desc.assign((size_t)c->ntiles * 8, 0);
  c->h_tb_meta.clear();
  for (int k = 0; k < c->ntiles; ++k) {
    const int v0 = c->h_tile_ptr[k], v1 = c->h_tile_ptr[k + 1];
    const int q0 = c->h_outptr[v0], q1 = c->h_outptr[v1];
    const int off = (int)c->h_tb_meta.size();
    for (int v = v0; v <= v1; ++v) c->h_tb_meta.push_back(c->h_outptr[v] - q0);
    while (c->h_tb_meta.size() % 4) c->h_tb_meta.push_back(0);
    for (int q = q0; q < q1; ++q) c->h_tb_meta.push_back(c->h_out_hidx[q]);
    while (c->h_tb_meta.size() % 4) c->h_tb_meta.push_back(0);
    int* d = &c->h_tb_desc[(size_t)k * 8];
    d[0] = v0;
    d[1] = v1 - v0;
    d[2] = q0;
    d[3] = q1 - q0;
    d[4] = c->h_hout_ptr[k];
    d[5] = c->h_hout_ptr[k + 1] - c->h_hout_ptr[k];
    d[6] = off;
    d[7] = (int)c->h_tb_meta.size() - off;
  }
  // tile forward: per tile 16 ints {v0, nv, qi0, nai, qo0, nao, hin0, nhin, hout0, nhout, moff, mn, o_inidx, o_outptr,
  // o_outidx, 0} and the block [nv + 1 in offsets | in-halo indices | nv + 1 out offsets | out-halo indices]
  c->h_tf_desc.assign((size_t)c->ntiles * 16, 0);
  c->h_tf_meta.clear();
  auto pad4 = [&]() { while (c->h_tf_meta.size() % 4) c->h_tf_meta.push_back(0); };
  for (int k = 0; k < c->ntiles; ++k) {
    const int v0 = c->h_tile_ptr[k], v1 = c->h_tile_ptr[k + 1];
    const int qi0 = c->h_inptr[v0], qi1 = c->h_inptr[v1], qo0 = c->h_outptr[v0], qo1 = c->h_outptr[v1];
    const int off = (int)c->h_tf_meta.size();
    for (int v = v0; v <= v1; ++v) c->h_tf_meta.push_back(c->h_inptr[v] - qi0);
    pad4();
    const int o_inidx = (int)c->h_tf_meta.size() - off;
    for (int q = qi0; q < qi1; ++q) c->h_tf_meta.push_back(c->h_in_hidx[q]);
    pad4();
    const int o_outptr = (int)c->h_tf_meta.size() - off;
    for (int v = v0; v <= v1; ++v) c->h_tf_meta.push_back(c->h_outptr[v] - qo0);
    pad4();
    const int o_outidx = (int)c->h_tf_meta.size() - off;
    for (int q = qo0; q < qo1; ++q) c->h_tf_meta.push_back(c->h_out_hidx[q]);
    pad4();
    int* d = &c->h_tf_desc[(size_t)k * 16];
    const int dv[16] = {v0, v1 - v0, qi0, qi1 - qi0, qo0, qo1 - qo0, c->h_hin_ptr[k], c->h_hin_ptr[k + 1] - c->h_hin_ptr[k],
                        c->h_hout_ptr[k], c->h_hout_ptr[k + 1] - c->h_hout_ptr[k], off, (int)c->h_tf_meta.size() - off,
                        o_inidx, o_outptr, o_outidx, 0};
    std::copy(dv, dv + 16, d);
  }
  c->prepared = true;
}

// walk the workspace layout; assign pointers when base != nullptr
// the multi-GPU exchange buffer holds the flows of the arcs with a finite capacity at some step only (SURVEY 8(e)
// mitigation 2: the all-reduce of a step moves |E| values, not |A|; [4]: 150,444 of 190,444)
static void build_fpos(mmf_ctx* c) {
  const int64_t A = c->A;
  const int TC = c->cap_tv ? c->T : 1;
  std::vector<char> capd(A, 0);
  for (int t = 0; t < TC; ++t)
    for (int64_t a = 0; a < A; ++a)
      if (std::isfinite(c->cap[(size_t)t * A + a])) capd[c->int_of_arc[a]] = 1;
  c->h_fpos.assign(A, -1);
  int64_t e = 0;
  for (int64_t k = 0; k < A; ++k)
    if (capd[k]) c->h_fpos[k] = (int)e++;
  c->Ecap = e;
  c->fpos_ok = true;
}

size_t layout(mmf_ctx* c, char* base) {
  if (!c->fpos_ok) build_fpos(c);
  Layout L;
  const size_t A = (size_t)c->A, N = (size_t)c->N, T = (size_t)c->T, Lp = (size_t)c->Lp;
  const size_t TK = c->cost_tv ? T : 1, TC = c->cap_tv ? T : 1;
  const size_t sm = c->sm(), se = c->se();
  DevPtrs& p = c->dp;
  TileMeta& tm = c->tm;
  auto at = [&](size_t o) -> char* { return base ? base + o : nullptr; };
  p.tail = (const int*)at(L.take(A * 4));
  p.in_ptr = (const int*)at(L.take((N + 1) * 4));
  p.out_ptr = (const int*)at(L.take((N + 1) * 4));
  p.out_arc = (const int*)at(L.take(A * 4));
  p.out_head = (const int*)at(L.take(A * 4));
  p.Km = at(L.take(TK * A * sm));
  p.Ke = (const int*)at(L.take(TK * A * 4));
  p.dcap = at(L.take(TC * A * sm));
  p.Wm = at(L.take(T * A * sm));
  p.We = (int*)at(L.take(T * A * 4));
  const size_t aslots = c->opt_schedule == 2 ? T + 1 : 2;  // (symmetric GS keeps every alpha_t)
  p.am = at(L.take(aslots * N * Lp * sm));
  p.ae = at(L.take(aslots * N * Lp * se));
  p.akeep = c->opt_schedule == 2 ? 1 : 0;
  p.bm = at(L.take((T + 1) * N * Lp * sm));
  p.be = at(L.take((T + 1) * N * Lp * se));
  p.u0m = at(L.take(N * Lp * sm));
  p.u0e = at(L.take(N * Lp * se));
  p.dnm = c->node_cost.empty() ? nullptr : at(L.take(N * Lp * sm));
  p.dne = c->node_cost.empty() ? nullptr : at(L.take(N * Lp * se));
  const bool ncap = !c->node_cap.empty();
  p.dnc = ncap ? at(L.take((c->node_cap_tv ? T + 1 : 1) * N * sm)) : nullptr;
  p.dnc_tv = c->node_cap_tv ? 1 : 0;
  p.unm = ncap ? at(L.take((T + 1) * N * sm)) : nullptr;
  p.une = ncap ? (int*)at(L.take((T + 1) * N * 4)) : nullptr;
  p.unlm = nullptr;
  p.unle = nullptr;
  if (!c->point) {
    p.mu0m = at(L.take(N * Lp * sm));
    p.mu0e = at(L.take(N * Lp * se));
    p.muTm = at(L.take(N * Lp * sm));
    p.muTe = at(L.take(N * Lp * se));
    p.psrc = p.pdst = nullptr;
    p.pmass = nullptr;
  } else {
    p.mu0m = p.mu0e = p.muTm = p.muTe = nullptr;
    p.psrc = (const int*)at(L.take((size_t)c->L * 4));
    p.pdst = (const int*)at(L.take((size_t)c->L * 4));
    p.pmass = (const double*)at(L.take((size_t)c->L * 8));
  }
  p.part = at(L.take((size_t)c->G * A * sm));
  p.Fsum = at(L.take(std::max<int64_t>(c->Ecap, 1) * sm));
  p.fpos = (const int*)at(L.take(A * 4));
  p.Ecap = (int)c->Ecap;
  p.Fout = at(L.take(T * A * sm));
  p.err = (unsigned*)at(L.take(8));
  p.errloc = (unsigned long long*)at(L.take(8));
  p.stats = (double*)at(L.take(8 * 8));
  const size_t nt = (size_t)c->ntiles;
  tm.tile_ptr = (const int*)at(L.take((nt + 1) * 4));
  tm.hin_ptr = (const int*)at(L.take((nt + 1) * 4));
  tm.hin_node = (const int*)at(L.take(c->h_hin_node.size() * 4 + 4));
  tm.hout_ptr = (const int*)at(L.take((nt + 1) * 4));
  tm.hout_node = (const int*)at(L.take(c->h_hout_node.size() * 4 + 4));
  tm.in_hidx = (const int*)at(L.take(A * 4));
  tm.out_hidx = (const int*)at(L.take(A * 4));
  c->d_tb_desc = (const int*)at(L.take(c->h_tb_desc.size() * 4 + 16));
  c->d_tb_meta = (const int*)at(L.take(c->h_tb_meta.size() * 4 + 16));
  c->d_tf_desc = (const int*)at(L.take(c->h_tf_desc.size() * 4 + 16));
  c->d_tf_meta = (const int*)at(L.take(c->h_tf_meta.size() * 4 + 16));
  c->d_tf_part = c->tile_fwd ? (float*)at(L.take((size_t)A * c->tfc.nch * 4)) : nullptr;
  tm.cnt = (int*)at(L.take(nt * 4));
  c->wc.cnt = (int*)at(L.take(((size_t)c->N + 1) * 4));
  tm.part = at(L.take(A * (size_t)c->nch * sm));
  c->wc.part = tm.part;
  {
    const bool recs = c->opt_kernels >= 3;
    const size_t rb = c->prec == MMF_FP32 ? sizeof(ArcKW<float>) : sizeof(ArcKW<double>);
    p.inrec = recs ? at(L.take(T * A * rb)) : nullptr;
    p.outrec = recs ? at(L.take(T * A * rb)) : nullptr;
    p.opos = (const int*)at(L.take(A * 4));
    c->wdo.ptr = p.out_ptr;
    c->wdo.src = c->win_bwd ? (const int*)at(L.take(A * 4)) : nullptr;
    c->wdo.fptr = c->win_bwd ? (const int*)at(L.take(c->h_wfptr_out.size() * 4)) : nullptr;
    c->wdo.fnode = c->win_bwd ? (const int*)at(L.take(c->h_wfnode_out.size() * 4 + 4)) : nullptr;
    const bool ell = c->pipe_bwd;
    p.Din = ell ? c->ell_din : 0;
    p.diag = c->opt_dry >= 2 ? c->opt_dry : 0;
    p.l2hint = c->opt_l2hint;
    p.theta = (float)c->opt_theta_milli / 1000.f;
    p.Dout = ell ? c->pb.D : 0;
    p.ell_in = ell ? at(L.take(T * N * (size_t)p.Din * 16)) : nullptr;
    p.ell_ops = ell && c->prec == MMF_FP32 ? at(L.take(T * N * (size_t)p.Din * 32)) : nullptr;
    p.ell_out = ell ? at(L.take(T * N * (size_t)p.Dout * 16)) : nullptr;
    p.ell_ipos = ell ? (const int*)at(L.take(A * 4)) : nullptr;
    p.ell_opos = ell ? (const int*)at(L.take(A * 4)) : nullptr;
  }
  tm.ntiles = c->ntiles;
  tm.max_hin = c->max_hin;
  tm.max_hout = c->max_hout;
  tm.max_ia = c->max_ia;
  tm.max_oa = c->max_oa;
  tm.B = c->tileB;
  tm.nch = c->nch;
  tm.LC = c->LC;
  p.N = c->N;
  p.Lp = c->Lp;
  p.L = c->L;
  p.A = (int)c->A;
  p.T = c->T;
  p.TK = (int)TK;
  p.TC = (int)TC;
  p.G = c->G;
  p.maxdeg_in = c->maxdeg_in;
  return L.off;
}

bool ready_for_layout(const mmf_ctx* c) { return c->N > 0 && c->have_cost && c->have_cap && c->have_marg; }

// ------------------------------------------------------------------------------------------------
// launch helpers (accounting + optional per-kernel event timing)

cudaEvent_t get_event(mmf_ctx* c) {
  if (!c->ev_pool.empty()) {
    cudaEvent_t e = c->ev_pool.back();
    c->ev_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

struct LaunchScope {
  mmf_ctx* c;
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  LaunchScope(mmf_ctx* cc, int k, cudaStream_t ss) : c(cc), kind(k), s(ss) {
    if (c->opt_profile && !c->capturing) {
      a = get_event(c);
      b = get_event(c);
      cudaEventRecord(a, s);
    }
  }
  ~LaunchScope() {
    if (c->capturing)
      c->graph_launch_tally[kind]++;
    else
      c->launches[kind]++;
    if (a) {
      cudaEventRecord(b, s);
      c->prof.push_back({kind, a, b});
    }
  }
};

struct VSum {
  void* f[8];
};
// F = sum over the virtual ranks' partial flows (fixed order), written back to every rank's buffer
template <class M> __global__ void k_vsum(VSum v, int G, int64_t A) {
  for (int64_t a = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; a < A; a += (int64_t)gridDim.x * blockDim.x) {
    M x = M(0);
    for (int g = 0; g < G; ++g) x += ((const M*)v.f[g])[a];
    for (int g = 0; g < G; ++g) ((M*)v.f[g])[a] = x;
  }
}

inline unsigned grid1d(size_t n, int bs) {
  size_t g = (n + bs - 1) / bs;
  if (g > 148u * 16u) g = 148u * 16u;
  return (unsigned)std::max<size_t>(g, 1);
}

template <class T_> struct Eng {
  typedef typename T_::M M;
  typedef typename T_::E E;

  // the device pointers for a launch whose output messages are layer `layer`: the commodity node factor D (NEXT-2,
  // reading R-N) applies at the intermediate layers 1..T-1 only
  // (with_u: the node-capacity dual u_layer (NEXT-3) too — backward and readout launches; the forward sweep's launches
  // write alpha without it and k_node_cap applies the updated u)
  static DevPtrs lay(const mmf_ctx* c, int layer, bool with_u = true) {
    DevPtrs d = c->dp;
    d.unlm = nullptr;
    d.unle = nullptr;
    if (layer < 1 || layer > c->T - 1) {
      d.dnm = nullptr;
      d.dne = nullptr;
    } else if (with_u && d.unm) {
      d.unlm = (const char*)d.unm + (size_t)layer * c->N * c->sm();
      d.unle = d.une + (size_t)layer * c->N;
    }
    return d;
  }
  // NEXT-3 node-capacity block of layer t (1..T-1): u_t from the marginal of alpha_t (written without u_t) and the
  // stored beta-hat_t, then alpha_t *= u_t
  static void node_cap(mmf_ctx* c, cudaStream_t s, int t) {
    if (!c->dp.unm || t < 1 || t > c->T - 1) return;
    LaunchScope ls(c, K_UPDATE, s);
    k_node_cap<T_><<<c->N, 256, 0, s>>>(c->dp, t);
  }

  static void zero_slot(mmf_ctx* c, cudaStream_t s, void* pm, void* pe) {
    LaunchScope ls(c, K_BOUNDARY, s);
    size_t n = (size_t)c->N * c->Lp;
    k_zero<T_><<<grid1d(n, 256), 256, 0, s>>>((M*)pm, (E*)pe, n);
  }

  static void boundary(mmf_ctx* c, cudaStream_t s, int which) {
    const DevPtrs& p = c->dp;
    if (!c->point) {
      LaunchScope ls(c, K_BOUNDARY, s);
      size_t n = (size_t)c->N * c->Lp;
      k_boundary_dense<T_><<<grid1d(n, 256), 256, 0, s>>>(p, which);
    } else {
      if (which == 0) {
        zero_slot(c, s, p.am, p.ae);
        zero_slot(c, s, p.u0m, p.u0e);
      } else {
        zero_slot(c, s, (M*)p.bm + (size_t)c->T * c->N * c->Lp, (E*)p.be + (size_t)c->T * c->N * c->Lp);
      }
      LaunchScope ls(c, K_BOUNDARY, s);
      k_boundary_point<T_><<<(c->L + 127) / 128, 128, 0, s>>>(p, which);
    }
  }

  static void bwd_pass(mmf_ctx* c, cudaStream_t s) {
    dim3 grid(c->N, c->G);
    for (int t = c->T - 1; t >= 0; --t) {
      LaunchScope ls(c, K_BWD, s);
      k_bwd<T_><<<grid, c->block, 0, s>>>(lay(c, t), t);
    }
  }

  // forward step t; readout = 1: flows of all arcs into Fout[t], no dual update
  static mmf_status fwd_step(mmf_ctx* ctx, cudaStream_t s, int t, int readout) {
    mmf_ctx* c = ctx;
    const DevPtrs& p = c->dp;
    dim3 grid(c->N, c->G);
    {
      LaunchScope ls(c, K_FLOW, s);
      k_flow<T_><<<grid, c->block, 0, s>>>(p, t, readout ? 0 : 1);
    }
    const unsigned ga = (unsigned)((c->A + 255) / 256);
    if (readout) {
      M* out = (M*)p.Fout + (size_t)t * c->A;
      {
        LaunchScope ls(c, K_REDUCE, s);
        k_reduce<T_><<<ga, 256, 0, s>>>(p, t, out, 0);
      }
      if (c->comm) {
        int r = nccl_api().AllReduce(out, out, (size_t)c->A, c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64,
                                     NCCL_SUM, c->comm, s);
        if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce failed");
      }
    } else if (c->comm) {
      {
        LaunchScope ls(c, K_REDUCE, s);
        k_reduce<T_><<<ga, 256, 0, s>>>(p, t, (M*)p.Fsum, 1);
      }
      int r = nccl_api().AllReduce(p.Fsum, p.Fsum, (size_t)c->Ecap, c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64,
                                   NCCL_SUM, c->comm, s);
      if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce failed");
      LaunchScope ls(c, K_REDUCE, s);
      k_dual<T_><<<ga, 256, 0, s>>>(p, t, 1);
    } else {
      LaunchScope ls(c, K_REDUCE, s);
      k_reduce<T_><<<ga, 256, 0, s>>>(p, t, nullptr, 2);
    }
    {
      LaunchScope ls(c, K_UPDATE, s);
      k_spmm_fwd<T_><<<grid, c->block, 0, s>>>(lay(c, t + 1, readout != 0), t);
    }
    return MMF_OK;
  }

  static constexpr bool is_f32() { return sizeof(M) == 4; }
  // ---------------- wide-lane path (opt_kernels == 3)
  template <int CPT, int MODE, int FMODE> static void launch_fwd_wide(mmf_ctx* c, cudaStream_t s, int t) {
    dim3 grid((c->N + c->wc.npc - 1) / c->wc.npc, c->wc.ngroup);
    k_fwd_wide<T_, CPT, MODE, FMODE><<<grid, WIDE_THREADS, wide_smem<M>(c->wc.max_oa, c->wc.cpcta), s>>>(lay(c, t, FMODE == 2), c->wc, t);
  }
  template <int CPT> static void wide_fwd_cpt(mmf_ctx* c, cudaStream_t s, int t, int fmode) {
    const int mode = t == 0 ? 0 : (t == c->T ? 2 : 1);
    switch (mode * 3 + fmode) {
      case 0: launch_fwd_wide<CPT, 0, 0>(c, s, t); break;
      case 1: launch_fwd_wide<CPT, 0, 1>(c, s, t); break;
      case 2: launch_fwd_wide<CPT, 0, 2>(c, s, t); break;
      case 3: launch_fwd_wide<CPT, 1, 0>(c, s, t); break;
      case 4: launch_fwd_wide<CPT, 1, 1>(c, s, t); break;
      case 5: launch_fwd_wide<CPT, 1, 2>(c, s, t); break;
      case 6: launch_fwd_wide<CPT, 2, 0>(c, s, t); break;
      case 7: launch_fwd_wide<CPT, 2, 1>(c, s, t); break;
      default: launch_fwd_wide<CPT, 2, 2>(c, s, t); break;
    }
  }
  template <int CPT> static void wide_bwd_cpt(mmf_ctx* c, cudaStream_t s, int t) {
    dim3 grid((c->N + c->wc.npc - 1) / c->wc.npc, c->wc.ngroup);
    k_bwd_wide<T_, CPT><<<grid, WIDE_THREADS, wide_smem<M>(0, 1), s>>>(lay(c, t), c->wc, t);
  }
  // ---------------- head-flow register-gather path (opt_kernels == 4)
  template <int CPT, int MODE, bool KEEP> static void launch_fwd_head(mmf_ctx* c, cudaStream_t s, int t) {
    const HeadCfg& h = c->hc;
    dim3 grid((c->N + h.npc - 1) / h.npc);
    k_fwd_head<T_, CPT, MODE, KEEP><<<grid, h.npc * h.wpn * 32, head_smem<M>(h.max_ia, h.nch), s>>>(lay(c, t, false), h, t);
  }
  template <int CPT> static void head_fwd_cpt(mmf_ctx* c, cudaStream_t s, int t) {
    const int mode = t == 0 ? 0 : (t == c->T ? 2 : 1);
    const bool keep = c->hc.nch <= HF_WARPS;
    switch (mode * 2 + (keep ? 1 : 0)) {
      case 0: launch_fwd_head<CPT, 0, false>(c, s, t); break;
      case 1: launch_fwd_head<CPT, 0, true>(c, s, t); break;
      case 2: launch_fwd_head<CPT, 1, false>(c, s, t); break;
      case 3: launch_fwd_head<CPT, 1, true>(c, s, t); break;
      case 4: launch_fwd_head<CPT, 2, false>(c, s, t); break;
      default: launch_fwd_head<CPT, 2, true>(c, s, t); break;
    }
  }
  static void head_fwd(mmf_ctx* c, cudaStream_t s, int t) {
    LaunchScope ls(c, K_FUSED, s);
    if (c->CPT == 1) head_fwd_cpt<1>(c, s, t);
    else if (c->CPT == 2 || !is_f32()) head_fwd_cpt<2>(c, s, t);
    else if (c->CPT == 4) head_fwd_cpt<is_f32() ? 4 : 2>(c, s, t);
    else head_fwd_cpt<is_f32() ? 8 : 2>(c, s, t);
  }
  template <int CPT> static void head_bwd_cpt(mmf_ctx* c, cudaStream_t s, int t) {
    const size_t warps = (size_t)c->N * c->hc.nch;
    k_bwd_head<T_, CPT><<<(unsigned)((warps + HF_WARPS - 1) / HF_WARPS), HF_WARPS * 32, 0, s>>>(lay(c, t), c->hc, t);
  }
  static void tiled_fwd(mmf_ctx* c, cudaStream_t s, int t, int fmode) {
    LaunchScope ls(c, K_FUSED, s);  // (kernels >= 3: the wide-lane forward)
    if (c->CPT == 1) wide_fwd_cpt<1>(c, s, t, fmode);
    else if (c->CPT == 2 || !is_f32()) wide_fwd_cpt<2>(c, s, t, fmode);
    else if (c->CPT == 4) wide_fwd_cpt<is_f32() ? 4 : 2>(c, s, t, fmode);
    else wide_fwd_cpt<is_f32() ? 8 : 2>(c, s, t, fmode);
  }
  template <int CPT, int GW, int NG, int NP, int MODE> static void pipe_fwd_launch(mmf_ctx* c, cudaStream_t s, int t) {
    const PipeCfg5& pc = c->pf;
    const unsigned grid = (unsigned)std::min((c->N + NP - 1) / NP, c->sms);
    k_fwd_pipe<CPT, GW, NG, NP, MODE>
        <<<grid, fwd_threads<GW, NG, NP>(), NP * pfwd_smem(pc.R, pc.D, pc.SW, NG).total, s>>>(lay(c, t, MODE == 3), pc, t);
  }
  template <int MODE> static void pipe_fwd_mode(mmf_ctx* c, cudaStream_t s, int t) {
    pipe_fwd_mode_launch<MODE>(c, s, t);
    // (the pipelined epilogues skip the layer's node factors: D here, and u in the readout; the sweep's u is
    // applied by k_node_cap)
    if (MODE == 1 || MODE == 3 || MODE == 5) apply_factors(c, s, t, 0, MODE == 3);
  }
  template <int MODE> static void pipe_fwd_mode_launch(mmf_ctx* c, cudaStream_t s, int t) {
    const int SW = c->pf.SW, gw = c->pf_gw, ng = c->pf_ng, np = c->pf_np;
#define MMF_FWD_COMBO(sw, cpt, g, n, q) \
  if (SW == sw && gw == g && ng == n && np == q) return pipe_fwd_launch<cpt, g, n, q, MODE>(c, s, t);
    MMF_FWD_COMBOS(MMF_FWD_COMBO)
#undef MMF_FWD_COMBO
  }
  // node factors of layer t applied to a stored layer (which = 0 alpha_t, 1 beta_t) after a pipelined launch
  static void apply_factors(mmf_ctx* c, cudaStream_t s, int t, int which, bool with_u) {
    if (t < 1 || t > c->T - 1) return;
    const DevPtrs d = lay(c, t, with_u);
    if (!d.dnm && !d.unlm) return;
    LaunchScope ls(c, K_OTHER, s);
    k_apply_factors<T_><<<grid1d((size_t)c->N * c->Lp, 256), 256, 0, s>>>(d, t, which);
  }
  static void pipe_fwd(mmf_ctx* c, cudaStream_t s, int t) {
    Nvtx r(t == 0 ? "a2" : t == c->T ? "a3 + a4 step" : "a3 step");
    if constexpr (sizeof(M) == 4) {
      if (t == 0) {  // a2: elementwise, the head kernel's MODE 0
        head_fwd(c, s, 0);
        return;
      }
      LaunchScope ls(c, K_FUSED, s);
      if (t == c->T) pipe_fwd_mode<2>(c, s, t);
      else pipe_fwd_mode<1>(c, s, t);
    }
  }
  template <int CPT> static void pipe2_bwd_cpt(mmf_ctx* c, cudaStream_t s, int t) {
    const PipeCfg5& pc = c->pb2;
    const size_t share = (pipe_smem(pc.R, FWD_SD, pc.D, pc.SW).total + 127) / 128 * 128;
    const unsigned grid = (unsigned)std::min((pc.nitems + BWD_NP - 1) / BWD_NP, c->sms);
    k_bwd_pipe2<CPT><<<grid, BWD_THREADS, BWD_NP * share, s>>>(lay(c, t), pc, t);
  }
  template <int CPT> static void pipe_bwd_cpt(mmf_ctx* c, cudaStream_t s, int t) {
    const PipeCfg5& pc = c->pb;
    const unsigned grid = (unsigned)std::min(pc.nitems, c->sms);
    k_bwd_pipe<CPT><<<grid, PIPE_THREADS, pipe_smem(pc.R, pc.SD, pc.D, pc.SW).total, s>>>(lay(c, t), pc, t);
  }
  static void tiled_bwd(mmf_ctx* c, cudaStream_t s, int t) {
    Nvtx r("a5 step");
    if (tiled_bwd_launch(c, s, t)) apply_factors(c, s, t, 1, true);  // (pipelined epilogues skip the factors)
  }
  // returns true for the pipelined families (their epilogues leave the layer's node factors out)
  static bool tiled_bwd_launch(mmf_ctx* c, cudaStream_t s, int t) {
    LaunchScope ls(c, K_BWD, s);
    if constexpr (sizeof(M) == 4) {
      if (c->tile_bwd) {
        TileCfg tc = c->tbc;
        tc.tile_ptr = c->tm.tile_ptr;
        tc.hout_ptr = c->tm.hout_ptr;
        tc.hout_node = c->tm.hout_node;
        tc.out_hidx = c->tm.out_hidx;
        tc.desc = c->d_tb_desc;
        tc.meta = c->d_tb_meta;
        const int SW = 32 * c->tb_cpt;
        const unsigned grid = (unsigned)std::min(tc.nitems, c->sms);
        const size_t sm = tb_smem(tc.nst, tc.H, SW, tc.MA, tc.MB);
        if (c->tb_cpt == 8) k_bwd_tile2<8><<<grid, TB_THREADS, sm, s>>>(lay(c, t), tc, t);
        else k_bwd_tile2<4><<<grid, TB_THREADS, sm, s>>>(lay(c, t), tc, t);
        return true;
      }
      if (c->win_bwd) {
        const WinCfg& w = c->wcb;
        const unsigned grid = (unsigned)(w.ns * w.nseg);
        const int tma = c->win_tma ? 1 : 0;
        if (c->win_cpt == 4)
          k_bwd_win<4><<<grid, WIN_THREADS, win_smem<4>(w).total, s>>>(lay(c, t), w, c->wdo, c->tmb, tma, t);
        else if (c->win_cpt == 2)
          k_bwd_win<2><<<grid, WIN_THREADS, win_smem<2>(w).total, s>>>(lay(c, t), w, c->wdo, c->tmb, tma, t);
        else
          k_bwd_win<1><<<grid, WIN_THREADS, win_smem<1>(w).total, s>>>(lay(c, t), w, c->wdo, c->tmb, tma, t);
        return true;
      }
      if (c->pipe2_bwd) {
        const int cp = c->pb2.SW / 256;
        if (cp == 4) pipe2_bwd_cpt<4>(c, s, t);
        else if (cp == 2) pipe2_bwd_cpt<2>(c, s, t);
        else pipe2_bwd_cpt<1>(c, s, t);
        return true;
      }
      if (c->pipe_bwd) {
        const int cp = c->pb.SW / 256;
        if (cp == 4) pipe_bwd_cpt<4>(c, s, t);
        else if (cp == 2) pipe_bwd_cpt<2>(c, s, t);
        else pipe_bwd_cpt<1>(c, s, t);
        return true;
      }
    }
    if (c->opt_kernels >= 4) {
      if (c->CPT == 1) head_bwd_cpt<1>(c, s, t);
      else if (c->CPT == 2 || !is_f32()) head_bwd_cpt<2>(c, s, t);
      else if (c->CPT == 4) head_bwd_cpt<is_f32() ? 4 : 2>(c, s, t);
      else head_bwd_cpt<is_f32() ? 8 : 2>(c, s, t);
      return false;
    }
    if (c->CPT == 1) wide_bwd_cpt<1>(c, s, t);  // (kernels == 3)
    else if (c->CPT == 2 || !is_f32()) wide_bwd_cpt<2>(c, s, t);
    else if (c->CPT == 4) wide_bwd_cpt<is_f32() ? 4 : 2>(c, s, t);
    else wide_bwd_cpt<is_f32() ? 8 : 2>(c, s, t);
    return false;
  }
  // node-tile forward launch t (alpha_t, flow partials of step t or a4) and, t < T, the dual update of step t
  static void tile_fwd_step(mmf_ctx* c, cudaStream_t s, int t) {
    if constexpr (sizeof(M) == 4) {
      TileCfgF tc = c->tfc;
      tc.desc = c->d_tf_desc;
      tc.meta = c->d_tf_meta;
      tc.hin_node = c->tm.hin_node;
      tc.hout_node = c->tm.hout_node;
      tc.part = c->d_tf_part;
      {
        LaunchScope ls(c, K_FUSED, s);
        const unsigned grid = (unsigned)std::min(tc.nitems, c->sms);
        k_fwd_tile2<4><<<grid, TB_THREADS, tf_smem(tc.nst, tc.Hin, tc.Hout, 128, tc.MAi, tc.MAo, tc.MM), s>>>(
            lay(c, t), tc, t);
      }
      if (t < c->T) {
        LaunchScope ls(c, K_UPDATE, s);
        k_tile_dual<<<(unsigned)((c->A + 255) / 256), 256, 0, s>>>(c->dp, tc.part, tc.nch, t);
      }
    }
  }
  // the multi-GPU exchange of one forward step: all-reduce the rank-partial F_t, then W_t update
  // the exchange path runs on the pipelined kernels (fp32, one slice per node) unless option pexch = 0
  static bool pipe_exchange(const mmf_ctx* c) {
    return sizeof(M) == 4 && c->opt_kernels >= 5 && c->pipe_fwd && c->comm && pexch_on(c);
  }
  static bool pexch_on(const mmf_ctx* c) { return c->opt_pexch > 0 || (c->opt_pexch < 0 && c->pf.SW >= 1024); }
  static mmf_status exchange(mmf_ctx* c, cudaStream_t s, int t) {
    const DevPtrs& p = c->dp;
    int r = nccl_api().AllReduce(p.Fsum, p.Fsum, (size_t)c->Ecap, c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64,
                                 NCCL_SUM, c->comm, s);  // (capacitated arcs only, SURVEY 8(e) mitigation 2)
    if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce failed");
    LaunchScope ls(c, K_REDUCE, s);
    k_dual<T_><<<(unsigned)((c->A + 255) / 256), 256, 0, s>>>(p, t, 1);
    return MMF_OK;
  }

  // virtual ranks: G contexts on one device, each one commodity shard, swept together with the
  // multi-GPU exchange path's kernels (partial flows of the shard -> sum -> dual update) and a device-side sum in
  // place of ncclAllReduce (fixed shard order)
  static mmf_status group_sweep(mmf_ctx* const* cs, int G, cudaStream_t s) {
    mmf_ctx* c0 = cs[0];
    VSum vs{};
    for (int g = 0; g < G; ++g) vs.f[g] = cs[g]->dp.Fsum;
    const unsigned ga = (unsigned)((c0->A + 255) / 256);
    bool pipe = true;
    for (int g = 0; g < G; ++g) pipe = pipe && sizeof(M) == 4 && cs[g]->opt_kernels >= 5 && cs[g]->pipe_fwd && pexch_on(cs[g]);
    if (pipe) {  // the pipelined exchange path (as pipe_exchange): MODE 4 partials, device sum, dual, MODE 5 / 6
      for (int g = 0; g < G; ++g) pipe_fwd(cs[g], s, 0);  // a2
      for (int t = 1; t <= c0->T; ++t) {
        for (int g = 0; g < G; ++g) {
          LaunchScope ls(cs[g], K_FUSED, s);
          pipe_fwd_mode<4>(cs[g], s, t);
        }
        {
          LaunchScope ls(c0, K_REDUCE, s);
          k_vsum<M><<<ga, 256, 0, s>>>(vs, G, c0->Ecap);
        }
        for (int g = 0; g < G; ++g) {
          LaunchScope ls(cs[g], K_REDUCE, s);
          k_dual<T_><<<ga, 256, 0, s>>>(cs[g]->dp, t - 1, 1);
        }
        for (int g = 0; g < G; ++g) {
          LaunchScope ls(cs[g], K_FUSED, s);
          if (t == c0->T) pipe_fwd_mode<6>(cs[g], s, t);
          else pipe_fwd_mode<5>(cs[g], s, t);
        }
      }
      for (int g = 0; g < G; ++g)
        for (int t = c0->T - 1; t >= 0; --t) tiled_bwd(cs[g], s, t);  // a5
      return MMF_OK;
    }
    for (int t = 0; t <= c0->T; ++t) {
      for (int g = 0; g < G; ++g) tiled_fwd(cs[g], s, t, 1);  // alpha_t of the shard; its partial F_t -> Fsum
      if (t < c0->T) {
        {
          LaunchScope ls(c0, K_REDUCE, s);
          k_vsum<M><<<ga, 256, 0, s>>>(vs, G, c0->Ecap);
        }
        for (int g = 0; g < G; ++g) {
          LaunchScope ls(cs[g], K_REDUCE, s);
          k_dual<T_><<<ga, 256, 0, s>>>(cs[g]->dp, t, 1);
        }
      }
    }
    for (int g = 0; g < G; ++g)
      for (int t = c0->T - 1; t >= 0; --t) tiled_bwd(cs[g], s, t);  // a5
    return MMF_OK;
  }

  static mmf_status enqueue_sweep(mmf_ctx* c, cudaStream_t s) {
    Nvtx r("mmf sweep");
    if (c->opt_schedule == 1) return jacobi_sweep(c, s);
    if (c->opt_schedule == 2) return symmetric_sweep(c, s);
    return gs_sweep(c, s, true);
  }

  // Algorithm 2's sweep (a2, forward with the W updates, a4, and the backward pass a5 when do_bwd)
  static mmf_status gs_sweep(mmf_ctx* c, cudaStream_t s, bool do_bwd) {
    if (c->tile_fwd && !c->comm) {  // node-tile forward: launch t = alpha_t + flow partials of step t, then its dual
      {
        Nvtx r("forward pass (a2, a3 on node tiles, a4)");
        tiled_fwd(c, s, 0, 0);  // a2 + flows + dual update of step 0 (wide-lane launch)
        for (int t = 1; t <= c->T; ++t) {
          tile_fwd_step(c, s, t);
          node_cap(c, s, t);
        }
      }
      if (do_bwd) {
        Nvtx r("backward pass (a5)");
        for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
      }
      return MMF_OK;
    }
    if (c->opt_kernels >= 5 && c->pipe_fwd && !c->comm) {
      {
        Nvtx r("forward pass (a2, a3, a4)");
        for (int t = 0; t <= c->T; ++t) {
          pipe_fwd(c, s, t);  // a2 in t = 0; a3 (W_{t-1}, alpha_t); a4 in t = T
          node_cap(c, s, t);  // (node capacities: u_t, P:1093 on the states)
        }
      }
      if (do_bwd) {
        Nvtx r("backward pass (a5)");
        for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
      }
      return MMF_OK;
    }
    if (pipe_exchange(c)) {  // multi-GPU Gauss-Seidel on the pipelined kernels: each step split around the exchange
      {
        Nvtx r("forward pass (a2, a3 + exchange, a4)");
        pipe_fwd(c, s, 0);  // a2
        for (int t = 1; t <= c->T; ++t) {
          {
            LaunchScope ls(c, K_FUSED, s);
            pipe_fwd_mode<4>(c, s, t);  // rank-partial F_{t-1} -> Fsum
          }
          mmf_status st = exchange(c, s, t - 1);  // all-reduce, W_{t-1} update
          if (st != MMF_OK) return st;
          LaunchScope ls(c, K_FUSED, s);
          if (t == c->T) pipe_fwd_mode<6>(c, s, t);  // alpha_T, a4
          else pipe_fwd_mode<5>(c, s, t);  // alpha_t with the updated W_{t-1}
        }
      }
      if (do_bwd) {
        Nvtx r("backward pass (a5)");
        for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
      }
      return MMF_OK;
    }
    if (c->opt_kernels == 4 && !c->comm) {
      for (int t = 0; t <= c->T; ++t) head_fwd(c, s, t);       // a2 in t = 0; a3 (W_{t-1}, alpha_t); a4 in t = T
      if (do_bwd)
        for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
      return MMF_OK;
    }
    if (c->opt_kernels >= 2) {
      const int fmode = c->comm ? 1 : 0;
      for (int t = 0; t <= c->T; ++t) {  // a2 fused in t = 0, a4 fused in t = T
        tiled_fwd(c, s, t, fmode);
        if (c->comm && t < c->T) {
          mmf_status st = exchange(c, s, t);
          if (st != MMF_OK) return st;
        }
      }
      if (do_bwd)
        for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
      return MMF_OK;
    }
    boundary(c, s, 0);  // a2
    for (int t = 0; t < c->T; ++t) {
      mmf_status st = fwd_step(c, s, t, 0);  // a3
      if (st != MMF_OK) return st;
      node_cap(c, s, t + 1);
    }
    boundary(c, s, 1);  // a4
    if (do_bwd) bwd_pass(c, s);  // a5
    return MMF_OK;
  }

  // symmetric Gauss-Seidel (option schedule = 2): Algorithm 2's forward pass, then a backward
  // pass that updates W_t again before forming beta_t: per step the flows F_t of the current tensor (alpha_t kept
  // from the forward pass: the alpha store has T + 1 slots; beta_{t+1} fresh), the dual update of W_t (all-reduced
  // flows on the multi-GPU path), the backward step
  static mmf_status symmetric_sweep(mmf_ctx* c, cudaStream_t s) {
    mmf_status st = gs_sweep(c, s, false);
    Nvtx r("symmetric backward pass");
    if (st != MMF_OK) return st;
    const bool pipe = sizeof(M) == 4 && c->opt_kernels >= 5 && c->pipe_fwd && !c->comm;
    const unsigned ga = (unsigned)((c->A + 255) / 256);
    for (int t = c->T - 1; t >= 0; --t) {
      // flows of step t into Fout[t] (the readout launches; the alpha they rewrite is unchanged: W_{<=t} are as the
      // forward pass left them)
      if (pipe) {
        LaunchScope ls(c, K_FUSED, s);
        pipe_fwd_mode<3>(c, s, t + 1);
      } else if (c->opt_kernels >= 2) {
        tiled_fwd(c, s, t, 2);
      } else {
        st = fwd_step(c, s, t, 1);
        if (st != MMF_OK) return st;
      }
      M* Ft = (M*)c->dp.Fout + (size_t)t * c->A;
      if (c->comm && (pipe || c->opt_kernels >= 2)) {  // (fwd_step all-reduced already)
        int r = nccl_api().AllReduce(Ft, Ft, (size_t)c->A, c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64, NCCL_SUM,
                                     c->comm, s);
        if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce failed");
      }
      {
        DevPtrs d = c->dp;
        d.Fsum = Ft;
        LaunchScope ls(c, K_UPDATE, s);
        k_dual<T_><<<ga, 256, 0, s>>>(d, t, 0);
      }
      if (c->opt_kernels >= 2) {
        tiled_bwd(c, s, t);
      } else {
        LaunchScope ls(c, K_BWD, s);
        k_bwd<T_><<<dim3(c->N, c->G), c->block, 0, s>>>(lay(c, t), t);
      }
    }
    return MMF_OK;
  }

  static mmf_status init_device(mmf_ctx* ctx, cudaStream_t s) {
    mmf_ctx* c = ctx;
    const DevPtrs& p = c->dp;
    if constexpr (sizeof(M) == 4) {
      if (c->tile_fwd) {
        const int sm = (int)tf_smem(c->tfc.nst, c->tfc.Hin, c->tfc.Hout, 128, c->tfc.MAi, c->tfc.MAo, c->tfc.MM);
        CU(cudaFuncSetAttribute(k_fwd_tile2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        if (getenv("MMF_VERBOSE"))
          fprintf(stderr, "[mmf] tile fwd: stages %d Hin %d Hout %d items %d smem %d\n", c->tfc.nst, c->tfc.Hin,
                  c->tfc.Hout, c->tfc.nitems, sm);
      }
      if (c->tile_bwd) {
        const int sm = (int)tb_smem(c->tbc.nst, c->tbc.H, 32 * c->tb_cpt, c->tbc.MA, c->tbc.MB);
        CU(cudaFuncSetAttribute(k_bwd_tile2<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CU(cudaFuncSetAttribute(k_bwd_tile2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        if (getenv("MMF_VERBOSE"))
          fprintf(stderr, "[mmf] tile bwd: cpt %d stages %d H %d tiles %d items %d smem %d\n", c->tb_cpt, c->tbc.nst,
                  c->tbc.H, c->ntiles, c->tbc.nitems, sm);
      }
      if (c->pipe_bwd) {
        const int sm = (int)pipe_smem(c->pb.R, c->pb.SD, c->pb.D, c->pb.SW).total;
        CU(cudaFuncSetAttribute(k_bwd_pipe<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CU(cudaFuncSetAttribute(k_bwd_pipe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CU(cudaFuncSetAttribute(k_bwd_pipe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      }
      if (c->win_bwd) {
        if (c->win_cpt == 4)
          CU(cudaFuncSetAttribute(k_bwd_win<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem<4>(c->wcb).total));
        else if (c->win_cpt == 2)
          CU(cudaFuncSetAttribute(k_bwd_win<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem<2>(c->wcb).total));
        else
          CU(cudaFuncSetAttribute(k_bwd_win<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)win_smem<1>(c->wcb).total));
        c->win_tma = c->opt_wintma && c->win_cpt >= 2 && make_tmaps(c, c->dp.bm, c->dp.be, c->T + 1, 32 * c->win_cpt, c->tmb);
        if (getenv("MMF_VERBOSE"))
          fprintf(stderr, "[mmf] window tma %d\n", (int)c->win_tma);
        if (getenv("MMF_VERBOSE"))
          fprintf(stderr, "[mmf] window bwd: cpt %d Wb %d RBa %d ns %d nseg %d segB %d farmax %d maxrec %d smem %zu\n",
                  c->win_cpt, c->wcb.Wb, c->wcb.RBa, c->wcb.ns, c->wcb.nseg, c->wcb.segB, c->wcb.farmax,
                  c->wcb.maxrec, c->win_cpt == 4 ? win_smem<4>(c->wcb).total : c->win_cpt == 2 ? win_smem<2>(c->wcb).total : win_smem<1>(c->wcb).total);
      }
      if (c->pipe2_bwd) {
        const int sm = BWD_NP * (int)((pipe_smem(c->pb2.R, FWD_SD, c->pb2.D, c->pb2.SW).total + 127) / 128 * 128);
        CU(cudaFuncSetAttribute(k_bwd_pipe2<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CU(cudaFuncSetAttribute(k_bwd_pipe2<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
        CU(cudaFuncSetAttribute(k_bwd_pipe2<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm));
      }
      if (c->pipe_fwd) {
        const int sm = c->pf_np * (int)pfwd_smem(c->pf.R, c->pf.D, c->pf.SW, c->pf_ng).total;
        const int SW = c->pf.SW, gw = c->pf_gw, ng = c->pf_ng, np = c->pf_np;
#define MMF_FWD_COMBO(sw, cpt, g, n, q)                                                                    \
  if (SW == sw && gw == g && ng == n && np == q) {                                                         \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
    CU(cudaFuncSetAttribute(k_fwd_pipe<cpt, g, n, q, 6>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm)); \
  }
        MMF_FWD_COMBOS(MMF_FWD_COMBO)
#undef MMF_FWD_COMBO
        if (getenv("MMF_VERBOSE"))
          fprintf(stderr, "[mmf] pipe fwd: SW %d GW %d NG %d NP %d R %d D %d smem %d\n", SW, gw, ng, np, c->pf.R, c->pf.D, sm);
      }
    }
    {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->T * c->A;
      k_init_w<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    }
    // U0 = 0 until the first a2 (the oracle's lam0 = -inf): a readout before any sweep sees the zero tensor
    zero_slot(c, s, p.u0m, p.u0e);
    if (p.inrec) {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->T * c->A;
      k_init_recs<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    }
    if (!c->point) {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->N * c->Lp;
      k_init_ut_dense<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    } else {
      zero_slot(c, s, (M*)p.bm + (size_t)c->T * c->N * c->Lp, (E*)p.be + (size_t)c->T * c->N * c->Lp);
      LaunchScope ls(c, K_OTHER, s);
      k_init_ut_point<T_><<<(c->L + 127) / 128, 128, 0, s>>>(p);
    }
    if (c->opt_kernels >= 2)
      for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);
    else
      bwd_pass(c, s);
    return MMF_OK;
  }

  // after a state load (W and UT written): records from W, then the backward pass (as mmf_init does with W = 1)
  static mmf_status restore(mmf_ctx* ctx, cudaStream_t s) {
    mmf_ctx* c = ctx;
    const DevPtrs& p = c->dp;
    if (p.inrec) {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->T * c->A;
      k_init_recs<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    }
    if (c->opt_kernels >= 2)
      for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);
    else
      bwd_pass(c, s);
    return MMF_OK;
  }

  static mmf_status readout(mmf_ctx* ctx, cudaStream_t s) { return forward_flows(ctx, s, true); }

  // Jacobi sweep: a2, one forward pass with the previous W (alpha_t and the flows F_t of
  // every step, this rank's commodities), a4, ONE exchange of the T x |A| flows, all W_t, the backward pass
  static mmf_status jacobi_sweep(mmf_ctx* c, cudaStream_t s) {
    boundary(c, s, 0);  // a2
    mmf_status st = forward_flows(c, s, false);
    if (st != MMF_OK) return st;
    boundary(c, s, 1);  // a4
    if (c->comm) {
      int r = nccl_api().AllReduce(c->dp.Fout, c->dp.Fout, (size_t)c->T * c->A,
                                   c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64, NCCL_SUM, c->comm, s);
      if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce(flows) failed");
    }
    {
      LaunchScope ls(c, K_UPDATE, s);
      size_t n = (size_t)c->T * c->A;
      k_jacobi_update<T_><<<grid1d(n, 256), 256, 0, s>>>(c->dp);
    }
    if (c->opt_kernels >= 2)
      for (int t = c->T - 1; t >= 0; --t) tiled_bwd(c, s, t);  // a5
    else
      bwd_pass(c, s);
    return MMF_OK;
  }

  // forward pass with the current factors (no dual update): alpha_t of the current state and the flows of every
  // step into Fout (exchanged per step over the ranks if asked)
  static mmf_status forward_flows(mmf_ctx* ctx, cudaStream_t s, bool exchange_each) {
    Nvtx r("readout forward pass");
    mmf_ctx* c = ctx;
    const DevPtrs& p = c->dp;
    if (c->opt_kernels >= 2) {
      // (the pipelined forward in readout mode where it applies; its launch t yields the flows of step t - 1, so
      // with a per-step exchange the wide-lane kernels are used)
      const bool pipe = sizeof(M) == 4 && c->opt_kernels >= 5 && c->pipe_fwd && !(c->comm && exchange_each) &&
                        !MMF_FWD_DEDUP;
      for (int t = 0; t <= c->T; ++t) {
        if (pipe && t > 0) {
          LaunchScope ls(c, K_FUSED, s);
          pipe_fwd_mode<3>(c, s, t);  // (MODE 3: flows of every arc into Fout, no dual update)
        } else {
          tiled_fwd(c, s, t, 2);
        }
        if (c->comm && exchange_each && t < c->T) {
          M* out = (M*)p.Fout + (size_t)t * c->A;
          int r = nccl_api().AllReduce(out, out, (size_t)c->A, c->prec == MMF_FP32 ? NCCL_FLOAT32 : NCCL_FLOAT64,
                                       NCCL_SUM, c->comm, s);
          if (r != 0) return fail(c, MMF_ENCCL, "ncclAllReduce failed");
        }
      }
      return MMF_OK;
    }
    const size_t n = (size_t)c->N * c->Lp;
    CU(cudaMemcpyAsync(p.am, p.u0m, n * sizeof(M), cudaMemcpyDeviceToDevice, s));
    CU(cudaMemcpyAsync(p.ae, p.u0e, n * sizeof(E), cudaMemcpyDeviceToDevice, s));
    for (int t = 0; t < c->T; ++t) {
      mmf_status st = fwd_step(c, s, t, 1);
      if (st != MMF_OK) return st;
    }
    return MMF_OK;
  }

  // forward messages of the end-of-sweep tensor up to step t (the readout pass's launches 0..t), then the
  // per-commodity flows of step t into d_out ([n_arcs][L] user arc order)
  static mmf_status commodity_flows(mmf_ctx* ctx, cudaStream_t s, int t, double* d_out) {
    mmf_ctx* c = ctx;
    if (c->opt_kernels >= 2) {
      for (int k = 0; k <= t; ++k) tiled_fwd(c, s, k, 2);
    } else {
      const size_t n = (size_t)c->N * c->Lp;
      CU(cudaMemcpyAsync(c->dp.am, c->dp.u0m, n * sizeof(M), cudaMemcpyDeviceToDevice, s));
      CU(cudaMemcpyAsync(c->dp.ae, c->dp.u0e, n * sizeof(E), cudaMemcpyDeviceToDevice, s));
      for (int k = 0; k < t; ++k) {
        mmf_status st = fwd_step(c, s, k, 1);
        if (st != MMF_OK) return st;
      }
    }
    LaunchScope ls(c, K_OTHER, s);
    const int64_t n = (int64_t)c->A * c->L;
    const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 8 * 148);
    k_commodity_flows<T_><<<grid, 256, 0, s>>>(c->dp, c->d_int_of_arc, t, d_out);
    return MMF_OK;
  }
  static mmf_status excess(mmf_ctx* ctx, cudaStream_t s) {
    LaunchScope ls(ctx, K_OTHER, s);
    size_t n = (size_t)ctx->T * ctx->A;
    k_stats_excess<T_><<<grid1d(n, 256), 256, 0, s>>>(ctx->dp);
    return MMF_OK;
  }
  static mmf_status stats(mmf_ctx* ctx, cudaStream_t s) {
    mmf_ctx* c = ctx;
    const DevPtrs& p = c->dp;
    CU(cudaMemsetAsync(p.stats, 0, 8 * sizeof(double), s));
    {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->N * c->Lp;
      k_stats_nodes<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    }
    {
      LaunchScope ls(c, K_OTHER, s);
      size_t n = (size_t)c->T * c->A;
      k_stats_arcs<T_><<<grid1d(n, 256), 256, 0, s>>>(p);
    }
    return MMF_OK;
  }
};

template <class F> mmf_status dispatch(mmf_ctx* c, F f) {
  if (c->prec == MMF_FP32) return f(Eng<TrF32>());
  return f(Eng<TrF64>());
}

mmf_status check_sticky(mmf_ctx* ctx) {
  mmf_ctx* c = ctx;
  unsigned err = 0;
  unsigned long long loc = 0;
  CU(cudaMemcpy(&err, c->dp.err, sizeof(err), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&loc, c->dp.errloc, sizeof(loc), cudaMemcpyDeviceToHost));
  if (err) {
    int commodity = (int)((loc >> 32) & 0x7fffffffull);
    int node_int = (int)(loc & 0xffffffffull);
    int node_user = node_int;
    if (node_int >= 0 && node_int < c->N && (err & (ERR_INFEASIBLE | ERR_RANGE)))
      for (int v = 0; v < c->N; ++v)
        if (c->newid[v] == node_int) {
          node_user = v;
          break;
        }
    char buf[256];
    if (err & ERR_INFEASIBLE) {
      snprintf(buf, sizeof buf, "infeasible boundary scaling (x/0, x>0): commodity %d, node %d",
               commodity + c->l_begin, node_user);
      return fail(c, MMF_EINFEASIBLE, buf);
    }
    if (err & ERR_RANGE) {
      snprintf(buf, sizeof buf, "extended exponent overflow: commodity %d, node %d", commodity + c->l_begin, node_user);
      return fail(c, MMF_ERANGE, buf);
    }
    snprintf(buf, sizeof buf, "NaN/inf edge flow (internal arc %d)", node_int);
    return fail(c, MMF_ERANGE, buf);
  }
  if (c->comm) {
    ncclResult_t_ r = 0;
    nccl_api().CommGetAsyncError(c->comm, &r);
    if (r != 0) return fail(c, MMF_ENCCL, "NCCL async error");
  }
  return MMF_OK;
}

mmf_status collect_profile(mmf_ctx* ctx) {
  mmf_ctx* c = ctx;
  for (auto& pr : c->prof) {
    float ms = 0;
    CU(cudaEventElapsedTime(&ms, pr.a, pr.b));
    c->ms[pr.kind] += ms;
    c->ev_pool.push_back(pr.a);
    c->ev_pool.push_back(pr.b);
  }
  c->prof.clear();
  return MMF_OK;
}

// build internal structures and upload (called by mmf_init)
mmf_status finalize(mmf_ctx* ctx) {
  HostTimer ht("finalize");
  mmf_ctx* c = ctx;
  const int N = c->N;
  const int64_t A = c->A;
  prepare(c);

  derive_shapes(c);
  size_t need = layout(c, nullptr);
  if (!c->ws) {
    void* d = nullptr;
    if (cudaMalloc(&d, need) != cudaSuccess) return fail(c, MMF_ENOMEM, "cudaMalloc of the workspace failed");
    c->ws = d;
    c->ws_bytes = need;
    c->ws_owned = true;
  } else if (c->ws_bytes < need) {
    return fail(c, MMF_ENOMEM, "workspace smaller than mmf_workspace_bytes");
  }
  layout(c, (char*)c->ws);
  DevPtrs& p = c->dp;
  cudaStream_t s = c->stream;

  CU(cudaMemcpyAsync((void*)p.tail, c->h_tail.data(), A * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.in_ptr, c->h_inptr.data(), (N + 1) * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.out_ptr, c->h_outptr.data(), (N + 1) * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.out_arc, c->h_outarc.data(), A * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.out_head, c->h_outhead.data(), A * 4, cudaMemcpyHostToDevice, s));
  {
    std::vector<int> opos(A);
    for (int64_t k = 0; k < A; ++k) opos[c->h_outarc[k]] = (int)k;
    CU(cudaMemcpyAsync((void*)p.opos, opos.data(), A * 4, cudaMemcpyHostToDevice, s));
    if (c->win_bwd) {
      CU(cudaMemcpyAsync((void*)c->wdo.src, c->h_wsrc_out.data(), A * 4, cudaMemcpyHostToDevice, s));
      CU(cudaMemcpyAsync((void*)c->wdo.fptr, c->h_wfptr_out.data(), c->h_wfptr_out.size() * 4, cudaMemcpyHostToDevice, s));
      if (!c->h_wfnode_out.empty())
        CU(cudaMemcpyAsync((void*)c->wdo.fnode, c->h_wfnode_out.data(), c->h_wfnode_out.size() * 4,
                           cudaMemcpyHostToDevice, s));
    }
    std::vector<int> eip, eop;
    if (p.ell_in) {
      eip.resize(A);
      eop.resize(A);
      for (int64_t k = 0; k < A; ++k) {
        const int hd = c->h_head[k], tl = c->h_tail[k];
        eip[k] = hd * p.Din + (int)(k - c->h_inptr[hd]);
        eop[k] = tl * p.Dout + (opos[k] - c->h_outptr[tl]);
      }
      CU(cudaMemcpyAsync((void*)p.ell_ipos, eip.data(), A * 4, cudaMemcpyHostToDevice, s));
      CU(cudaMemcpyAsync((void*)p.ell_opos, eop.data(), A * 4, cudaMemcpyHostToDevice, s));
      // unused ELL slots: node = -1, km = NaN (never > 0)
      CU(cudaMemsetAsync(p.ell_in, 0xff, (size_t)c->T * N * p.Din * 16, s));
      CU(cudaMemsetAsync(p.ell_out, 0xff, (size_t)c->T * N * p.Dout * 16, s));
    }
    CU(cudaStreamSynchronize(s));
  }
  {
    const TileMeta& tm = c->tm;
    const size_t nt = (size_t)c->ntiles;
    CU(cudaMemcpyAsync((void*)tm.tile_ptr, c->h_tile_ptr.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)tm.hin_ptr, c->h_hin_ptr.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)tm.hout_ptr, c->h_hout_ptr.data(), (nt + 1) * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_hin_node.empty())
      CU(cudaMemcpyAsync((void*)tm.hin_node, c->h_hin_node.data(), c->h_hin_node.size() * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_hout_node.empty())
      CU(cudaMemcpyAsync((void*)tm.hout_node, c->h_hout_node.data(), c->h_hout_node.size() * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)tm.in_hidx, c->h_in_hidx.data(), A * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)tm.out_hidx, c->h_out_hidx.data(), A * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_tb_desc.empty())
      CU(cudaMemcpyAsync((void*)c->d_tb_desc, c->h_tb_desc.data(), c->h_tb_desc.size() * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_tb_meta.empty())
      CU(cudaMemcpyAsync((void*)c->d_tb_meta, c->h_tb_meta.data(), c->h_tb_meta.size() * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_tf_desc.empty())
      CU(cudaMemcpyAsync((void*)c->d_tf_desc, c->h_tf_desc.data(), c->h_tf_desc.size() * 4, cudaMemcpyHostToDevice, s));
    if (!c->h_tf_meta.empty())
      CU(cudaMemcpyAsync((void*)c->d_tf_meta, c->h_tf_meta.data(), c->h_tf_meta.size() * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemsetAsync(tm.cnt, 0, nt * 4, s));
    CU(cudaMemsetAsync(c->wc.cnt, 0, ((size_t)c->N + 1) * 4, s));
  }

  const bool f32 = c->prec == MMF_FP32;
  const size_t sm = c->sm(), se = c->se();
  // K = exp(-C/eps) (fp64 on host), capacities
  const int TK = c->cost_tv ? c->T : 1, TC = c->cap_tv ? c->T : 1;
  std::vector<char> hKm((size_t)TK * A * sm), hdc((size_t)TC * A * sm);
  std::vector<int> hKe((size_t)TK * A);
  for (int t = 0; t < TK; ++t)
    for (int64_t a = 0; a < A; ++a) {
      double m = 0.0;
      int e = 0;
      const double ca = c->cost[(size_t)t * A + a];
      if (std::isfinite(ca)) k_to_xf(-ca / c->eps, m, e);  // (+inf: an arc absent at this step, K = 0)
      size_t k = (size_t)t * A + c->int_of_arc[a];
      if (f32)
        ((float*)hKm.data())[k] = (float)m;
      else
        ((double*)hKm.data())[k] = m;
      hKe[k] = e;
    }
  for (int t = 0; t < TC; ++t)
    for (int64_t a = 0; a < A; ++a) {
      double d = c->cap[(size_t)t * A + a];
      size_t k = (size_t)t * A + c->int_of_arc[a];
      if (f32)
        ((float*)hdc.data())[k] = (float)d;
      else
        ((double*)hdc.data())[k] = d;
    }
  CU(cudaMemcpyAsync((void*)p.Km, hKm.data(), hKm.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.Ke, hKe.data(), hKe.size() * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.dcap, hdc.data(), hdc.size(), cudaMemcpyHostToDevice, s));
  CU(cudaMemcpyAsync((void*)p.fpos, c->h_fpos.data(), (size_t)A * 4, cudaMemcpyHostToDevice, s));
  CU(cudaMemsetAsync(p.Fsum, 0, (size_t)std::max<int64_t>(c->Ecap, 1) * sm, s));

  // marginals
  std::vector<char> h0, h0e, hT, hTe;
  std::vector<int> hs, hd;
  if (!c->point) {
    const size_t n = (size_t)N * c->Lp;
    h0.assign(n * sm, 0);
    hT.assign(n * sm, 0);
    h0e.assign(n * se, 0);
    hTe.assign(n * se, 0);
    for (int l = 0; l < c->Lp; ++l)
      for (int v = 0; v < N; ++v) {
        size_t k = (size_t)c->newid[v] * c->Lp + l;
        double m0 = 0, mT = 0;
        int e0 = EZERO, eT = EZERO;
        if (l < c->L) {
          to_xf(c->mu0[(size_t)l * N + v], m0, e0);
          to_xf(c->muT[(size_t)l * N + v], mT, eT);
        }
        if (f32) {
          ((float*)h0.data())[k] = (float)m0;
          ((float*)hT.data())[k] = (float)mT;
          ((int16_t*)h0e.data())[k] = (int16_t)e0;
          ((int16_t*)hTe.data())[k] = (int16_t)eT;
        } else {
          ((double*)h0.data())[k] = m0;
          ((double*)hT.data())[k] = mT;
          ((int32_t*)h0e.data())[k] = e0;
          ((int32_t*)hTe.data())[k] = eT;
        }
      }
    CU(cudaMemcpyAsync((void*)p.mu0m, h0.data(), h0.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.mu0e, h0e.data(), h0e.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.muTm, hT.data(), hT.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.muTe, hTe.data(), hTe.size(), cudaMemcpyHostToDevice, s));
  } else {
    hs.resize(c->L);
    hd.resize(c->L);
    for (int l = 0; l < c->L; ++l) {
      hs[l] = c->newid[c->src[l]];
      hd[l] = c->newid[c->dst[l]];
    }
    CU(cudaMemcpyAsync((void*)p.psrc, hs.data(), c->L * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.pdst, hd.data(), c->L * 4, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.pmass, c->mass.data(), c->L * 8, cudaMemcpyHostToDevice, s));
  }
  // commodity node factors D[l, j] = exp(-c[l, j] / eps) (NEXT-2), formed in fp64 like K, [N][Lp] internal order;
  // padded commodities carry D = 1
  std::vector<char> hDm, hDe;
  if (!c->node_cost.empty()) {
    const size_t n = (size_t)N * c->Lp;
    hDm.assign(n * sm, 0);
    hDe.assign(n * se, 0);
    for (int v = 0; v < N; ++v)
      for (int l = 0; l < c->Lp; ++l) {
        double m = 1.0;
        int e = 0;
        if (l < c->L) k_to_xf(-c->node_cost[(size_t)l * N + v] / c->eps, m, e);
        const size_t k = (size_t)c->newid[v] * c->Lp + l;
        if (f32) {
          ((float*)hDm.data())[k] = (float)m;
          ((int16_t*)hDe.data())[k] = (int16_t)e;
        } else {
          ((double*)hDm.data())[k] = m;
          ((int32_t*)hDe.data())[k] = e;
        }
      }
    CU(cudaMemcpyAsync((void*)p.dnm, hDm.data(), hDm.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync((void*)p.dne, hDe.data(), hDe.size(), cudaMemcpyHostToDevice, s));
  }
  std::vector<char> hdn;
  if (p.dnc) {  // node capacities (internal node order); u = 1
    const int TN = c->node_cap_tv ? c->T + 1 : 1;
    hdn.assign((size_t)TN * N * sm, 0);
    for (int t = 0; t < TN; ++t)
      for (int v = 0; v < N; ++v) {
        const double d = c->node_cap[(size_t)t * N + v];
        const size_t k = (size_t)t * N + c->newid[v];
        if (f32)
          ((float*)hdn.data())[k] = (float)d;
        else
          ((double*)hdn.data())[k] = d;
      }
    CU(cudaMemcpyAsync((void*)p.dnc, hdn.data(), hdn.size(), cudaMemcpyHostToDevice, s));
  }
  std::vector<char> hum;
  if (p.unm) {  // u = 1 (significand 1, exponent 0)
    const size_t n = (size_t)(c->T + 1) * N;
    hum.assign(n * sm, 0);
    for (size_t k = 0; k < n; ++k) {
      if (f32)
        ((float*)hum.data())[k] = 1.f;
      else
        ((double*)hum.data())[k] = 1.0;
    }
    CU(cudaMemcpyAsync(p.unm, hum.data(), hum.size(), cudaMemcpyHostToDevice, s));
    CU(cudaMemsetAsync(p.une, 0, n * 4, s));
  }
  CU(cudaMemsetAsync(p.err, 0, 8, s));
  CU(cudaMemsetAsync(p.errloc, 0, 8, s));
  // host staging buffers die at return: wait for the copies
  CU(cudaStreamSynchronize(s));
  return MMF_OK;
}

}  // namespace

// ================================================================================================
// C ABI

namespace mmf {
// readouts in user arc order, converted to fp64 on the device ([T][A]: t * A + user arc <- t * A + internal arc)
template <class M>
__global__ void k_export_flows(const M* __restrict__ src, const int* __restrict__ ioa, double* __restrict__ out,
                               int64_t A, int64_t Au, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = k / Au, a = k - t * Au;  // (Au = user arcs: the first Au of the A internal ones' user order)
    out[k] = (double)src[t * A + ioa[a]];
  }
}
template <class M>
__global__ void k_export_duals(const M* __restrict__ wm, const int* __restrict__ we, const int* __restrict__ ioa,
                               double* __restrict__ out, int64_t A, int64_t Au, int64_t n) {
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = k / Au, a = k - t * Au;
    const int64_t i = t * A + ioa[a];
    const double m = (double)wm[i];
    out[k] = m == 0.0 ? 0.0 : ldexp(m, we[i]);  // (values below 2^-1074 read 0)
  }
}
// device -> pageable host copy of a readout through a pinned bounce buffer (two halves: the DMA of one chunk
// overlaps the host threads' copy of the other into the caller's buffer); a plain pageable cudaMemcpy runs at a few
// GB/s on the [T][A] fp64 readouts (305 MB on [4])
static cudaError_t d2h_staged(mmf_ctx* ctx, void* out, const void* dev, size_t bytes) {
  constexpr size_t CH = 16u << 20;  // bytes per half
  if (bytes < 2 * CH) {
    cudaError_t e = cudaMemcpyAsync(out, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream);
    return e == cudaSuccess ? cudaStreamSynchronize(ctx->stream) : e;
  }
  if (!ctx->pinned) {
    cudaError_t e = cudaMallocHost(&ctx->pinned, 2 * CH);
    if (e != cudaSuccess) {
      ctx->pinned = nullptr;
      cudaGetLastError();
      e = cudaMemcpyAsync(out, dev, bytes, cudaMemcpyDeviceToHost, ctx->stream);
      return e == cudaSuccess ? cudaStreamSynchronize(ctx->stream) : e;
    }
    if (!ctx->ev_d2h[0]) {
      cudaEventCreateWithFlags(&ctx->ev_d2h[0], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ctx->ev_d2h[1], cudaEventDisableTiming);
    }
  }
  char* pin = (char*)ctx->pinned;
  const char* src = (const char*)dev;
  char* dst = (char*)out;
  const size_t nch = (bytes + CH - 1) / CH;
  auto issue = [&](size_t k) {
    const size_t off = k * CH, len = std::min(CH, bytes - off);
    cudaError_t e = cudaMemcpyAsync(pin + (k & 1) * CH, src + off, len, cudaMemcpyDeviceToHost, ctx->stream);
    if (e == cudaSuccess) e = cudaEventRecord(ctx->ev_d2h[k & 1], ctx->stream);
    return e;
  };
  cudaError_t e = issue(0);
  for (size_t k = 0; k < nch && e == cudaSuccess; ++k) {
    e = cudaEventSynchronize(ctx->ev_d2h[k & 1]);
    if (e != cudaSuccess) break;
    if (k + 1 < nch) e = issue(k + 1);  // (the other half is free: its copy-out finished last iteration)
    const size_t off = k * CH, len = std::min(CH, bytes - off);
    const int nt = 4;
    std::vector<std::thread> th;
    for (int i = 0; i < nt; ++i)
      th.emplace_back([&, i]() {
        const size_t a = len * i / nt, b = len * (i + 1) / nt;
        memcpy(dst + off + a, pin + (k & 1) * CH + a, b - a);
      });
    for (auto& x : th) x.join();
  }
  return e;
}

// what: 0 edge flows (one readout pass first), 1 capacity duals
static mmf_status read_export(mmf_ctx* ctx, double* out, int what) {
  if (!ctx || !out) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  CU(cudaSetDevice(ctx->device));
  if (what == 0) {
    mmf_status st = dispatch(ctx, [&](auto eng) { return decltype(eng)::readout(ctx, ctx->stream); });
    if (st != MMF_OK) return st;
  }
  mmf_status st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  const int64_t A = ctx->A, Au = ctx->A_user, n = (int64_t)ctx->T * Au;
  if (!ctx->d_int_of_arc) {
    CU(cudaMalloc(&ctx->d_int_of_arc, (size_t)A * sizeof(int)));
    CU(cudaMemcpy(ctx->d_int_of_arc, ctx->int_of_arc.data(), (size_t)A * sizeof(int), cudaMemcpyHostToDevice));
  }
  if (!ctx->d_export) CU(cudaMalloc(&ctx->d_export, (size_t)n * sizeof(double)));
  double* d = ctx->d_export;
  const unsigned grid = (unsigned)std::min<int64_t>((n + 255) / 256, 8 * 148);
  if (ctx->prec == MMF_FP32) {
    if (what == 0) k_export_flows<float><<<grid, 256, 0, ctx->stream>>>((const float*)ctx->dp.Fout, ctx->d_int_of_arc, d, A, Au, n);
    else k_export_duals<float><<<grid, 256, 0, ctx->stream>>>((const float*)ctx->dp.Wm, ctx->dp.We, ctx->d_int_of_arc, d, A, Au, n);
  } else {
    if (what == 0) k_export_flows<double><<<grid, 256, 0, ctx->stream>>>((const double*)ctx->dp.Fout, ctx->d_int_of_arc, d, A, Au, n);
    else k_export_duals<double><<<grid, 256, 0, ctx->stream>>>((const double*)ctx->dp.Wm, ctx->dp.We, ctx->d_int_of_arc, d, A, Au, n);
  }
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = d2h_staged(ctx, out, d, (size_t)n * sizeof(double));
  if (e != cudaSuccess) return fail(ctx, MMF_ECUDA, std::string("readout: ") + cudaGetErrorString(e));
  return MMF_OK;
}
}  // namespace mmf

namespace mmf {
// ---- checkpoint / resume: W [T][A] (user arc order) and UT = beta_T [N][Lp] (user node
// order) of the end-of-sweep state; everything else is recomputed from them on load
struct StateHdr {
  char magic[8];  // "MMFSTAT2"
  int32_t prec, N, T, L, Lp, l_begin;
  int64_t A, sweeps;
  uint64_t graph_hash;    // N, A, arcs
  uint64_t problem_hash;  // T, eps, costs, capacities (bit patterns)
};
struct Fnv {
  uint64_t h = 1469598103934665603ull;
  void mix(uint64_t x) {
    h ^= x;
    h *= 1099511628211ull;
  }
  void mixd(double d) {
    uint64_t u;
    memcpy(&u, &d, 8);
    mix(u);
  }
};
static uint64_t graph_hash(const mmf_ctx* c) {
  Fnv f;
  f.mix((uint64_t)c->N);
  f.mix((uint64_t)c->A);
  for (int64_t a = 0; a < c->A; ++a) f.mix(((uint64_t)(uint32_t)c->tail[a] << 32) | (uint32_t)c->head[a]);
  return f.h;
}
static uint64_t problem_hash(const mmf_ctx* c) {
  Fnv f;
  f.mix((uint64_t)c->T);
  f.mixd(c->eps);
  f.mix((uint64_t)c->cost_tv);
  for (double x : c->cost) f.mixd(x);
  f.mix((uint64_t)c->cap_tv);
  for (double x : c->cap) f.mixd(x);
  f.mix((uint64_t)c->node_cost.size());
  for (double x : c->node_cost) f.mixd(x);
  for (double x : c->node_cap) f.mixd(x);
  return f.h;
}
// W [T][A] (user arc order), then UT = beta_T and U0 (the last a2's source scaling; readouts before the next sweep
// start from it), each [N][Lp] significand + exponent planes in user node order
static size_t state_bytes(const mmf_ctx* c) {
  const size_t se = c->prec == MMF_FP32 ? 2 : 4;
  return sizeof(StateHdr) + (size_t)c->T * c->A * (c->sm() + 4) + 2 * (size_t)c->N * c->Lp * (c->sm() + se);
}
}  // namespace mmf

extern "C" {

const char* mmf_version(void) { return "mmf 0.1 (sm_100a, XF f32/i16 + f64/i32)"; }

const char* mmf_last_error(const mmf_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_error.c_str(); }

mmf_status mmf_create(mmf_ctx** out, int device, mmf_prec prec, void* cuda_stream) {
  if (!out) {
    g_create_error = "out is NULL";
    return MMF_EINVAL;
  }
  *out = nullptr;
  if (prec != MMF_FP32 && prec != MMF_FP64) {
    g_create_error = "unknown precision";
    return MMF_EINVAL;
  }
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    g_create_error = "no such CUDA device";
    return MMF_ECUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    g_create_error = "cudaSetDevice failed";
    return MMF_ECUDA;
  }
  mmf_ctx* c = new mmf_ctx();
  c->device = device;
  c->prec = prec;
  cudaDeviceGetAttribute(&c->sms, cudaDevAttrMultiProcessorCount, device);
  if (c->sms <= 0) c->sms = 148;
  c->stream = (cudaStream_t)cuda_stream;
  if (cudaStreamCreateWithFlags(&c->priv, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_user, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_priv, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    g_create_error = "stream/event creation failed";
    return MMF_ECUDA;
  }
  *out = c;
  return MMF_OK;
}

mmf_status mmf_set_option(mmf_ctx* ctx, const char* key, int64_t value) {
  if (!ctx || !key) return MMF_EINVAL;
  std::string k(key);
  if (k == "graph")
    ctx->opt_graph = value != 0;
  else if (k == "profile")
    ctx->opt_profile = value != 0;
  else if (k == "prefetch") {
    ctx->opt_prefetch = value != 0;
    ctx->wc.prefetch = ctx->opt_prefetch;
    if (ctx->gexec) {  // the captured graph bakes kernel arguments: recapture
      cudaGraphExecDestroy(ctx->gexec);
      cudaGraphDestroy(ctx->graph);
      ctx->gexec = nullptr;
      ctx->graph = nullptr;
    }
  }
  else if (k == "reorder" || k == "dry" || k == "copy" || k == "wintma" || k == "bwd" || k == "fgw" || k == "wrap" || k == "stripw" || k == "schedule" || k == "theta_milli" || k == "fng" || k == "fnp" || k == "l2hint" || k == "kernels" || k == "tile" || k == "cpt" || k == "halo" || k == "cpc" || k == "order" || k == "pexch" || k == "tbwd" || k == "tfwd" || k == "wcp") {
    if (ctx->inited) return fail(ctx, MMF_ESTATE, k + " must be set before mmf_init");
    if (k == "reorder") ctx->opt_reorder = value != 0;
    if (k == "dry") ctx->opt_dry = (int)value;
    if (k == "copy") ctx->opt_copy = (int)value;
    if (k == "wintma") ctx->opt_wintma = (int)value;
    if (k == "bwd") {
      if (value < 0 || value > 3) return fail(ctx, MMF_EINVAL, "bwd must be 0 .. 3");
      ctx->opt_bwd = (int)value;
    }
    if (k == "fgw") {
      if (value != 0 && value != 2 && value != 4 && value != 8) return fail(ctx, MMF_EINVAL, "fgw must be 0, 2, 4 or 8");
      ctx->opt_fgw = (int)value;
    }
    if (k == "fng") {
      if (value < 0 || value > 6) return fail(ctx, MMF_EINVAL, "fng must be in [0, 6]");
      ctx->opt_fng = (int)value;
    }
    if (k == "schedule") {
      if (value < 0 || value > 2)
        return fail(ctx, MMF_EINVAL, "schedule must be 0 (Gauss-Seidel), 1 (Jacobi) or 2 (symmetric Gauss-Seidel)");
      ctx->opt_schedule = (int)value;
    }
    if (k == "theta_milli") {
      if (value < 0 || value > 1000) return fail(ctx, MMF_EINVAL, "theta_milli must be in [0, 1000]");
      ctx->opt_theta_milli = (int)value;
    }
    if (k == "stripw") {
      if (value < 0 || value > 64) return fail(ctx, MMF_EINVAL, "stripw must be in [0, 64]");
      ctx->opt_stripw = (int)value;
    }
    if (k == "wrap") {
      if (value < -1 || value > 1) return fail(ctx, MMF_EINVAL, "wrap must be -1, 0 or 1");
      ctx->opt_wrap = (int)value;
    }
    if (k == "l2hint") ctx->opt_l2hint = value != 0;
    if (k == "wcp") {
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
        return fail(ctx, MMF_EINVAL, "wcp must be 0, 1, 2, 4 or 8");
      ctx->opt_wcp = (int)value;
    }
    if (k == "tfwd") {
      if (value < -1 || value > 1) return fail(ctx, MMF_EINVAL, "tfwd must be -1 (auto), 0 or 1");
      ctx->opt_tfwd = (int)value;
    }
    if (k == "tbwd") {
      if (value < -1 || value > 1) return fail(ctx, MMF_EINVAL, "tbwd must be -1 (auto), 0 or 1");
      ctx->opt_tbwd = (int)value;
    }
    if (k == "pexch") {
      if (value < -1 || value > 1) return fail(ctx, MMF_EINVAL, "pexch must be -1 (auto), 0 or 1");
      ctx->opt_pexch = (int)value;
    }
    if (k == "fnp") {
      if (value < 0 || value > 3) return fail(ctx, MMF_EINVAL, "fnp must be in [0, 3]");
      ctx->opt_fnp = (int)value;
    }
    if (k == "kernels") {
      if (value < 1 || value > 6 || value == 2)
        return fail(ctx, MMF_EINVAL, "kernels must be 1 or 3 .. 6 (the node-tile family 2 was removed)");
      ctx->opt_kernels = (int)value;
    }
    if (k == "tile") {
      if (value < 1 || value > 256) return fail(ctx, MMF_EINVAL, "tile must be in [1, 256]");
      ctx->opt_tile = (int)value;
    }
    if (k == "order") {
      if (value < 0 || value > 4) return fail(ctx, MMF_EINVAL, "order must be in [0, 4]");
      ctx->opt_order = (int)value;
    }
    if (k == "cpc") {
      if (value < 0) return fail(ctx, MMF_EINVAL, "cpc must be >= 0");
      ctx->opt_cpc = (int)value;
    }
    if (k == "halo") {
      if (value < 0 || value > 4096) return fail(ctx, MMF_EINVAL, "halo must be in [0, 4096]");
      ctx->opt_halo = (int)value;
    }
    if (k == "cpt") {
      if (value != 0 && value != 1 && value != 2 && value != 4 && value != 8)
        return fail(ctx, MMF_EINVAL, "cpt must be 0, 1, 2, 4 or 8");
      ctx->opt_cpt = (int)value;
    }
    ctx->prepared = false;
  } else
    return fail(ctx, MMF_EINVAL, "unknown option " + k);
  return MMF_OK;
}

mmf_status mmf_set_graph(mmf_ctx* ctx, int32_t N, int64_t n_arcs, const int32_t* tail, const int32_t* head) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->augmented) return fail(ctx, MMF_ESTATE, "problem fixed once the layout was taken with commodity times");
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "graph already initialised");
  if (N < 1) return fail(ctx, MMF_EINVAL, "N must be >= 1");
  if (n_arcs < 1 || n_arcs > (int64_t)0x7fffffff) return fail(ctx, MMF_EINVAL, "n_arcs out of range");
  if (!tail || !head) return fail(ctx, MMF_EINVAL, "tail/head NULL");
  std::vector<int64_t> key(n_arcs);
  for (int64_t a = 0; a < n_arcs; ++a) {
    if (tail[a] < 0 || tail[a] >= N || head[a] < 0 || head[a] >= N)
      return fail(ctx, MMF_EINVAL, "arc " + std::to_string(a) + ": node id out of range");
    key[a] = (int64_t)tail[a] * N + head[a];
  }
  std::sort(key.begin(), key.end());
  for (int64_t a = 1; a < n_arcs; ++a)
    if (key[a] == key[a - 1]) return fail(ctx, MMF_EINVAL, "duplicate (tail, head) arc");
  ctx->N = N;
  ctx->A = n_arcs;
  ctx->tail.assign(tail, tail + n_arcs);
  ctx->head.assign(head, head + n_arcs);
  ctx->have_cost = ctx->have_cap = false;
  ctx->prepared = false;
  return MMF_OK;
}

mmf_status mmf_set_costs(mmf_ctx* ctx, int32_t T, double eps, const double* cost, int time_varying) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->augmented) return fail(ctx, MMF_ESTATE, "problem fixed once the layout was taken with commodity times");
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (ctx->N == 0) return fail(ctx, MMF_ESTATE, "mmf_set_graph first");
  if (T < 1) return fail(ctx, MMF_EINVAL, "T must be >= 1");
  if (!(eps > 0) || !std::isfinite(eps)) return fail(ctx, MMF_EINVAL, "eps must be finite and > 0");
  if (!cost) return fail(ctx, MMF_EINVAL, "cost NULL");
  const size_t n = (size_t)(time_varying ? T : 1) * ctx->A;
  for (size_t k = 0; k < n; ++k)
    if (!std::isfinite(cost[k])) return fail(ctx, MMF_EINVAL, "non-finite cost");
  ctx->T = T;
  ctx->eps = eps;
  ctx->cost.assign(cost, cost + n);
  ctx->cost_tv = time_varying != 0;
  ctx->have_cost = true;
  if (ctx->have_cap && ctx->cap_tv && ctx->cap.size() != (size_t)T * ctx->A) ctx->have_cap = false;
  return MMF_OK;
}

mmf_status mmf_set_capacity(mmf_ctx* ctx, const double* cap, int time_varying) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->augmented) return fail(ctx, MMF_ESTATE, "problem fixed once the layout was taken with commodity times");
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (!ctx->have_cost) return fail(ctx, MMF_ESTATE, "mmf_set_costs first");
  if (!cap) return fail(ctx, MMF_EINVAL, "cap NULL");
  const size_t n = (size_t)(time_varying ? ctx->T : 1) * ctx->A;
  for (size_t k = 0; k < n; ++k)
    if (!(cap[k] >= 0)) return fail(ctx, MMF_EINVAL, "capacity < 0 or NaN");
  ctx->cap.assign(cap, cap + n);
  ctx->cap_tv = time_varying != 0;
  ctx->fpos_ok = false;
  ctx->have_cap = true;
  return MMF_OK;
}

static mmf_status check_slice(mmf_ctx* ctx, int32_t L_global, int32_t l_begin, int32_t l_count) {
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (ctx->augmented) return fail(ctx, MMF_ESTATE, "problem fixed once the layout was taken with commodity times");
  if (ctx->N == 0) return fail(ctx, MMF_ESTATE, "mmf_set_graph first");
  if (L_global < 1 || l_count < 1 || l_begin < 0 || l_begin + l_count > L_global)
    return fail(ctx, MMF_EINVAL, "bad commodity slice");
  return MMF_OK;
}

mmf_status mmf_set_marginals(mmf_ctx* ctx, int32_t L_global, int32_t l_begin, int32_t l_count, const double* mu0,
                             const double* muT) {
  if (!ctx) return MMF_EINVAL;
  mmf_status st = check_slice(ctx, L_global, l_begin, l_count);
  if (st != MMF_OK) return st;
  if (!mu0 || !muT) return fail(ctx, MMF_EINVAL, "mu0/muT NULL");
  const int N = ctx->N;
  for (int l = 0; l < l_count; ++l) {
    double s0 = 0, sT = 0;
    for (int v = 0; v < N; ++v) {
      double a = mu0[(size_t)l * N + v], b = muT[(size_t)l * N + v];
      if (!(a >= 0) || !(b >= 0) || !std::isfinite(a) || !std::isfinite(b))
        return fail(ctx, MMF_EINVAL, "marginal entries must be finite and >= 0");
      s0 += a;
      sT += b;
    }
    if (std::fabs(s0 - sT) > 1e-12 * std::max(s0, sT))
      return fail(ctx, MMF_EINVAL, "commodity " + std::to_string(l + l_begin) + ": mass imbalance (S:112)");
  }
  ctx->Lg = L_global;
  ctx->l_begin = l_begin;
  ctx->L = l_count;
  ctx->point = false;
  ctx->prepared = false;  // (the node order is chosen from L and the precision)
  if (ctx->node_cost.size() != (size_t)l_count * N) ctx->node_cost.clear();
  ctx->mu0.assign(mu0, mu0 + (size_t)l_count * N);
  ctx->muT.assign(muT, muT + (size_t)l_count * N);
  ctx->have_marg = true;
  return MMF_OK;
}

mmf_status mmf_set_point_marginals(mmf_ctx* ctx, int32_t L_global, int32_t l_begin, int32_t l_count,
                                   const int32_t* src, const int32_t* dst, const double* mass) {
  if (!ctx) return MMF_EINVAL;
  mmf_status st = check_slice(ctx, L_global, l_begin, l_count);
  if (st != MMF_OK) return st;
  if (!src || !dst || !mass) return fail(ctx, MMF_EINVAL, "src/dst/mass NULL");
  for (int l = 0; l < l_count; ++l) {
    if (src[l] < 0 || src[l] >= ctx->N || dst[l] < 0 || dst[l] >= ctx->N)
      return fail(ctx, MMF_EINVAL, "point marginal node out of range");
    if (!(mass[l] > 0) || !std::isfinite(mass[l])) return fail(ctx, MMF_EINVAL, "mass must be finite and > 0");
  }
  ctx->Lg = L_global;
  ctx->l_begin = l_begin;
  ctx->L = l_count;
  ctx->point = true;
  ctx->prepared = false;  // (the node order is chosen from L and the precision)
  if (ctx->node_cost.size() != (size_t)l_count * ctx->N) ctx->node_cost.clear();
  ctx->src.assign(src, src + l_count);
  ctx->dst.assign(dst, dst + l_count);
  ctx->mass.assign(mass, mass + l_count);
  ctx->have_marg = true;
  return MMF_OK;
}

mmf_status mmf_set_node_costs(mmf_ctx* ctx, const double* c) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->augmented) return fail(ctx, MMF_ESTATE, "problem fixed once the layout was taken with commodity times");
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (!ctx->have_marg || !ctx->have_cost) return fail(ctx, MMF_ESTATE, "mmf_set_costs and the marginals first");
  if (!c) {
    ctx->node_cost.clear();
    ctx->prepared = false;
    return MMF_OK;
  }
  const size_t n = (size_t)ctx->L * ctx->N;
  // D = exp(-c / eps) must be representable as an extended-range factor: |c / eps| log2(e) <= ELIM / 2
  const double lim = 0.5 * ELIM / 1.4426950408889634;
  for (size_t k = 0; k < n; ++k)
    if (!std::isfinite(c[k]) || std::fabs(c[k] / ctx->eps) > lim)
      return fail(ctx, MMF_EINVAL, "node cost not finite or |c / eps| beyond the extended range");
  ctx->node_cost.assign(c, c + n);
  ctx->prepared = false;
  return MMF_OK;
}

mmf_status mmf_set_node_capacity(mmf_ctx* ctx, const double* cap, int time_varying) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->inited || ctx->augmented) return fail(ctx, MMF_ESTATE, "node capacities must be set before the layout");
  if (!ctx->have_cost) return fail(ctx, MMF_ESTATE, "mmf_set_costs first");
  if (!cap) {
    ctx->node_cap.clear();
    ctx->prepared = false;
    return MMF_OK;
  }
  const size_t n = (size_t)(time_varying ? ctx->T + 1 : 1) * ctx->N;
  for (size_t k = 0; k < n; ++k)
    if (!(cap[k] >= 0)) return fail(ctx, MMF_EINVAL, "node capacity < 0 or NaN");
  ctx->node_cap.assign(cap, cap + n);
  ctx->node_cap_tv = time_varying != 0;
  ctx->prepared = false;
  return MMF_OK;
}

mmf_status mmf_read_node_duals(mmf_ctx* ctx, double* out) {
  if (!ctx || !out) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (ctx->node_cap.empty()) return fail(ctx, MMF_EINVAL, "no node capacities");
  mmf_status st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  const size_t n = (size_t)(ctx->T + 1) * ctx->N;
  std::vector<char> m(n * ctx->sm());
  std::vector<int> e(n);
  CU(cudaMemcpy(m.data(), ctx->dp.unm, m.size(), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(e.data(), ctx->dp.une, n * 4, cudaMemcpyDeviceToHost));
  for (int t = 0; t <= ctx->T; ++t)
    for (int v = 0; v < ctx->N_user; ++v) {
      const size_t k = (size_t)t * ctx->N + ctx->newid[v];
      const double mm = ctx->prec == MMF_FP32 ? (double)((const float*)m.data())[k] : ((const double*)m.data())[k];
      out[(size_t)t * ctx->N_user + v] = mm == 0.0 ? 0.0 : std::ldexp(mm, e[k]);
    }
  return MMF_OK;
}

mmf_status mmf_set_commodity_times(mmf_ctx* ctx, const int32_t* t_in, const int32_t* t_out) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->inited || ctx->augmented) return fail(ctx, MMF_ESTATE, "commodity times must be set before the layout");
  if (!ctx->have_marg || !ctx->have_cost) return fail(ctx, MMF_ESTATE, "mmf_set_costs and the marginals first");
  if (!t_in || !t_out) {
    ctx->t_in.clear();
    ctx->t_out.clear();
    return MMF_OK;
  }
  if (!ctx->point) return fail(ctx, MMF_EINVAL, "commodity times need point-mass commodities");
  if (ctx->comm) return fail(ctx, MMF_EINVAL, "commodity times: single rank (the holding nodes are per commodity)");
  for (int l = 0; l < ctx->L; ++l)
    if (!(t_in[l] >= 0 && t_in[l] < t_out[l] && t_out[l] <= ctx->T))
      return fail(ctx, MMF_EINVAL, "commodity " + std::to_string(l + ctx->l_begin) + ": need 0 <= t_in < t_out <= T");
  ctx->t_in.assign(t_in, t_in + ctx->L);
  ctx->t_out.assign(t_out, t_out + ctx->L);
  ctx->prepared = false;
  return MMF_OK;
}

mmf_status mmf_workspace_bytes(const mmf_ctx* cctx, size_t* bytes) {
  if (!cctx || !bytes) return MMF_EINVAL;
  mmf_ctx* ctx = const_cast<mmf_ctx*>(cctx);
  if (!ready_for_layout(ctx)) return fail(ctx, MMF_ESTATE, "graph, costs, capacity and marginals must be set");
  prepare(ctx);
  derive_shapes(ctx);
  DevPtrs saved = ctx->dp;
  TileMeta savedt = ctx->tm;
  *bytes = layout(ctx, nullptr);
  ctx->dp = saved;
  ctx->tm = savedt;
  return MMF_OK;
}

mmf_status mmf_set_workspace(mmf_ctx* ctx, void* dptr, size_t bytes) {
  if (!ctx) return MMF_EINVAL;
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (!dptr || ((uintptr_t)dptr & 255)) return fail(ctx, MMF_EINVAL, "workspace must be non-NULL and 256-byte aligned");
  if (ctx->ws_owned) {
    cudaFree(ctx->ws);
    ctx->ws_owned = false;
  }
  ctx->ws = dptr;
  ctx->ws_bytes = bytes;
  return MMF_OK;
}

mmf_status mmf_nccl_unique_id(void* out128) {
  if (!out128) return MMF_EINVAL;
  NcclApi& api = nccl_api();
  if (!api.ok || !api.GetUniqueId) {
    g_create_error = "libnccl.so.2 not found in the process";
    return MMF_ENCCL;
  }
  NcclUid uid;
  if (api.GetUniqueId(&uid) != 0) {
    g_create_error = "ncclGetUniqueId failed";
    return MMF_ENCCL;
  }
  memcpy(out128, uid.internal, 128);
  return MMF_OK;
}

mmf_status mmf_attach_nccl(mmf_ctx* ctx, const void* unique_id128, int nranks, int rank) {
  if (!ctx || !unique_id128) return MMF_EINVAL;
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "attach NCCL before mmf_init");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(ctx, MMF_EINVAL, "bad nranks/rank");
  if (!ctx->t_in.empty()) return fail(ctx, MMF_EINVAL, "commodity times: single rank");
  NcclApi& api = nccl_api();
  if (!api.ok) return fail(ctx, MMF_ENCCL, "libnccl.so.2 not found in the process");
  NcclUid uid;
  memcpy(uid.internal, unique_id128, 128);
  ncclComm_t_ comm = nullptr;
  int r = api.CommInitRank(&comm, nranks, uid, rank);
  if (r != 0)
    return fail(ctx, MMF_ENCCL,
                std::string("ncclCommInitRank: ") + (api.GetErrorString ? api.GetErrorString(r) : "error"));
  ctx->comm = comm;
  ctx->nranks = nranks;
  ctx->rank = rank;
  return MMF_OK;
}

mmf_status mmf_init(mmf_ctx* ctx) {
  if (!ctx) return MMF_EINVAL;
  Nvtx r("mmf_init");
  if (ctx->inited) return fail(ctx, MMF_ESTATE, "already initialised");
  if (!ready_for_layout(ctx)) return fail(ctx, MMF_ESTATE, "graph, costs, capacity and marginals must be set");
  CU(cudaSetDevice(ctx->device));
  mmf_status st = finalize(ctx);
  if (st != MMF_OK) return st;
  if (!ctx->node_cap.empty()) {
    const bool fam = ctx->opt_kernels == 1 || (ctx->prec == MMF_FP32 && ctx->opt_kernels >= 5 && ctx->pipe_fwd);
    if (!fam || ctx->opt_schedule == 1 || ctx->comm)
      return fail(ctx, MMF_EINVAL, "node capacities: the pipelined fp32 path (L >= 256) or kernels = 1, Gauss-Seidel "
                                   "or symmetric schedule, one rank");
  }
  st = dispatch(ctx, [&](auto eng) { return decltype(eng)::init_device(ctx, ctx->stream); });
  if (st != MMF_OK) return st;
  CU(cudaGetLastError());
  ctx->inited = true;
  ctx->sweeps = 0;
  return MMF_OK;
}

mmf_status mmf_sweep(mmf_ctx* ctx, int32_t n) {
  if (!ctx) return MMF_EINVAL;
  Nvtx r("mmf_sweep");
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (n < 0) return fail(ctx, MMF_EINVAL, "n < 0");
  if (n == 0) return MMF_OK;
  CU(cudaSetDevice(ctx->device));
  const bool use_graph = ctx->opt_graph && !ctx->opt_profile;
  if (!use_graph) {
    for (int k = 0; k < n; ++k) {
      mmf_status st = dispatch(ctx, [&](auto eng) { return decltype(eng)::enqueue_sweep(ctx, ctx->stream); });
      if (st != MMF_OK) return st;
    }
    CU(cudaGetLastError());
    ctx->sweeps += n;
    return MMF_OK;
  }
  if (!ctx->gexec) {
    ctx->capturing = true;
    std::fill(ctx->graph_launch_tally, ctx->graph_launch_tally + K_NKINDS, 0);
    cudaError_t e = cudaStreamBeginCapture(ctx->priv, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) {
      ctx->capturing = false;
      return fail(ctx, MMF_ECUDA, std::string("cudaStreamBeginCapture: ") + cudaGetErrorString(e));
    }
    mmf_status st = dispatch(ctx, [&](auto eng) { return decltype(eng)::enqueue_sweep(ctx, ctx->priv); });
    cudaGraph_t g = nullptr;
    e = cudaStreamEndCapture(ctx->priv, &g);
    ctx->capturing = false;
    if (st != MMF_OK) return st;
    if (e != cudaSuccess) return fail(ctx, MMF_ECUDA, std::string("cudaStreamEndCapture: ") + cudaGetErrorString(e));
    ctx->graph = g;
    CU(cudaGraphInstantiate(&ctx->gexec, g, 0));
  }
  CU(cudaEventRecord(ctx->ev_user, ctx->stream));
  CU(cudaStreamWaitEvent(ctx->priv, ctx->ev_user, 0));
  for (int k = 0; k < n; ++k) {
    CU(cudaGraphLaunch(ctx->gexec, ctx->priv));
    for (int q = 0; q < K_NKINDS; ++q) ctx->launches[q] += ctx->graph_launch_tally[q];
  }
  CU(cudaEventRecord(ctx->ev_priv, ctx->priv));
  CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_priv, 0));
  ctx->sweeps += n;
  return MMF_OK;
}

mmf_status mmf_sweep_group(mmf_ctx* const* ctxs, int32_t G, int32_t n) {
  if (!ctxs || G < 1 || G > 8) return MMF_EINVAL;
  mmf_ctx* c0 = ctxs[0];
  if (!c0) return MMF_EINVAL;
  for (int g = 0; g < G; ++g) {
    mmf_ctx* c = ctxs[g];
    if (!c || !c->inited) return fail(c0, MMF_ESTATE, "every context must be initialised");
    if (c->comm) return fail(c0, MMF_EINVAL, "virtual ranks do not use NCCL");
    if (c->device != c0->device || c->stream != c0->stream || c->prec != c0->prec || c->N != c0->N ||
        c->A != c0->A || c->T != c0->T || c->opt_schedule != 0 || c->opt_kernels < 3 || c->opt_kernels != c0->opt_kernels)
      return fail(c0, MMF_EINVAL, "virtual ranks: same device, stream, precision, problem shape; kernels >= 3; GS");
  }
  if (n < 0) return fail(c0, MMF_EINVAL, "n < 0");
  CU2(c0, cudaSetDevice(c0->device));
  for (int k = 0; k < n; ++k) {
    mmf_status st = dispatch(c0, [&](auto eng) { return decltype(eng)::group_sweep(ctxs, G, c0->stream); });
    if (st != MMF_OK) return st;
  }
  CU2(c0, cudaGetLastError());
  for (int g = 0; g < G; ++g) ctxs[g]->sweeps += n;
  return MMF_OK;
}

mmf_status mmf_sync(mmf_ctx* ctx) {
  if (!ctx) return MMF_EINVAL;
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));
  CU(cudaGetLastError());
  if (!ctx->inited) return MMF_OK;
  mmf_status st = collect_profile(ctx);
  if (st != MMF_OK) return st;
  return check_sticky(ctx);
}

mmf_status mmf_read_edge_flows(mmf_ctx* ctx, double* out) {
  return mmf::read_export(ctx, out, 0);
}

mmf_status mmf_read_cap_duals(mmf_ctx* ctx, double* out) {
  return mmf::read_export(ctx, out, 1);
}

mmf_status mmf_solve(mmf_ctx* ctx, double tol, int32_t max_sweeps, int32_t check_every, int32_t* sweeps_done,
                     double* err_out, double* err_hist) {
  if (!ctx || !sweeps_done || !err_out) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (max_sweeps < 0 || check_every < 1 || !(tol >= 0)) return fail(ctx, MMF_EINVAL, "max_sweeps >= 0, check_every >= 1, tol >= 0");
  CU(cudaSetDevice(ctx->device));
  int done = 0, h = 0;
  double err = INFINITY;
  for (;;) {
    if (done > 0) {  // error of the end-of-sweep state, reduced on the device
      mmf_status st = dispatch(ctx, [&](auto eng) { return decltype(eng)::readout(ctx, ctx->stream); });
      if (st != MMF_OK) return st;
      st = dispatch(ctx, [&](auto eng) { return decltype(eng)::stats(ctx, ctx->stream); });
      if (st != MMF_OK) return st;
      st = dispatch(ctx, [&](auto eng) { return decltype(eng)::excess(ctx, ctx->stream); });
      if (st != MMF_OK) return st;
      if (ctx->comm) {  // (mass and marginal mismatches are per-rank partial sums; the flows are already global)
        int r = nccl_api().AllReduce(ctx->dp.stats, ctx->dp.stats, 5, NCCL_FLOAT64, NCCL_SUM, ctx->comm, ctx->stream);
        if (r != 0) return fail(ctx, MMF_ENCCL, "ncclAllReduce(stats) failed");
      }
      st = mmf_sync(ctx);
      if (st != MMF_OK) return st;
      double s[8];
      CU(cudaMemcpy(s, ctx->dp.stats, sizeof s, cudaMemcpyDeviceToHost));
      err = s[0] > 0 ? (s[1] + s[2] + s[6]) / s[0] : INFINITY;
      if (err_hist) err_hist[h] = err;
      ++h;
      if (err < tol) break;
    }
    if (done >= max_sweeps) break;
    const int n = std::min(check_every, max_sweeps - done);
    mmf_status st = mmf_sweep(ctx, n);
    if (st != MMF_OK) return st;
    done += n;
  }
  *sweeps_done = done;
  *err_out = err;
  return err < tol ? MMF_OK : MMF_ENOTCONV;
}

mmf_status mmf_read_commodity_flows(mmf_ctx* ctx, int32_t t, double* out) {
  if (!ctx || !out) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (t < 0 || t >= ctx->T) return fail(ctx, MMF_EINVAL, "t must be in [0, T)");
  CU(cudaSetDevice(ctx->device));
  mmf_status st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  const int64_t A = ctx->A, n = A * ctx->L;
  if (!ctx->d_int_of_arc) {
    CU(cudaMalloc(&ctx->d_int_of_arc, (size_t)A * sizeof(int)));
    CU(cudaMemcpy(ctx->d_int_of_arc, ctx->int_of_arc.data(), (size_t)A * sizeof(int), cudaMemcpyHostToDevice));
  }
  double* d = nullptr;
  CU(cudaMalloc(&d, (size_t)n * sizeof(double)));
  st = dispatch(ctx, [&](auto eng) { return decltype(eng)::commodity_flows(ctx, ctx->stream, t, d); });
  cudaError_t e = st == MMF_OK ? cudaGetLastError() : cudaSuccess;
  if (st == MMF_OK && e == cudaSuccess)
    e = cudaMemcpyAsync(out, d, (size_t)ctx->A_user * ctx->L * sizeof(double), cudaMemcpyDeviceToHost, ctx->stream);
  if (st == MMF_OK && e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
  cudaFree(d);
  if (st != MMF_OK) return st;
  if (e != cudaSuccess) return fail(ctx, MMF_ECUDA, std::string("commodity flows: ") + cudaGetErrorString(e));
  return mmf_sync(ctx);
}

mmf_status mmf_state_bytes(const mmf_ctx* ctx, size_t* bytes) {
  if (!ctx || !bytes) return MMF_EINVAL;
  if (!ctx->inited) return MMF_ESTATE;
  *bytes = mmf::state_bytes(ctx);
  return MMF_OK;
}

mmf_status mmf_save_state(mmf_ctx* ctx, void* buf, size_t bytes) {
  if (!ctx || !buf) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (!ctx->node_cap.empty()) return fail(ctx, MMF_EINVAL, "checkpoints do not cover node capacities");
  if (bytes < mmf::state_bytes(ctx)) return fail(ctx, MMF_EINVAL, "state buffer too small (mmf_state_bytes)");
  mmf_status st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  mmf::StateHdr h{};
  memcpy(h.magic, "MMFSTAT2", 8);
  h.prec = (int32_t)ctx->prec;
  h.N = ctx->N;
  h.T = ctx->T;
  h.L = ctx->L;
  h.Lp = ctx->Lp;
  h.l_begin = ctx->l_begin;
  h.A = ctx->A;
  h.sweeps = ctx->sweeps;
  h.graph_hash = mmf::graph_hash(ctx);
  h.problem_hash = mmf::problem_hash(ctx);
  char* o = (char*)buf;
  memcpy(o, &h, sizeof h);
  o += sizeof h;
  const size_t TA = (size_t)ctx->T * ctx->A, sm = ctx->sm(), se = ctx->prec == MMF_FP32 ? 2 : 4;
  const size_t NL = (size_t)ctx->N * ctx->Lp;
  std::vector<char> wm(TA * sm), bm(NL * sm), be(NL * se);
  std::vector<int> we(TA);
  CU(cudaMemcpy(wm.data(), ctx->dp.Wm, wm.size(), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(we.data(), ctx->dp.We, TA * 4, cudaMemcpyDeviceToHost));
  char* owm = o;
  char* owe = owm + TA * sm;
  for (int t = 0; t < ctx->T; ++t)
    for (int64_t a = 0; a < ctx->A; ++a) {
      const size_t k = (size_t)t * ctx->A + ctx->int_of_arc[a], u = (size_t)t * ctx->A + a;
      memcpy(owm + u * sm, wm.data() + k * sm, sm);
      memcpy(owe + u * 4, &we[k], 4);
    }
  const size_t row_m = (size_t)ctx->Lp * sm, row_e = (size_t)ctx->Lp * se;
  char* ob = owe + TA * 4;
  // UT = beta_T, then U0
  const void* planes[2][2] = {{(char*)ctx->dp.bm + (size_t)ctx->T * NL * sm, (char*)ctx->dp.be + (size_t)ctx->T * NL * se},
                              {ctx->dp.u0m, ctx->dp.u0e}};
  for (int q = 0; q < 2; ++q) {
    CU(cudaMemcpy(bm.data(), planes[q][0], bm.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(be.data(), planes[q][1], be.size(), cudaMemcpyDeviceToHost));
    char* obm = ob;
    char* obe = obm + NL * sm;
    for (int v = 0; v < ctx->N; ++v) {
      memcpy(obm + (size_t)v * row_m, bm.data() + (size_t)ctx->newid[v] * row_m, row_m);
      memcpy(obe + (size_t)v * row_e, be.data() + (size_t)ctx->newid[v] * row_e, row_e);
    }
    ob = obe + NL * se;
  }
  return MMF_OK;
}

mmf_status mmf_load_state(mmf_ctx* ctx, const void* buf, size_t bytes) {
  if (!ctx || !buf) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  if (bytes < sizeof(mmf::StateHdr)) return fail(ctx, MMF_EINVAL, "state buffer too small");
  mmf::StateHdr h;
  memcpy(&h, buf, sizeof h);
  if (memcmp(h.magic, "MMFSTAT2", 8) != 0) return fail(ctx, MMF_EINVAL, "not an mmf state (MMFSTAT2)");
  if (h.prec != (int32_t)ctx->prec || h.N != ctx->N || h.T != ctx->T || h.L != ctx->L || h.A != ctx->A ||
      h.l_begin != ctx->l_begin || h.graph_hash != mmf::graph_hash(ctx))
    return fail(ctx, MMF_EINVAL, "state was saved for another problem (graph, T, commodity slice or precision)");
  if (h.problem_hash != mmf::problem_hash(ctx))
    return fail(ctx, MMF_EINVAL, "state was saved for another problem (eps, costs or capacities differ)");
  if (h.Lp <= 0 || h.Lp < h.L || h.sweeps < 0) return fail(ctx, MMF_EINVAL, "corrupt state header");
  const size_t TA = (size_t)ctx->T * ctx->A, sm = ctx->sm(), se = ctx->prec == MMF_FP32 ? 2 : 4;
  const size_t NL = (size_t)ctx->N * ctx->Lp, NLs = (size_t)ctx->N * h.Lp;
  if (bytes < sizeof h + TA * (sm + 4) + 2 * NLs * (sm + se)) return fail(ctx, MMF_EINVAL, "state buffer truncated");
  mmf_status st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  const char* o = (const char*)buf + sizeof h;
  const char* owm = o;
  const char* owe = owm + TA * sm;
  std::vector<char> wm(TA * sm), bm(NL * sm, 0), be(NL * se, 0);
  std::vector<int> we(TA);
  for (int t = 0; t < ctx->T; ++t)
    for (int64_t a = 0; a < ctx->A; ++a) {
      const size_t k = (size_t)t * ctx->A + ctx->int_of_arc[a], u = (size_t)t * ctx->A + a;
      memcpy(wm.data() + k * sm, owm + u * sm, sm);
      memcpy(&we[k], owe + u * 4, 4);
    }
  CU(cudaMemcpy(ctx->dp.Wm, wm.data(), wm.size(), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(ctx->dp.We, we.data(), TA * 4, cudaMemcpyHostToDevice));
  const int Lc = std::min(ctx->Lp, (int)h.Lp);  // (padding may differ between kernel configurations)
  void* planes[2][2] = {{(char*)ctx->dp.bm + (size_t)ctx->T * NL * sm, (char*)ctx->dp.be + (size_t)ctx->T * NL * se},
                        {ctx->dp.u0m, ctx->dp.u0e}};
  const char* ob = owe + TA * 4;
  for (int q = 0; q < 2; ++q) {
    const char* obm = ob;
    const char* obe = obm + NLs * sm;
    std::fill(bm.begin(), bm.end(), 0);
    std::fill(be.begin(), be.end(), 0);
    if (ctx->prec == MMF_FP32)  // (padding lanes: exact zeros, exponent EZERO)
      for (size_t k = 0; k < NL; ++k) ((int16_t*)be.data())[k] = (int16_t)EZERO;
    else
      for (size_t k = 0; k < NL; ++k) ((int32_t*)be.data())[k] = EZERO;
    for (int v = 0; v < ctx->N; ++v) {
      memcpy(bm.data() + (size_t)ctx->newid[v] * ctx->Lp * sm, obm + (size_t)v * h.Lp * sm, (size_t)Lc * sm);
      memcpy(be.data() + (size_t)ctx->newid[v] * ctx->Lp * se, obe + (size_t)v * h.Lp * se, (size_t)Lc * se);
    }
    CU(cudaMemcpy(planes[q][0], bm.data(), bm.size(), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(planes[q][1], be.data(), be.size(), cudaMemcpyHostToDevice));
    ob = obe + NLs * se;
  }
  st = dispatch(ctx, [&](auto eng) { return decltype(eng)::restore(ctx, ctx->stream); });
  if (st != MMF_OK) return st;
  ctx->sweeps = h.sweeps;
  return mmf_sync(ctx);
}

mmf_status mmf_read_stats(mmf_ctx* ctx, mmf_stats* out) {
  if (!ctx || !out) return MMF_EINVAL;
  if (!ctx->inited) return fail(ctx, MMF_ESTATE, "mmf_init first");
  const size_t TA = (size_t)ctx->T * ctx->A_user;
  std::vector<double> F(TA);
  mmf_status st = mmf_read_edge_flows(ctx, F.data());  // also leaves alpha_T of the end-of-sweep state
  if (st != MMF_OK) return st;
  st = dispatch(ctx, [&](auto eng) { return decltype(eng)::stats(ctx, ctx->stream); });
  if (st != MMF_OK) return st;
  if (ctx->comm) {
    int r = nccl_api().AllReduce(ctx->dp.stats, ctx->dp.stats, 5, NCCL_FLOAT64, NCCL_SUM, ctx->comm, ctx->stream);
    if (r != 0) return fail(ctx, MMF_ENCCL, "ncclAllReduce(stats) failed");
  }
  st = mmf_sync(ctx);
  if (st != MMF_OK) return st;
  double s[8];
  CU(cudaMemcpy(s, ctx->dp.stats, sizeof s, cudaMemcpyDeviceToHost));
  double primal = 0, viol = 0;
  const int64_t A = ctx->A_user;  // (user arcs; the user's cost / capacity arrays)
  const bool ctv = ctx->cost_user.size() > (size_t)A, ktv = ctx->cap_user.size() > (size_t)A;
  for (int t = 0; t < ctx->T; ++t)
    for (int64_t a = 0; a < A; ++a) {
      const double f = F[(size_t)t * A + a];
      primal += ctx->cost_user[(ctv ? (size_t)t * A : 0) + a] * f;
      const double d = ctx->cap_user[(ktv ? (size_t)t * A : 0) + a];
      if (std::isfinite(d)) viol = std::max(viol, f - d);
    }
  out->sweeps = ctx->sweeps;
  out->mass = s[0];
  out->src_mismatch = s[1];
  out->sink_mismatch = s[2];
  out->cap_violation = viol;
  double snode = 0.0;  // NEXT-3: sum_t <d_t, log u_t> over finite positive node capacities
  if (!ctx->node_cap.empty()) {
    const size_t n = (size_t)(ctx->T + 1) * ctx->N;
    std::vector<char> m(n * ctx->sm());
    std::vector<int> e(n);
    CU(cudaMemcpy(m.data(), ctx->dp.unm, m.size(), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(e.data(), ctx->dp.une, n * 4, cudaMemcpyDeviceToHost));
    for (int t = 1; t < ctx->T; ++t)
      for (int v = 0; v < ctx->N; ++v) {
        const double d = ctx->node_cap[(size_t)(ctx->node_cap_tv ? t : 0) * ctx->N + v];
        if (!(d > 0) || std::isinf(d)) continue;
        const size_t k = (size_t)t * ctx->N + ctx->newid[v];
        const double mm = ctx->prec == MMF_FP32 ? (double)((const float*)m.data())[k] : ((const double*)m.data())[k];
        snode += d * (std::log(mm) + e[k] * 0.69314718055994530942);
      }
  }
  out->dual = ctx->eps * (-s[0] + s[3] + s[4] + s[5] + snode);
  out->primal = primal;
  return MMF_OK;
}

mmf_status mmf_read_kernel_stats(mmf_ctx* ctx, int64_t* launches, double* ms, int n) {
  if (!ctx) return MMF_EINVAL;
  CU(cudaSetDevice(ctx->device));
  CU(cudaStreamSynchronize(ctx->stream));  // (accounting only: sticky solver errors surface at mmf_sync)
  if (ctx->inited) {
    mmf_status st = collect_profile(ctx);
    if (st != MMF_OK) return st;
  }
  for (int k = 0; k < n && k < K_NKINDS; ++k) {
    if (launches) launches[k] = ctx->launches[k];
    if (ms) ms[k] = ctx->ms[k];
  }
  return MMF_OK;
}

mmf_status mmf_sweep_bytes(const mmf_ctx* ctx, double* total, double* per_kind, int n) {
  if (!ctx) return MMF_EINVAL;
  // Algorithmic bytes (SURVEY §8(d) byte model; what the method must move with no cross-step reuse), with
  // B_e = significand + exponent bytes of a message element, B_w = W significand + exponent, true L:
  //   forward step : read alpha_{t-1}, read beta_t, write alpha_t  = 3 N L B_e + 2 |A| B_w (W read + write)
  //   backward step: read beta_{t+1}, write beta_t                 = 2 N L B_e +   |A| B_w
  //   boundaries   : 4 N L B_e for dense marginals (a2 / a4), ~0 for point masses
  // per sweep = T (5 N L B_e + 3 |A| B_w) + boundaries.  Per-kind entries attribute the same bytes to the
  // kernel kinds of the production path (fused forward, backward); the split reference kernels
  // (kernels=1) get their own shares for their attribution passes.
  const double Be = (double)(ctx->sm() + ctx->se());
  const double NL = (double)ctx->N * ctx->L;
  const double Bw = (double)(ctx->sm() + 4);
  const double A = (double)ctx->A;
  const double bnd = ctx->point ? 0.0 : 4 * NL * Be;
  double k[K_NKINDS] = {};
  k[K_FUSED] = ctx->T * (3 * NL * Be + 2 * A * Bw) + bnd;
  k[K_BWD] = ctx->T * (2 * NL * Be + A * Bw);
  k[K_FLOW] = ctx->T * (2 * NL * Be + A * Bw);
  k[K_UPDATE] = ctx->T * (2 * NL * Be + A * Bw);
  k[K_REDUCE] = ctx->T * (2 * A * Bw);
  k[K_BOUNDARY] = bnd;
  const double tot = ctx->T * (5 * NL * Be + 3 * A * Bw) + bnd;
  if (total) *total = tot;
  for (int q = 0; q < n && q < K_NKINDS; ++q)
    if (per_kind) per_kind[q] = k[q];
  return MMF_OK;
}

mmf_status mmf_destroy(mmf_ctx* ctx) {
  if (!ctx) return MMF_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream || ctx->priv) {
    cudaStreamSynchronize(ctx->stream);
    cudaStreamSynchronize(ctx->priv);
  }
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  if (ctx->graph) cudaGraphDestroy(ctx->graph);
  for (auto& pr : ctx->prof) {
    cudaEventDestroy(pr.a);
    cudaEventDestroy(pr.b);
  }
  for (auto e : ctx->ev_pool) cudaEventDestroy(e);
  if (ctx->ev_user) cudaEventDestroy(ctx->ev_user);
  if (ctx->ev_priv) cudaEventDestroy(ctx->ev_priv);
  if (ctx->comm) nccl_api().CommDestroy(ctx->comm);
  if (ctx->ws_owned) cudaFree(ctx->ws);
  if (ctx->d_int_of_arc) cudaFree(ctx->d_int_of_arc);
  if (ctx->d_export) cudaFree(ctx->d_export);
  if (ctx->pinned) cudaFreeHost(ctx->pinned);
  for (auto e : ctx->ev_d2h)
    if (e) cudaEventDestroy(e);
  if (ctx->priv) cudaStreamDestroy(ctx->priv);
  delete ctx;
  return MMF_OK;
}

}  // extern "C"
