// pipefwd.cuh — TMA-pipelined persistent forward step (kernels >= 5, fp32, one slice of Lp commodities per
// node), and the three-pipeline backward (k_bwd_pipe2, at the end of the file).
//
// Forward kernel of step t (1 <= t <= T), one item per node j (all Lp commodities), Algorithm 2's
// Gauss-Seidel order:
//   (i)   F_{t-1}[a] = K W_{t-1}[a] sum_l alpha_{t-1}[i_a,l] beta_t[j,l] for the in-arcs a -> j  (cor:proj P:1078)
//   (ii)  W_{t-1}[a] <- min(W_{t-1}[a] d[a] / F_{t-1}[a], 1)                         (eq:sinkhorn_graph_Vineq P:861)
//   (iii) alpha_t[j] = sum_{a -> j} alpha_{t-1}[i_a] K W_{t-1}[a] with the updated W    (eq:psi_hat P:1031-1036)
// MODE 1: (i)-(iii); MODE 2: also a4 (t = T); MODE 3 (readout, Jacobi pass): (i) into Fout for every arc and
// (iii) with the current factors, no update.  The multi-GPU Gauss-Seidel exchange (rem:multi_tensor_scheme
// P:1139-1147) splits a step in two launches around the all-reduce of the rank-partial flows: MODE 4 computes
// (i) over the rank's commodities into the compact exchange buffer Fsum (capacitated arcs), k_dual applies (ii)
// to the all-reduced sums, then MODE 5 computes (iii) with the updated factors (MODE 6: also a4).
// (earlier note:)
// (iii) with the current factors, no update.
//
// Each CTA runs NP pipelines; a pipeline is one producer warp and NG consumer groups of GW warps (default 2 x
// (1 x 8)).  The producer stages, per item: the compacted rows alpha_{t-1}[i_a] (nonzero factor) by
// cp.async.bulk into contiguous ring slots (items never wrap), the arc records and dual-update operands by
// cp.async into a prefetch ring (8 items ahead), and prefetches the node's own row beta_t[j] into L2; the
// consumers load that row from global memory at the start of the item.
//
// Consumers compute the per-row terms
//   t_q[c] = alpha_q[c] K W_q 2^-E[c]     (E[c] = max_q exponent of alpha_q[c] K W_q, extended range)
// once, in registers (the row count is a compile-time constant of the code path, switch on n).  Then
//   flows:  F_q = sum_c t_q[c] * beta_lin[c],   beta_lin[c] = beta[j,c] 2^E[c]  (one FMA per element),
//           reduced over the lanes by a transposed butterfly (9 shuffles for up to 8 rows) and over the
//           group's warps in shared memory (fixed order: deterministic);
//   update: one lane per arc applies (ii) branch-free, warp 0 refreshes the arc's records; r_q = W_new / W_old;
//   alpha:  alpha_t[j,c] = 2^E[c] sum_q r_q t_q[c]   (one FMA per element)
// — valid while every |log2 r_q| <= 40 (the dropped terms, below 2^-126 of the old maximum, stay below
// 2^-46 of the new one); otherwise the item is recomputed from shared memory with the new factors.
#pragma once
#include "pipe.cuh"

namespace mmf {

// Pipelines have their own share of the shared memory (row ring, descriptors, record ring): one producer warp
// per SM cannot feed the consumers (its per-item issue of the TMA copies is serial), two can.
constexpr int FWD_NP = 2;  // (pipelines per CTA of the backward's structure)
constexpr int FWD_PW = PIPE_NWC + 1;  // warps per pipeline of the backward (8 consumers + producer)
constexpr int FWD_SD = 8;             // item descriptors per pipeline of the backward (power of two)
#ifndef MMF_FWD_SDF
#define MMF_FWD_SDF 8  // (4: [3] forward 8 % slower, [4] 2 %)
#endif
constexpr int FWD_SDF = MMF_FWD_SDF;  // item descriptors per pipeline of the forward (power of two)
#ifndef MMF_FWD_P
#define MMF_FWD_P 6
#endif
constexpr int FWD_P = MMF_FWD_P;      // record prefetch distance of the forward (items; PIPE_RP > FWD_P + FWD_SDF)
static_assert(PIPE_RP > FWD_P + FWD_SDF, "record-ring slots are read by the consumers until released");
#ifndef MMF_NORM_PACKED
#define MMF_NORM_PACKED 0  // packed normalise-and-store of the pipelined kernels' output rows (measured: no gain)
#endif
#ifndef MMF_BWD_NOWRAP_PATH
#define MMF_BWD_NOWRAP_PATH 1  // compile the backward's never-wrapping item path
#endif
#ifndef MMF_FWD_PREACC
#define MMF_FWD_PREACC 0  // (measured no gain) alpha with the old factors before the barrier, corrected for changed factors after
#endif
#ifndef MMF_FWD_ILP
#define MMF_FWD_ILP 0  // (measured 1% slower) split dependency chains (maximum, alpha accumulation) of the forward's register path
#endif
#ifndef MMF_FWD_LEAN_UPDATE
#define MMF_FWD_LEAN_UPDATE 1  // branch-light dual update in the pipelined forward
#endif
#ifndef MMF_L2PF
#define MMF_L2PF 0  // producers prefetch into L2 the gathered row of the node this many positions ahead (0: off)
#endif
#ifndef MMF_FWD_BPRE
#define MMF_FWD_BPRE 0  // (measured: no gain on [4], 4 % slower on [3]) consumers load the own row beta_t[j] of their next item one item ahead (registers)
#endif
#ifndef MMF_ALT_ORDER
#define MMF_ALT_ORDER 0  // odd steps visit the nodes in reverse order (the rows written last by the previous launch
                         // are still in L2 when the next launch starts)
#endif
__device__ __forceinline__ int alt_node(int x, int N, int t) { return (MMF_ALT_ORDER && (t & 1)) ? N - 1 - x : x; }
#ifndef MMF_FWD_OWNG
#define MMF_FWD_OWNG 1  // 1: the node's own row beta_t[j] is loaded by the consumers from global memory (L2-
                        // prefetched by the producer) instead of staged in the ring
#endif
// forward pipelines: NG consumer groups of GW warps (a group takes every NG-th item of its pipeline; a warp
// owns 32 CPT commodities of the item, SW = 32 GW CPT) + one producer warp
template <int GW, int NG, int NP> constexpr int fwd_threads() { return NP * (GW * NG + 1) * 32; }
// compiled (SW, CPT, GW, NG, NP) combinations: NP pipelines per CTA, each NG groups of GW warps (a warp owns
// CPT commodities per lane); the first of each SW is the default
#define MMF_FWD_COMBOS(X)                                                                           \
  X(1024, 4, 8, 1, 2) X(1024, 4, 8, 1, 3) X(1024, 4, 8, 2, 1) X(1024, 8, 4, 2, 2) X(1024, 8, 4, 3, 1)  \
  X(512, 2, 8, 1, 2)                                                                                \
  X(512, 4, 4, 2, 2)                                                                                \
  X(256, 4, 2, 4, 2)
inline bool fwd_combo_ok(int SW, int gw, int ng, int np) {
#define MMF_FWD_OK(sw, cpt, g, n, q) \
  if (SW == sw && gw == g && ng == n && np == q) return true;
  MMF_FWD_COMBOS(MMF_FWD_OK)
#undef MMF_FWD_OK
  return false;
}

struct __align__(16) FwdHdr {
  unsigned kb[32];  // rows (compacted, nonzero factor): K W significand bits
  unsigned k2[32];  //   ... exponent, packed twice (int16x2)
  int rarc[32];     //   ... arc position of the row
  int rowof[32];    // arcs (all in-arcs, q < na): row index or -1
  int aux[32];      //   ... arc id | bit 31 uncapacitated
  int rtail[32];    //   ... tail node
  unsigned capmask; // bit q: row q's arc is capacitated
  int nr, na, start, end;
  int oslot;        // record-ring slot of the item (its dual-update operands, ArcOps, stay there until released)
  int pad[2];
};

// per consumer group scratch: flow partials (row, warp), double-buffered by the group's item parity (a
// warp may start the group's next item while another still reads this item's partials)
struct FwdGrp {
  float fpart[2][32][PIPE_NWC];
  // the update's results per arc (written by the group's warp 0 between the two barriers of an item)
  float rq[2][32];
  unsigned nkb[2][32], nk2[2][32];
  int big[2];
  int pad[2];
};
#ifndef MMF_FWD_DEDUP
#define MMF_FWD_DEDUP 0  // 1: warp 0 alone evaluates the dual update (second barrier); 0: every warp does
#endif

struct PFwdSmem {
  size_t off_full, off_empty, off_ring, off_oring, off_hdr, off_grp, off_sig, off_exp, total;
};

__host__ __device__ inline PFwdSmem pfwd_smem(int R, int D, int SW, int NG) {
  PFwdSmem m;
  size_t o = 0;
  m.off_full = o;
  o += 8 * (size_t)FWD_SDF;
  m.off_empty = o;
  o += 8 * (size_t)FWD_SDF;
  o = (o + 15) / 16 * 16;
  m.off_ring = o;
  o += (size_t)PIPE_RP * D * 16;
  m.off_oring = o;
  o += (size_t)PIPE_RP * D * 32;
  m.off_hdr = o;
  o += (size_t)FWD_SDF * sizeof(FwdHdr);
  o = (o + 15) / 16 * 16;
  m.off_grp = o;
  o += (size_t)NG * sizeof(FwdGrp);
  o = (o + 127) / 128 * 128;
  m.off_sig = o;
  o += (size_t)R * SW * 4;
  m.off_exp = o;
  o += (size_t)R * SW * 2;
  m.total = (o + 127) / 128 * 128;
  return m;
}

// L2 cache policy for the gathered message rows (option "l2hint"): a row of step t's messages is read by every
// neighbour of its node within a short band of items, while the node's own row and the output rows stream once
__device__ __forceinline__ unsigned long long l2_policy_keep() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s_h(void* dst, const void* src, unsigned bytes, unsigned long long* bar, bool hint,
                                           unsigned long long pol) {
  if (hint)
    bulk_g2s_hint(dst, src, bytes, bar, pol);
  else
    bulk_g2s(dst, src, bytes, bar);
}

__device__ __forceinline__ void bulk_prefetch_l2(const void* g, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(g), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

// sums over the 32 lanes of up to 8 per-lane values at once (transposed butterfly: 4 + 2 + 1 + 1 + 1
// shuffles); the total of value q ends in the lanes with (lane & 3) == 0 and bfly_row(lane) == q
__device__ __forceinline__ int bfly_row(int lane) {
  return ((lane >> 4) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 2) & 1);
}
__device__ __forceinline__ float bfly8(const float* v, int lane) {
  const bool b4 = lane & 16, b3 = lane & 8, b2 = lane & 4;
  float u[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float send = b4 ? v[i] : v[i + 4];
    const float keep = b4 ? v[i + 4] : v[i];
    u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float w[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b3 ? u[i] : u[i + 2];
    const float keep = b3 ? u[i + 2] : u[i];
    w[i] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
  }
  float r = (b2 ? w[1] : w[0]) + __shfl_xor_sync(0xffffffffu, b2 ? w[0] : w[1], 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}

// the same for up to 4 values (2 + 1 + 1 + 1 + 1 shuffles); total of value q in the lanes with (lane & 7) == 0
// and bfly_row4(lane) == q
__device__ __forceinline__ int bfly_row4(int lane) { return ((lane >> 4) & 1) * 2 + ((lane >> 3) & 1); }
__device__ __forceinline__ float bfly4(const float* v, int lane) {
  const bool b4 = lane & 16, b3 = lane & 8;
  float u[2];
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const float send = b4 ? v[i] : v[i + 2];
    const float keep = b4 ? v[i + 2] : v[i];
    u[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
  }
  float r = (b3 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b3 ? u[0] : u[1], 8);
  r += __shfl_xor_sync(0xffffffffu, r, 4);
  r += __shfl_xor_sync(0xffffffffu, r, 2);
  r += __shfl_xor_sync(0xffffffffu, r, 1);
  return r;
}

// W_new = min(W_old d / F, 1) in fp32 (d = 0 -> 0, F = 0 -> 1), W = wm 2^we with wm in [1, 2):
// the ratio d / F is formed in fp32 (its exponent range covers every flow and capacity of the fp32 mode;
// an overflow means W_new = 1), then W_old's significand is applied and the result renormalised.
__device__ __forceinline__ void w_new_f32(float d, float wm0, int we0, float F, float& wm, int& we) {
  if (d == 0.f) {
    wm = 0.f;
    we = EZERO;
    return;
  }
  if (!(F > 0.f)) {
    wm = 1.f;
    we = 0;
    return;
  }
  const float x = wm0 * (d / F);
  if (!(x < 3.0e38f)) {  // (inf) W d / F >= 1
    wm = 1.f;
    we = 0;
    return;
  }
  const unsigned u = __float_as_uint(x);  // x > 0 normal or subnormal
  int e;
  float m;
  if ((u >> 23) == 0u) {  // subnormal: scale up by 2^64
    const unsigned v = __float_as_uint(x * 18446744073709551616.f);
    m = __uint_as_float((v & 0x007fffffu) | 0x3f800000u);
    e = we0 + (int)(v >> 23) - 127 - 64;
  } else {
    m = __uint_as_float((u & 0x007fffffu) | 0x3f800000u);
    e = we0 + (int)(u >> 23) - 127;
  }
  if (e >= 0) {
    wm = 1.f;
    we = 0;
  } else {
    wm = m;
    we = e;
  }
}

// capacity-dual update of the item's in-arcs, lane = arc position.  Every warp of the group evaluates it
// (cheap, and no second barrier is needed); warp 0 alone stores W and refreshes the records.  Returns, in
// the arc's lane, the ratio r = W_new / W_old (linear; 1 for uncapacitated arcs) and the new factor K W;
// *big: some |log2 r| > 40 (the item then takes the recompute path).
struct FwdUpd {
  float rq;
  unsigned nkb, nk2;
};
// the dual-update operands of the lane's arc (plain loads issued at the start of the item: their latency
// overlaps the flow computation)
struct FwdOps {
  float d, wm, Km;
  int we, Ke, eopos, copos;
  float wd, rw;  // W_old d and 1 / W_old (approximate), formed before the item's barrier
};
__device__ __forceinline__ FwdOps fwd_ops(const ArcOps* hops, const FwdHdr& h, int lane) {
  FwdOps o{0.f, 1.f, 0.f, 0, 0, 0, 0, 0.f, 1.f};
  if (lane < h.na) {
    const ArcOps a = hops[lane];
    o.d = a.d;
    o.wm = a.wm;
    o.we = a.we;
    o.Km = a.Km;
    o.Ke = a.Ke;
    o.eopos = a.eopos;
    o.copos = a.copos;
  }
  o.wd = o.wm * o.d;
  o.rw = __fdividef(1.f, o.wm);
  return o;
}
template <int GW>
__device__ __forceinline__ FwdUpd fwd_update(const DevPtrs& p, const FwdHdr& h, const FwdOps& o,
                                             const float (*fp)[PIPE_NWC], int t, int j, int D, int lane, int writer_wg,
                                             bool* big_out) {
  const bool writer = writer_wg == 0;
#if MMF_FWD_LEAN_UPDATE
  // branch-light form (same arithmetic as below up to the rounding of d / F, computed as an approximate
  // quotient (2 ulp) instead of an IEEE one): every arc lane evaluates, selects pick the case
  FwdUpd u{1.f, 0x3f800000u, 0u};
  const bool act = lane < h.na;
  const int aux = act ? h.aux[lane] : -1;
  const int row = act ? h.rowof[lane] : -1;
  const bool cap = aux >= 0;
  if (row >= 0) {
    u.nkb = h.kb[row];
    u.nk2 = h.k2[row];
  }
  float F = 0.f;
  if (cap && row >= 0) {
    if constexpr (GW == 8) {
      const float4 a = *reinterpret_cast<const float4*>(&fp[row][0]);
      const float4 b = *reinterpret_cast<const float4*>(&fp[row][4]);
      F = ((a.x + a.y) + (a.z + a.w)) + ((b.x + b.y) + (b.z + b.w));
    } else {
#pragma unroll
      for (int w = 0; w < GW; ++w) F += fp[row][w];
    }
  }
  const float d = o.d, w0 = o.wm;
  const int e0 = o.we;
  // x = W_old d / F; W_new = min(x, 1) with W = wm 2^we, wm in [1, 2)
  float x = __fdividef(o.wd, F);
  const bool sub = x < 1.17549435e-38f;  // (subnormal or 0: rescale by 2^64)
  x = sub ? x * 18446744073709551616.f : x;
  const unsigned ux = __float_as_uint(x);
  const int ex = e0 + (int)(ux >> 23) - 127 - (sub ? 64 : 0);
  const float mx = __uint_as_float((ux & 0x007fffffu) | 0x3f800000u);
  const bool one = !(F > 0.f) || !(x < 3.0e38f) || ex >= 0;  // (F = 0 or W d / F >= 1)
  const bool zero = d == 0.f;
  float wm = zero ? 0.f : one ? 1.f : mx;
  int we = zero ? EZERO : one ? 0 : ex;
  if (!cap) {
    wm = w0;
    we = e0;
  }
  float km = o.Km * wm;
  int ke = o.Ke + we;
  const bool kz = !(km > 0.f) || ke < -ELIM;
  km = kz ? 0.f : km;
  ke = kz ? -ELIM : min(ke, ELIM);
  bool big = false;
  if (cap) {
    // the new W and the refreshed records are stored by one warp of the group (SP = 1; spreading the stores
    // over the warps measured slower)
    const int wg = writer_wg == 0 ? 0 : 1 + writer_wg;
    ArcKW<float> rr;
    rr.km = km;
    rr.ke = ke;
    rr.aux = aux;
    rr.node = j;
    const size_t ell = (size_t)(t - 1) * p.N * D + (size_t)j * D + lane;
    if (wg == 0) {
      View<TrF32> v(p);
      v.Wm(t - 1)[aux] = wm;
      v.We(t - 1)[aux] = we;
    }
    if (wg == 0) {
      ArcOps* op = (ArcOps*)p.ell_ops + ell;
      op->wm = wm;
      op->we = we;
    }
    if (wg == 0) ((ArcKW<float>*)p.ell_out)[(size_t)(t - 1) * p.N * p.Dout + o.eopos] = rr;
    if (wg == 0) ((ArcKW<float>*)p.outrec)[(size_t)(t - 1) * p.A + o.copos] = rr;
    if (wg == 0) {
      if (!(F == F) || isinf(F)) set_error(p, ERR_NAN, -1, aux);
    }
    rr.node = h.rtail[lane];
    if (wg == 0) ((ArcKW<float>*)p.ell_in)[ell] = rr;
    if (wg == 0) ((ArcKW<float>*)p.inrec)[(size_t)(t - 1) * p.A + aux] = rr;
    if (row >= 0) {
      const int de = we - e0;
      const bool ok = w0 > 0.f && wm > 0.f && de <= 40 && de >= -40;
      big = !ok;
      u.rq = ok ? wm * o.rw * __uint_as_float((unsigned)(de + 127) << 23) : 0.f;
      u.nkb = __float_as_uint(km);
      u.nk2 = pack2(ke);
    }
  }
  *big_out = __any_sync(0xffffffffu, big);
  return u;
#else

  typedef float M;
  View<TrF32> v(p);
  bool big = false;
  FwdUpd u{1.f, 0x3f800000u, 0u};
  if (lane < h.na) {
    const int aux = h.aux[lane];
    const int row = h.rowof[lane];
    if (row >= 0) {
      u.nkb = h.kb[row];
      u.nk2 = h.k2[row];
    }
    if (aux >= 0) {
      const int a = aux;
      float s = 0.f;
      if (row >= 0)
#pragma unroll
        for (int w = 0; w < GW; ++w) s += fp[row][w];
      const float d = o.d, w0 = o.wm;
      const int e0 = o.we;
      float wm;
      int we;
      w_new_f32(d, w0, e0, s, wm, we);
      ArcKW<M> rr;
      kw_clamp<TrF32>(o.Km, o.Ke, wm, we, rr.km, rr.ke);
      if (writer) {
        if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, a);
        v.Wm(t - 1)[a] = wm;
        v.We(t - 1)[a] = we;
        // refresh the step's records: ELL (in: this node's slot; out: the tail's slot) and CSR (in: arc id;
        // out: the arc's out-CSR position)
        rr.aux = aux;
        rr.node = h.rtail[lane];
        ((ArcKW<M>*)p.ell_in)[(size_t)(t - 1) * p.N * D + (size_t)j * D + lane] = rr;
        {
          ArcOps* op = (ArcOps*)p.ell_ops + (size_t)(t - 1) * p.N * D + (size_t)j * D + lane;
          op->wm = wm;
          op->we = we;
        }
        ((ArcKW<M>*)p.inrec)[(size_t)(t - 1) * p.A + a] = rr;
        rr.node = j;
        ((ArcKW<M>*)p.ell_out)[(size_t)(t - 1) * p.N * p.Dout + o.eopos] = rr;
        ((ArcKW<M>*)p.outrec)[(size_t)(t - 1) * p.A + o.copos] = rr;
      }
      if (row >= 0) {
        u.rq = 0.f;
        if (w0 > 0.f && wm > 0.f) {
          const int de = we - e0;
          big = de > 40 || de < -40;
          if (!big) u.rq = __fdividef(wm, w0) * __uint_as_float((unsigned)(de + 127) << 23);
        } else {
          big = true;  // W changed from / to exact zero
        }
        u.nkb = __float_as_uint(rr.km);
        u.nk2 = pack2(rr.ke);
      }
    }
  }
  *big_out = __any_sync(0xffffffffu, big);
  return u;
#endif
}

// alpha from the new factors (gathered from the arcs' lanes), two passes over shared memory
// the own row beta_t[j] scaled to the terms' exponents: beta_lin[c] = beta[j,c] 2^E[c] (flows are bounded
// by the mass: the exponent is clamped to the normal range)
template <int CPT>
__device__ __forceinline__ void beta_lin(const Row<TrF32, CPT>& b, const XPre<CPT>& P, float* bl) {
  if constexpr (CPT % 2 == 0) {  // two at a time: biased exponent e + E + 127 clamped to [0, 254] (0: flushed)
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) {
#if MMF_XPRE_FAST
      const unsigned es = __vmins2(__viaddmax_s16x2((unsigned)b.w[w], P.Ep2[w], 0u), 0x00fe00feu);  // (XPre::set)
#else
      const unsigned es = __vmins2(__vmaxs2(__vaddss2((unsigned)b.w[w], P.Ep2[w]), 0u), 0x00fe00feu);
#endif
      mul2(bl[2 * w], bl[2 * w + 1], b.m[2 * w], b.m[2 * w + 1], __uint_as_float(es << 23),
           __uint_as_float((es >> 16) << 23));
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int es = b.e(c) + P.E[c];
      bl[c] = (es < -126 || !(b.m[c] > 0.f)) ? 0.f : b.m[c] * __uint_as_float((unsigned)(min(es, 127) + 127) << 23);
    }
  }
}

// the flows + update + alpha of one item with N (compile-time) rows; returns (s, Ex)
// ring row of an item's q-th row: items may wrap around the ring
struct RingRows {
  const float* sig;
  const int16_t* sex;
  int start, R, col, SW;
  __device__ __forceinline__ int off(int q) const {
    const int r = start + q;
    return (r >= R ? r - R : r) * SW + col;
  }
};
// an item's rows are contiguous ring slots start .. start + n - 1 (the producers never wrap an item: they
// skip to slot 0 instead), so row q is at a compile-time offset from the item's base
template <int SW> struct RingRowsF {
  const float* sig;
  const int16_t* sex;
  __device__ __forceinline__ RingRowsF(const RingRows& r)
      : sig(r.sig + r.start * SW + r.col), sex(r.sex + r.start * SW + r.col) {}
  __device__ __forceinline__ int off(int q) const { return q * SW; }
};

// the dual update's per-arc results as every warp of the group sees them: from the group's shared scratch
// (MMF_FWD_DEDUP: written by warp 0) or from the arcs' lanes (every warp evaluated the update)
struct UpdView {
  const float* rq_;
  const unsigned *kb_, *k2_;
  FwdUpd u;
  __device__ __forceinline__ float rq(int src) const {
    return MMF_FWD_DEDUP ? rq_[src] : __shfl_sync(0xffffffffu, u.rq, src);
  }
  __device__ __forceinline__ unsigned kb(int src) const {
    return MMF_FWD_DEDUP ? kb_[src] : __shfl_sync(0xffffffffu, u.nkb, src);
  }
  __device__ __forceinline__ unsigned k2(int src) const {
    return MMF_FWD_DEDUP ? k2_[src] : __shfl_sync(0xffffffffu, u.nk2, src);
  }
};
// the update phase of an item (after the flow partials are in fp and the group's barrier has passed)
template <int GW>
__device__ __forceinline__ UpdView fwd_update_phase(const DevPtrs& p, const FwdHdr& h, const FwdOps& o0,
                                                    const ArcOps* hops, FwdGrp& G, int par, int t, int j, int D,
                                                    int lane, int wg, int bar_id, bool* big) {
  UpdView v;
#if MMF_FWD_DEDUP
  if (wg == 0) {
    const FwdOps o = fwd_ops(hops, h, lane);
    bool b;
    const FwdUpd u = fwd_update<GW>(p, h, o, G.fpart[par], t, j, D, lane, 0, &b);
    G.rq[par][lane] = u.rq;
    G.nkb[par][lane] = u.nkb;
    G.nk2[par][lane] = u.nk2;
    if (lane == 0) G.big[par] = b;
  }
  named_bar(bar_id, GW * 32);
  v.rq_ = G.rq[par];
  v.kb_ = G.nkb[par];
  v.k2_ = G.nk2[par];
  *big = G.big[par] != 0;
#else
  v.u = fwd_update<GW>(p, h, o0, G.fpart[par], t, j, D, lane, wg, big);
#endif
  return v;
}

template <int MODE> constexpr bool fwd_has_flows() { return MODE <= 4; }   // (MODE 5, 6: alpha only)
template <int MODE> constexpr bool fwd_alpha_only() { return MODE == 5 || MODE == 6; }
// exchange mode (MODE 4): the rank-partial flow of every capacitated in-arc (0 for zero-factor arcs) -> Fsum[fpos]
template <int GW>
__device__ __forceinline__ void fwd_exchange_store(const DevPtrs& p, const FwdHdr& h, const float (*fp)[PIPE_NWC],
                                                   int lane, int wg) {
  if (wg != 0 || lane >= h.na) return;
  const int aux = h.aux[lane];
  if (aux < 0) return;  // (uncapacitated at this step: not exchanged)
  const int row = h.rowof[lane];
  float F = 0.f;
  if (row >= 0)
#pragma unroll
    for (int w = 0; w < GW; ++w) F += fp[row][w];
  ((float*)p.Fsum)[p.fpos[aux]] = F;
}

// readout mode (MODE 3): the flow of every in-arc of the item (0 for zero-factor arcs) -> Fout[t - 1][arc], by
// warp 0; the dual update is skipped and alpha uses the current factors
template <int GW>
__device__ __forceinline__ void fwd_readout_store(const DevPtrs& p, const FwdHdr& h, const float (*fp)[PIPE_NWC],
                                                  int t, int lane, int wg) {
  if (wg != 0 || lane >= h.na) return;
  const int row = h.rowof[lane];
  float F = 0.f;
  if (row >= 0)
#pragma unroll
    for (int w = 0; w < GW; ++w) F += fp[row][w];
  ((float*)p.Fout)[(size_t)(t - 1) * p.A + (h.aux[lane] & 0x7fffffff)] = F;
}
__device__ __forceinline__ UpdView fwd_old_view(const FwdHdr& h, int lane) {
  UpdView v;
  v.u = FwdUpd{1.f, 0x3f800000u, 0u};
  if (lane < h.na && h.rowof[lane] >= 0) {
    v.u.nkb = h.kb[h.rowof[lane]];
    v.u.nk2 = h.k2[h.rowof[lane]];
  }
  return v;
}

// alpha from the new factors, two passes over shared memory
template <int CPT, class RW>
__device__ __forceinline__ void fwd_alpha_new(const RW& rw, const FwdHdr& h, const UpdView& u, int nr, float* s,
                                              int* Ex) {
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < nr; ++q) {
    const int src = h.rarc[q];
    const unsigned kb = u.kb(src), k2 = u.k2(src);
    if (!(__uint_as_float(kb) > 0.f)) continue;
    Row<TrF32, CPT> x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xmax_add<CPT>(E2, x, k2, k2_to_ke(k2));
  }
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
  for (int q = 0; q < nr; ++q) {
    const int src = h.rarc[q];
    const unsigned kb = u.kb(src), k2 = u.k2(src);
    if (!(__uint_as_float(kb) > 0.f)) continue;
    Row<TrF32, CPT> x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xacc<CPT>(x, kb, k2, k2_to_ke(k2), P, s);
  }
}

// a lane's CPT significands / packed exponent words of a shared-memory row
template <int CPT> __device__ __forceinline__ void load_sig(const float* pm, float* m) {
  typedef typename VecM<float, CPT>::T VM;
  const VM vm = *reinterpret_cast<const VM*>(pm);
  const float* sm = reinterpret_cast<const float*>(&vm);
#pragma unroll
  for (int c = 0; c < CPT; ++c) m[c] = sm[c];
}
template <int CPT> __device__ __forceinline__ void load_exps(const int16_t* pe, int* w) {
  typedef typename VecE<int16_t, CPT>::T VE;
  const VE ve = *reinterpret_cast<const VE*>(pe);
  const int* sw = reinterpret_cast<const int*>(&ve);
#pragma unroll
  for (int k = 0; k < CPT / 2; ++k) w[k] = sw[k];
}
// in place: m[c] <- m[c] K W 2^(e[c] + ke - E[c]) (xterms on separately loaded words)
template <int CPT>
__device__ __forceinline__ void xterms_w(const int* w, float* m, unsigned kb, unsigned k2, const XPre<CPT>& P) {
#pragma unroll
  for (int k = 0; k < CPT / 2; ++k) {
    const unsigned u = __viaddmax_s16x2((unsigned)w[k], k2, P.Lo2[k]);
    const unsigned d2 = __viaddmax_s16x2(u, P.nE2[k], 0xff82ff82u);
    mul2(m[2 * k], m[2 * k + 1], m[2 * k], m[2 * k + 1], __uint_as_float(kb + (d2 << 23)),
         __uint_as_float(kb + MMF_HI23(d2)));
  }
}

// register path, N (compile-time) rows held in registers: the maximum exponent, the terms in place
template <int CPT, int GW, int N, int MODE>
__device__ __forceinline__ void fwd_body(const DevPtrs& p, const RingRows& rw0, const FwdHdr& h, const ArcOps* hops,
                                         const Row<TrF32, CPT>& bown, FwdGrp& G, int par, int t, int j, int D,
                                         int lane, int wg, int bar_id, float* s, int* Ex) {
  typedef Row<TrF32, CPT> R_;
  constexpr int NQ = N > 0 ? N : 1;
  const RingRowsF<32 * GW * CPT> rw(rw0);
  const FwdOps o0 = MMF_FWD_DEDUP ? FwdOps{} : fwd_ops(hops, h, lane);
  float tq[NQ][CPT];
  XPre<CPT> P;
  {
    int xw[NQ][CPT / 2];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const int o = rw.off(q);
      load_exps<CPT>(rw.sex + o, xw[q]);
      load_sig<CPT>(rw.sig + o, tq[q]);
    }
    unsigned E2[CPT / 2];
#if MMF_FWD_ILP
    {  // two interleaved maximum chains (halves the dependency depth)
      unsigned Eb[CPT / 2];
      xmax_init<CPT>(E2);
      xmax_init<CPT>(Eb);
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const unsigned k2 = h.k2[q];
#pragma unroll
        for (int k = 0; k < CPT / 2; ++k) {
          if (q & 1) Eb[k] = __viaddmax_s16x2((unsigned)xw[q][k], k2, Eb[k]);
          else E2[k] = __viaddmax_s16x2((unsigned)xw[q][k], k2, E2[k]);
        }
      }
#pragma unroll
      for (int k = 0; k < CPT / 2; ++k) E2[k] = __vmaxs2(E2[k], Eb[k]);
    }
#else
    xmax_init<CPT>(E2);
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const unsigned k2 = h.k2[q];
#pragma unroll
      for (int k = 0; k < CPT / 2; ++k) E2[k] = __viaddmax_s16x2((unsigned)xw[q][k], k2, E2[k]);
    }
#endif
    P.set(E2);
#pragma unroll
    for (int q = 0; q < N; ++q) xterms_w<CPT>(xw[q], tq[q], h.kb[q], h.k2[q], P);
  }
  float bl[CPT];
  if constexpr (!fwd_has_flows<MODE>()) {
  } else if constexpr (MMF_FWD_OWNG) {
    beta_lin<CPT>(bown, P, bl);
  } else {
    R_ b;
    const int o = rw.off(N);
    b.load(rw.sig + o, rw.sex + o);  // own row beta_t[j]
    beta_lin<CPT>(b, P, bl);
  }
  const unsigned cap = h.capmask;
  float (*fp)[PIPE_NWC] = G.fpart[par];
  if (p.diag == 2) {  // diagnostics (results invalid): alpha with the old factors only
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = 0.f;
      Ex[c] = P.E[c];
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) s[c] += tq[q][c] * bl[c];
    return;
  }
  if (fwd_has_flows<MODE>() && N > 0 && cap != 0u) {
    constexpr int NF = N <= 4 ? 4 : 8;
    float f[NF];
#pragma unroll
    for (int q = 0; q < NF; ++q) {
      f[q] = 0.f;
      if (q < N) {
#if MMF_F2
        float f0 = 0.f, f1 = 0.f;  // (pairs of commodities: two partial sums)
#pragma unroll
        for (int c = 0; c < CPT; c += 2) fma2(f0, f1, tq[q < N ? q : 0][c], tq[q < N ? q : 0][c + 1], bl[c], bl[c + 1]);
        f[q] = f0 + f1;
#else
#pragma unroll
        for (int c = 0; c < CPT; ++c) f[q] = fmaf(tq[q < N ? q : 0][c], bl[c], f[q]);
#endif
      }
    }
    if constexpr (NF == 4) {
      const float r = bfly4(f, lane);
      const int row = bfly_row4(lane);
      if ((lane & 7) == 0 && row < N && ((cap >> row) & 1u)) fp[row][wg] = r;
    } else {
      const float r = bfly8(f, lane);
      const int row = bfly_row(lane);
      if ((lane & 3) == 0 && row < N && ((cap >> row) & 1u)) fp[row][wg] = r;
    }
  }
#if MMF_FWD_PREACC && !MMF_FWD_DEDUP
  // alpha with the old factors, accumulated before the barrier (off the update's critical path); after the
  // update only the rows whose factor changed (ratio r != 1: saturated arcs) are corrected by (r - 1) t_q
  float sp[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) sp[c] = 0.f;
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int c = 0; c < CPT; ++c) sp[c] += tq[q][c];
#endif
  if constexpr (fwd_has_flows<MODE>()) named_bar(bar_id, GW * 32);
  if constexpr (MODE == 4) {  // exchange: the rank-partial flows out, no alpha
    fwd_exchange_store<GW>(p, h, fp, lane, wg);
    return;
  }
  if constexpr (MODE == 3 || fwd_alpha_only<MODE>()) {  // readout: flows out, alpha with the current factors
    if constexpr (MODE == 3) fwd_readout_store<GW>(p, h, fp, t, lane, wg);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = 0.f;
      Ex[c] = P.E[c];
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) s[c] += tq[q][c];
    return;
  }
  if (p.diag == 3) {  // diagnostics (results invalid): flows and their reduction, no dual update
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = fp[0][c];
      Ex[c] = P.E[c];
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int c = 0; c < CPT; ++c) s[c] = fmaf(tq[q][c], bl[c], s[c]);
    return;
  }
  bool big;
  const UpdView u = fwd_update_phase<GW>(p, h, o0, hops, G, par, t, j, D, lane, wg, bar_id, &big);
  if (!big) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = 0.f;
      Ex[c] = P.E[c];
    }
#if MMF_FWD_PREACC && !MMF_FWD_DEDUP
    const unsigned chg = __ballot_sync(0xffffffffu, lane < h.na && u.u.rq != 1.f);
#pragma unroll
    for (int c = 0; c < CPT; ++c) s[c] = sp[c];
    if (chg) {
#pragma unroll
      for (int q = 0; q < N; ++q) {
        const int src = h.rarc[q];
        const float r = __shfl_sync(0xffffffffu, u.u.rq, src) - 1.f;
        if ((chg >> src) & 1u)
#pragma unroll
          for (int c = 0; c < CPT; ++c) s[c] = fmaf(r, tq[q][c], s[c]);
      }
    }
#elif MMF_FWD_ILP
    float s2[CPT];  // (two interleaved accumulation chains)
#pragma unroll
    for (int c = 0; c < CPT; ++c) s2[c] = 0.f;
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float r = u.rq(h.rarc[q]);
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        if (q & 1) s2[c] = fmaf(r, tq[q][c], s2[c]);
        else s[c] = fmaf(r, tq[q][c], s[c]);
      }
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) s[c] += s2[c];
#else
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float r = u.rq(h.rarc[q]);
#pragma unroll
      for (int c = 0; c < CPT; c += 2) fma2(s[c], s[c + 1], r, r, tq[q][c], tq[q][c + 1]);
    }
#endif
  } else {  // large ratios: recompute from shared memory with the new factors
    fwd_alpha_new<CPT>(rw, h, u, N, s, Ex);
  }
}

// any row count (more than the register path's): streaming flows, then the update, then alpha from shared
// memory
template <int CPT, int GW, int MODE>
__device__ __forceinline__ void fwd_body_any(const DevPtrs& p, const RingRows& rw0, const FwdHdr& h, const ArcOps* hops,
                                             const Row<TrF32, CPT>& bown, FwdGrp& G, int par, int t, int j, int D,
                                             int lane, int wg, int bar_id, int nr, float* s, int* Ex) {
  const RingRowsF<32 * GW * CPT> rw(rw0);
  typedef Row<TrF32, CPT> R_;
  const FwdOps o0 = MMF_FWD_DEDUP ? FwdOps{} : fwd_ops(hops, h, lane);
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < nr; ++q) {
    R_ x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xmax_add<CPT>(E2, x, h.k2[q], k2_to_ke(h.k2[q]));
  }
  XPre<CPT> P;
  P.set(E2);
  float bl[CPT];
  if constexpr (!fwd_has_flows<MODE>()) {
    fwd_alpha_new<CPT>(rw, h, fwd_old_view(h, lane), nr, s, Ex);  // (alpha only: the current factors)
    return;
  } else if constexpr (MMF_FWD_OWNG) {
    beta_lin<CPT>(bown, P, bl);
  } else {
    R_ b;
    b.load(rw.sig + rw.off(nr), rw.sex + rw.off(nr));
    beta_lin<CPT>(b, P, bl);
  }
  float (*fp)[PIPE_NWC] = G.fpart[par];
  for (int q = 0; q < nr; ++q) {
    if (!((h.capmask >> q) & 1u)) continue;
    R_ x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    float tt[CPT];
    xterms<CPT>(x, h.kb[q], h.k2[q], k2_to_ke(h.k2[q]), P, tt);
    float f = 0.f;
#pragma unroll
    for (int c = 0; c < CPT; ++c) f = fmaf(tt[c], bl[c], f);
    f = warp_sum<float>(f);
    if (lane == 0) fp[q][wg] = f;
  }
  named_bar(bar_id, GW * 32);
  if constexpr (MODE == 4) {
    fwd_exchange_store<GW>(p, h, fp, lane, wg);
    return;
  }
  if constexpr (MODE == 3) {
    fwd_readout_store<GW>(p, h, fp, t, lane, wg);
    fwd_alpha_new<CPT>(rw, h, fwd_old_view(h, lane), nr, s, Ex);
    return;
  }
  bool big;
  const UpdView u = fwd_update_phase<GW>(p, h, o0, hops, G, par, t, j, D, lane, wg, bar_id, &big);
  fwd_alpha_new<CPT>(rw, h, u, nr, s, Ex);
}

template <int CPT, int GW, int NG, int NP, int MODE>
__global__ void __launch_bounds__(fwd_threads<GW, NG, NP>(), 1) k_fwd_pipe(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  constexpr int SW = 32 * GW * CPT;
  constexpr int PW = GW * NG + 1;                             // warps per pipeline
  constexpr int NMAX = fwd_threads<GW, NG, NP>() > 640 ? 5 : CPT >= 8 && fwd_threads<GW, NG, NP>() > 448 ? 6 : 8;
  extern __shared__ __align__(16) unsigned char smem_all[];
  const PFwdSmem L = pfwd_smem(pc.R, pc.D, SW, NG);
  const int pl = (threadIdx.x >> 5) / PW;                     // pipeline of this warp
  unsigned char* smem = smem_all + (size_t)pl * L.total;      // its share of the shared memory
  const int jstep = NP * gridDim.x, j0 = blockIdx.x + pl * gridDim.x;
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  ArcOps* oring = (ArcOps*)(smem + L.off_oring);
  FwdHdr* hdr = (FwdHdr*)(smem + L.off_hdr);
  FwdGrp* grps = (FwdGrp*)(smem + L.off_grp);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % PW;  // (warp within the pipeline)
  const int D = pc.D, R = pc.R;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < FWD_SDF; ++s) {
      mbar_init(&full[s], 1);          // expect_tx arrive (all rows land by TMA)
      mbar_init(&empty[s], GW);        // one consumer group per item
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);

  if (warp == GW * NG) {  // ---------------- producer
    const ArcKW<M>* ell = (const ArcKW<M>*)p.ell_in + (size_t)(t - 1) * p.N * D;
    const M* gm = v.am(t - 1);
    const E* ge = v.ae(t - 1);
    const M* bm = v.bm(t);
    const E* be = v.be(t);
    const M* dc = v.dcap(t - 1);
    const M* Wm = v.Wm(t - 1);
    const int* We = v.We(t - 1);
    const M* Km = v.Km(t - 1);
    const int* Ke = v.Ke(t - 1);
    const unsigned long long pol = l2_policy_keep();
    int pnode = j0, pslot = 0;
    auto prefetch = [&]() {
      const int pn = alt_node(pnode, p.N, t);
      if (pnode < p.N && lane < D) {
        cp_async16(&ring[pslot * D + lane], ell + (size_t)pn * D + lane);
        const ArcOps* go = (const ArcOps*)p.ell_ops + (size_t)(t - 1) * p.N * D + (size_t)pn * D + lane;
        cp_async16(&oring[pslot * D + lane], go);
        cp_async16((char*)&oring[pslot * D + lane] + 16, (const char*)go + 16);
      }
      if (MMF_FWD_OWNG && fwd_has_flows<MODE>() && pnode < p.N && lane >= 30) {  // the item's own row beta_t[j] -> L2 (read at its start)
        const size_t g = (size_t)pn * p.Lp;
        if (lane == 30) bulk_prefetch_l2(bm + g, SW * 4);
        else bulk_prefetch_l2(be + g, SW * 2);
      }
      cp_async_commit();
      pnode += jstep;
      pslot = pslot + 1 == PIPE_RP ? 0 : pslot + 1;
    };
#pragma unroll 1
    for (int k = 0; k < FWD_P; ++k) prefetch();
    RowRing rr;
    auto release = [&]() {
      const int ds = rr.kold & (FWD_SDF - 1);
      mbar_wait(&empty[ds], (rr.kold / FWD_SDF) & 1);
      rr.tail = (unsigned)hdr[ds].end;
      ++rr.kold;
    };
    int k = 0, cslot = 0;
    for (int jpos = j0; jpos < p.N; jpos += jstep, ++k) {
      const int j = alt_node(jpos, p.N, t);
      cp_async_wait<FWD_P - 1>();
      __syncwarp();
      ArcKW<M> r;
      r.node = -1;
      r.km = M(0);
      r.ke = 0;
      r.aux = 0;
      if (lane < D) r = ring[cslot * D + lane];
      const int oslot = cslot;
      cslot = cslot + 1 == PIPE_RP ? 0 : cslot + 1;
      __syncwarp();
      const bool valid = lane < D && r.node >= 0;
      const bool ok = valid && r.km > M(0);
      const unsigned vbal = __ballot_sync(0xffffffffu, valid);
      const unsigned obal = __ballot_sync(0xffffffffu, ok);
      const unsigned cbal = __ballot_sync(0xffffffffu, ok && (r.aux >= 0 || MODE == 3));  // (readout: every arc)
      const int na = __popc(vbal), nr = __popc(obal);
      while (rr.kold <= k - FWD_SDF) release();
      constexpr int OWN = MMF_FWD_OWNG ? 0 : 1;  // ring rows per item: nr (+ the own row)
      const int nrow = nr + OWN;
      {  // items never wrap: skip the ring's last rpos..R-1 slots (counted with this item) if it does not fit
        unsigned pad = rr.rpos + nrow > R ? (unsigned)(R - rr.rpos) : 0u;
        while (rr.head + pad + (unsigned)nrow - rr.tail > (unsigned)R && rr.kold < k) release();  // (R >= D + OWN)
        if (rr.head + pad + (unsigned)nrow - rr.tail > (unsigned)R) pad = 0u;  // (all released: start over at 0)
        if (rr.rpos + nrow > R) rr.rpos = 0;
        rr.head += pad;
      }
      const int ds = k & (FWD_SDF - 1);
      FwdHdr& h = hdr[ds];
      const int rs = __popc(obal & ((1u << lane) - 1u));
      MMF_DASSERT(rr.rpos >= 0 && rr.rpos + nrow <= R);                 // (items never wrap)
      MMF_DASSERT(!valid || (r.node >= 0 && r.node < p.N && lane < D));  // (ELL record: a node of the graph)
      if (ok) {
        h.kb[rs] = __float_as_uint(r.km);
        h.k2[rs] = pack2(r.ke);
        h.rarc[rs] = lane;
      }
      if (valid) {
        h.rowof[lane] = ok ? rs : -1;
        h.aux[lane] = r.aux;
        h.rtail[lane] = r.node;
      }
      // capmask over rows (row order = lane order of the nonzero-factor arcs)
      const unsigned cm = __reduce_or_sync(0xffffffffu, ok && ((cbal >> lane) & 1u) ? 1u << rs : 0u);
      if (lane == 0) {
        h.capmask = cm;
        h.nr = nr;
        h.na = na;
        h.start = rr.rpos;
        h.end = (int)(rr.head + (unsigned)nrow);
        h.oslot = oslot;
      }
      __syncwarp();  // (the header writes of every lane precede lane 0's releasing arrive)
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)(nr + OWN) * (unsigned)SW * 6u);
      __syncwarp();
      prefetch();
      if (ok) {
        const size_t g = (size_t)r.node * p.Lp;
        const int q = rr.rpos + rs;
        bulk_g2s_h(sig + q * SW, gm + g, SW * 4, &full[ds], p.l2hint, pol);
        bulk_g2s_h(sex + q * SW, ge + g, SW * 2, &full[ds], p.l2hint, pol);
      }
      if (!MMF_FWD_OWNG && lane == 31) {  // the node's own beta_t row -> slot nr
        const size_t g = (size_t)j * p.Lp;
        const int q = rr.rpos + nr;
        bulk_g2s(sig + q * SW, bm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, be + g, SW * 2, &full[ds]);
      }
      if (MMF_L2PF > 0 && lane >= 28 && lane < 30 && j + MMF_L2PF < p.N) {  // first touch of an upcoming row
        const size_t g = (size_t)(j + MMF_L2PF) * p.Lp;
        if (lane == 28) bulk_prefetch_l2(gm + g, SW * 4);
        else bulk_prefetch_l2(ge + g, SW * 2);
      }
      rr.head += (unsigned)nrow;
      rr.rpos += nrow;
      if (rr.rpos >= R) rr.rpos = 0;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers
  const int grp = warp / GW, wg = warp % GW;
  FwdGrp& G = grps[grp];
  const int col = wg * 32 * CPT + lane * CPT;
  const int bar_id = 1 + pl * NG + grp;
  int k = grp;
  Row<TrF32, CPT> bnext;  // (MMF_FWD_BPRE) own row of the group's next item, loaded one item ahead
  if (MMF_FWD_OWNG && MMF_FWD_BPRE && j0 + grp * jstep < p.N) {
    const size_t g = (size_t)alt_node(j0 + grp * jstep, p.N, t) * p.Lp + col;
    bnext.load(v.bm(t) + g, v.be(t) + g);
  }
  for (int jpos = j0 + grp * jstep; jpos < p.N; jpos += NG * jstep, k += NG) {
    const int j = alt_node(jpos, p.N, t);
    const int ds = k & (FWD_SDF - 1);
    Row<TrF32, CPT> bown;  // own row beta_t[j] (global; its latency overlaps the wait and the row math)
    if constexpr (MMF_FWD_OWNG && MMF_FWD_BPRE) {
      bown = bnext;
      if (jpos + NG * jstep < p.N) {
        const size_t g = (size_t)alt_node(jpos + NG * jstep, p.N, t) * p.Lp + col;
        bnext.load(v.bm(t) + g, v.be(t) + g);
      }
    } else if constexpr (MMF_FWD_OWNG && fwd_has_flows<MODE>()) {
      const size_t g = (size_t)j * p.Lp + col;
      bown.load(v.bm(t) + g, v.be(t) + g);
    }
    mbar_wait_sleep(&full[ds], (k / FWD_SDF) & 1);
    const FwdHdr& h = hdr[ds];
    const ArcOps* hops = oring + h.oslot * D;
    MMF_DASSERT(h.start >= 0 && h.start + h.nr <= R && h.nr <= h.na && h.na <= D && h.oslot < PIPE_RP);
    if (pc.dry == 1) {  // diagnostics: delivery rate of the producer / TMA alone
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ds]);
      continue;
    }
    const int nr = h.nr;
    const RingRows rw{sig, sex, h.start, R, col, SW};
    const int par = (k / NG) & 1;
    M s[CPT];
    int Ex[CPT];
    switch (nr) {
      case 0: fwd_body<CPT, GW, 0, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 1: fwd_body<CPT, GW, 1, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 2: fwd_body<CPT, GW, 2, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 3: fwd_body<CPT, GW, 3, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 4: fwd_body<CPT, GW, 4, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 5: fwd_body<CPT, GW, 5, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 6: fwd_body<CPT, GW, 6, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 7:
        if constexpr (NMAX >= 7) fwd_body<CPT, GW, 7, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex);
        else fwd_body_any<CPT, GW, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, nr, s, Ex);
        break;
      case 8:
        if constexpr (NMAX >= 8) fwd_body<CPT, GW, 8, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, s, Ex);
        else fwd_body_any<CPT, GW, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, nr, s, Ex);
        break;
      default: fwd_body_any<CPT, GW, MODE>(p, rw, h, hops, bown, G, par, t, j, D, lane, wg, bar_id, nr, s, Ex); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    // s is 0 or a normal float (ratios are within 2^+-40 of the previous terms): bit-level normalisation
    const size_t g = (size_t)j * p.Lp + col;
    if constexpr (MODE == 4) {  // (exchange: flows only)
    } else if constexpr (MODE == 2 || MODE == 6) {  // a4: UT = muT ./ alpha_T -> beta_T
      Lane<M, E, CPT> a;
      norm_lane<TrF32, CPT, false>(p, s, Ex, a, col, j);
      a.store(v.am(t) + g, v.ae(t) + g);
      Lane<M, E, CPT> ut;
      boundary_lane<TrF32, CPT>(p, 1, j, col, g, a, ut);
      ut.store(v.bm(p.T) + g, v.be(p.T) + g);
    } else if constexpr (MMF_NORM_PACKED) {
      norm_store_f32<CPT>(p, s, Ex, v.am(t) + g, v.ae(t) + g, col, j);
    } else {
      Lane<M, E, CPT> a;
      norm_lane<TrF32, CPT, false>(p, s, Ex, a, col, j);
      a.store(v.am(t) + g, v.ae(t) + g);
    }
  }
}

}  // namespace mmf

namespace mmf {

// ------------------------------------------------------------------------------------------------
// Pipelined backward with FWD_NP producer/consumer pipelines per CTA (the structure of k_fwd_pipe):
//   beta_t[i, slice] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a, slice]   (eq:psi P:1038-1043)
// items = (node, slice) pairs in grid-stride order, rows staged by TMA bulk copies into each pipeline's
// ring (items may wrap), arc records prefetched with cp.async.
template <int CPT, int N, class RW>
__device__ __forceinline__ void ring_sum_n(const RW& rw, const PipeHdr& h, float* s, int* Ex) {
  Row<TrF32, CPT> x[N > 0 ? N : 1];
#pragma unroll
  for (int q = 0; q < N; ++q) x[q].load(rw.sig + rw.off(q), rw.sex + rw.off(q));
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
#pragma unroll
  for (int q = 0; q < N; ++q) xmax_add<CPT>(E2, x[q], h.k2[q], k2_to_ke(h.k2[q]));
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
#pragma unroll
  for (int q = 0; q < N; ++q) xacc<CPT>(x[q], h.kb[q], h.k2[q], k2_to_ke(h.k2[q]), P, s);
}
template <int CPT, class RW>
__device__ __forceinline__ void ring_sum_any(const RW& rw, const PipeHdr& h, int n, float* s, int* Ex) {
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < n; ++q) {
    Row<TrF32, CPT> x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xmax_add<CPT>(E2, x, h.k2[q], k2_to_ke(h.k2[q]));
  }
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
  for (int q = 0; q < n; ++q) {
    Row<TrF32, CPT> x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xacc<CPT>(x, h.kb[q], h.k2[q], k2_to_ke(h.k2[q]), P, s);
  }
}
template <int CPT, class RW>
__device__ __forceinline__ void ring_sum(const RW& rw, const PipeHdr& h, int n, float* s, int* Ex) {
  switch (n) {
    case 0: ring_sum_n<CPT, 0>(rw, h, s, Ex); break;
    case 1: ring_sum_n<CPT, 1>(rw, h, s, Ex); break;
    case 2: ring_sum_n<CPT, 2>(rw, h, s, Ex); break;
    case 3: ring_sum_n<CPT, 3>(rw, h, s, Ex); break;
    case 4: ring_sum_n<CPT, 4>(rw, h, s, Ex); break;
    case 5: ring_sum_n<CPT, 5>(rw, h, s, Ex); break;
    case 6: ring_sum_n<CPT, 6>(rw, h, s, Ex); break;
    case 7: ring_sum_n<CPT, 7>(rw, h, s, Ex); break;
    case 8: ring_sum_n<CPT, 8>(rw, h, s, Ex); break;
    default: ring_sum_any<CPT>(rw, h, n, s, Ex); break;
  }
}

constexpr int BWD_NP = 3;  // pipelines per CTA of the backward (56 registers per thread: three fit)
constexpr int BWD_THREADS = BWD_NP * FWD_PW * 32;

template <int CPT>
__global__ void __launch_bounds__(BWD_THREADS, 1) k_bwd_pipe2(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  constexpr int SW = pipe_sw<CPT>();
  extern __shared__ __align__(16) unsigned char smem_all[];
  const PipeSmem L = pipe_smem(pc.R, FWD_SD, pc.D, SW);
  const size_t share = (L.total + 127) / 128 * 128;
  const int pl = (threadIdx.x >> 5) / FWD_PW;
  unsigned char* smem = smem_all + (size_t)pl * share;
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  PipeHdr* hdr = (PipeHdr*)(smem + L.off_hdr);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % FWD_PW;
  const int D = pc.D, R = pc.R;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < FWD_SD; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PIPE_NWC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);
  const ArcKW<M>* ell = (const ArcKW<M>*)p.ell_out + (size_t)t * p.N * D;
  const M* gm = v.bm(t + 1);
  const E* ge = v.be(t + 1);
  const int step = BWD_NP * gridDim.x, item0 = blockIdx.x + pl * gridDim.x;

  if (warp == PIPE_NWC) {  // ---------------- producer
    ItemIt pf, cur;
    pf.init(item0, step, pc.ns);
    cur = pf;
    const unsigned long long pol = l2_policy_keep();
    int pslot = 0;
    auto prefetch = [&]() {
      if (pf.node < p.N && lane < D)
        cp_async16(&ring[pslot * D + lane], ell + (size_t)alt_node(pf.node, p.N, t) * D + lane);
      cp_async_commit();
      pf.next();
      pslot = pslot + 1 == PIPE_RP ? 0 : pslot + 1;
    };
#pragma unroll 1
    for (int k = 0; k < PIPE_P; ++k) prefetch();
    RowRing rr;
    auto release = [&]() {
      const int ds = rr.kold & (FWD_SD - 1);
      mbar_wait(&empty[ds], (rr.kold / FWD_SD) & 1);
      rr.tail = (unsigned)hdr[ds].end;
      ++rr.kold;
    };
    int cslot = 0;
    for (int k = 0; cur.node < p.N; ++k, cur.next()) {
      cp_async_wait<PIPE_P - 1>();
      __syncwarp();
      ArcKW<M> r;
      r.node = -1;
      r.km = M(0);
      r.ke = 0;
      if (lane < D) r = ring[cslot * D + lane];
      cslot = cslot + 1 == PIPE_RP ? 0 : cslot + 1;
      __syncwarp();
      prefetch();
      const bool ok = lane < D && r.node >= 0 && r.km > M(0);
      const unsigned bal = __ballot_sync(0xffffffffu, ok);
      const int n = __popc(bal);
      while (rr.kold <= k - FWD_SD) release();
      {  // items never wrap (as in the forward) unless pc.wrap
        unsigned pad = !pc.wrap && rr.rpos + n > R ? (unsigned)(R - rr.rpos) : 0u;
        while (rr.head + pad + (unsigned)n - rr.tail > (unsigned)R && rr.kold < k) release();  // (R >= D)
        if (rr.head + pad + (unsigned)n - rr.tail > (unsigned)R) pad = 0u;
        if (!pc.wrap && rr.rpos + n > R) rr.rpos = 0;
        rr.head += pad;
      }
      const int ds = k & (FWD_SD - 1);
      const int slot = __popc(bal & ((1u << lane) - 1u));
      MMF_DASSERT(!ok || (r.node >= 0 && r.node < p.N));
      MMF_DASSERT(rr.rpos >= 0 && rr.rpos < R && n <= R);
      if (ok) {
        hdr[ds].kb[slot] = __float_as_uint(r.km);
        hdr[ds].k2[slot] = pack2(r.ke);
      }
      if (lane == 0) {
        hdr[ds].n = n;
        hdr[ds].start = rr.rpos;
        hdr[ds].end = (int)(rr.head + (unsigned)n);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)n * (unsigned)SW * 6u);
      __syncwarp();
      if (ok) {
        const size_t g = (size_t)r.node * p.Lp + (size_t)cur.sl * SW;
        int q = rr.rpos + slot;
        if (q >= R) q -= R;
        bulk_g2s_h(sig + q * SW, gm + g, SW * 4, &full[ds], p.l2hint, pol);
        bulk_g2s_h(sex + q * SW, ge + g, SW * 2, &full[ds], p.l2hint, pol);
      }
      if (MMF_L2PF > 0 && lane >= 28 && lane < 30 && cur.node + MMF_L2PF < p.N) {  // first touch of an upcoming row
        const size_t g = (size_t)(cur.node + MMF_L2PF) * p.Lp + (size_t)cur.sl * SW;
        if (lane == 28) bulk_prefetch_l2(gm + g, SW * 4);
        else bulk_prefetch_l2(ge + g, SW * 2);
      }
      rr.head += (unsigned)n;
      rr.rpos += n;
      if (rr.rpos >= R) rr.rpos -= R;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers
  const int col = warp * 32 * CPT + lane * CPT;
  ItemIt it;
  it.init(item0, step, pc.ns);
  M* const bmt = v.bm(t);
  E* const bet = v.be(t);
  for (int k = 0; it.node < p.N; ++k, it.next()) {
    const int ds = k & (FWD_SD - 1);
    mbar_wait_sleep(&full[ds], (k / FWD_SD) & 1);
    if (pc.dry == 1) {  // diagnostics: delivery rate of the producer / TMA alone
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ds]);
      continue;
    }
    const PipeHdr& h = hdr[ds];
    const RingRows rw0{sig, sex, h.start, R, col, SW};
    M s[CPT];
    int Ex[CPT];
    if (MMF_BWD_NOWRAP_PATH == 0 || pc.wrap) ring_sum<CPT>(rw0, h, h.n, s, Ex);
    else ring_sum<CPT>(RingRowsF<SW>(rw0), h, h.n, s, Ex);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    const int node = alt_node(it.node, p.N, t);
    const size_t g = (size_t)node * p.Lp + (size_t)(it.sl * SW + col);
    if constexpr (CPT % 2 == 0 && MMF_NORM_PACKED) {
      norm_store_f32<CPT>(p, s, Ex, bmt + g, bet + g, it.sl * SW + col, node);
    } else {
      Lane<M, E, CPT> out;
      norm_lane<TrF32, CPT, false>(p, s, Ex, out, it.sl * SW + col, node);
      out.store(bmt + g, bet + g);
    }
  }
}

}  // namespace mmf
