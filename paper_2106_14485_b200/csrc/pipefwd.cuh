// pipefwd.cuh — TMA-pipelined persistent forward step (option kernels = 5, fp32, one slice per node).
//
// Forward kernel of step t (1 <= t <= T), one item per node j (all Lp commodities), the head-flow order of
// headflow.cuh (Algorithm 2's Gauss-Seidel order):
//   (i)   F_{t-1}[a] = K W_{t-1}[a] sum_l alpha_{t-1}[i_a,l] beta_t[j,l] for the in-arcs a -> j  (cor:proj P:1078)
//   (ii)  W_{t-1}[a] <- min(W_{t-1}[a] d[a] / F_{t-1}[a], 1)                         (eq:sinkhorn_graph_Vineq P:861)
//   (iii) alpha_t[j] = sum_{a -> j} alpha_{t-1}[i_a] K W_{t-1}[a] with the updated W    (eq:psi_hat P:1031-1036)
// The producer warp stages, per item: the compacted rows alpha_{t-1}[i_a] (nonzero factor) and the node's
// own row beta_t[j] (cp.async.bulk; contiguous ring slots) and the arc records (cp.async ring, prefetched);
// the consumers load the dual-update operands d, W, K (and record slots) of their arcs with plain loads
// at the start of the item, overlapped with the flow computation.
//
// Consumers (a group of 8 warps per item, 2 groups alternating items) compute the per-row terms
//   t_q[c] = alpha_q[c] K W_q 2^-E[c]     (E[c] = max_q exponent of alpha_q[c] K W_q, extended range)
// once, in registers (the row count is a compile-time constant of the code path, switch on n).  Then
//   flows:  F_q = sum_c t_q[c] * beta_lin[c],   beta_lin[c] = beta[j,c] 2^E[c]  (one FMA per element),
//           reduced over the lanes by a transposed butterfly (9 shuffles for up to 8 rows) and over the
//           group's warps in shared memory (fixed order: deterministic);
//   update: one lane per arc applies (ii), refreshes the arc's ELL records and publishes r_q = W_new / W_old;
//   alpha:  alpha_t[j,c] = 2^E[c] sum_q r_q t_q[c]   (one FMA per element)
// — valid while every |log2 r_q| <= 40 (the dropped terms, below 2^-126 of the old maximum, stay below
// 2^-46 of the new one); otherwise the item is recomputed from shared memory with the new factors.
#pragma once
#include "pipe.cuh"

namespace mmf {

// The forward CTA runs FWD_NP independent pipelines, each one producer warp + one consumer group of 8 warps
// with its own share of the shared memory (row ring, descriptors, record ring): the producer's per-item
// serial latency (~0.9 us, mostly issuing the item's ~12 TMA copies; measured with idle consumers) is what
// limits a single pipeline.  An item's rows may wrap around its ring (consumers resolve the wrap per row),
// so a ring needs only D + 1 slots.
constexpr int FWD_NG = 1;
constexpr int FWD_NP = 2;
constexpr int FWD_PW = PIPE_NWC * FWD_NG + 1;  // warps per pipeline
constexpr int FWD_THREADS = FWD_NP * FWD_PW * 32;
constexpr int FWD_SD = 8;  // item descriptors per pipeline (power of two)

struct __align__(16) FwdHdr {
  unsigned kb[32];  // rows (compacted, nonzero factor): K W significand bits
  unsigned k2[32];  //   ... exponent, packed twice (int16x2)
  int rarc[32];     //   ... arc position of the row
  int rowof[32];    // arcs (all in-arcs, q < na): row index or -1
  int aux[32];      //   ... arc id | bit 31 uncapacitated
  int rtail[32];    //   ... tail node
  ArcOps ops[32];   //   ... dual-update operands (prefetched with the records)

  unsigned capmask; // bit q: row q's arc is capacitated
  int nr, na, start, end;
  int pad[3];
};

// per consumer group scratch: flow partials (row, warp), double-buffered by the group's item parity (a
// warp may start the group's next item while another still reads this item's partials)
struct FwdGrp {
  float fpart[2][32][PIPE_NWC];
};

struct PFwdSmem {
  size_t off_full, off_empty, off_ring, off_oring, off_hdr, off_grp, off_sig, off_exp, total;
};

__host__ __device__ inline PFwdSmem pfwd_smem(int R, int D, int SW) {
  PFwdSmem m;
  size_t o = 0;
  m.off_full = o;
  o += 8 * (size_t)FWD_SD;
  m.off_empty = o;
  o += 8 * (size_t)FWD_SD;
  o = (o + 15) / 16 * 16;
  m.off_ring = o;
  o += (size_t)PIPE_RP * D * 16;
  m.off_oring = o;
  o += (size_t)PIPE_RP * D * 32;
  m.off_hdr = o;
  o += (size_t)FWD_SD * sizeof(FwdHdr);
  o = (o + 15) / 16 * 16;
  m.off_grp = o;
  o += (size_t)FWD_NG * sizeof(FwdGrp);
  o = (o + 127) / 128 * 128;
  m.off_sig = o;
  o += (size_t)R * SW * 4;
  m.off_exp = o;
  o += (size_t)R * SW * 2;
  m.total = (o + 127) / 128 * 128;
  return m;
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
};
__device__ __forceinline__ FwdOps fwd_ops(const DevPtrs& p, const FwdHdr& h, int t, int lane) {
  FwdOps o{0.f, 1.f, 0.f, 0, 0, 0, 0};
  if (lane < h.na) {
    const ArcOps a = h.ops[lane];
    o.d = a.d;
    o.wm = a.wm;
    o.we = a.we;
    o.Km = a.Km;
    o.Ke = a.Ke;
    o.eopos = a.eopos;
    o.copos = a.copos;
  }
  return o;
}
__device__ __forceinline__ FwdUpd fwd_update(const DevPtrs& p, const FwdHdr& h, const FwdOps& o,
                                             const float (*fp)[PIPE_NWC], int t, int j, int D, int lane, bool writer,
                                             bool* big_out) {
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
        for (int w = 0; w < PIPE_NWC; ++w) s += fp[row][w];
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
}

// alpha from the new factors (gathered from the arcs' lanes), two passes over shared memory
// the own row beta_t[j] scaled to the terms' exponents: beta_lin[c] = beta[j,c] 2^E[c] (flows are bounded
// by the mass: the exponent is clamped to the normal range)
template <int CPT>
__device__ __forceinline__ void beta_lin(const Row<TrF32, CPT>& b, const XPre<CPT>& P, float* bl) {
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int es = b.e(c) + P.E[c];
    bl[c] = (es < -126 || !(b.m[c] > 0.f)) ? 0.f : b.m[c] * __uint_as_float((unsigned)(min(es, 127) + 127) << 23);
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

// alpha from the new factors (gathered from the arcs' lanes), two passes over shared memory
template <int CPT>
__device__ __forceinline__ void fwd_alpha_new(const RingRows& rw, const FwdHdr& h, const FwdUpd& u, int nr, int lane,
                                              float* s, int* Ex) {
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < nr; ++q) {
    const int src = h.rarc[q];
    const unsigned kb = __shfl_sync(0xffffffffu, u.nkb, src), k2 = __shfl_sync(0xffffffffu, u.nk2, src);
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
    const unsigned kb = __shfl_sync(0xffffffffu, u.nkb, src), k2 = __shfl_sync(0xffffffffu, u.nk2, src);
    if (!(__uint_as_float(kb) > 0.f)) continue;
    Row<TrF32, CPT> x;
    x.load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    xacc<CPT>(x, kb, k2, k2_to_ke(k2), P, s);
  }
}

template <int CPT, int N>
__device__ __forceinline__ void fwd_body(const DevPtrs& p, const RingRows& rw, const FwdHdr& h,
                                         float (*fp)[PIPE_NWC], int t, int j, int D, int lane, int wg, int bar_id,
                                         float* s, int* Ex) {
  typedef Row<TrF32, CPT> R_;
  const FwdOps o = fwd_ops(p, h, t, lane);
  R_ b;
  b.load(rw.sig + rw.off(N), rw.sex + rw.off(N));  // own row beta_t[j]
  float tq[N > 0 ? N : 1][CPT];
  XPre<CPT> P;
  {
    R_ x[N > 0 ? N : 1];
#pragma unroll
    for (int q = 0; q < N; ++q) x[q].load(rw.sig + rw.off(q), rw.sex + rw.off(q));
    unsigned E2[CPT];
    xmax_init<CPT>(E2);
#pragma unroll
    for (int q = 0; q < N; ++q) xmax_add<CPT>(E2, x[q], h.k2[q], k2_to_ke(h.k2[q]));
    P.set(E2);
#pragma unroll
    for (int q = 0; q < N; ++q) xterms<CPT>(x[q], h.kb[q], h.k2[q], k2_to_ke(h.k2[q]), P, tq[q]);
  }
  float bl[CPT];
  beta_lin<CPT>(b, P, bl);
  const unsigned cap = h.capmask;
  if (N > 0 && cap != 0u) {
    float f[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      f[q] = 0.f;
      if (q < N)
#pragma unroll
        for (int c = 0; c < CPT; ++c) f[q] = fmaf(tq[q < N ? q : 0][c], bl[c], f[q]);
    }
    const float r = bfly8(f, lane);
    const int row = bfly_row(lane);
    if ((lane & 3) == 0 && row < N && ((cap >> row) & 1u)) fp[row][wg] = r;
  }
  named_bar(bar_id, PIPE_NWC * 32);
  bool big;
  const FwdUpd u = fwd_update(p, h, o, fp, t, j, D, lane, wg == 0, &big);
  if (!big) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = 0.f;
      Ex[c] = P.E[c];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      const float r = __shfl_sync(0xffffffffu, u.rq, h.rarc[q]);
#pragma unroll
      for (int c = 0; c < CPT; ++c) s[c] = fmaf(r, tq[q][c], s[c]);
    }
  } else {  // large ratios: recompute from shared memory with the new factors
    fwd_alpha_new<CPT>(rw, h, u, N, lane, s, Ex);
  }
}

// any row count (more than 8 rows): streaming flows, then the update, then alpha from shared memory
template <int CPT>
__device__ __forceinline__ void fwd_body_any(const DevPtrs& p, const RingRows& rw, const FwdHdr& h,
                                             float (*fp)[PIPE_NWC], int t, int j, int D, int lane, int wg, int bar_id,
                                             int nr, float* s, int* Ex) {
  typedef Row<TrF32, CPT> R_;
  const FwdOps o = fwd_ops(p, h, t, lane);
  R_ b;
  b.load(rw.sig + rw.off(nr), rw.sex + rw.off(nr));
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
  beta_lin<CPT>(b, P, bl);
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
  named_bar(bar_id, PIPE_NWC * 32);
  bool big;
  const FwdUpd u = fwd_update(p, h, o, fp, t, j, D, lane, wg == 0, &big);
  fwd_alpha_new<CPT>(rw, h, u, nr, lane, s, Ex);
}

template <int CPT, int MODE>
__global__ void __launch_bounds__(FWD_THREADS, 1) k_fwd_pipe(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  constexpr int SW = pipe_sw<CPT>();
  extern __shared__ __align__(16) unsigned char smem_all[];
  const PFwdSmem L = pfwd_smem(pc.R, pc.D, SW);
  const int pl = (threadIdx.x >> 5) / FWD_PW;                 // pipeline of this warp
  unsigned char* smem = smem_all + (size_t)pl * L.total;      // its share of the shared memory
  const int jstep = FWD_NP * gridDim.x, j0 = blockIdx.x + pl * gridDim.x;
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  ArcOps* oring = (ArcOps*)(smem + L.off_oring);
  FwdHdr* hdr = (FwdHdr*)(smem + L.off_hdr);
  FwdGrp* grps = (FwdGrp*)(smem + L.off_grp);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % FWD_PW;  // (warp within the pipeline)
  const int D = pc.D, R = pc.R;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < FWD_SD; ++s) {
      mbar_init(&full[s], 1);          // expect_tx arrive (all rows land by TMA)
      mbar_init(&empty[s], PIPE_NWC);  // one consumer group per item
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);

  if (warp == PIPE_NWC * FWD_NG) {  // ---------------- producer
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
    int pnode = j0, pslot = 0;
    auto prefetch = [&]() {
      if (pnode < p.N && lane < D) {
        cp_async16(&ring[pslot * D + lane], ell + (size_t)pnode * D + lane);
        const ArcOps* go = (const ArcOps*)p.ell_ops + (size_t)(t - 1) * p.N * D + (size_t)pnode * D + lane;
        cp_async16(&oring[pslot * D + lane], go);
        cp_async16((char*)&oring[pslot * D + lane] + 16, (const char*)go + 16);
      }
      cp_async_commit();
      pnode += jstep;
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
    int k = 0, cslot = 0;
    for (int j = j0; j < p.N; j += jstep, ++k) {
      cp_async_wait<PIPE_P - 1>();
      __syncwarp();
      ArcKW<M> r;
      r.node = -1;
      r.km = M(0);
      r.ke = 0;
      r.aux = 0;
      ArcOps ro;
      if (lane < D) {
        r = ring[cslot * D + lane];
        ro = oring[cslot * D + lane];
      }
      cslot = cslot + 1 == PIPE_RP ? 0 : cslot + 1;
      __syncwarp();
      const bool valid = lane < D && r.node >= 0;
      const bool ok = valid && r.km > M(0);
      const unsigned vbal = __ballot_sync(0xffffffffu, valid);
      const unsigned obal = __ballot_sync(0xffffffffu, ok);
      const unsigned cbal = __ballot_sync(0xffffffffu, ok && r.aux >= 0);
      const int na = __popc(vbal), nr = __popc(obal);
      while (rr.kold <= k - FWD_SD) release();
      while (rr.head + (unsigned)(nr + 1) - rr.tail > (unsigned)R && rr.kold < k) release();  // (R >= D + 1)
      const int ds = k & (FWD_SD - 1);
      FwdHdr& h = hdr[ds];
      const int rs = __popc(obal & ((1u << lane) - 1u));
      if (ok) {
        h.kb[rs] = __float_as_uint(r.km);
        h.k2[rs] = pack2(r.ke);
        h.rarc[rs] = lane;
      }
      if (valid) {
        h.rowof[lane] = ok ? rs : -1;
        h.aux[lane] = r.aux;
        h.rtail[lane] = r.node;
        h.ops[lane] = ro;
      }
      if (lane == 0) {
        // capmask over rows (row order = lane order of the nonzero-factor arcs)
        unsigned cm = 0u, ob = obal;
        for (int q = 0; ob; ++q) {
          const int l = __ffs(ob) - 1;
          if ((cbal >> l) & 1u) cm |= 1u << q;
          ob &= ob - 1u;
        }
        h.capmask = cm;
        h.nr = nr;
        h.na = na;
        h.start = rr.rpos;
        h.end = (int)(rr.head + (unsigned)(nr + 1));
      }
      __syncwarp();  // (the header writes of every lane precede lane 0's releasing arrive)
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)(nr + 1) * (unsigned)SW * 6u);
      __syncwarp();
      prefetch();
      if (ok) {
        const size_t g = (size_t)r.node * p.Lp;
        int q = rr.rpos + rs;
        if (q >= R) q -= R;
        bulk_g2s(sig + q * SW, gm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, ge + g, SW * 2, &full[ds]);
      }
      if (lane == 31) {  // the node's own beta_t row -> slot nr
        const size_t g = (size_t)j * p.Lp;
        int q = rr.rpos + nr;
        if (q >= R) q -= R;
        bulk_g2s(sig + q * SW, bm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, be + g, SW * 2, &full[ds]);
      }
      rr.head += (unsigned)(nr + 1);
      rr.rpos += nr + 1;
      if (rr.rpos >= R) rr.rpos -= R;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers
  const int grp = warp / PIPE_NWC, wg = warp % PIPE_NWC;
  FwdGrp& G = grps[grp];
  const int col = wg * 32 * CPT + lane * CPT;
  const int bar_id = 1 + pl;
  int k = grp;
  for (int j = j0; j < p.N; j += jstep, k += FWD_NG) {
    const int ds = k & (FWD_SD - 1);
    mbar_wait(&full[ds], (k / FWD_SD) & 1);
    const FwdHdr& h = hdr[ds];
    if (pc.dry) {  // diagnostics: delivery rate of the producer / TMA alone
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ds]);
      continue;
    }
    const int nr = h.nr;
    const RingRows rw{sig, sex, h.start, R, col, SW};
    float (*fp)[PIPE_NWC] = G.fpart[(k / FWD_NG) & 1];
    M s[CPT];
    int Ex[CPT];
    switch (nr) {
      case 0: fwd_body<CPT, 0>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 1: fwd_body<CPT, 1>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 2: fwd_body<CPT, 2>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 3: fwd_body<CPT, 3>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 4: fwd_body<CPT, 4>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 5: fwd_body<CPT, 5>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 6: fwd_body<CPT, 6>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 7: fwd_body<CPT, 7>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      case 8: fwd_body<CPT, 8>(p, rw, h, fp, t, j, D, lane, wg, bar_id, s, Ex); break;
      default: fwd_body_any<CPT>(p, rw, h, fp, t, j, D, lane, wg, bar_id, nr, s, Ex); break;
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    // s is 0 or a normal float (ratios are within 2^+-40 of the previous terms): bit-level normalisation
    Lane<M, E, CPT> a;
    norm_lane<TrF32, CPT>(p, s, Ex, a, col, j);
    const size_t g = (size_t)j * p.Lp + col;
    a.store(v.am(t) + g, v.ae(t) + g);
    if (MODE == 2) {  // a4: UT = muT ./ alpha_T -> beta_T
      Lane<M, E, CPT> ut;
      boundary_lane<TrF32, CPT>(p, 1, j, col, g, a, ut);
      ut.store(v.bm(p.T) + g, v.be(p.T) + g);
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
template <int CPT, int N>
__device__ __forceinline__ void ring_sum_n(const RingRows& rw, const PipeHdr& h, float* s, int* Ex) {
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
template <int CPT>
__device__ __forceinline__ void ring_sum_any(const RingRows& rw, const PipeHdr& h, int n, float* s, int* Ex) {
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
template <int CPT>
__device__ __forceinline__ void ring_sum(const RingRows& rw, const PipeHdr& h, int n, float* s, int* Ex) {
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
    int pslot = 0;
    auto prefetch = [&]() {
      if (pf.node < p.N && lane < D) cp_async16(&ring[pslot * D + lane], ell + (size_t)pf.node * D + lane);
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
      while (rr.head + (unsigned)n - rr.tail > (unsigned)R && rr.kold < k) release();  // (R >= D)
      const int ds = k & (FWD_SD - 1);
      const int slot = __popc(bal & ((1u << lane) - 1u));
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
        bulk_g2s(sig + q * SW, gm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, ge + g, SW * 2, &full[ds]);
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
    mbar_wait(&full[ds], (k / FWD_SD) & 1);
    const PipeHdr& h = hdr[ds];
    const RingRows rw{sig, sex, h.start, R, col, SW};
    M s[CPT];
    int Ex[CPT];
    ring_sum<CPT>(rw, h, h.n, s, Ex);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    Lane<M, E, CPT> out;
    norm_lane<TrF32, CPT>(p, s, Ex, out, it.sl * SW + col, it.node);
    const size_t g = (size_t)it.node * p.Lp + (size_t)(it.sl * SW + col);
    out.store(bmt + g, bet + g);
  }
}

}  // namespace mmf
