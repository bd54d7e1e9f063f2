// reuse.cuh — row-reuse rings for the pipelined kernels (fp32 mode).
//
// The pipelined kernels (pipe.cuh, pipefwd.cuh) stage every gathered row of an item in shared memory by TMA.
// Each row is needed by all |A|/N neighbours that gather it, so the L2 -> SM traffic of a step is |A|/N times
// the message plane (4.8x on [4], 10.3x on [5]) and the gather kernels run close to the L2 (LTS) throughput
// cap.  Here a pipeline walks a contiguous block of nodes (node order chosen for neighbour overlap of
// consecutive nodes, mmf.cu choose_reuse_order), and its producer keeps a directory of the rows resident in
// its ring: a row already there (loaded for one of the last few items) is referenced, not loaded again.
//
// Ring bookkeeping (counters are monotonic, slot = counter mod R):
//   * an item references rows at counters >= lo (its oldest referenced row); rows at counters >= the
//     minimum lo over the unreleased items are protected; a new row may be allocated at counter c once
//     c - R is below that minimum;
//   * an item may reuse a resident row at counter pos only if head + n_new - pos <= R: its own allocation
//     cannot overwrite the row, and with every older item released its new rows fit (no deadlock); the
//     oldest reuses are dropped (reloaded) until this holds;
//   * a reused row may still be in flight (loaded for an earlier item): the consumers of a pipeline form
//     ONE group and take the items in order, so they have already observed the earlier item's full
//     barrier — the row has landed.
//
// Backward step (eq:psi): beta_t[i, slice] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a, slice].
#pragma once
#include "pipefwd.cuh"

namespace mmf {

#ifndef MMF_RU_NP
#define MMF_RU_NP 3
#endif
constexpr int RU_NP = MMF_RU_NP;  // pipelines per CTA of the backward
constexpr int RU_PW = PIPE_NWC + 1;
constexpr int RU_THREADS = RU_NP * RU_PW * 32;
constexpr int RU_SD = 8;  // item descriptors per pipeline (power of two)
constexpr int RU_P = 8;   // record prefetch distance (items; PIPE_RP > RU_P + RU_SD)
static_assert(PIPE_RP >= RU_P + RU_SD, "record ring");

// item descriptor: n rows (compacted, nonzero factor) with their ring offsets (slot * SW) and factors
struct RuHdr {
  unsigned kb[32];
  unsigned k2[32];
  int roff[32];
  int n;
  int pad[3];
};

// directory entry of a resident row
struct RuDir {
  int node;
  unsigned pos;  // ring counter
  int slot;
  int pad;
};

struct RuSmem {
  size_t off_full, off_empty, off_ring, off_hdr, off_dir, off_lo, off_sig, off_exp, total;
};
__host__ __device__ inline RuSmem ru_smem(int R, int D, int SW) {
  RuSmem m;
  size_t o = 0;
  m.off_full = o;
  o += 8 * (size_t)RU_SD;
  m.off_empty = o;
  o += 8 * (size_t)RU_SD;
  o = (o + 15) / 16 * 16;
  m.off_ring = o;
  o += (size_t)PIPE_RP * D * 16;
  m.off_hdr = o;
  o += (size_t)RU_SD * sizeof(RuHdr);
  m.off_dir = o;
  o += 32 * sizeof(RuDir);
  m.off_lo = o;
  o += 4 * (size_t)RU_SD;
  o = (o + 127) / 128 * 128;
  m.off_sig = o;
  o += (size_t)R * SW * 4;
  m.off_exp = o;
  o += (size_t)R * SW * 2;
  m.total = (o + 127) / 128 * 128;
  return m;
}

// node block of pipeline g of P (contiguous, equal counts)
__device__ __forceinline__ int ru_blk(int g, int P, int N) { return (int)(((long long)g * N) / P); }

// walk of a pipeline's items: slices outer, nodes of the block inner
struct RuIt {
  int j, s, j0, j1, ns;
  __device__ __forceinline__ void init(int g, int P, int N, int ns_) {
    j0 = ru_blk(g, P, N);
    j1 = ru_blk(g + 1, P, N);
    ns = ns_;
    j = j0;
    s = j0 < j1 ? 0 : ns_;
  }
  __device__ __forceinline__ bool ok() const { return s < ns; }
  __device__ __forceinline__ void next() {
    if (++j == j1) {
      j = j0;
      ++s;
    }
  }
};

// producer-side row allocation with reuse (warp-wide; lane < D: the item's arc `lane`, needing the row of
// `node` if `need`).  Returns, in the arc lanes, the row's ring slot; sets n_new / lo (oldest referenced
// counter) and, for new rows, isnew.  The directory lives in shared memory (entries 0 .. 31 - D).
struct RuAlloc {
  int slot;
  bool isnew;
  int nnew;
  unsigned lo;
  unsigned newmask;
};
__device__ __forceinline__ RuAlloc ru_lookup(RuDir* dir, int lane, int D, int R, unsigned head, int rpos, bool need,
                                             int node) {
  RuAlloc a;
  const bool isdir = lane >= D;
  RuDir e{-1, 0u, 0, 0};
  if (isdir) e = dir[lane - D];
  // candidates: rows still resident (no allocation has reached counter pos + R yet)
  const bool dvalid = isdir && e.node >= 0 && (int)(e.pos + (unsigned)R - head) > 0;
  const int key = isdir ? (dvalid ? e.node : -2 - lane) : (need ? node : -100 - lane);
  const unsigned m = __match_any_sync(0xffffffffu, key);
  const unsigned dm = D < 32 ? (m >> D) : 0u;
  bool hit = need && dm != 0u;
  const int src = hit ? (__ffs(dm) - 1 + D) : lane;
  const unsigned hpos = __shfl_sync(0xffffffffu, e.pos, src);
  const int hslot = __shfl_sync(0xffffffffu, e.slot, src);
  // the item's own allocation must not overwrite a row it reuses, and with every older item released it
  // must fit (no deadlock): both are head + nnew - lo <= R; drop the oldest reuses (load those rows again)
  // until it holds
  for (;;) {
    const unsigned nn = (unsigned)__popc(__ballot_sync(0xffffffffu, need && !hit));
    const unsigned dd = hit ? head - hpos : 0u;
    const unsigned dmax = __reduce_max_sync(0xffffffffu, dd);
    if (nn + dmax <= (unsigned)R) break;
    if (hit && dd == dmax) hit = false;
  }
  a.newmask = __ballot_sync(0xffffffffu, need && !hit);
  a.nnew = __popc(a.newmask);
  const int nrank = __popc(a.newmask & ((1u << lane) - 1u));
  int ns_ = rpos + nrank;
  if (ns_ >= R) ns_ -= R;
  a.isnew = need && !hit;
  a.slot = hit ? hslot : ns_;
  const unsigned dist = hit ? head - hpos : 0u;  // (new rows are at counters >= head)
  a.lo = head - __reduce_max_sync(0xffffffffu, dist);
  return a;
}
// insert the item's new rows into the directory (FIFO over the DL = 32 - D entries); wp is warp-uniform
__device__ __forceinline__ void ru_insert(RuDir* dir, int lane, int D, unsigned head, const RuAlloc& a, int node,
                                          int& wp) {
  const int DL = 32 - D;
  if (DL <= 0) return;
  if (a.isnew) {
    const int nrank = __popc(a.newmask & ((1u << lane) - 1u));
    if (a.nnew - nrank <= DL) {  // (only the last DL new rows are kept)
      int e = wp + nrank - (a.nnew > DL ? a.nnew - DL : 0);
      e %= DL;
      dir[e] = RuDir{node, head + (unsigned)nrank, a.slot, 0};
    }
  }
  wp = (wp + min(a.nnew, DL)) % DL;
  __syncwarp();
}
// ring space: protected counters start at min(lo of the unreleased items, lo of the current item)
__device__ __forceinline__ unsigned ru_tail(const unsigned* lo_arr, int kold, int k, unsigned head, unsigned lo_cur,
                                            int lane) {
  unsigned d = head - lo_cur;
  const int n_in = k - kold;  // (<= RU_SD)
  if (lane < n_in) d = max(d, head - lo_arr[(kold + lane) & (RU_SD - 1)]);
  return head - __reduce_max_sync(0xffffffffu, d);
}

// rows of an item addressed by per-row ring offsets (header), column col of the lane
struct RuRows {
  const float* sig;
  const int16_t* sex;
  const int* roff;
  int col;
  __device__ __forceinline__ int off(int q) const { return roff[q] + col; }
};

template <int CPT, int N>
__device__ __forceinline__ void ru_sum_n(const RuRows& rw, const RuHdr& h, float* s, int* Ex) {
  constexpr int NQ = N > 0 ? N : 1;
  float xm[NQ][CPT];
  int xw[NQ][CPT / 2];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const int o = rw.off(q);
    load_exps<CPT>(rw.sex + o, xw[q]);
    load_sig<CPT>(rw.sig + o, xm[q]);
  }
  unsigned E2[CPT / 2];
  xmax_init<CPT>(E2);
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const unsigned k2 = h.k2[q];
#pragma unroll
    for (int k = 0; k < CPT / 2; ++k) E2[k] = __viaddmax_s16x2((unsigned)xw[q][k], k2, E2[k]);
  }
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const unsigned kb = h.kb[q], k2 = h.k2[q];
#pragma unroll
    for (int k = 0; k < CPT / 2; ++k) {
      const unsigned u = __viaddmax_s16x2((unsigned)xw[q][k], k2, P.Lo2[k]);
      const unsigned d2 = __viaddmax_s16x2(u, P.nE2[k], 0xff82ff82u);
      s[2 * k] = fmaf(xm[q][2 * k], __uint_as_float(kb + (d2 << 23)), s[2 * k]);
      s[2 * k + 1] = fmaf(xm[q][2 * k + 1], __uint_as_float(kb + MMF_HI23(d2)), s[2 * k + 1]);
    }
  }
}
template <int CPT>
__device__ __forceinline__ void ru_sum_any(const RuRows& rw, const RuHdr& h, int n, float* s, int* Ex) {
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
__device__ __forceinline__ void ru_sum(const RuRows& rw, const RuHdr& h, int n, float* s, int* Ex) {
  switch (n) {
    case 0: ru_sum_n<CPT, 0>(rw, h, s, Ex); break;
    case 1: ru_sum_n<CPT, 1>(rw, h, s, Ex); break;
    case 2: ru_sum_n<CPT, 2>(rw, h, s, Ex); break;
    case 3: ru_sum_n<CPT, 3>(rw, h, s, Ex); break;
    case 4: ru_sum_n<CPT, 4>(rw, h, s, Ex); break;
    case 5: ru_sum_n<CPT, 5>(rw, h, s, Ex); break;
    case 6: ru_sum_n<CPT, 6>(rw, h, s, Ex); break;
    case 7: ru_sum_n<CPT, 7>(rw, h, s, Ex); break;
    case 8: ru_sum_n<CPT, 8>(rw, h, s, Ex); break;
    default: ru_sum_any<CPT>(rw, h, n, s, Ex); break;
  }
}

template <int CPT>
__global__ void __launch_bounds__(RU_THREADS, 1) k_bwd_reuse(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  constexpr int SW = pipe_sw<CPT>();
  extern __shared__ __align__(16) unsigned char smem_all[];
  const RuSmem L = ru_smem(pc.R, pc.D, SW);
  const int pl = (threadIdx.x >> 5) / RU_PW;
  unsigned char* smem = smem_all + (size_t)pl * L.total;
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  RuHdr* hdr = (RuHdr*)(smem + L.off_hdr);
  RuDir* dir = (RuDir*)(smem + L.off_dir);
  unsigned* lo_arr = (unsigned*)(smem + L.off_lo);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = (threadIdx.x >> 5) % RU_PW;
  const int D = pc.D, R = pc.R;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < RU_SD; ++s) {
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
  const int P = RU_NP * gridDim.x, g = blockIdx.x * RU_NP + pl;  // (adjacent blocks in one CTA)

  if (warp == PIPE_NWC) {  // ---------------- producer
    RuIt pf, cur;
    pf.init(g, P, p.N, pc.ns);
    cur = pf;
    int pslot = 0;
    auto prefetch = [&]() {
      if (pf.ok() && lane < D) cp_async16(&ring[pslot * D + lane], ell + (size_t)pf.j * D + lane);
      cp_async_commit();
      if (pf.ok()) pf.next();
      pslot = pslot + 1 == PIPE_RP ? 0 : pslot + 1;
    };
#pragma unroll 1
    for (int k = 0; k < RU_P; ++k) prefetch();
    for (int e = lane; e < 32; e += 32) dir[e] = RuDir{-1, 0u, 0, 0};
    __syncwarp();
    unsigned head = 0;
    int rpos = 0, kold = 0, wp = 0, cslot = 0, sprev = cur.s;
    for (int k = 0; cur.ok(); ++k, cur.next()) {
      cp_async_wait<RU_P - 1>();
      __syncwarp();
      ArcKW<M> r;
      r.node = -1;
      r.km = M(0);
      r.ke = 0;
      if (lane < D) r = ring[cslot * D + lane];
      cslot = cslot + 1 == PIPE_RP ? 0 : cslot + 1;
      __syncwarp();
      prefetch();
      if (cur.s != sprev) {  // new slice: other rows
        dir[lane] = RuDir{-1, 0u, 0, 0};
        sprev = cur.s;
        __syncwarp();
      }
      const bool need = lane < D && r.node >= 0 && r.km > M(0);
      while (kold <= k - RU_SD) {  // descriptor slot reuse
        mbar_wait(&empty[kold & (RU_SD - 1)], (kold / RU_SD) & 1);
        ++kold;
      }
      const RuAlloc a = ru_lookup(dir, lane, D, R, head, rpos, need, r.node);
      for (;;) {
        const unsigned tail = ru_tail(lo_arr, kold, k, head, a.lo, lane);
        if (head + (unsigned)a.nnew - tail <= (unsigned)R || kold >= k) break;
        mbar_wait(&empty[kold & (RU_SD - 1)], (kold / RU_SD) & 1);
        ++kold;
      }
      const int ds = k & (RU_SD - 1);
      RuHdr& h = hdr[ds];
      const unsigned okm = __ballot_sync(0xffffffffu, need);
      const int q = __popc(okm & ((1u << lane) - 1u));
      if (need) {
        h.kb[q] = __float_as_uint(r.km);
        h.k2[q] = pack2(r.ke);
        h.roff[q] = a.slot * SW;
      }
      if (lane == 0) {
        h.n = __popc(okm);
        lo_arr[ds] = a.lo;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)a.nnew * (unsigned)SW * 6u);
      __syncwarp();
      if (a.isnew) {
        const size_t go = (size_t)r.node * p.Lp + (size_t)cur.s * SW;
        bulk_g2s(sig + a.slot * SW, gm + go, SW * 4, &full[ds]);
        bulk_g2s(sex + a.slot * SW, ge + go, SW * 2, &full[ds]);
      }
      ru_insert(dir, lane, D, head, a, r.node, wp);
      head += (unsigned)a.nnew;
      rpos += a.nnew;
      if (rpos >= R) rpos -= R;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers (one group per pipeline: items in order)
  const int col = warp * 32 * CPT + lane * CPT;
  RuIt it;
  it.init(g, P, p.N, pc.ns);
  M* const bmt = v.bm(t);
  E* const bet = v.be(t);
  for (int k = 0; it.ok(); ++k, it.next()) {
    const int ds = k & (RU_SD - 1);
    mbar_wait(&full[ds], (k / RU_SD) & 1);
    const RuHdr& h = hdr[ds];
    const RuRows rw{sig, sex, h.roff, col};
    M s[CPT];
    int Ex[CPT];
    ru_sum<CPT>(rw, h, h.n, s, Ex);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    const size_t go = (size_t)it.j * p.Lp + (size_t)(it.s * SW + col);
    norm_store_f32<CPT>(p, s, Ex, bmt + go, bet + go, it.s * SW + col, it.j);
  }
}

}  // namespace mmf
