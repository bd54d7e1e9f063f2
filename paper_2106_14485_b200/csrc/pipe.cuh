// pipe.cuh — warp-specialised, TMA-pipelined persistent sweep kernels (option kernels = 5, fp32 mode).
//
// Why: the gather of a step is latency-bound when each warp walks its own dependent chain
// (CSR pointer -> arc records -> neighbour rows -> arithmetic) with the rows landing in registers:
// bytes in flight per SM are capped by the register file (ncu on [4]: 25-37 % occupancy, long-scoreboard
// stalls, 28-34 % of DRAM bandwidth).  Here one producer warp per CTA runs ahead of the arithmetic:
//   * the arc records of upcoming items (ELL layout [T][N][D], no CSR pointer round trip) are prefetched
//     P items ahead with cp.async into a small ring;
//   * the neighbour rows of an item (slice of SW commodities of each gathered node: significand plane +
//     exponent plane) are fetched with cp.async.bulk (TMA bulk copies, SASS UBLKCP) into a ring of R row
//     slots in shared memory (an item's rows are contiguous), completion tracked by mbarrier transaction
//     counts in a ring of item descriptors;
// and consumer warps compute from shared memory and release the item.  Work items are visited in
// grid-stride order (item = blockIdx.x + k * gridDim.x over node-major (node, slice) pairs), so at any
// moment the whole GPU works on a narrow band of consecutive nodes: a gathered row is reused from L2 by
// the neighbouring nodes' CTAs while it is still resident (nodes are numbered for locality).
//
// Backward step (eq:psi):  beta_t[i, slice] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a, slice].
#pragma once
#include "headflow.cuh"

namespace mmf {

constexpr int PIPE_NWC = 8;                                  // consumer warps per group (one group = one item)
constexpr int PIPE_NG = 2;                                   // consumer groups (alternate items)
constexpr int PIPE_THREADS = (PIPE_NWC * PIPE_NG + 1) * 32;  // + one producer warp
#ifndef MMF_PIPE_P
#define MMF_PIPE_P 12
#endif
#ifndef MMF_PIPE_RP
#define MMF_PIPE_RP 16
#endif
constexpr int PIPE_P = MMF_PIPE_P;                           // record prefetch distance (items)
constexpr int PIPE_RP = MMF_PIPE_RP;                         // record ring slots (> PIPE_P)
constexpr int PIPE_NR = 8;                                   // rows a consumer holds in registers (fast path)
constexpr int PIPE_SD = 16;                                  // item descriptors (power of two)

// slice width of the pipelined kernels: 8 consumer warps x 32 lanes x CPT commodities
template <int CPT> constexpr int pipe_sw() { return 32 * CPT * PIPE_NWC; }

struct PipeCfg5 {
  int R;       // row slots in the shared-memory ring (each SW significands + SW exponents)
  int SD;      // item descriptors (= PIPE_SD)
  int D;       // ELL width of the gathered arc lists (max degree, <= 32)
  int SW;      // commodities per item (slice) = 32 * CPT * PIPE_NWC
  int ns;      // slices per node = Lp / SW
  int nitems;  // N * ns
  int dry;     // diagnostics: consumers only wait and release (measures the producer / TMA delivery rate)
  int copy;    // row staging: 0 = cp.async.bulk (TMA, one per row plane), 1 = cp.async 16 B per lane (LDGSTS)
  int wrap;    // k_bwd_pipe2: 1 = an item's rows may wrap around the ring (offsets computed per row), 0 = items
               // never wrap (the producer skips to slot 0; compile-time row offsets, fewer ring slots usable)
};

// item descriptor: the n present rows (compacted, nonzero factor; ring slots start .. start + n - 1, never
// wrapping) and their arc factors K W (bits of the significand, exponent packed twice as int16x2)
struct PipeHdr {
  unsigned kb[32];
  unsigned k2[32];
  int n;
  int start;  // first ring slot
  int end;    // producer's monotonic slot counter after this item
  int pad;
};

struct PipeSmem {
  size_t off_full, off_empty, off_ring, off_hdr, off_sig, off_exp, total;
};

__host__ __device__ inline PipeSmem pipe_smem(int R, int SD, int D, int SW) {
  PipeSmem m;
  size_t o = 0;
  m.off_full = o;
  o += 8 * (size_t)SD;
  m.off_empty = o;
  o += 8 * (size_t)SD;
  o = (o + 15) / 16 * 16;
  m.off_ring = o;
  o += (size_t)PIPE_RP * D * 16;
  m.off_hdr = o;
  o += (size_t)SD * sizeof(PipeHdr);
  o = (o + 127) / 128 * 128;
  m.off_sig = o;
  o += (size_t)R * SW * 4;
  m.off_exp = o;
  o += (size_t)R * SW * 2;
  m.total = o;
  return m;
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N> __device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// warp-cooperative copy of one row slice (SW significands + SW exponents) with 16-byte cp.async per lane
template <int SW>
__device__ __forceinline__ void row_cp_async(float* dsig, int16_t* dexp, const float* gsig, const int16_t* gexp,
                                             int lane) {
#pragma unroll
  for (int o = lane * 4; o < SW; o += 128) cp_async16(dsig + o, gsig + o);
#pragma unroll
  for (int o = lane * 8; o < SW; o += 256) cp_async16(dexp + o, gexp + o);
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

// grid-stride walk over node-major (node, slice) items without divisions in the loop
struct ItemIt {
  int node, sl, dn, ds, ns;
  __device__ __forceinline__ void init(int item0, int step, int ns_) {
    ns = ns_;
    node = item0 / ns;
    sl = item0 - node * ns;
    dn = step / ns;
    ds = step - dn * ns;
  }
  __device__ __forceinline__ void next() {
    node += dn;
    sl += ds;
    if (sl >= ns) {
      sl -= ns;
      ++node;
    }
  }
};

// normalise a lane's sums (s[c] * 2^Ex[c], s[c] = 0 or a normal float) into [1, 2) significands and int16
// exponents two at a time, and store them (norm_lane's semantics: zero -> (0, EZERO); an exponent outside
// [-ELIM, ELIM] is clamped and raises the sticky ERR_RANGE — checked once per lane)
template <int CPT>
__device__ __forceinline__ void norm_store_f32(const DevPtrs& p, const float* s, const int* Ex, float* pm,
                                               int16_t* pe, int l0, int node) {
  static_assert(CPT % 2 == 0, "packed exponents");
  typedef typename VecM<float, CPT>::T VM;
  typedef typename VecE<int16_t, CPT>::T VE;
  VM vm;
  VE ve;
  float* m = reinterpret_cast<float*>(&vm);
  unsigned* e2 = reinterpret_cast<unsigned*>(&ve);
  unsigned hi = 0x80008000u, lo = 0x7fff7fffu;
#pragma unroll
  for (int w = 0; w < CPT / 2; ++w) {
    const unsigned u0 = __float_as_uint(s[2 * w]), u1 = __float_as_uint(s[2 * w + 1]);
    const unsigned E2 = __byte_perm((unsigned)Ex[2 * w], (unsigned)Ex[2 * w + 1], 0x5410);
    const unsigned f2 = (u0 >> 23) | ((u1 >> 7) & 0x00ff0000u);  // float exponent fields (0: the sum is 0)
    const unsigned z2 = __vcmpeq2(f2, 0u);
    const unsigned er = __vsub2(__vadd2(E2, f2), 0x007f007fu);
    e2[w] = (er & ~z2) | (0xc000c000u & z2);  // (EZERO = -16384)
    const unsigned enz = er & ~z2;
    hi = __vmaxs2(hi, enz);
    lo = __vmins2(lo, enz);
    m[2 * w] = u0 ? __uint_as_float((u0 & 0x007fffffu) | 0x3f800000u) : 0.f;
    m[2 * w + 1] = u1 ? __uint_as_float((u1 & 0x007fffffu) | 0x3f800000u) : 0.f;
  }
  const int emax = max((int)(short)(hi & 0xffffu), (int)hi >> 16);
  const int emin = min((int)(short)(lo & 0xffffu), (int)lo >> 16);
  if (emax > ELIM || emin < -ELIM) {  // (rare) clamp and report, element by element
    int16_t* es = reinterpret_cast<int16_t*>(&ve);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int e = es[c];
      if (m[c] != 0.f && (e > ELIM || e < -ELIM)) {
        set_error(p, ERR_RANGE, l0 + c, node);
        es[c] = (int16_t)(e > 0 ? ELIM : -ELIM);
      }
    }
  }
  *reinterpret_cast<VM*>(pm) = vm;
  *reinterpret_cast<VE*>(pe) = ve;
}

// sum over N (compile-time) contiguous rows sg + q * SW of an item: (s, E) per commodity
template <int CPT, int N>
__device__ __forceinline__ void sum_rows_n(const float* sg, const int16_t* se, const unsigned* kb, const unsigned* k2,
                                           float* s, int* Ex) {
  constexpr int SW = pipe_sw<CPT>();
  Row<TrF32, CPT> x[N > 0 ? N : 1];
#pragma unroll
  for (int q = 0; q < N; ++q) x[q].load(sg + q * SW, se + q * SW);
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
#pragma unroll
  for (int q = 0; q < N; ++q) xmax_add<CPT>(E2, x[q], k2[q], k2_to_ke(k2[q]));
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
#pragma unroll
  for (int q = 0; q < N; ++q) xacc<CPT>(x[q], kb[q], k2[q], k2_to_ke(k2[q]), P, s);
}
// any n (high degree): two passes over shared memory
template <int CPT>
__device__ __forceinline__ void sum_rows_any(const float* sg, const int16_t* se, const unsigned* kb,
                                             const unsigned* k2, int n, float* s, int* Ex) {
  constexpr int SW = pipe_sw<CPT>();
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < n; ++q) {
    Row<TrF32, CPT> x;
    x.load(sg + q * SW, se + q * SW);
    xmax_add<CPT>(E2, x, k2[q], k2_to_ke(k2[q]));
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
    x.load(sg + q * SW, se + q * SW);
    xacc<CPT>(x, kb[q], k2[q], k2_to_ke(k2[q]), P, s);
  }
}
template <int CPT>
__device__ __forceinline__ void sum_rows(const float* sg, const int16_t* se, const unsigned* kb, const unsigned* k2,
                                         int n, float* s, int* Ex) {
  switch (n) {
    case 0: sum_rows_n<CPT, 0>(sg, se, kb, k2, s, Ex); break;
    case 1: sum_rows_n<CPT, 1>(sg, se, kb, k2, s, Ex); break;
    case 2: sum_rows_n<CPT, 2>(sg, se, kb, k2, s, Ex); break;
    case 3: sum_rows_n<CPT, 3>(sg, se, kb, k2, s, Ex); break;
    case 4: sum_rows_n<CPT, 4>(sg, se, kb, k2, s, Ex); break;
    case 5: sum_rows_n<CPT, 5>(sg, se, kb, k2, s, Ex); break;
    case 6: sum_rows_n<CPT, 6>(sg, se, kb, k2, s, Ex); break;
    case 7: sum_rows_n<CPT, 7>(sg, se, kb, k2, s, Ex); break;
    case 8: sum_rows_n<CPT, 8>(sg, se, kb, k2, s, Ex); break;
    default: sum_rows_any<CPT>(sg, se, kb, k2, n, s, Ex); break;
  }
}

// producer-side row-slot ring: monotonic counters, [tail, head) in use; rpos = head mod R
struct RowRing {
  unsigned head = 0, tail = 0;
  int rpos = 0;
  int kold = 0;  // items < kold are known to be released
};

// ------------------------------------------------------------------------------------------------
template <int CPT>
__global__ void __launch_bounds__(PIPE_THREADS, 1) k_bwd_pipe(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  constexpr int SW = pipe_sw<CPT>();
  extern __shared__ __align__(16) unsigned char smem[];
  const PipeSmem L = pipe_smem(pc.R, PIPE_SD, pc.D, SW);
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  PipeHdr* hdr = (PipeHdr*)(smem + L.off_hdr);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int D = pc.D, R = pc.R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_SD; ++s) {
      mbar_init(&full[s], pc.copy ? 1 + 32 : 1);  // (+ one cp.async noinc arrive per producer lane)
      mbar_init(&empty[s], PIPE_NWC);             // one consumer group per item
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);
  const ArcKW<M>* ell = (const ArcKW<M>*)p.ell_out + (size_t)t * p.N * D;
  const M* gm = v.bm(t + 1);
  const E* ge = v.be(t + 1);

  if (warp == PIPE_NWC * PIPE_NG) {  // ---------------- producer
    ItemIt pf, cur;  // record prefetch runs PIPE_P items ahead of the issue position
    pf.init(blockIdx.x, gridDim.x, pc.ns);
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
      const int ds = rr.kold & (PIPE_SD - 1);
      mbar_wait(&empty[ds], (rr.kold / PIPE_SD) & 1);
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
      while (rr.kold <= k - PIPE_SD) release();  // descriptor reuse
      if (rr.rpos + n > R) {                     // keep the item's rows contiguous
        rr.head += (unsigned)(R - rr.rpos);
        rr.rpos = 0;
      }
      while (rr.head + (unsigned)n - rr.tail > (unsigned)R && rr.kold < k) release();  // row space (R >= 2 D)
      const int ds = k & (PIPE_SD - 1);
      const int slot = __popc(bal & ((1u << lane) - 1u));
      if (ok) {
        hdr[ds].kb[slot] = __float_as_uint(r.km);
        hdr[ds].k2[slot] = pack2(r.ke);
      }
      if (lane == 0) {
        hdr[ds].n = n;
        hdr[ds].start = rr.rpos;
        hdr[ds].end = (int)(rr.head + (unsigned)n);  // monotonic row counter after this item (producer only)
      }
      __syncwarp();
      if (pc.copy) {  // LDGSTS: the warp copies the rows together; completion via cp.async arrive (noinc)
        for (int q = 0; q < n; ++q) {
          const int src = __shfl_sync(0xffffffffu, r.node, __fns(bal, 0, q + 1));
          const size_t g = (size_t)src * p.Lp + (size_t)cur.sl * SW;
          const int rs = rr.rpos + q;
          row_cp_async<SW>(sig + rs * SW, sex + rs * SW, gm + g, ge + g, lane);
        }
        cp_async_mbar_arrive_noinc(&full[ds]);
        if (lane == 0) mbar_arrive(&full[ds]);
      } else {
        if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)n * (unsigned)SW * 6u);
        __syncwarp();
        if (ok) {
          const size_t g = (size_t)r.node * p.Lp + (size_t)cur.sl * SW;
          const int rs = rr.rpos + slot;
          bulk_g2s(sig + rs * SW, gm + g, SW * 4, &full[ds]);
          bulk_g2s(sex + rs * SW, ge + g, SW * 2, &full[ds]);
        }
      }
      rr.head += (unsigned)n;
      rr.rpos += n;
      if (rr.rpos >= R) rr.rpos -= R;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers: group g takes items k = g, g + NG, ...; warp w of the group owns commodities
  // [w * 32 * CPT, (w + 1) * 32 * CPT) of the item's slice
  const int grp = warp / PIPE_NWC, wg = warp % PIPE_NWC;
  const int col = wg * 32 * CPT + lane * CPT;
  ItemIt it;
  it.init(blockIdx.x + grp * gridDim.x, PIPE_NG * gridDim.x, pc.ns);
  M* const bmt = v.bm(t);
  E* const bet = v.be(t);
  for (int k = grp; it.node < p.N; k += PIPE_NG, it.next()) {
    const int ds = k & (PIPE_SD - 1);
    mbar_wait(&full[ds], (k / PIPE_SD) & 1);
    const PipeHdr& h = hdr[ds];
    if (pc.dry) {
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[ds]);
      continue;
    }
    const int base = h.start * SW + col;
    M s[CPT];
    int Ex[CPT];
    sum_rows<CPT>(sig + base, sex + base, h.kb, h.k2, h.n, s, Ex);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    Lane<M, E, CPT> out;
    norm_lane<TrF32, CPT, false>(p, s, Ex, out, it.sl * SW + col, it.node);
    const size_t g = (size_t)it.node * p.Lp + (size_t)(it.sl * SW + col);
    out.store(bmt + g, bet + g);
  }
}

}  // namespace mmf
