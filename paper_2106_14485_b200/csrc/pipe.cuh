// pipe.cuh — warp-specialised, TMA-pipelined persistent sweep kernels (option kernels = 5, fp32 mode).
//
// Why: the gather of a step is latency-bound when each warp walks its own dependent chain
// (CSR pointer -> arc records -> neighbour rows -> arithmetic) with the rows landing in registers:
// bytes in flight per SM are capped by the register file (ncu on [4]: 25-37 % occupancy, long-scoreboard
// stalls, 28-34 % of DRAM bandwidth).  Here one producer warp per CTA runs ahead of the arithmetic:
//   * the arc records of upcoming items (ELL layout [T][N][D], no CSR pointer round trip) are prefetched
//     P items ahead with cp.async into a small ring;
//   * the neighbour rows of an item (slice of SW commodities of each gathered node: significand plane +
//     exponent plane) are fetched with cp.async.bulk (TMA bulk copies, SASS UBLKCP) into an S-stage
//     shared-memory ring, completion tracked by mbarrier transaction counts;
// and NWC consumer warps compute from shared memory and release the stage.  Work items are visited in
// grid-stride order (item = blockIdx.x + k * gridDim.x over node-major (node, slice) pairs), so at any
// moment the whole GPU works on a narrow band of consecutive nodes: a gathered row is reused from L2 by
// the neighbouring nodes' CTAs while it is still resident (nodes are numbered for locality).
//
// Backward step (eq:psi):  beta_t[i, slice] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a, slice].
#pragma once
#include "headflow.cuh"

namespace mmf {

constexpr int PIPE_NWC = 8;                       // consumer warps per group (one group = one item)
constexpr int PIPE_NG = 2;                        // consumer groups (alternate items)
constexpr int PIPE_THREADS = (PIPE_NWC * PIPE_NG + 1) * 32;  // + one producer warp
constexpr int PIPE_P = 12;                        // record prefetch distance (items)
constexpr int PIPE_RP = 16;                       // record ring slots (> PIPE_P)
constexpr int PIPE_NR = 8;                        // rows a consumer holds in registers (fast path)
constexpr int PIPE_SD = 16;                       // item descriptors (power of two)

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

struct PipeCfg5 {
  int R;       // row slots in the shared-memory ring (each SW significands + SW exponents)
  int SD;      // item descriptors (= PIPE_SD)
  int D;       // ELL width of the gathered arc lists (max degree, <= 32)
  int SW;      // commodities per item (slice) = 32 * CPT * PIPE_NWC
  int ns;      // slices per node = Lp / SW
  int nitems;  // N * ns
};

// item descriptor: the n present rows (compacted, nonzero factor; ring slots start .. start + n - 1 mod R)
// and their arc factors K W
struct PipeHdr {
  float km[32];
  int ke[32];
  int n;
  int start;  // first ring slot (mod R)
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

// lane-row of a stage: CPT significands + CPT int16 exponents (packed two per word when CPT is even)
template <int CPT> __device__ __forceinline__ void lds_row(const float* sm, const int16_t* se, Row<TrF32, CPT>& x) {
  x.load(sm, se);  // (generic pointers into shared memory: LDS after address-space inference)
}

// extended-range sum over the n compacted rows of a stage (rows q < n, factors in the header):
//   out = sum_q x_q * KW_q   as (s, E) per commodity, E = max_q (e_q + ke_q)
// fp32 packed arithmetic (CPT even), per pair of commodities and row: one VIADDMNMX.S16x2 for the max
// (e + ke is exact in int16: |e| <= 16384, |ke| <= 16000); in the sum pass d = max(max(e + ke, E - 32512)
// - E, -126) by two more (no 16-bit wrap), the scale KW * 2^d by an integer add into the float's exponent
// field (mod 2^32 the low / high half of d << 23 equals d2 << 23 / (d2 & 0xffff0000) << 7), then FFMA.
template <int CPT>
__device__ __forceinline__ void stage_sum(const float* sig, const int16_t* sex, int col, int SW, int nslots,
                                          const PipeHdr& h, int n, float* s, int* Ex) {
  const int start = h.start;
  auto slot = [&](int q) {
    const int r = start + q;
    return (r >= nslots ? r - nslots : r) * SW + col;  // (shared-memory index: 32-bit)
  };
  typedef Row<TrF32, CPT> R;
  if constexpr (R::PACKED) {
    constexpr int NW = R::NW;
    unsigned E2[NW];
#pragma unroll
    for (int w = 0; w < NW; ++w) E2[w] = 0x80008000u;
    float acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
    if (n <= PIPE_NR) {
      R x[PIPE_NR];
#pragma unroll
      for (int q = 0; q < PIPE_NR; ++q)
        if (q < n) lds_row<CPT>(sig + slot(q), sex + slot(q), x[q]);
#pragma unroll
      for (int q = 0; q < PIPE_NR; ++q)
        if (q < n) {
          const unsigned k2 = pack2(h.ke[q]);
#pragma unroll
          for (int w = 0; w < NW; ++w) E2[w] = __viaddmax_s16x2((unsigned)x[q].w[w], k2, E2[w]);
        }
      unsigned nE2[NW], Lo2[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        nE2[w] = __vneg2(E2[w]);
        Lo2[w] = __vsubss2(E2[w], 0x7f007f00u);  // E - 32512 (saturated): e + ke below it is negligible
      }
#pragma unroll
      for (int q = 0; q < PIPE_NR; ++q)
        if (q < n) {
          const unsigned k2 = pack2(h.ke[q]);
          const unsigned kb = __float_as_uint(h.km[q]);
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            // d = max(max(e + ke, E - 32512) - E, -126): every 16-bit intermediate in range, no wrap
            const unsigned tq = __viaddmax_s16x2((unsigned)x[q].w[w], k2, Lo2[w]);
            const unsigned d2 = __viaddmax_s16x2(tq, nE2[w], 0xff82ff82u);
            acc[2 * w] = fmaf(x[q].m[2 * w], __uint_as_float(kb + (d2 << 23)), acc[2 * w]);
            acc[2 * w + 1] = fmaf(x[q].m[2 * w + 1], __uint_as_float(kb + ((d2 & 0xffff0000u) << 7)), acc[2 * w + 1]);
          }
        }
    } else {  // high degree: two passes over shared memory
      for (int q = 0; q < n; ++q) {
        R x;
        lds_row<CPT>(sig + slot(q), sex + slot(q), x);
        const unsigned k2 = pack2(h.ke[q]);
#pragma unroll
        for (int w = 0; w < NW; ++w) E2[w] = __viaddmax_s16x2((unsigned)x.w[w], k2, E2[w]);
      }
      unsigned nE2[NW], Lo2[NW];
#pragma unroll
      for (int w = 0; w < NW; ++w) {
        nE2[w] = __vneg2(E2[w]);
        Lo2[w] = __vsubss2(E2[w], 0x7f007f00u);
      }
      for (int q = 0; q < n; ++q) {
        R x;
        lds_row<CPT>(sig + slot(q), sex + slot(q), x);
        const unsigned k2 = pack2(h.ke[q]);
        const unsigned kb = __float_as_uint(h.km[q]);
#pragma unroll
        for (int w = 0; w < NW; ++w) {
          const unsigned tq = __viaddmax_s16x2((unsigned)x.w[w], k2, Lo2[w]);
          const unsigned d2 = __viaddmax_s16x2(tq, nE2[w], 0xff82ff82u);
          acc[2 * w] = fmaf(x.m[2 * w], __uint_as_float(kb + (d2 << 23)), acc[2 * w]);
          acc[2 * w + 1] = fmaf(x.m[2 * w + 1], __uint_as_float(kb + ((d2 & 0xffff0000u) << 7)), acc[2 * w + 1]);
        }
      }
    }
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      Ex[2 * w] = (int)(short)(E2[w] & 0xffffu);
      Ex[2 * w + 1] = (int)E2[w] >> 16;
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) s[c] = acc[c];
  } else {  // CPT = 1: plain ints
    int E = EZERO - 4 * ELIM;
    for (int q = 0; q < n; ++q) E = max(E, (int)sex[slot(q)] + h.ke[q]);
    float a = 0.f;
    for (int q = 0; q < n; ++q) {
      const int d = max((int)sex[slot(q)] + h.ke[q] - E, -126);
      a = fmaf(sig[slot(q)], __uint_as_float(__float_as_uint(h.km[q]) + ((unsigned)d << 23)), a);
    }
    s[0] = a;
    Ex[0] = E;
  }
}

// ------------------------------------------------------------------------------------------------
template <int CPT>
__global__ void __launch_bounds__(PIPE_THREADS, 1) k_bwd_pipe(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  extern __shared__ __align__(16) unsigned char smem[];
  const PipeSmem L = pipe_smem(pc.R, pc.SD, pc.D, pc.SW);
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  PipeHdr* hdr = (PipeHdr*)(smem + L.off_hdr);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int D = pc.D, SW = pc.SW, R = pc.R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_SD; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], PIPE_NWC);  // one consumer group per item
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
    unsigned head = 0, tail = 0;  // row-slot counters (monotonic); slots [tail, head) are in use
    int rpos = 0;                 // head mod R
    int kold = 0;                 // items < kold are known to be released
    auto release = [&]() {        // wait for item kold's consumers, free its rows
      const int ds = kold & (PIPE_SD - 1);
      mbar_wait(&empty[ds], (kold / PIPE_SD) & 1);
      tail = (unsigned)hdr[ds].end;
      ++kold;
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
      while (kold <= k - PIPE_SD) release();                      // descriptor reuse
      while (head + (unsigned)n - tail > (unsigned)R) release();  // row space
      const int ds = k & (PIPE_SD - 1);
      const int slot = __popc(bal & ((1u << lane) - 1u));
      if (ok) {
        hdr[ds].km[slot] = r.km;
        hdr[ds].ke[slot] = r.ke;
      }
      if (lane == 0) {
        hdr[ds].n = n;
        hdr[ds].start = rpos;
        hdr[ds].end = (int)(head + (unsigned)n);  // monotonic row counter after this item (producer only)
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)n * (unsigned)SW * 6u);
      __syncwarp();
      if (ok) {
        const size_t g = (size_t)r.node * p.Lp + (size_t)cur.sl * SW;
        int rs = rpos + slot;
        if (rs >= R) rs -= R;
        bulk_g2s(sig + rs * SW, gm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + rs * SW, ge + g, SW * 2, &full[ds]);
      }
      head += (unsigned)n;
      rpos += n;
      if (rpos >= R) rpos -= R;
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
    M s[CPT];
    int Ex[CPT];
    stage_sum<CPT>(sig, sex, col, SW, R, h, h.n, s, Ex);
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    Lane<M, E, CPT> out;
    norm_lane<TrF32, CPT>(p, s, Ex, out, it.sl * SW + col, it.node);
    const size_t g = (size_t)it.node * p.Lp + (size_t)(it.sl * SW + col);
    out.store(bmt + g, bet + g);
  }
}

}  // namespace mmf
