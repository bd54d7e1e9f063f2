// win.cuh — sliding-window sweep kernels (option kernels = 6, fp32 mode).
//
// Why: a step's gather reads every message row ~|A|/N times (4.8 on [4], 10.3 on [5]); served from L2 the
// pipelined kernels reach only ~5.4 TB/s into the SMs.  Here a CTA owns one commodity slice
// (SW = 32 * CPT commodities) of one node segment, visits the segment's node blocks (32 consecutive
// nodes) in order and keeps a window of message rows in shared memory: the rows of the node blocks
// [b - Wb, b + Wb] around the current block b, streamed in once per CTA with cp.async (row blocks are
// prefetched PD blocks ahead through commit groups).  Nodes are numbered so that almost every arc joins
// nodes at most Wb blocks apart (a strip ordering on [4], reverse Cuthill-McKee elsewhere, chosen by the
// host); the few arcs that leave the window ("far" arcs: highways, strip seams) gather their rows through
// a per-block far list, prefetched like the window.  All gathers then read shared memory; DRAM and L2
// traffic is ~1x the algorithmic bytes plus the far rows.
//
// Per-record tables (window slot or far index of the gathered row) are static and built on the host.
#pragma once
#include <cuda.h>
#include "pipefwd.cuh"

namespace mmf {

constexpr int WIN_BR = 32;        // nodes per block (= rows per row block)
constexpr int WIN_WARPS = 16;
constexpr int WIN_THREADS = WIN_WARPS * 32;
constexpr int WIN_PD = 3;         // prefetch distance (blocks)

struct WinCfg {
  int ns;      // commodity slices of SW
  int nseg;    // node segments
  int segB;    // node blocks per segment
  int Wb;      // window half-width (blocks)
  int RBa;     // ring blocks of the gathered window = 2 Wb + 1 + PD
  int farmax;  // far rows per block (capacity)
  int maxrec;  // records per block (capacity)
  int nblk;    // node blocks = ceil(N / 32)
  int dry;     // diagnostics: 1 = stream only (no arithmetic), 2 = no normalisation / store
};

// 2-D TMA views of the gathered message planes: significand (fp32) and exponent (u16) planes as
// [rows = slots * N][Lp] tensors, box = 32 rows x SW commodities (one window row block per operation)
struct WinTmaps {
  CUtensorMap sig;
  CUtensorMap exp;
};

struct WinDir {        // static tables of one gather direction (in-arcs or out-arcs)
  const int* ptr;      // [N + 1] CSR pointer of the direction (in_ptr / out_ptr)
  const int* src;      // [A] per CSR record: window slot (< RBa * 32) or RBa * 32 + far index
  const int* fptr;     // [nblk + 1] far-list offsets
  const int* fnode;    // far nodes (unique per block)
};

template <int CPT> struct WinSmem {
  size_t off_sig, off_exp, off_rec, off_src, off_ptr, off_desc, off_flist, off_meta, off_bar, total;
  int rows;  // window rows + far rows + one zero row
};
// row space of the window arrays: [0, RBa*32) window ring, then (PD+1) far buffers of farmax rows, then a
// zero row (significand 0, exponent EZERO: the target of zero-factor arcs, so the sums need no branches)
template <int CPT> __host__ __device__ inline WinSmem<CPT> win_smem(const WinCfg& c) {
  constexpr int SW = 32 * CPT;
  WinSmem<CPT> m;
  size_t o = 0;
  auto take = [&](size_t b) {
    size_t r = o;
    o += (b + 127) / 128 * 128;
    return r;
  };
  m.rows = c.RBa * WIN_BR + (WIN_PD + 1) * c.farmax + 1;
  m.off_sig = take((size_t)m.rows * SW * 4);
  m.off_exp = take((size_t)m.rows * SW * 2);
  m.off_rec = take((size_t)(WIN_PD + 2) * c.maxrec * 16);
  m.off_src = take((size_t)(WIN_PD + 2) * c.maxrec * 4);
  m.off_ptr = take((size_t)(WIN_PD + 2) * (WIN_BR + 1) * 4);
  m.off_desc = take((size_t)2 * c.maxrec * 16);
  m.off_flist = take((size_t)(2 * WIN_PD + 1) * c.farmax * 4);
  m.off_meta = take((size_t)2 * (c.segB + 2 * WIN_PD + 3) * 4);
  m.off_bar = take((size_t)c.RBa * 8);
  m.total = o;
  return m;
}

// per-row descriptor of a block (built once per block by all threads): the row's index in the window
// arrays and the arc factor K W (significand bits, exponent packed twice as int16x2)
struct WinDesc {
  int row;
  unsigned kb;
  unsigned k2;
  int pad;
};

__device__ __forceinline__ void cp_async4s(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
template <int N> __device__ __forceinline__ void cp_async_wait_n() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// The window machinery of one CTA (slice s, segment g) over the gathered plane (gm, ge).
template <int CPT> struct Win {
  static constexpr int SW = 32 * CPT;
  const DevPtrs& p;
  const WinCfg& c;
  const WinDir& d;
  const ArcKW<float>* grec;  // CSR records of the step
  const float* gm;
  const int16_t* ge;
  int col0, bs, be, nrb, wr, zrow;
  float* sig;
  int16_t* sex;
  ArcKW<float>* rec;
  int* src;
  int* ptr;
  WinDesc* desc;
  int* flist;
  int* mb;   // record offset of block bs + i
  int* mf;   // far-list offset of block bs + i
  unsigned long long* bar;  // [RBa] completion of the ring slots' TMA row-block loads
  const WinTmaps* tm;       // (or null: cp.async row blocks)
  int trow0;                // tensor row of node 0 of the gathered slot
  __device__ __forceinline__ Win(const DevPtrs& p_, const WinCfg& c_, const WinDir& d_, unsigned char* smem,
                                 const ArcKW<float>* grec_, const float* gm_, const int16_t* ge_, int s, int g,
                                 const WinTmaps* tm_ = nullptr, int trow0_ = 0)
      : p(p_), c(c_), d(d_), grec(grec_), gm(gm_), ge(ge_), tm(tm_), trow0(trow0_) {
    const WinSmem<CPT> L = win_smem<CPT>(c);
    sig = (float*)(smem + L.off_sig);
    sex = (int16_t*)(smem + L.off_exp);
    rec = (ArcKW<float>*)(smem + L.off_rec);
    src = (int*)(smem + L.off_src);
    ptr = (int*)(smem + L.off_ptr);
    desc = (WinDesc*)(smem + L.off_desc);
    flist = (int*)(smem + L.off_flist);
    bar = (unsigned long long*)(smem + L.off_bar);
    mb = (int*)(smem + L.off_meta);
    mf = mb + (c.segB + 2 * WIN_PD + 3);
    col0 = s * SW;
    bs = g * c.segB;
    be = min(bs + c.segB, c.nblk);
    nrb = c.nblk;
    wr = c.RBa * WIN_BR;
    zrow = L.rows - 1;
  }
  __device__ __forceinline__ void preload_meta() {
    const int n = be - bs + 2 * WIN_PD + 2;
    for (int i = threadIdx.x; i <= n; i += blockDim.x) {
      const int b = min(bs + i, nrb);
      mb[i] = d.ptr[min(b * WIN_BR, p.N)];
      mf[i] = d.fptr[b];
    }
    for (int k = threadIdx.x; k < SW; k += blockDim.x) {
      sig[(size_t)zrow * SW + k] = 0.f;
      sex[(size_t)zrow * SW + k] = (int16_t)EZERO;
    }
  }
  __device__ __forceinline__ void issue_rowblock(int rb) {
    if (rb < 0 || rb >= nrb) return;
    const int slot = rb % c.RBa;
    if (tm) {  // one 2-D TMA load per plane: rows rb*32 .. rb*32+31 of the slot, commodities col0 .. col0+SW
      if (threadIdx.x == 0) {
        fence_proxy_async();  // (the slot's previous generic-proxy reads precede the async-proxy write)
        mbar_arrive_expect_tx(&bar[slot], (unsigned)(WIN_BR * SW * 6));
        const int y = trow0 + rb * WIN_BR;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                smem_u32(sig + slot * WIN_BR * SW)),
            "l"(&tm->sig), "r"(col0), "r"(y), "r"(smem_u32(&bar[slot]))
            : "memory");
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];\n" ::"r"(
                smem_u32(sex + slot * WIN_BR * SW)),
            "l"(&tm->exp), "r"(col0), "r"(y), "r"(smem_u32(&bar[slot]))
            : "memory");
      }
      return;
    }
    constexpr int CS = SW / 4, CE = SW / 8 > 0 ? SW / 8 : 1;  // 16-byte chunks per row
    for (int k = threadIdx.x; k < WIN_BR * CS; k += blockDim.x) {
      const int r = k / CS, q = k - r * CS;
      const int row = rb * WIN_BR + r;
      if (row < p.N) cp_async16(sig + (slot * WIN_BR + r) * SW + q * 4, gm + (size_t)row * p.Lp + col0 + q * 4);
    }
    if constexpr (SW >= 8) {
      for (int k = threadIdx.x; k < WIN_BR * CE; k += blockDim.x) {
        const int r = k / CE, q = k - r * CE;
        const int row = rb * WIN_BR + r;
        if (row < p.N) cp_async16(sex + (slot * WIN_BR + r) * SW + q * 8, ge + (size_t)row * p.Lp + col0 + q * 8);
      }
    }
  }
  // records, source slots and node offsets of block b
  __device__ __forceinline__ void issue_records(int b) {
    if (b >= be) return;
    const int bf = (b - bs) % (WIN_PD + 2);
    const int r0 = mb[b - bs], r1 = mb[b - bs + 1];
    for (int k = threadIdx.x; k < r1 - r0; k += blockDim.x) {
      cp_async16(rec + bf * c.maxrec + k, grec + r0 + k);
      cp_async4s(src + bf * c.maxrec + k, d.src + r0 + k);
    }
    for (int k = threadIdx.x; k <= WIN_BR; k += blockDim.x)
      cp_async4s(ptr + bf * (WIN_BR + 1) + k, d.ptr + min(b * WIN_BR + k, p.N));
  }
  __device__ __forceinline__ void issue_farlist(int b) {
    if (b >= be) return;
    const int bf = (b - bs) % (2 * WIN_PD + 1);
    const int f0 = mf[b - bs], f1 = mf[b - bs + 1];
    for (int k = threadIdx.x; k < f1 - f0; k += blockDim.x) cp_async4s(flist + bf * c.farmax + k, d.fnode + f0 + k);
  }
  __device__ __forceinline__ int far_row(int b, int f) const { return wr + ((b - bs) % (WIN_PD + 1)) * c.farmax + f; }
  __device__ __forceinline__ void issue_farrows(int b) {
    if (b >= be) return;
    const int bl = (b - bs) % (2 * WIN_PD + 1);
    const int nf = mf[b - bs + 1] - mf[b - bs];
    constexpr int CS = SW / 4, CE = SW / 8 > 0 ? SW / 8 : 1;
    for (int k = threadIdx.x; k < nf * CS; k += blockDim.x) {
      const int f = k / CS, q = k - f * CS;
      const int node = flist[bl * c.farmax + f];
      cp_async16(sig + far_row(b, f) * SW + q * 4, gm + (size_t)node * p.Lp + col0 + q * 4);
    }
    if constexpr (SW >= 8) {
      for (int k = threadIdx.x; k < nf * CE; k += blockDim.x) {
        const int f = k / CE, q = k - f * CE;
        const int node = flist[bl * c.farmax + f];
        cp_async16(sex + far_row(b, f) * SW + q * 8, ge + (size_t)node * p.Lp + col0 + q * 8);
      }
    }
  }
  // descriptors of block b (records of b complete)
  __device__ __forceinline__ void prepass(int b) {
    if (b >= be) return;
    const int bf = (b - bs) % (WIN_PD + 2);
    const int nrec = mb[b - bs + 1] - mb[b - bs];
    WinDesc* ds = desc + ((b - bs) & 1) * c.maxrec;
    for (int k = threadIdx.x; k < nrec; k += blockDim.x) {
      const ArcKW<float> r = rec[bf * c.maxrec + k];
      const int v = src[bf * c.maxrec + k];
      WinDesc e;
      if (r.km > 0.f) {
        e.row = v < wr ? v : far_row(b, v - wr);
        e.kb = __float_as_uint(r.km);
        e.k2 = pack2(r.ke);
      } else {  // zero factor: the zero row, factor 1 * 2^-ELIM (never the maximum, contributes 0)
        e.row = zrow;
        e.kb = 0x3f800000u;
        e.k2 = pack2(-ELIM);
      }
      e.pad = 0;
      ds[k] = e;
    }
  }
  __device__ __forceinline__ void prologue() {
    if (tm && threadIdx.x == 0) {
      for (int k = 0; k < c.RBa; ++k) mbar_init(&bar[k], 1);
      mbar_fence_init();
    }
    preload_meta();
    __syncthreads();
    for (int rb = bs - c.Wb; rb < bs + c.Wb + WIN_PD; ++rb) issue_rowblock(rb);
    for (int b = bs; b <= bs + WIN_PD; ++b) issue_records(b);
    for (int b = bs; b < bs + 2 * WIN_PD; ++b) issue_farlist(b);
    cp_async_commit();
    cp_async_wait_n<0>();
    __syncthreads();
    for (int b = bs; b < bs + WIN_PD; ++b) issue_farrows(b);
    cp_async_commit();
    prepass(bs);
    cp_async_wait_n<0>();
    for (int rb = bs - c.Wb; rb <= bs + c.Wb; ++rb) wait_rowblock(rb);
    __syncthreads();
  }
  // iteration b, after the top wait + barrier: prefetch ahead, then the descriptors of block b + 1
  __device__ __forceinline__ void issue_ahead(int b) {
    issue_rowblock(b + c.Wb + WIN_PD);
    issue_records(b + WIN_PD + 1);
    issue_farlist(b + 2 * WIN_PD);
    issue_farrows(b + WIN_PD);
    cp_async_commit();
    prepass(b + 1);
  }
  // TMA row blocks: wait for row block rb.  This CTA loads row blocks rb0, rb0 + 1, ... in order, so the load
  // of rb is use number (rb - rb0) / RBa of its ring slot's barrier -> phase parity
  __device__ __forceinline__ void wait_rowblock(int rb) {
    if (!tm || rb < 0 || rb >= nrb) return;
    const int rb0 = max(bs - c.Wb, 0);
    mbar_wait(&bar[rb % c.RBa], ((rb - rb0) / c.RBa) & 1);
  }
  __device__ __forceinline__ void top(int b) {
    if (b > bs) {
      cp_async_wait_n<WIN_PD - 1>();
      wait_rowblock(b + c.Wb);
      __syncthreads();
    }
  }
  __device__ __forceinline__ const WinDesc* block_desc(int b) const { return desc + ((b - bs) & 1) * c.maxrec; }
  __device__ __forceinline__ const int* block_ptr(int b) const { return ptr + ((b - bs) % (WIN_PD + 2)) * (WIN_BR + 1); }
};

// extended-range sum of a node's n rows (descriptors ds[0 .. n)), compile-time n: rows read once
template <int CPT, int N>
__device__ __forceinline__ void win_sum_n(const float* sig, const int16_t* sex, const WinDesc* ds, int lane, float* s,
                                          int* Ex) {
  constexpr int SW = 32 * CPT;
  Row<TrF32, CPT> x[N > 0 ? N : 1];
  unsigned kb[N > 0 ? N : 1], k2[N > 0 ? N : 1];
#pragma unroll
  for (int q = 0; q < N; ++q) {
    const WinDesc e = ds[q];
    kb[q] = e.kb;
    k2[q] = e.k2;
    x[q].load(sig + e.row * SW + lane * CPT, sex + e.row * SW + lane * CPT);
  }
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
template <int CPT>
__device__ __forceinline__ void win_sum_any(const float* sig, const int16_t* sex, const WinDesc* ds, int n, int lane,
                                            float* s, int* Ex) {
  constexpr int SW = 32 * CPT;
  unsigned E2[CPT];
  xmax_init<CPT>(E2);
  for (int q = 0; q < n; ++q) {
    const WinDesc e = ds[q];
    Row<TrF32, CPT> x;
    x.load(sig + e.row * SW + lane * CPT, sex + e.row * SW + lane * CPT);
    xmax_add<CPT>(E2, x, e.k2, k2_to_ke(e.k2));
  }
  XPre<CPT> P;
  P.set(E2);
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = 0.f;
    Ex[c] = P.E[c];
  }
  for (int q = 0; q < n; ++q) {
    const WinDesc e = ds[q];
    Row<TrF32, CPT> x;
    x.load(sig + e.row * SW + lane * CPT, sex + e.row * SW + lane * CPT);
    xacc<CPT>(x, e.kb, e.k2, k2_to_ke(e.k2), P, s);
  }
}
template <int CPT>
__device__ __forceinline__ void win_sum(const float* sig, const int16_t* sex, const WinDesc* ds, int n, int lane,
                                        float* s, int* Ex) {
  switch (n) {
    case 0: win_sum_n<CPT, 0>(sig, sex, ds, lane, s, Ex); break;
    case 1: win_sum_n<CPT, 1>(sig, sex, ds, lane, s, Ex); break;
    case 2: win_sum_n<CPT, 2>(sig, sex, ds, lane, s, Ex); break;
    case 3: win_sum_n<CPT, 3>(sig, sex, ds, lane, s, Ex); break;
    case 4: win_sum_n<CPT, 4>(sig, sex, ds, lane, s, Ex); break;
    case 5: win_sum_n<CPT, 5>(sig, sex, ds, lane, s, Ex); break;
    case 6: win_sum_n<CPT, 6>(sig, sex, ds, lane, s, Ex); break;
    case 7: win_sum_n<CPT, 7>(sig, sex, ds, lane, s, Ex); break;
    case 8: win_sum_n<CPT, 8>(sig, sex, ds, lane, s, Ex); break;
    default: win_sum_any<CPT>(sig, sex, ds, n, lane, s, Ex); break;
  }
}

// backward step t: beta_t[i] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a]  (eq:psi P:1038-1043)
template <int CPT>
__global__ void __launch_bounds__(WIN_THREADS, 1) k_bwd_win(DevPtrs p, WinCfg c, WinDir d, const __grid_constant__ WinTmaps tmb,
                                                            int use_tma, int t) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int s = blockIdx.x % c.ns, g = blockIdx.x / c.ns;
  if (g * c.segB >= c.nblk) return;
  View<TrF32> v(p);
  Win<CPT> w(p, c, d, smem, (const ArcKW<float>*)p.outrec + (size_t)t * p.A, v.bm(t + 1), v.be(t + 1), s, g,
             use_tma ? &tmb : nullptr, (t + 1) * p.N);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  w.prologue();
  float* const bmt = v.bm(t);
  int16_t* const bet = v.be(t);
  for (int b = w.bs; b < w.be; ++b) {
    w.top(b);
    w.issue_ahead(b);
    const int* pb = w.block_ptr(b);
    const WinDesc* db = w.block_desc(b);
    if (c.dry == 1) continue;
    for (int u = warp; u < WIN_BR; u += WIN_WARPS) {
      const int i = b * WIN_BR + u;
      if (i >= p.N) break;
      const int k0 = pb[u] - pb[0], k1 = pb[u + 1] - pb[0];
      float sm[CPT];
      int Ex[CPT];
      win_sum<CPT>(w.sig, w.sex, db + k0, k1 - k0, lane, sm, Ex);
      if (c.dry == 2) {
        if (sm[0] == 12345.f) bmt[0] = 0.f;  // keep the sum alive
        continue;
      }
      Lane<float, int16_t, CPT> out;
      norm_lane<TrF32, CPT, false>(p, sm, Ex, out, w.col0 + lane * CPT, i);
      const size_t gidx = (size_t)i * p.Lp + w.col0 + lane * CPT;
      out.store(bmt + gidx, bet + gidx);
    }
  }
  cp_async_wait_n<0>();
}

}  // namespace mmf
