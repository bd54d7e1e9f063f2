// tiled.cuh — node-tile kernels of the sweep (the production path).
//
// Nodes are renumbered into compact tiles (BFS-grown blobs with a bounded halo; host side).  A CTA owns
// one tile J and a range of commodity chunks (LC = 32*CPT commodities per chunk: a warp covers a
// chunk, CPT commodities per lane).  For every chunk, the message rows it gathers — alpha_{t-1} over
// the tile's in-halo H_in(J) and beta_{t+1} over its out-halo H_out(J) — are brought into shared
// memory by TMA bulk copies (cp.async.bulk + mbarrier), double-buffered so the copies of chunk c+1
// overlap the arithmetic of chunk c.  Each gathered row crosses L2->SM once per CTA and chunk instead
// of once per arc (halo amplification |H|/|J| instead of the mean degree); the tile's arc metadata
// (halo indices, K W factors) is staged once per CTA.
//
// Forward kernel K_t (one launch per step, SURVEY §8(a) a3 re-associated):
//   1. alpha_t[J]  = sum_{a->j} alpha_{t-1}[i_a] K_{t-1}[a] W_{t-1}[a]     (SpMM^T of step t-1, eq:psi_hat)
//      (t = 0: alpha_0 = U0 = mu0 ./ beta_0, a2 fused)
//   2. the chunk's flow F_t[a] contributions of the tile's out-arcs a = (i -> k), i in J:
//        sum_l alpha_t[i,l] K_t[a] W_t[a] beta_{t+1}[k,l]                (cor:proj P:1078)
//      accumulated in shared memory over the CTA's chunks (warp-shuffle commodity reduction);
//   3. capacity-dual update W_t[a] <- min(W_t d_t / F_t, 1) by the CTA itself when it covers
//      all commodities, else by the last CTA of the tile to arrive (fixed-order sum of the group
//      partials: deterministic, no extra launch).
//   (t = T: step 1 only, then UT = muT ./ alpha_T -> beta_T, a4 fused.)
// so a forward step moves alpha_{t-1} (read), alpha_t (write), beta_{t+1} (read): 3 N L B_e.
// Backward kernel: beta_t[J] = sum_{a: i_a in J} K_t W_t beta_{t+1}[j_a] over the staged out-halo.
//
// Arithmetic (fp32 significand + int16 exponent messages, CPT even): extended-range sums are done in
// two passes — pass 1 takes the per-commodity maximum exponent with the packed 16x2 max-plus
// (VIADDMNMX.S16x2, two commodities per instruction), pass 2 adds x * (K W 2^(e - E)) where the scale
// is built by an integer add into the float exponent field, ~4 ALU ops per term.  Arcs whose factor
// is zero point at an all-zero staged row, so the inner loops have no branches.
#pragma once
#include "kernels.cuh"

namespace mmf {

constexpr int TILE_THREADS = 256;

struct TileMeta {
  int ntiles, B, nch, LC;
  const int* tile_ptr;   // [ntiles+1] node ranges (internal ids)
  const int* hin_ptr;    // [ntiles+1]
  const int* hin_node;   // halo-in nodes (tails of the tile's in-arcs), sorted per tile
  const int* hout_ptr;   // [ntiles+1]
  const int* hout_node;  // halo-out nodes (heads of the tile's out-arcs)
  const int* in_hidx;    // [A] internal arc -> index of its tail in the head tile's halo-in
  const int* out_hidx;   // [A] out-CSR position -> index of the head in the tail tile's halo-out
  int* cnt;              // [ntiles] arrival counters (zero between launches)
  void* part;            // [A][ngroup] group partial flows (M)
  int max_hin, max_hout; // largest halos (shared-memory sizing)
  int max_ia, max_oa;    // largest per-tile in-arc / out-arc counts
};

struct PipeCfg {
  int cpc;     // commodity chunks per CTA
  int ngroup;  // chunk groups per tile (= gridDim.y); > 1 -> partial flows + last arriver
};

template <class M, int CPT> struct VecM;
template <> struct VecM<float, 1> { typedef float T; };
template <> struct VecM<float, 2> { typedef float2 T; };
template <> struct VecM<float, 4> { typedef float4 T; };
struct __align__(16) float8v {
  float4 a, b;
};
template <> struct VecM<float, 8> { typedef float8v T; };
template <> struct VecM<double, 1> { typedef double T; };
template <> struct VecM<double, 2> { typedef double2 T; };
template <class E, int CPT> struct VecE;
template <> struct VecE<int16_t, 1> { typedef int16_t T; };
template <> struct VecE<int16_t, 2> { typedef unsigned T; };  // two int16 in one word
template <> struct VecE<int16_t, 4> { typedef uint2 T; };
template <> struct VecE<int16_t, 8> { typedef uint4 T; };
template <> struct VecE<int32_t, 1> { typedef int T; };
template <> struct VecE<int32_t, 2> { typedef int2 T; };

// CPT consecutive significands / exponents of one lane
template <class M, class E, int CPT> struct Lane {
  M m[CPT];
  E e[CPT];
  __device__ __forceinline__ void load(const M* pm, const E* pe) {
    typedef typename VecM<M, CPT>::T VM;
    typedef typename VecE<E, CPT>::T VE;
    VM vm = *reinterpret_cast<const VM*>(pm);
    VE ve = *reinterpret_cast<const VE*>(pe);
    const M* sm = reinterpret_cast<const M*>(&vm);
    const E* se = reinterpret_cast<const E*>(&ve);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      m[c] = sm[c];
      e[c] = se[c];
    }
  }
  __device__ __forceinline__ void store(M* pm, E* pe) const {
    typedef typename VecM<M, CPT>::T VM;
    typedef typename VecE<E, CPT>::T VE;
    VM vm;
    VE ve;
    M* sm = reinterpret_cast<M*>(&vm);
    E* se = reinterpret_cast<E*>(&ve);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      sm[c] = m[c];
      se[c] = e[c];
    }
    *reinterpret_cast<VM*>(pm) = vm;
    *reinterpret_cast<VE*>(pe) = ve;
  }
};

// ------------------------------------------------------------------------------------------------
// TMA bulk copies + mbarrier (async proxy) for the chunk pipeline

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
#ifndef MMF_WAIT_HINT
#define MMF_WAIT_HINT 0  // suspend-time hint (ns) of the consumers' full-barrier waits (0: the default)
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// a wait that suspends the warp until the phase completes or `hint` ns pass (no spinning issue slots: the
// waiting consumers leave them to the producer and to the consumers that have data)
__device__ __forceinline__ void mbar_wait_sleep(unsigned long long* bar, unsigned parity) {
#if MMF_WAIT_HINT > 0
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity), "n"(MMF_WAIT_HINT)
      : "memory");
#else
  mbar_wait(bar, parity);
#endif
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// issue (warp-wide) the bulk copies of one chunk's halo rows: rows r of `nodes` -> smem row r
template <class M, class E, int LC>
__device__ __forceinline__ void issue_rows(const M* gm, const E* ge, int Lp, size_t chunk0, const int* nodes, int n,
                                           M* sm, E* se, unsigned long long* bar, int lane) {
  for (int r = lane; r < n; r += 32) {
    const size_t g = (size_t)nodes[r] * Lp + chunk0;
    bulk_g2s(sm + (size_t)r * LC, gm + g, LC * sizeof(M), bar);
    bulk_g2s(se + (size_t)r * LC, ge + g, LC * sizeof(E), bar);
  }
}

// ------------------------------------------------------------------------------------------------

// FAC: apply the node factors of the launch's output layer (NEXT-2 commodity node factor D, NEXT-3 node-capacity
// dual u) here; the pipelined kernels instantiate FAC = false (their launches are followed by k_apply_factors when a
// problem has such factors): the per-element checks cost their epilogues up to 17 % (measured on [4])
template <class T_, int CPT, bool FAC = true>
__device__ __forceinline__ void norm_lane(const DevPtrs& p, const typename T_::M* s, const int* E,
                                          Lane<typename T_::M, typename T_::E, CPT>& out, int l0, int node) {
  typedef typename T_::M M;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    M m;
    int e;
    if constexpr (sizeof(M) == 4) {
      // the sum is 0 or >= 1 (its largest term has K W x >= 1): no subnormal case
      const unsigned u = __float_as_uint(s[c]);
      m = __uint_as_float((u & 0x007fffffu) | 0x3f800000u);
      e = E[c] + (int)(u >> 23) - 127;
      if (u == 0u) {
        m = 0.f;
        e = EZERO;
      }
    } else {
      xf_norm<M>(s[c], E[c], m, e);
    }
    if constexpr (FAC) {
      if (p.dnm && m != M(0)) {  // commodity node factor of this layer (NEXT-2)
        const size_t k = (size_t)node * p.Lp + l0 + c;
        m *= ((const M*)p.dnm)[k];
        e += (int)((const typename T_::E*)p.dne)[k];
        if (m >= M(2)) {
          m *= M(0.5);
          e += 1;
        }
      }
      if (p.unlm && m != M(0)) {  // node-capacity dual of this layer (NEXT-3)
        m *= ((const M*)p.unlm)[node];
        e += p.unle[node];
        if (m >= M(2)) {
          m *= M(0.5);
          e += 1;
        }
        if (m == M(0)) e = EZERO;
      }
    }
    if (e > ELIM || (m != M(0) && e < -ELIM)) {
      set_error(p, ERR_RANGE, l0 + c, node);
      e = e > 0 ? ELIM : -ELIM;
    }
    MMF_DASSERT(m == M(0) ? true : (m >= M(1) && m < M(2) && e >= -ELIM && e <= ELIM));
    MMF_DASSERT(node >= 0 && node < p.N && l0 + c < p.Lp);
    out.m[c] = m;
    out.e[c] = (typename T_::E)e;
  }
}

// the node factors of layer t applied in place to a stored message layer (after the pipelined kernels, whose
// epilogues skip them): which = 0 alpha_t, 1 beta_t; the pointers in p are the launch's (lay: D, and u if set)
template <class T_> __global__ void k_apply_factors(DevPtrs p, int t, int which) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  View<T_> v(p);
  M* pm = which ? v.bm(t) : v.am(t);
  E* pe = which ? v.be(t) : v.ae(t);
  const size_t n = (size_t)p.N * p.Lp;
  for (size_t k = (size_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += (size_t)gridDim.x * blockDim.x) {
    M m = pm[k];
    if (m == M(0)) continue;
    int e = (int)pe[k];
    const int node = (int)(k / p.Lp);
    if (p.dnm) {
      m *= ((const M*)p.dnm)[k];
      e += (int)((const E*)p.dne)[k];
      if (m >= M(2)) {
        m *= M(0.5);
        e += 1;
      }
    }
    if (p.unlm) {
      m *= ((const M*)p.unlm)[node];
      e += p.unle[node];
      if (m >= M(2)) {
        m *= M(0.5);
        e += 1;
      }
    }
    if (m == M(0)) {
      e = EZERO;
    } else if (e > ELIM || e < -ELIM) {
      set_error(p, ERR_RANGE, (int)(k % p.Lp), node);
      e = e > 0 ? ELIM : -ELIM;
    }
    pm[k] = m;
    pe[k] = (E)e;
  }
}

// boundary scaling of one lane: x = mu / msg with 0/0 := 0 (a2 / a4)
template <class T_, int CPT>
__device__ __forceinline__ void boundary_lane(const DevPtrs& p, int which, int node, int l0, size_t g,
                                              const Lane<typename T_::M, typename T_::E, CPT>& msg,
                                              Lane<typename T_::M, typename T_::E, CPT>& out) {
  typedef typename T_::M M;
  typedef typename T_::E E;
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    const int l = l0 + c;
    M mu_m = M(0);
    int mu_e = EZERO;
    if (p.psrc) {
      if (l < p.L && (which == 0 ? p.psrc[l] : p.pdst[l]) == node) {
        int ex;
        const double fr = frexp(p.pmass[l], &ex);
        mu_m = (M)(fr * 2.0);
        mu_e = ex - 1;
      }
    } else {
      mu_m = ((const M*)(which == 0 ? p.mu0m : p.muTm))[g + c];
      mu_e = (int)((const E*)(which == 0 ? p.mu0e : p.muTe))[g + c];
    }
    M m = M(0);
    int e = EZERO;
    if (mu_m > M(0)) {
      if (msg.m[c] > M(0)) {
        xf_norm<M>(mu_m / msg.m[c], mu_e - (int)msg.e[c], m, e);
        if (e > ELIM || e < -ELIM) {
          set_error(p, ERR_RANGE, l, node);
          e = e > 0 ? ELIM : -ELIM;
        }
      } else {
        set_error(p, ERR_INFEASIBLE, l, node);
      }
    }
    out.m[c] = m;
    out.e[c] = (E)e;
  }
}

// per-arc metadata in shared memory: one 16-byte record per arc
//   h   : staged-row index of the gathered message (the all-zero row if the arc factor is 0)
//   kb  : K W significand (bits of a float in [1, 4); 1.0 for zero factors)
//   ke  : K W exponent (clamped to [-ELIM, ELIM])
//   k2  : ke packed twice into int16x2 (for the 16x2 max-plus)
// M = double: kb holds nothing; the double significand lives in a parallel array.
struct ArcRec {
  int h;
  unsigned kb;
  int ke;
  unsigned k2;
};

__device__ __forceinline__ unsigned pack2(int e) { return ((unsigned)e & 0xffffu) * 0x10001u; }

template <class M>
__device__ __forceinline__ void arc_rec(M km, int ke, M wm, int we, int h, int zero_row, ArcRec& r, M& mm) {
  M m = km * wm;
  int e = ke + we;
  const bool zero = !(m > M(0)) || e < -ELIM;
  if (zero) {
    m = M(1);
    e = -ELIM;
  }
  if (e > ELIM) e = ELIM;  // K > 2^ELIM (cost far below zero): clamp, ERANGE-level input
  r.h = zero ? zero_row : h;
  r.kb = sizeof(M) == 4 ? __float_as_uint((float)m) : 0u;
  r.ke = e;
  r.k2 = pack2(e);
  mm = m;
}

// smem region for the tile's arcs: in-arcs (forward SpMM), out-arcs (flow pass / backward SpMM)
template <class M> struct ArcSmem {
  int* iptr;     // [B+1] in-arc offsets of the tile's nodes
  int* optr;     // [B+1] out-arc offsets
  int* oa;       // [max_oa] arc id of out-arc q
  int* of;       // [max_oa] flow code: staged row of the head, -1 skip (uncapacitated), -2 zero factor
  ArcRec* ir;    // [max_ia]
  ArcRec* orr;   // [max_oa]
  M* im;         // [max_ia] K W significand (used by the generic / fp64 path)
  M* om;         // [max_oa]
  static __host__ __device__ size_t bytes(int B, int max_ia, int max_oa) {
    size_t b = (size_t)(2 * (B + 1) + 2 * max_oa) * 4;
    b = (b + 15) & ~size_t(15);
    b += (size_t)(max_ia + max_oa) * sizeof(ArcRec);
    b += ((size_t)(max_ia + max_oa) * sizeof(M) + 15) / 16 * 16;
    return b;
  }
  __device__ __forceinline__ void carve(unsigned char* base, int B, int max_ia, int max_oa) {
    iptr = (int*)base;
    optr = iptr + B + 1;
    oa = optr + B + 1;
    of = oa + max_oa;
    size_t off = (size_t)(2 * (B + 1) + 2 * max_oa) * 4;
    off = (off + 15) & ~size_t(15);
    ir = (ArcRec*)(base + off);
    orr = ir + max_ia;
    im = (M*)(orr + max_oa);
    om = im + max_ia;
  }
};

// stage the arc metadata of the tile (one thread per arc; independent loads)
template <class T_>
__device__ __forceinline__ void stage_arcs(const DevPtrs& p, const TileMeta& tm, ArcSmem<typename T_::M>& sa, int j0,
                                           int nb, int t_in, int t_out, bool want_in, bool want_out, bool all_out,
                                           int in_base, int zrow_in, int zrow_out) {
  typedef typename T_::M M;
  View<T_> v(p);
  for (int r = threadIdx.x; r <= nb; r += blockDim.x) {
    sa.iptr[r] = p.in_ptr[j0 + r] - p.in_ptr[j0];
    sa.optr[r] = p.out_ptr[j0 + r] - p.out_ptr[j0];
  }
  if (want_in) {
    const int a0 = p.in_ptr[j0], n = p.in_ptr[j0 + nb] - a0;
    const M* Km = v.Km(t_in);
    const int* Ke = v.Ke(t_in);
    const M* Wm = v.Wm(t_in);
    const int* We = v.We(t_in);
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int a = a0 + q;
      ArcRec r;
      M m;
      arc_rec<M>(Km[a], Ke[a], Wm[a], We[a], in_base + tm.in_hidx[a], zrow_in, r, m);
      sa.ir[q] = r;
      sa.im[q] = m;
    }
  }
  if (want_out) {
    const int k0 = p.out_ptr[j0], n = p.out_ptr[j0 + nb] - k0;
    const M* Km = v.Km(t_out);
    const int* Ke = v.Ke(t_out);
    const M* Wm = v.Wm(t_out);
    const int* We = v.We(t_out);
    const M* dc = v.dcap(t_out);
    for (int q = threadIdx.x; q < n; q += blockDim.x) {
      const int k = k0 + q;
      const int arc = p.out_arc[k];
      ArcRec r;
      M m;
      arc_rec<M>(Km[arc], Ke[arc], Wm[arc], We[arc], tm.out_hidx[k], zrow_out, r, m);
      sa.oa[q] = arc;
      sa.of[q] = (all_out || !isinf(dc[arc])) ? (r.h == zrow_out ? -2 : r.h) : -1;
      sa.orr[q] = r;
      sa.om[q] = m;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// extended-range weighted row sums over the staged halo: out = sum_q KW_q * x[h_q]

// generic path (any M / E / CPT): running-max accumulator
template <class T_, int CPT>
__device__ __forceinline__ void row_sum_generic(const typename T_::M* xm, const typename T_::E* xe, int lane,
                                                const ArcRec* rec, const typename T_::M* km, int q0, int q1,
                                                typename T_::M* s, int* E) {
  typedef typename T_::M M;
  typedef typename T_::E E_;
  constexpr int LC = 32 * CPT;
  XAcc<M> acc[CPT];
  for (int q = q0; q < q1; ++q) {
    const ArcRec r = rec[q];
    const M kwm = km[q];
    Lane<M, E_, CPT> x;
    x.load(xm + (size_t)r.h * LC + lane * CPT, xe + (size_t)r.h * LC + lane * CPT);
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c].add(x.m[c] * kwm, (int)x.e[c] + r.ke);
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = acc[c].s;
    E[c] = acc[c].E;
  }
}

// fp32 / int16 path, CPT even: two passes with packed exponents
template <int CPT>
__device__ __forceinline__ void row_sum_f32(const float* xm, const int16_t* xe, int lane, const ArcRec* rec, int q0,
                                            int q1, float* s, int* E) {
  constexpr int LC = 32 * CPT;
  constexpr int NP = CPT / 2;
  typedef typename VecE<int16_t, CPT>::T VE;
  unsigned E2[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) E2[k] = 0x80008000u;
  for (int q = q0; q < q1; ++q) {
    const ArcRec r = rec[q];
    const VE ev = *reinterpret_cast<const VE*>(xe + (size_t)r.h * LC + lane * CPT);
    const unsigned* ew = reinterpret_cast<const unsigned*>(&ev);
#pragma unroll
    for (int k = 0; k < NP; ++k) E2[k] = __viaddmax_s16x2(ew[k], r.k2, E2[k]);
  }
  int nE[CPT];
#pragma unroll
  for (int k = 0; k < NP; ++k) {
    E[2 * k] = (int)(short)(E2[k] & 0xffffu);
    E[2 * k + 1] = (int)E2[k] >> 16;
    nE[2 * k] = -E[2 * k];
    nE[2 * k + 1] = -E[2 * k + 1];
  }
  float acc[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
  for (int q = q0; q < q1; ++q) {
    const ArcRec r = rec[q];
    Lane<float, int16_t, CPT> x;
    x.load(xm + (size_t)r.h * LC + lane * CPT, xe + (size_t)r.h * LC + lane * CPT);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int d = max((int)x.e[c] + r.ke + nE[c], -126);          // <= 0 by construction of E
      const float sc = __uint_as_float(r.kb + ((unsigned)d << 23));  // K W 2^d, a normal float
      acc[c] = fmaf(x.m[c], sc, acc[c]);
    }
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) s[c] = acc[c];
}

template <class T_, int CPT>
__device__ __forceinline__ void row_sum(const typename T_::M* xm, const typename T_::E* xe, int lane, const ArcRec* rec,
                                        const typename T_::M* km, int q0, int q1, typename T_::M* s, int* E) {
  if constexpr (sizeof(typename T_::M) == 4 && sizeof(typename T_::E) == 2 && CPT % 2 == 0)
    row_sum_f32<CPT>(xm, xe, lane, rec, q0, q1, s, E);
  else
    row_sum_generic<T_, CPT>(xm, xe, lane, rec, km, q0, q1, s, E);
}

// flow term of one lane: sum_c lin(a_c * b_c * KW) over its CPT commodities
template <class T_, int CPT>
__device__ __forceinline__ typename T_::M flow_terms(const Lane<typename T_::M, typename T_::E, CPT>& a,
                                                     const Lane<typename T_::M, typename T_::E, CPT>& b,
                                                     typename T_::M kwm, int kwe) {
  typedef typename T_::M M;
  M f = M(0);
  if constexpr (sizeof(M) == 4) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      // scale 2^es as a float: es clamped to -127 gives exactly 0 (flows < 2^-126 are dropped)
      const int es = max((int)a.e[c] + (int)b.e[c] + kwe, -127);
      const float sc = __uint_as_float((unsigned)(es + 127) << 23);
      f = fmaf(a.m[c] * kwm * b.m[c], sc, f);
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) f += xf_to_lin<M>(a.m[c] * b.m[c] * kwm, (int)a.e[c] + (int)b.e[c] + kwe);
  }
  return f;
}

// zero-fill one staged row (significand 0, exponent EZERO): the target of zero-factor arcs
template <class M, class E, int LC> __device__ __forceinline__ void zero_row(M* sm, E* se, int row) {
  for (int k = threadIdx.x; k < LC; k += blockDim.x) {
    sm[(size_t)row * LC + k] = M(0);
    se[(size_t)row * LC + k] = (E)EZERO;
  }
}

template <class T_, int CPT> struct FwdSmem {
  // [2 stages x (hout rows + zero row + hin rows + zero row)] [arc metadata] [flow accumulators] [2 mbarriers]
  static __host__ __device__ size_t stage_rows_n(int max_hout, int max_hin) { return (size_t)max_hout + max_hin + 2; }
  static __host__ __device__ size_t row_bytes() { return (size_t)32 * CPT * (sizeof(typename T_::M) + sizeof(typename T_::E)); }
  static __host__ __device__ size_t bytes(int max_hout, int B, int max_hin, int max_ia, int max_oa) {
    return 2 * stage_rows_n(max_hout, max_hin) * row_bytes() + ArcSmem<typename T_::M>::bytes(B, max_ia, max_oa) +
           ((size_t)max_oa * sizeof(typename T_::M) + 15) / 16 * 16 + 16;
  }
};

// MODE 0: t = 0 (a2 fused, or U0 reload in readout); MODE 1: 0 < t < T; MODE 2: t = T (a4 fused)
// FMODE (flow handling): 0 dual update in place, 1 write Fsum (multi-GPU), 2 readout (Fout[t], all arcs)
template <class T_, int CPT, int MODE, int FMODE>
__global__ void __launch_bounds__(TILE_THREADS, 2) k_fwd_tile(DevPtrs p, TileMeta tm, PipeCfg pc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  constexpr int LC = 32 * CPT;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  View<T_> v(p);
  const int tile = blockIdx.x, grp = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j0 = tm.tile_ptr[tile], nb = tm.tile_ptr[tile + 1] - j0;
  const int hi0 = tm.hin_ptr[tile], nhi = tm.hin_ptr[tile + 1] - hi0;
  const int ho0 = tm.hout_ptr[tile], nho = tm.hout_ptr[tile + 1] - ho0;
  const int c0 = grp * pc.cpc, c1 = min(c0 + pc.cpc, tm.nch);
  // stage layout (rows): [0, max_hout) beta halo, max_hout zero row, [max_hout+1, +max_hin) alpha halo, then zero row
  const int zout = tm.max_hout, hin_base = tm.max_hout + 1, zin = hin_base + tm.max_hin;
  const size_t stride = FwdSmem<T_, CPT>::stage_rows_n(tm.max_hout, tm.max_hin) * LC;  // elements per stage
  M* stm = (M*)smem;
  E* ste = (E*)(stm + 2 * stride);
  unsigned char* after = (unsigned char*)(ste + 2 * stride);
  ArcSmem<M> sa;
  sa.carve(after, tm.B, tm.max_ia, tm.max_oa);
  M* facc = (M*)(after + ArcSmem<M>::bytes(tm.B, tm.max_ia, tm.max_oa));
  unsigned long long* bar = (unsigned long long*)((unsigned char*)facc + ((size_t)tm.max_oa * sizeof(M) + 15) / 16 * 16);

  const unsigned chunk_bytes =
      (unsigned)(((MODE != 2 ? nho : 0) + (MODE != 0 ? nhi : 0)) * FwdSmem<T_, CPT>::row_bytes());
  auto issue = [&](int c, int buf) {
    if (chunk_bytes == 0) return;
    if (lane == 0) mbar_arrive_expect_tx(&bar[buf], chunk_bytes);
    __syncwarp();
    M* bm_s = stm + buf * stride;
    E* be_s = ste + buf * stride;
    if (MODE != 2)
      issue_rows<M, E, LC>(v.bm(t + 1), v.be(t + 1), p.Lp, (size_t)c * LC, tm.hout_node + ho0, nho, bm_s, be_s,
                           &bar[buf], lane);
    if (MODE != 0)
      issue_rows<M, E, LC>(v.am(t - 1), v.ae(t - 1), p.Lp, (size_t)c * LC, tm.hin_node + hi0, nhi,
                           bm_s + (size_t)hin_base * LC, be_s + (size_t)hin_base * LC, &bar[buf], lane);
  };

  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  for (int b = 0; b < 2; ++b) {
    zero_row<M, E, LC>(stm + b * stride, ste + b * stride, zout);
    zero_row<M, E, LC>(stm + b * stride, ste + b * stride, zin);
  }
  __syncthreads();
  if (warp == 0) issue(c0, 0);
  stage_arcs<T_>(p, tm, sa, j0, nb, MODE == 0 ? 0 : t - 1, MODE == 2 ? t - 1 : t, MODE != 0, MODE != 2, FMODE == 2,
                 hin_base, zin, zout);
  for (int q = threadIdx.x; q < tm.max_oa; q += blockDim.x) facc[q] = M(0);
  __syncthreads();

  for (int c = c0; c < c1; ++c) {
    const int k = c - c0, buf = k & 1;
    if (warp == 0 && c + 1 < c1) {
      fence_proxy_async();  // generic reads of buffer buf^1 (previous chunk) precede the async writes
      issue(c + 1, buf ^ 1);
    }
    if (chunk_bytes) mbar_wait(&bar[buf], (k >> 1) & 1);
    const M* sbm = stm + buf * stride;
    const E* sbe = ste + buf * stride;
    const size_t col = (size_t)c * LC + lane * CPT;
    const int l0 = c * LC + lane * CPT;

    for (int r = warp; r < nb; r += nw) {
      const int j = j0 + r;
      const size_t g = (size_t)j * p.Lp + col;
      // 1. alpha_t of node j for this chunk
      Lane<M, E, CPT> a;
      if (MODE == 0) {
        if (FMODE == 2) {
          a.load((const M*)p.u0m + g, (const E*)p.u0e + g);
        } else {
          Lane<M, E, CPT> b0;
          b0.load(v.bm(0) + g, v.be(0) + g);
          boundary_lane<T_, CPT>(p, 0, j, l0, g, b0, a);
          a.store((M*)p.u0m + g, (E*)p.u0e + g);
        }
      } else {
        M s[CPT];
        int Ex[CPT];
        row_sum<T_, CPT>(sbm, sbe, lane, sa.ir, sa.im, sa.iptr[r], sa.iptr[r + 1], s, Ex);
        norm_lane<T_, CPT>(p, s, Ex, a, l0, j);
      }
      a.store(v.am(t) + g, v.ae(t) + g);
      if (MODE == 2) {
        if (FMODE != 2) {
          Lane<M, E, CPT> ut;
          boundary_lane<T_, CPT>(p, 1, j, l0, g, a, ut);
          ut.store(v.bm(p.T) + g, v.be(p.T) + g);
        }
      } else {
        // 2. this chunk's flow contributions of node j's out-arcs (the warp owning j owns its arcs)
        const int q1 = sa.optr[r + 1];
        for (int q = sa.optr[r]; q < q1; ++q) {
          const int h = sa.of[q];
          if (h < 0) continue;
          Lane<M, E, CPT> b;
          b.load(sbm + (size_t)h * LC + lane * CPT, sbe + (size_t)h * LC + lane * CPT);
          M f = flow_terms<T_, CPT>(a, b, sa.om[q], sa.orr[q].ke);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
          if (lane == 0) facc[q] += f;
        }
      }
    }
    __syncthreads();  // buffer buf is free for the chunk after next
  }
  if (MODE == 2) return;

  // 3. the tile's flows: complete here (one group) or via the last-arriving group
  const int nq = sa.optr[nb];
  M* part = (M*)tm.part;
  if (pc.ngroup > 1) {
    for (int q = threadIdx.x; q < nq; q += blockDim.x)
      if (sa.of[q] != -1) part[(size_t)sa.oa[q] * pc.ngroup + grp] = facc[q];
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int tk = atomicAdd(&tm.cnt[tile], 1);
      s_last = tk == pc.ngroup - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
  }
  for (int q = threadIdx.x; q < nq; q += blockDim.x) {
    if (sa.of[q] == -1) continue;
    const int arc = sa.oa[q];
    M s = facc[q];
    if (pc.ngroup > 1) {
      s = M(0);
      for (int g = 0; g < pc.ngroup; ++g) s += __ldcg(part + (size_t)arc * pc.ngroup + g);
    }
    if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, arc);
    if (FMODE == 0)
      dual_update<T_>(p, t, arc, (double)s);
    else if (FMODE == 1)
      ((M*)p.Fsum)[p.fpos[arc]] = s;  // (finite capacity at t: fpos >= 0)
    else
      ((M*)p.Fout)[(size_t)t * p.A + arc] = s;
  }
  if (pc.ngroup > 1 && threadIdx.x == 0) tm.cnt[tile] = 0;
}

template <class T_, int CPT> struct BwdSmem {
  static __host__ __device__ size_t bytes(int max_hout, int B, int max_oa) {
    return 2 * ((size_t)max_hout + 1) * FwdSmem<T_, CPT>::row_bytes() + ArcSmem<typename T_::M>::bytes(B, 0, max_oa) +
           16;
  }
};

// backward step: beta_t[i] = sum_{a: i_a = i} K_t[a] W_t[a] beta_{t+1}[j_a]   (eq:psi P:1038-1043)
template <class T_, int CPT>
__global__ void __launch_bounds__(TILE_THREADS, 2) k_bwd_tile(DevPtrs p, TileMeta tm, PipeCfg pc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  constexpr int LC = 32 * CPT;
  extern __shared__ __align__(16) unsigned char smem[];
  View<T_> v(p);
  const int tile = blockIdx.x, grp = blockIdx.y;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int j0 = tm.tile_ptr[tile], nb = tm.tile_ptr[tile + 1] - j0;
  const int ho0 = tm.hout_ptr[tile], nho = tm.hout_ptr[tile + 1] - ho0;
  const int c0 = grp * pc.cpc, c1 = min(c0 + pc.cpc, tm.nch);
  const int zout = tm.max_hout;
  const size_t stride = ((size_t)tm.max_hout + 1) * LC;
  M* stm = (M*)smem;
  E* ste = (E*)(stm + 2 * stride);
  unsigned char* after = (unsigned char*)(ste + 2 * stride);
  ArcSmem<M> sa;
  sa.carve(after, tm.B, 0, tm.max_oa);
  unsigned long long* bar = (unsigned long long*)(after + ArcSmem<M>::bytes(tm.B, 0, tm.max_oa));
  const unsigned chunk_bytes = (unsigned)(nho * FwdSmem<T_, CPT>::row_bytes());
  auto issue = [&](int c, int buf) {
    if (chunk_bytes == 0) return;
    if (lane == 0) mbar_arrive_expect_tx(&bar[buf], chunk_bytes);
    __syncwarp();
    issue_rows<M, E, LC>(v.bm(t + 1), v.be(t + 1), p.Lp, (size_t)c * LC, tm.hout_node + ho0, nho, stm + buf * stride,
                         ste + buf * stride, &bar[buf], lane);
  };
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    mbar_fence_init();
  }
  for (int b = 0; b < 2; ++b) zero_row<M, E, LC>(stm + b * stride, ste + b * stride, zout);
  __syncthreads();
  if (warp == 0) issue(c0, 0);
  stage_arcs<T_>(p, tm, sa, j0, nb, t, t, false, true, true, 0, zout, zout);
  __syncthreads();
  for (int c = c0; c < c1; ++c) {
    const int k = c - c0, buf = k & 1;
    if (warp == 0 && c + 1 < c1) {
      fence_proxy_async();
      issue(c + 1, buf ^ 1);
    }
    if (chunk_bytes) mbar_wait(&bar[buf], (k >> 1) & 1);
    const M* sbm = stm + buf * stride;
    const E* sbe = ste + buf * stride;
    const size_t col = (size_t)c * LC + lane * CPT;
    const int l0 = c * LC + lane * CPT;
    for (int r = warp; r < nb; r += nw) {
      const int i = j0 + r;
      M s[CPT];
      int Ex[CPT];
      row_sum<T_, CPT>(sbm, sbe, lane, sa.orr, sa.om, sa.optr[r], sa.optr[r + 1], s, Ex);
      Lane<M, E, CPT> out;
      norm_lane<T_, CPT>(p, s, Ex, out, l0, i);
      const size_t g = (size_t)i * p.Lp + col;
      out.store(v.bm(t) + g, v.be(t) + g);
    }
    __syncthreads();
  }
}

}  // namespace mmf
