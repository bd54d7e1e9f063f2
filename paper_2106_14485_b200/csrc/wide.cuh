// wide.cuh — "wide-lane" sweep kernels (the production path): one warp per (node, commodity chunk),
// CPT commodities per lane (up to 8: a lane reads 32 B of significands + 16 B of exponents per
// gathered row), gathers straight from global memory through the L1 (nodes are numbered for locality,
// so a CTA's warps and neighbouring CTAs share gathered rows in L1 / L2).  No shared-memory staging
// and no block barriers inside the step's arithmetic; the per-arc bookkeeping (neighbour index, K W
// factor) is fetched once per warp into a compacted shared-memory list (zero-factor / uncapacitated
// arcs dropped) and amortised over the warp's 32 x CPT commodities.
//
// Forward kernel (per step t, SURVEY §8(a) a3 re-associated as in tiled.cuh):
//   alpha_t[j] = sum_{a->j} alpha_{t-1}[i_a] K_{t-1} W_{t-1}   (t = 0: U0 = mu0 ./ beta_0, a2 fused)
//   F_t[a] chunk contributions of j's capacitated out-arcs, reduced over the warp (commodities) and
//   over the CTA's chunks in shared memory (fixed order), then W_t[a] <- min(W_t d_t / F_t, 1) by the
//   CTA (all chunks in one CTA) or by the last-arriving CTA of the node group (deterministic sums).
//   (t = T: alpha_T then UT = muT ./ alpha_T -> beta_T, a4 fused.)
// Backward kernel: beta_t[i] = sum_{a: i_a = i} K_t W_t beta_{t+1}[j_a].
//
// fp32 arithmetic per term (CPT even): pass 1 max-plus of packed int16 exponents (VIADDMNMX.S16x2,
// two commodities per instruction); pass 2 d = max(e + ke - E, -126), scale = K W 2^d built by an
// integer add into the float's exponent field, acc = fma(x, scale, acc).
#pragma once
#include "tiled.cuh"
#include "xpack.cuh"

namespace mmf {

struct WideCfg {
  int npc;     // nodes per CTA
  int cpcta;   // chunks per CTA (npc * cpcta = warps per CTA)
  int ngroup;  // chunk groups (gridDim.y); > 1 -> global partials + last arriver per node group
  int nch;     // chunks of LC commodities
  int max_oa;  // largest out-arc count of a node group (shared-memory sizing)
  int* cnt;    // [node groups] arrival counters
  void* part;  // [A][ngroup] partial flows (M)
  int prefetch;  // 1: pass 1 also prefetches the significand rows into L1
};

#ifndef MMF_WIDE_XFAST
#define MMF_WIDE_XFAST false  // native 16x2 form of the per-item exponent constants (XPre::set)
#endif
#ifndef MMF_WIDE_THREADS
#define MMF_WIDE_THREADS 256
#endif
constexpr int WIDE_THREADS = MMF_WIDE_THREADS;  // (warps per CTA = nodes x chunks per CTA)
constexpr int WARP_ARCS = 64;  // arcs per warp scratch batch
#ifndef MMF_U1
#define MMF_U1 4  // unroll of the exponent pass (loads in flight per warp)
#endif
#ifndef MMF_U2
#define MMF_U2 2  // unroll of the accumulation pass
#endif
constexpr int kUnroll1 = MMF_U1;
constexpr int kUnroll2 = MMF_U2;
#ifndef MMF_WIDE_MINB
#define MMF_WIDE_MINB 3  // CTAs per SM the register budget is sized for
#endif
#ifndef MMF_WIDE_MINB_F32X8
#define MMF_WIDE_MINB_F32X8 4  // ... for the fp32, 8-commodity-per-lane forward ([5]): 64 registers, 32 warps per SM
                               // (measured 62.5 -> 58.1 ms per sweep on [5]; the latency-bound gathers want warps)
#endif
template <class T_, int CPT> constexpr int wide_fwd_minb() {
  return sizeof(typename T_::M) == 4 && CPT == 8 ? MMF_WIDE_MINB_F32X8 : MMF_WIDE_MINB;
}

// compacted per-warp arc list: gathered node, K W factor, position of the arc (flow slot)
template <class M> struct WarpArcs {
  int node[WARP_ARCS];
  int ke[WARP_ARCS];
  int pos[WARP_ARCS];
  M km[WARP_ARCS];
};

template <class M> __host__ __device__ inline size_t wide_smem(int max_oa, int cpcta) {
  return (size_t)(WIDE_THREADS / 32) * sizeof(WarpArcs<M>) + ((size_t)max_oa * cpcta * sizeof(M) + 15) / 16 * 16;
}

// per-arc factor (m, e) of arc a at step t: K_t W_t, zero -> m = 0
template <class T_>
__device__ __forceinline__ void kw_factor(const View<T_>& v, int t, int a, typename T_::M& m, int& e) {
  typedef typename T_::M M;
  m = v.Km(t)[a] * v.Wm(t)[a];
  e = v.Ke(t)[a] + v.We(t)[a];
  if (!(m > M(0)) || e < -ELIM) {
    m = M(0);
    e = -ELIM;
  }
  if (e > ELIM) e = ELIM;
}

// Fill the warp scratch with the records rec[k0, k0 + n) (n <= WARP_ARCS), keeping only arcs with a
// nonzero factor (and, if cap_only, a finite capacity: aux bit 31 clear); pos = k - pos0.
// One 16-byte record load per lane, no dependent loads.  Returns the kept count (warp-uniform).
template <class M>
__device__ __forceinline__ int warp_arcs(const ArcKW<M>* rec, int k0, int n, int pos0, WarpArcs<M>& w, int lane,
                                         bool cap_only) {
  int kept = 0;
  for (int base = 0; base < n; base += 32) {
    const int q = base + lane;
    bool keep = false;
    ArcKW<M> r;
    if (q < n) {
      r = rec[k0 + q];
      keep = r.km > M(0) && !(cap_only && r.aux < 0);
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (keep) {
      const int slot = kept + __popc(bal & ((1u << lane) - 1u));
      w.node[slot] = r.node;
      w.ke[slot] = r.ke;
      w.pos[slot] = k0 + q - pos0;
      w.km[slot] = r.km;
    }
    kept += __popc(bal);
  }
  __syncwarp();
  return kept;
}

// extended-range row sum over gathered global rows: out = sum_q KW_q x[node_q] (q < n, all nonzero)
template <class T_, int CPT>
__device__ __forceinline__ void gather_sum(const typename T_::M* gm, const typename T_::E* ge, int Lp, size_t col,
                                          int n, const WarpArcs<typename T_::M>& w, typename T_::M* s, int* E,
                                          int prefetch = 0) {
  typedef typename T_::M M;
  typedef typename T_::E Ex;
  if constexpr (sizeof(M) == 4 && sizeof(Ex) == 2 && CPT % 2 == 0) {
    constexpr int NP = CPT / 2;
    typedef typename VecE<int16_t, CPT>::T VE;
    unsigned E2[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) E2[k] = 0x80008000u;
    // pass 1: per-commodity max exponent (packed 16x2 max-plus)
#pragma unroll kUnroll1
    for (int q = 0; q < n; ++q) {
      const unsigned k2 = pack2(w.ke[q]);
      if (prefetch) asm volatile("prefetch.global.L1 [%0];" ::"l"(gm + (size_t)w.node[q] * Lp + col));
      const VE ev = __ldg(reinterpret_cast<const VE*>(ge + (size_t)w.node[q] * Lp + col));
      const unsigned* ew = reinterpret_cast<const unsigned*>(&ev);
#pragma unroll
      for (int j = 0; j < NP; ++j) E2[j] = __viaddmax_s16x2(ew[j], k2, E2[j]);
    }
    XPre<CPT> P;
    P.template set<MMF_WIDE_XFAST>(E2);  // (see XPre::set)
#pragma unroll
    for (int c = 0; c < CPT; ++c) E[c] = P.E[c];
    float acc[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
    // pass 2: sum x * K W 2^(e - E) (packed: the scale of a commodity pair by two 16x2 max-plus operations,
    // the products by FFMA2; same arithmetic as the pipelined kernels' xacc)
#pragma unroll kUnroll2
    for (int q = 0; q < n; ++q) {
      const unsigned kb = __float_as_uint((float)w.km[q]);
      const unsigned k2 = pack2(w.ke[q]);
      const size_t g = (size_t)w.node[q] * Lp + col;
      Row<TrF32, CPT> x;
      x.load(gm + g, ge + g);
      xacc<CPT>(x, kb, k2, w.ke[q], P, acc);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) s[c] = acc[c];
  } else {
    XAcc<M> acc[CPT];
    for (int q = 0; q < n; ++q) {
      const size_t g = (size_t)w.node[q] * Lp + col;
      Lane<M, Ex, CPT> x;
      x.load(gm + g, ge + g);
      const M kwm = w.km[q];
      const int kwe = w.ke[q];
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c].add(x.m[c] * kwm, (int)x.e[c] + kwe);
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      s[c] = acc[c].s;
      E[c] = acc[c].E;
    }
  }
}

// full SpMM row of one node over records rec[k0, k1) (any degree: batches of WARP_ARCS through the
// scratch, merged in XF)
template <class T_, int CPT>
__device__ __forceinline__ void node_sum(const ArcKW<typename T_::M>* rec, int k0, int k1, const typename T_::M* gm,
                                        const typename T_::E* ge, int Lp, size_t col, WarpArcs<typename T_::M>& w,
                                        int lane, typename T_::M* s, int* E, int prefetch) {
  typedef typename T_::M M;
  if (k1 - k0 <= WARP_ARCS) {
    const int n = warp_arcs<M>(rec, k0, k1 - k0, k0, w, lane, false);
    gather_sum<T_, CPT>(gm, ge, Lp, col, n, w, s, E, prefetch);
    return;
  }
  XAcc<M> tot[CPT];
  for (int b = k0; b < k1; b += WARP_ARCS) {
    const int n = warp_arcs<M>(rec, b, min(WARP_ARCS, k1 - b), b, w, lane, false);
    M bs[CPT];
    int bE[CPT];
    gather_sum<T_, CPT>(gm, ge, Lp, col, n, w, bs, bE);
#pragma unroll
    for (int c = 0; c < CPT; ++c) tot[c].add(bs[c], bE[c]);
    __syncwarp();
  }
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    s[c] = tot[c].s;
    E[c] = tot[c].E;
  }
}

// MODE 0: t = 0 (a2 fused, or U0 reload in readout); MODE 1: 0 < t < T; MODE 2: t = T (a4 fused)
// FMODE: 0 dual update in place, 1 write Fsum (multi-GPU), 2 readout (Fout[t], all arcs)
template <class T_, int CPT, int MODE, int FMODE>
__global__ void __launch_bounds__(WIDE_THREADS, wide_fwd_minb<T_, CPT>()) k_fwd_wide(DevPtrs p, WideCfg wc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  constexpr int LC = 32 * CPT;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ int s_last;
  View<T_> v(p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpArcs<M>& wa = ((WarpArcs<M>*)smem)[warp];
  M* fpart = (M*)(smem + (WIDE_THREADS / 32) * sizeof(WarpArcs<M>));
  const int jg0 = blockIdx.x * wc.npc;  // first node of the CTA
  const int jloc = warp / wc.cpcta, cloc = warp % wc.cpcta;
  const int j = jg0 + jloc;
  const int c = blockIdx.y * wc.cpcta + cloc;
  const int jend = min(jg0 + wc.npc, p.N);
  const int oq0 = p.out_ptr[jg0];  // the CTA's out-arcs are contiguous in out-CSR order
  const int noq = p.out_ptr[jend] - oq0;
  const bool active = j < p.N && c < wc.nch;
  if (MODE != 2)
    for (int q = threadIdx.x; q < noq * wc.cpcta; q += blockDim.x) fpart[q] = M(0);
  __syncthreads();
  if (active) {
    const size_t col = (size_t)c * LC + lane * CPT;
    const int l0 = c * LC + lane * CPT;
    const size_t g = (size_t)j * p.Lp + col;
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
      MMF_DASSERT(p.in_ptr[j] >= 0 && p.in_ptr[j] <= p.in_ptr[j + 1] && p.in_ptr[j + 1] <= p.A);  // (CSR row)
      node_sum<T_, CPT>((const ArcKW<M>*)p.inrec + (size_t)(t - 1) * p.A, p.in_ptr[j], p.in_ptr[j + 1], v.am(t - 1),
                        v.ae(t - 1), p.Lp, col, wa, lane, s, Ex, wc.prefetch);
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
      // flow contributions of j's (capacitated, nonzero) out-arcs for this chunk
      const int k0 = p.out_ptr[j], k1 = p.out_ptr[j + 1];
      unsigned aw[CPT / 2 > 0 ? CPT / 2 : 1];  // (fp32: the own row's exponents packed 16x2 for flow_terms_f2)
      if constexpr (sizeof(M) == 4 && CPT % 2 == 0) {
#pragma unroll
        for (int k = 0; k < CPT / 2; ++k) aw[k] = pack_e2((int)a.e[2 * k], (int)a.e[2 * k + 1]);
      }
      __syncwarp();
      for (int b = k0; b < k1; b += WARP_ARCS) {
        const int n = warp_arcs<M>((const ArcKW<M>*)p.outrec + (size_t)t * p.A, b, min(WARP_ARCS, k1 - b), oq0, wa,
                                   lane, FMODE != 2);
        for (int q = 0; q < n; ++q) {
          const size_t gg = (size_t)wa.node[q] * p.Lp + col;
          M f;
          if constexpr (sizeof(M) == 4 && CPT % 2 == 0) {
            Row<TrF32, CPT> bb;
            bb.load((const float*)(v.bm(t + 1) + gg), v.be(t + 1) + gg);
            f = flow_terms_f2<CPT>((const float*)a.m, aw, bb, (float)wa.km[q], wa.ke[q]);
          } else {
            Lane<M, E, CPT> bb;
            bb.load(v.bm(t + 1) + gg, v.be(t + 1) + gg);
            f = flow_terms<T_, CPT>(a, bb, wa.km[q], wa.ke[q]);
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
          if (lane == 0) fpart[wa.pos[q] * wc.cpcta + cloc] = f;
        }
        __syncwarp();
      }
    }
  }
  if (MODE == 2) return;
  __syncthreads();
  // the CTA's out-arcs: fixed-order sum over its chunks, then over groups (last arriver)
  M* part = (M*)wc.part;
  const int nvalid = min(wc.cpcta, wc.nch - blockIdx.y * wc.cpcta);
  const M* dc = v.dcap(t);
  if (wc.ngroup > 1) {
    for (int q = threadIdx.x; q < noq; q += blockDim.x) {
      M s = M(0);
      for (int k = 0; k < nvalid; ++k) s += fpart[q * wc.cpcta + k];
      part[(size_t)p.out_arc[oq0 + q] * wc.ngroup + blockIdx.y] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      const int tk = atomicAdd(&wc.cnt[blockIdx.x], 1);
      s_last = tk == wc.ngroup - 1;
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
  }
  for (int q = threadIdx.x; q < noq; q += blockDim.x) {
    const int arc = p.out_arc[oq0 + q];
    if (FMODE != 2 && isinf(dc[arc])) continue;
    M s = M(0);
    if (wc.ngroup > 1) {
      for (int gidx = 0; gidx < wc.ngroup; ++gidx) s += __ldcg(part + (size_t)arc * wc.ngroup + gidx);
    } else {
      for (int k = 0; k < nvalid; ++k) s += fpart[q * wc.cpcta + k];
    }
    if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, arc);
    if (FMODE == 0)
      dual_update<T_>(p, t, arc, (double)s);
    else if (FMODE == 1)
      ((M*)p.Fsum)[p.fpos[arc]] = s;  // (finite capacity at t: fpos >= 0)
    else
      ((M*)p.Fout)[(size_t)t * p.A + arc] = s;
  }
  if (wc.ngroup > 1 && threadIdx.x == 0) wc.cnt[blockIdx.x] = 0;
}

// backward step: beta_t[i] = sum_{a: i_a = i} K_t[a] W_t[a] beta_{t+1}[j_a]   (eq:psi P:1038-1043)
template <class T_, int CPT>
__global__ void __launch_bounds__(WIDE_THREADS, MMF_WIDE_MINB) k_bwd_wide(DevPtrs p, WideCfg wc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  constexpr int LC = 32 * CPT;
  extern __shared__ __align__(16) unsigned char smem[];
  View<T_> v(p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpArcs<M>& wa = ((WarpArcs<M>*)smem)[warp];
  const int i = blockIdx.x * wc.npc + warp / wc.cpcta;
  const int c = blockIdx.y * wc.cpcta + warp % wc.cpcta;
  if (i >= p.N || c >= wc.nch) return;
  const size_t col = (size_t)c * LC + lane * CPT;
  const int l0 = c * LC + lane * CPT;
  M s[CPT];
  int Ex[CPT];
  node_sum<T_, CPT>((const ArcKW<M>*)p.outrec + (size_t)t * p.A, p.out_ptr[i], p.out_ptr[i + 1], v.bm(t + 1),
                    v.be(t + 1), p.Lp, col, wa, lane, s, Ex, wc.prefetch);
  Lane<M, E, CPT> out;
  norm_lane<T_, CPT>(p, s, Ex, out, l0, i);
  const size_t g = (size_t)i * p.Lp + col;
  out.store(v.bm(t) + g, v.be(t) + g);
}

}  // namespace mmf
