// headflow.cuh — register-gather sweep kernels (the production path, option kernels = 4).
//
// Forward kernel of step t (t = 1..T) computes, for the nodes j of its CTA and ALL their commodity chunks:
//   (i)   F_{t-1}[a] = K W_{t-1}[a] sum_l alpha_{t-1}[i_a,l] beta_t[j,l]   for the in-arcs a -> j
//         (cor:proj P:1078, evaluated at the head: the gathered rows alpha_{t-1}[i_a] are the ones (iii)
//         needs anyway, and beta_t[j] is the node's own row — no second gather);
//   (ii)  W_{t-1}[a] <- min(W_{t-1}[a] d[a] / F_{t-1}[a], 1)   (eq:sinkhorn_graph_Vineq P:861),
//         the commodity sum finished in shared memory in a fixed order (deterministic);
//   (iii) alpha_t[j] = sum_{a -> j} alpha_{t-1}[i_a] K W_{t-1}[a]   with the UPDATED W (eq:psi_hat
//         P:1031-1036), from the rows still held in registers.
// That is exactly Algorithm 2's Gauss-Seidel order: W_{t-1} is updated after alpha_{t-1}
// and before alpha_t.  t = 0 is a2 (U0 = mu0 ./ beta_0); t = T also does a4 (UT = muT ./ alpha_T,
// P:1096).  So one sweep is T + 1 forward launches and T backward launches, as before.
//
// Backward kernel of step t: beta_t[i] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a]  (eq:psi P:1038-1043).
//
// Both gather each (arc, chunk) row ONCE: all rows of a node's arcs (up to NB per batch) are loaded into
// registers with independent 16-byte loads before any arithmetic (one memory round trip instead of the
// two-pass exponent-then-significand walk of wide.cuh), then the extended-range sum is formed from the
// registers: max of (row exponent + arc exponent) per commodity (packed 16x2 max-plus for fp32), then
// sum m * KW * 2^(e + ke - E) with the scale built by an integer add into the float exponent field.
// Per-arc metadata is one coalesced 16-byte record load per lane, broadcast with shuffles.
#pragma once
#include "wide.cuh"

namespace mmf {

#ifndef MMF_NB
#define MMF_NB 6  // arcs held in registers per batch
#endif
#ifndef MMF_HF_MINB
#define MMF_HF_MINB 2
#endif
constexpr int HF_NB = MMF_NB;
constexpr int HF_WARPS = 8;

struct HeadCfg {
  int nch;     // commodity chunks of 32 * CPT
  int npc;     // nodes per CTA (forward)
  int wpn;     // warps per node (forward): nch if nch <= 8 (rows stay in registers), else 8 (chunk loop)
  int max_ia;  // largest in-arc count of a CTA's node group (shared-memory sizing)
};

template <class M> struct KwEnt {
  M m;
  int e;
};

template <class M> __host__ __device__ inline size_t head_smem(int max_ia, int nch) {
  return ((size_t)max_ia * nch * sizeof(M) + 15) / 16 * 16 + (size_t)max_ia * sizeof(KwEnt<M>) + 16;
}

// 16-bit-exponent-safe max-plus state (fp32 packed path) or plain ints
template <class T_, int CPT> struct RowMax {
  typedef Row<T_, CPT> R;
  int E[R::NW];
  __device__ __forceinline__ void init() {
#pragma unroll
    for (int k = 0; k < R::NW; ++k) E[k] = R::PACKED ? (int)0x80008000u : (EZERO - 4 * ELIM);
  }
  __device__ __forceinline__ void add(const R& x, int ke) {
    if constexpr (R::PACKED) {
      const unsigned k2 = pack2(ke);
#pragma unroll
      for (int k = 0; k < R::NW; ++k) E[k] = (int)__viaddmax_s16x2((unsigned)x.w[k], k2, (unsigned)E[k]);
    } else {
#pragma unroll
      for (int k = 0; k < R::NW; ++k) E[k] = max(E[k], x.w[k] + ke);
    }
  }
  __device__ __forceinline__ int get(int c) const {
    if constexpr (R::PACKED)
      return (c & 1) ? (E[c >> 1] >> 16) : (int)(short)(E[c >> 1] & 0xffff);
    else
      return E[c];
  }
};

// acc[c] += x.m[c] * KW * 2^(x.e[c] + ke - E[c])   (E[c] >= x.e[c] + ke; terms below 2^-126 relative dropped)
template <class T_, int CPT>
__device__ __forceinline__ void row_acc(const Row<T_, CPT>& x, typename T_::M km, int ke, const int* nE,
                                        typename T_::M* acc) {
  typedef typename T_::M M;
  if constexpr (sizeof(M) == 4) {
    const unsigned kb = __float_as_uint(km);
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int d = max(x.e(c) + ke + nE[c], -126);
      acc[c] = fmaf(x.m[c], __uint_as_float(kb + ((unsigned)d << 23)), acc[c]);
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) acc[c] += x.m[c] * km * pow2_nonpos<M>(x.e(c) + ke + nE[c]);
  }
}

// linear flow term of one lane: sum_c lin(a_c * b_c * KW)
template <class T_, int CPT>
__device__ __forceinline__ typename T_::M row_flow(const Row<T_, CPT>& a, const Row<T_, CPT>& b,
                                                   typename T_::M km, int ke) {
  typedef typename T_::M M;
  M f = M(0);
  if constexpr (sizeof(M) == 4) {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int es = max(a.e(c) + b.e(c) + ke, -127);  // -127 -> scale exactly 0
      f = fmaf(a.m[c] * km * b.m[c], __uint_as_float((unsigned)(es + 127) << 23), f);
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) f += xf_to_lin<M>(a.m[c] * b.m[c] * km, a.e(c) + b.e(c) + ke);
  }
  return f;
}

template <class M> __device__ __forceinline__ M warp_sum(M f) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) f += __shfl_xor_sync(0xffffffffu, f, o);
  return f;
}

// (s, E) of a register batch: kw(q, km, ke) returns false for arcs that do not contribute (absent or zero
// factor); factors are re-fetched per pass (shared memory / shuffles) to keep register live ranges short
template <class T_, int CPT, int NB, class KW>
__device__ __forceinline__ void batch_sum(const Row<T_, CPT> (&x)[NB], KW kw, typename T_::M* s, int* Eo) {
  typedef typename T_::M M;
  RowMax<T_, CPT> mx;
  mx.init();
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    M km;
    int ke;
    if (kw(q, km, ke)) mx.add(x[q], ke);
  }
  int nE[CPT];
#pragma unroll
  for (int c = 0; c < CPT; ++c) {
    Eo[c] = mx.get(c);
    nE[c] = -Eo[c];
    s[c] = M(0);
  }
#pragma unroll
  for (int q = 0; q < NB; ++q) {
    M km;
    int ke;
    if (kw(q, km, ke)) row_acc<T_, CPT>(x[q], km, ke, nE, s);
  }
}

// merge a batch result into a running total (multi-batch nodes)
template <class M> __device__ __forceinline__ void merge_xf(M& s, int& E, M s2, int E2) {
  if (!(s2 > M(0))) return;
  if (!(s > M(0))) {
    s = s2;
    E = E2;
    return;
  }
  const int nE = max(E, E2);
  s = s * pow2_nonpos<M>(E - nE) + s2 * pow2_nonpos<M>(E2 - nE);
  E = nE;
}

// broadcast of lane q's record fields
template <class M> struct RecB {
  int node, ke, aux;
  M km;
};
template <class M> __device__ __forceinline__ RecB<M> rec_bcast(const ArcKW<M>& r, int q) {
  RecB<M> b;
  b.node = __shfl_sync(0xffffffffu, r.node, q);
  b.ke = __shfl_sync(0xffffffffu, r.ke, q);
  b.aux = __shfl_sync(0xffffffffu, r.aux, q);
  b.km = __shfl_sync(0xffffffffu, r.km, q);
  return b;
}
// record q of a node's arc list [k0, k0 + deg): from the lane-held window r (deg <= 32, warp-uniform) or
// straight from memory (high-degree nodes)
template <class M>
__device__ __forceinline__ RecB<M> rec_get(const ArcKW<M>& r, const ArcKW<M>* rec, int k0, int deg, int q) {
  if (deg <= 32) return rec_bcast<M>(r, q & 31);
  RecB<M> b{0, 0, 0, M(0)};
  if (q < deg) {
    const ArcKW<M> x = rec[k0 + q];
    b.node = x.node;
    b.ke = x.ke;
    b.aux = x.aux;
    b.km = x.km;
  }
  return b;
}

// record of arc a's factor K W (the same clamps as write_recs)
template <class T_>
__device__ __forceinline__ void kw_clamp(typename T_::M km, int ke, typename T_::M wm, int we, typename T_::M& m,
                                         int& e) {
  typedef typename T_::M M;
  m = km * wm;
  e = ke + we;
  if (!(m > M(0)) || e < -ELIM) {
    m = M(0);
    e = -ELIM;
  }
  if (e > ELIM) e = ELIM;
}

// new W from the old one and the flow: min(W d / F, 1); d = 0 -> 0; F = 0 -> 1
template <class T_>
__device__ __forceinline__ void w_new(typename T_::M d, typename T_::M wm0, int we0, double F, typename T_::M& wm,
                                      int& we) {
  typedef typename T_::M M;
  if (d == M(0)) {
    wm = M(0);
    we = EZERO;
  } else if (!(F > 0.0)) {
    wm = M(1);
    we = 0;
  } else {
    double m;
    int e;
    const double x = (double)wm0 * ((double)d / F);
    xf_norm<double>(x, we0, m, e);
    if (isinf(x)) e = 0;
    wm = (M)m;
    if (wm >= M(2)) {
      wm = M(1);
      e += 1;
    }
    we = e;
    if (e >= 0) {
      wm = M(1);
      we = 0;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// forward step t.  MODE 0: t = 0 (a2);  MODE 1: 0 < t < T;  MODE 2: t = T (a4 fused).
// KEEP: every warp owns exactly one chunk of one node (nch <= 8) and keeps its gathered rows in registers
// from the flow phase to the message phase; otherwise warps loop over chunks and re-gather in phase 3.
template <class T_, int CPT, int MODE, bool KEEP>
__global__ void __launch_bounds__(HF_WARPS * 32, MMF_HF_MINB) k_fwd_head(DevPtrs p, HeadCfg hc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  typedef Row<T_, CPT> R;
  constexpr int LC = 32 * CPT;
  constexpr int NB = HF_NB;
  extern __shared__ __align__(16) unsigned char smem[];
  View<T_> v(p);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int j0 = blockIdx.x * hc.npc;
  const int jloc = warp / hc.wpn, wloc = warp % hc.wpn;
  const int j = j0 + jloc;
  const bool jok = jloc < hc.npc && j < p.N;

  if (MODE == 0) {  // a2: alpha_0 = U0 = mu0 ./ beta_0 (also kept as U0 for the readout)
    if (!jok) return;
    for (int c = wloc; c < hc.nch; c += hc.wpn) {
      const size_t g = (size_t)j * p.Lp + (size_t)c * LC + lane * CPT;
      Lane<M, E, CPT> b0, a;
      b0.load(v.bm(0) + g, v.be(0) + g);
      boundary_lane<T_, CPT>(p, 0, j, c * LC + lane * CPT, g, b0, a);
      a.store((M*)p.u0m + g, (E*)p.u0e + g);
      a.store(v.am(0) + g, v.ae(0) + g);
    }
    return;
  }

  const int jend = min(j0 + hc.npc, p.N);
  const int ia0 = p.in_ptr[j0];
  const int nia = p.in_ptr[jend] - ia0;
  M* fpart = (M*)smem;                                                           // [max_ia][nch]
  KwEnt<M>* kwt = (KwEnt<M>*)(smem + ((size_t)hc.max_ia * hc.nch * sizeof(M) + 15) / 16 * 16);  // [max_ia]
  const ArcKW<M>* rec = (const ArcKW<M>*)p.inrec + (size_t)(t - 1) * p.A;

  // dual-update operands of this thread's arc, loaded early (their latency overlaps the gathers)
  const int qa = threadIdx.x;
  const bool has_arc = qa < nia;
  M d_a = M(0), wm_a = M(1), km_a = M(0);
  int we_a = 0, ke_a = 0;
  if (has_arc) {
    const int a = ia0 + qa;
    d_a = v.dcap(t - 1)[a];
    wm_a = v.Wm(t - 1)[a];
    we_a = v.We(t - 1)[a];
    km_a = v.Km(t - 1)[a];
    ke_a = v.Ke(t - 1)[a];
  }

  int k0 = 0, k1 = 0;
  if (jok) {
    k0 = p.in_ptr[j];
    k1 = p.in_ptr[j + 1];
  }
  const int deg = k1 - k0;
  const bool fast = KEEP && deg <= NB;  // warp-uniform
  R x[NB];
  bool ok[NB];
  ArcKW<M> r{};
  if (jok && lane < deg) r = rec[k0 + lane];

  // ---- phase 1: flows of step t-1 on the in-arcs of j, per chunk
  if (jok) {
    if (fast) {  // one chunk per warp, all rows into registers (kept for phase 3)
      const int c = wloc;
      const size_t col = (size_t)c * LC + lane * CPT;
      R b;
      b.load(v.bm(t) + (size_t)j * p.Lp + col, v.be(t) + (size_t)j * p.Lp + col);
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        const RecB<M> rb = rec_bcast<M>(r, q);
        ok[q] = q < deg && rb.km > M(0);
        if (ok[q]) x[q].load(v.am(t - 1) + (size_t)rb.node * p.Lp + col, v.ae(t - 1) + (size_t)rb.node * p.Lp + col);
      }
#pragma unroll
      for (int q = 0; q < NB; ++q) {
        if (q >= deg) break;
        const RecB<M> rb = rec_bcast<M>(r, q);  // (re-broadcast: short live ranges)
        if (rb.aux < 0) continue;               // uncapacitated: no flow needed
        M f = ok[q] ? row_flow<T_, CPT>(x[q], b, rb.km, rb.ke) : M(0);
        f = warp_sum<M>(f);
        if (lane == 0) fpart[(size_t)(k0 - ia0 + q) * hc.nch + c] = f;
      }
    } else {  // streaming: one arc at a time, any degree, any number of chunks per warp
      for (int c = wloc; c < hc.nch; c += hc.wpn) {
        const size_t col = (size_t)c * LC + lane * CPT;
        R b;
        b.load(v.bm(t) + (size_t)j * p.Lp + col, v.be(t) + (size_t)j * p.Lp + col);
        for (int q = 0; q < deg; ++q) {
          const RecB<M> rb = rec_get<M>(r, rec, k0, deg, q);
          if (rb.aux < 0) continue;
          M f = M(0);
          if (rb.km > M(0)) {
            R y;
            y.load(v.am(t - 1) + (size_t)rb.node * p.Lp + col, v.ae(t - 1) + (size_t)rb.node * p.Lp + col);
            f = row_flow<T_, CPT>(y, b, rb.km, rb.ke);
          }
          f = warp_sum<M>(f);
          if (lane == 0) fpart[(size_t)(k0 - ia0 + q) * hc.nch + c] = f;
        }
      }
    }
  }
  __syncthreads();

  // ---- phase 2: capacity-dual update of the CTA's in-arcs (one thread per arc), new K W into smem
  for (int q = threadIdx.x; q < nia; q += blockDim.x) {
    const int a = ia0 + q;
    M dd = d_a, w0 = wm_a, kk = km_a;
    int e0 = we_a, kke = ke_a;
    if (q != qa) {
      dd = v.dcap(t - 1)[a];
      w0 = v.Wm(t - 1)[a];
      e0 = v.We(t - 1)[a];
      kk = v.Km(t - 1)[a];
      kke = v.Ke(t - 1)[a];
    }
    M wm = w0;
    int we = e0;
    if (!isinf(dd)) {
      M s = M(0);
      for (int c = 0; c < hc.nch; ++c) s += fpart[(size_t)q * hc.nch + c];
      if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, a);
      w_new<T_>(dd, w0, e0, (double)s, wm, we);
      v.Wm(t - 1)[a] = wm;
      v.We(t - 1)[a] = we;
      write_recs<T_>(p, t - 1, a, wm, we);
    }
    M m;
    int e;
    kw_clamp<T_>(kk, kke, wm, we, m, e);
    kwt[q].m = m;
    kwt[q].e = e;
  }
  __syncthreads();
  if (!jok) return;

  // ---- phase 3: alpha_t[j] = sum_a alpha_{t-1}[i_a] K W_{t-1}[a] (updated factors)
  const KwEnt<M>* kwj = kwt + (k0 - ia0);
  for (int c = wloc; c < hc.nch; c += hc.wpn) {  // (fast: exactly one chunk per warp)
    const size_t col = (size_t)c * LC + lane * CPT;
    const int l0 = c * LC + lane * CPT;
    M s[CPT];
    int Ex[CPT];
    if (fast) {
#pragma unroll
      for (int q = 0; q < NB; ++q)
        if (q < deg && !ok[q] && kwj[q].m > M(0)) {  // factor was zero before the update (rare): gather now
          const int nd = __shfl_sync(__activemask(), r.node, q);
          x[q].load(v.am(t - 1) + (size_t)nd * p.Lp + col, v.ae(t - 1) + (size_t)nd * p.Lp + col);
          ok[q] = true;
        }
      batch_sum<T_, CPT, NB>(
          x,
          [&](int q, M& km, int& ke) {
            if (!ok[q]) return false;
            const KwEnt<M> e = kwj[q];
            km = e.m;
            ke = e.e;
            return e.m > M(0);
          },
          s, Ex);
    } else {
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        s[cc] = M(0);
        Ex[cc] = EZERO;
      }
      for (int q0 = 0; q0 < deg; q0 += NB) {
        R y[NB];
#pragma unroll
        for (int q = 0; q < NB; ++q)
          if (q0 + q < deg && kwj[q0 + q].m > M(0)) {
            const int nd = rec[k0 + q0 + q].node;
            y[q].load(v.am(t - 1) + (size_t)nd * p.Lp + col, v.ae(t - 1) + (size_t)nd * p.Lp + col);
          }
        M bs[CPT];
        int bE[CPT];
        batch_sum<T_, CPT, NB>(
            y,
            [&](int q, M& km, int& ke) {
              if (q0 + q >= deg) return false;
              const KwEnt<M> e = kwj[q0 + q];
              km = e.m;
              ke = e.e;
              return e.m > M(0);
            },
            bs, bE);
#pragma unroll
        for (int cc = 0; cc < CPT; ++cc) merge_xf<M>(s[cc], Ex[cc], bs[cc], bE[cc]);
      }
    }
    Lane<M, E, CPT> a;
    norm_lane<T_, CPT>(p, s, Ex, a, l0, j);
    const size_t g = (size_t)j * p.Lp + col;
    a.store(v.am(t) + g, v.ae(t) + g);
    if (MODE == 2) {  // a4: UT = muT ./ alpha_T -> beta_T
      Lane<M, E, CPT> ut;
      boundary_lane<T_, CPT>(p, 1, j, l0, g, a, ut);
      ut.store(v.bm(p.T) + g, v.be(p.T) + g);
    }
  }
}

// backward step t: one warp per (node, chunk), flattened over the grid
template <class T_, int CPT>
__global__ void __launch_bounds__(HF_WARPS * 32, MMF_HF_MINB) k_bwd_head(DevPtrs p, HeadCfg hc, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  typedef Row<T_, CPT> R;
  constexpr int LC = 32 * CPT;
  constexpr int NB = HF_NB;
  View<T_> v(p);
  const int lane = threadIdx.x & 31;
  const int gw = blockIdx.x * HF_WARPS + (threadIdx.x >> 5);
  const int i = gw / hc.nch, c = gw % hc.nch;
  if (i >= p.N) return;
  const int k0 = p.out_ptr[i], k1 = p.out_ptr[i + 1];
  const int deg = k1 - k0;
  const ArcKW<M>* rec = (const ArcKW<M>*)p.outrec + (size_t)t * p.A;
  const size_t col = (size_t)c * LC + lane * CPT;
  const int l0 = c * LC + lane * CPT;
  const M* bm = v.bm(t + 1);
  const E* be = v.be(t + 1);
  M s[CPT];
  int Ex[CPT];
#pragma unroll
  for (int cc = 0; cc < CPT; ++cc) {
    s[cc] = M(0);
    Ex[cc] = EZERO;
  }
  ArcKW<M> r{};
  if (lane < deg) r = rec[k0 + lane];
  for (int q0 = 0; q0 < deg; q0 += NB) {
    R x[NB];
#pragma unroll
    for (int q = 0; q < NB; ++q) {
      const RecB<M> rb = rec_get<M>(r, rec, k0, deg, q0 + q);
      if (q0 + q < deg && rb.km > M(0)) x[q].load(bm + (size_t)rb.node * p.Lp + col, be + (size_t)rb.node * p.Lp + col);
    }
    M bs[CPT];
    int bE[CPT];
    batch_sum<T_, CPT, NB>(
        x,
        [&](int q, M& km, int& ke) {
          const RecB<M> rb = rec_get<M>(r, rec, k0, deg, q0 + q);
          km = rb.km;
          ke = rb.ke;
          return q0 + q < deg && rb.km > M(0);
        },
        bs, bE);
    if (q0 == 0) {
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) {
        s[cc] = bs[cc];
        Ex[cc] = bE[cc];
      }
    } else {
#pragma unroll
      for (int cc = 0; cc < CPT; ++cc) merge_xf<M>(s[cc], Ex[cc], bs[cc], bE[cc]);
    }
  }
  Lane<M, E, CPT> out;
  norm_lane<T_, CPT>(p, s, Ex, out, l0, i);
  const size_t g = (size_t)i * p.Lp + col;
  out.store(v.bm(t) + g, v.be(t) + g);
}

}  // namespace mmf
