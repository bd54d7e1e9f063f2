// tiled.cuh — shared building blocks of the sweep kernels: the per-lane message vectors (Lane, VecM / VecE), the
// mbarrier + TMA bulk-copy wrappers (cp.async.bulk, mbarrier try_wait / expect_tx) used by the pipelined and
// window kernels, the extended-range normalisation of a lane's sums into [1, 2) significands and int16 / int32
// exponents (norm_lane, with the node factors of NEXT-2 / NEXT-3), the boundary scalings a2 / a4 of one lane
// (boundary_lane, P:1090 / P:1096), the elementwise node-factor pass (k_apply_factors) and the linear flow term of
// one lane (flow_terms, cor:proj P:1078).  The host side still groups nodes into tiles (TileMeta: the BFS-tile
// node order of kernels 3..5); the node-tile kernels themselves (kernels = 2, smem halos staged per tile) were
// removed in round 2: measured 2-7x slower than the pipelined and wide-lane kernels on [3]-[5].
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

// ------------------------------------------------------------------------------------------------

// FAC: apply the node factors of the launch's output layer (NEXT-2 commodity node factor D, NEXT-3 node-capacity
// dual u) here; the pipelined kernels instantiate FAC = false (their launches are followed by k_apply_factors when a
// problem has such factors): the per-element checks cost their epilogues up to 17 % (measured on [4])
template <class T_, int CPT, bool FAC = true>
__device__ __forceinline__ void norm_lane(const DevPtrs& p, const typename T_::M* s, const int* E,
                                          Lane<typename T_::M, typename T_::E, CPT>& out, int l0, int node) {
  typedef typename T_::M M;
  if constexpr (sizeof(M) == 4 && !FAC) {
    // (the pipelined epilogues) one range flag per lane and a single rare branch instead of a compare-and-branch
    // per element; same results: a nonzero element with |e| > ELIM sets ERR_RANGE and is clamped
    bool bad = false;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const unsigned u = __float_as_uint(s[c]);
      const int e = E[c] + (int)(u >> 23) - 127;
      bad |= u != 0u && (unsigned)(e + ELIM) > 2u * ELIM;
      out.m[c] = u == 0u ? 0.f : __uint_as_float((u & 0x007fffffu) | 0x3f800000u);
      out.e[c] = (typename T_::E)(u == 0u ? EZERO : e);
      MMF_DASSERT(node >= 0 && node < p.N && l0 + c < p.Lp);
    }
    if (bad) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        const unsigned u = __float_as_uint(s[c]);
        const int e = E[c] + (int)(u >> 23) - 127;
        if (u != 0u && (e > ELIM || e < -ELIM)) {
          set_error(p, ERR_RANGE, l0 + c, node);
          out.e[c] = (typename T_::E)(e > 0 ? ELIM : -ELIM);
        }
      }
    }
    return;
  }
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

__device__ __forceinline__ unsigned pack2(int e) { return ((unsigned)e & 0xffffu) * 0x10001u; }

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

}  // namespace mmf
