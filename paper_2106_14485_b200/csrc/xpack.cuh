// xpack.cuh — a lane's CPT commodities of a message row in the fp32 extended-range format (significand in
// [1, 2) + int16 exponent, exponents packed two per 32-bit word) and the packed arithmetic on them shared by the
// pipelined and the wide-lane kernels: 16x2 max-plus exponents (VIADDMNMX.S16x2), scales built by an integer add
// into the float exponent field, and products / sums by FFMA2 / FMUL2 on commodity pairs.
#pragma once
#include "tiled.cuh"

namespace mmf {

// one lane's CPT consecutive commodities of a row; fp32 exponents kept packed two per word
template <class T_, int CPT> struct Row {
  typedef typename T_::M M;
  typedef typename T_::E E;
  static constexpr bool PACKED = sizeof(M) == 4 && sizeof(E) == 2 && CPT % 2 == 0;
  static constexpr int NW = PACKED ? CPT / 2 : CPT;
  M m[CPT];
  int w[NW];  // PACKED: int16x2 words; else one exponent per commodity
  __device__ __forceinline__ void load(const M* pm, const E* pe) {
    typedef typename VecM<M, CPT>::T VM;
    VM vm = *reinterpret_cast<const VM*>(pm);
    const M* sm = reinterpret_cast<const M*>(&vm);
#pragma unroll
    for (int c = 0; c < CPT; ++c) m[c] = sm[c];
    if constexpr (PACKED) {
      typedef typename VecE<int16_t, CPT>::T VE;
      VE ve = *reinterpret_cast<const VE*>(pe);
      const int* sw = reinterpret_cast<const int*>(&ve);
#pragma unroll
      for (int k = 0; k < NW; ++k) w[k] = sw[k];
    } else {
      typedef typename VecE<E, CPT>::T VE;
      VE ve = *reinterpret_cast<const VE*>(pe);
      const E* se = reinterpret_cast<const E*>(&ve);
#pragma unroll
      for (int c = 0; c < CPT; ++c) w[c] = (int)se[c];
    }
  }
  __device__ __forceinline__ int e(int c) const {
    if constexpr (PACKED)
      return (c & 1) ? (w[c >> 1] >> 16) : (int)(short)(w[c >> 1] & 0xffff);
    else
      return w[c];
  }
};


// ------------------------------------------------------------------------------------------------
// Extended-range arithmetic on a lane's CPT commodities (fp32 significand, int16 exponent).
// Exponents are handled two per 32-bit word (CPT even): the max of (row exponent + arc exponent) by one
// VIADDMNMX.S16x2 per pair (exact: |e| <= 16384, |ke| <= 16000); the scale 2^d, d = max(max(e + ke,
// E - 32512) - E, -126) (no 16-bit wrap) by two more; then K W 2^d by an integer add into the float's
// exponent field — mod 2^32 the low / high half of d << 23 equals d2 << 23 / (d2 >> 16) << 23 (PRMT + LEA).

#ifndef MMF_HI_SHF
#define MMF_HI_SHF 2
#endif
#if MMF_HI_SHF == 2
// (PRMT + LEA: written as a shift, ptxas folds it into SHL + LOP3 + IADD; the byte permute [b2 b3 b2 b3] is
// opaque to it and its low half is d2's high half, the copy above shifts out)
#define MMF_HI23(d2) (__byte_perm((d2), 0u, 0x3232) << 23)
#elif MMF_HI_SHF
#define MMF_HI23(d2) (((d2) >> 16) << 23)
#else
#define MMF_HI23(d2) (((d2)&0xffff0000u) << 7)
#endif
#ifndef MMF_XPRE_FAST
#define MMF_XPRE_FAST 1
#endif
template <int CPT> struct XPre {  // per-item constants of a lane: -E and the low clamp E - 126 (E - 32512 saturated in the emulated form), packed
  unsigned nE2[CPT / 2 > 0 ? CPT / 2 : 1], Lo2[CPT / 2 > 0 ? CPT / 2 : 1], Ep2[CPT / 2 > 0 ? CPT / 2 : 1];
  int nE[CPT];
  int E[CPT];
  // FAST = false: the emulated saturating form (kept for the register-capped wide-lane kernels, whose allocation
  // spills more with the native form: 284 vs 188 bytes in the 64-register fp32 forward, [5] forward 62.1 vs 58.0 ms
  // per sweep measured; option MMF_WIDE_XFAST)
  template <bool FAST = (MMF_XPRE_FAST != 0)> __device__ __forceinline__ void set(const unsigned* E2) {
    if constexpr (CPT % 2 == 0) {
#pragma unroll
      for (int w = 0; w < CPT / 2; ++w) {
        nE2[w] = __vneg2(E2[w]);
        if constexpr (FAST) {
        // (native VIMNMX / VIADD.16x2 instead of the emulated saturating __vsubss2 / __vaddss2, 6-7 instructions
        // each; same results) Lo2 = E - 126: the terms' low clamp u = max(e + ke, E - 126) keeps u - E in
        // [-126, 0] (E >= -32384 whenever a row exists: e >= EZERO, ke >= -ELIM; the floor only guards the
        // row-less maximum 0x8000, whose terms are never formed).  Ep2 = clamp(E, +-16131) + 127: for a nonzero
        // beta (|e_b| <= ELIM) e_b + E + 127 clamped to [0, 254] is unchanged by the clamp of E, and
        // e_b + Ep2 stays inside int16 (beta_lin adds it without saturation)
        Lo2[w] = __vadd2(__vmaxs2(E2[w], 0x81808180u), 0xff82ff82u);
        Ep2[w] = __vadd2(__vmins2(__vmaxs2(E2[w], 0xc0fdc0fdu), 0x3f033f03u), 0x007f007fu);
        } else {
        Lo2[w] = __vsubss2(E2[w], 0x7f007f00u);
        Ep2[w] = __vaddss2(E2[w], 0x007f007fu);  // E + 127 (float exponent bias), saturated
        }
        E[2 * w] = (int)(short)(E2[w] & 0xffffu);
        E[2 * w + 1] = (int)E2[w] >> 16;
      }
    } else {
#pragma unroll
      for (int c = 0; c < CPT; ++c) E[c] = (int)E2[c];
    }
#pragma unroll
    for (int c = 0; c < CPT; ++c) nE[c] = -E[c];
  }
};

template <int CPT> __device__ __forceinline__ void xmax_init(unsigned* E2) {
  if constexpr (CPT % 2 == 0) {
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) E2[w] = 0x80008000u;
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) E2[c] = (unsigned)(EZERO - 4 * ELIM);
  }
}
template <int CPT>
__device__ __forceinline__ void xmax_add(unsigned* E2, const Row<TrF32, CPT>& x, unsigned k2, int ke) {
  if constexpr (CPT % 2 == 0) {
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) E2[w] = __viaddmax_s16x2((unsigned)x.w[w], k2, E2[w]);
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) E2[c] = (unsigned)max((int)E2[c], x.e(c) + ke);
  }
}
// packed fp32x2 arithmetic (sm_100 FFMA2 / FMUL2: two IEEE fp32 operations per instruction, same rounding as
// the scalar ones) on commodity pairs
#ifndef MMF_F2
#define MMF_F2 1
#endif
__device__ __forceinline__ void fma2(float& a0, float& a1, float x0, float x1, float y0, float y1) {
#if MMF_F2
  const float2 r = __ffma2_rn(make_float2(x0, x1), make_float2(y0, y1), make_float2(a0, a1));
  a0 = r.x;
  a1 = r.y;
#else
  a0 = fmaf(x0, y0, a0);
  a1 = fmaf(x1, y1, a1);
#endif
}
__device__ __forceinline__ void mul2(float& a0, float& a1, float x0, float x1, float y0, float y1) {
#if MMF_F2
  const float2 r = __fmul2_rn(make_float2(x0, x1), make_float2(y0, y1));
  a0 = r.x;
  a1 = r.y;
#else
  a0 = x0 * y0;
  a1 = x1 * y1;
#endif
}

// t[c] = x.m[c] * K W * 2^(x.e[c] + ke - E[c]) (flushed below 2^-126 of the maximum)
template <int CPT>
__device__ __forceinline__ void xterms(const Row<TrF32, CPT>& x, unsigned kb, unsigned k2, int ke,
                                       const XPre<CPT>& P, float* tq) {
  if constexpr (CPT % 2 == 0) {
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) {
      const unsigned u = __viaddmax_s16x2((unsigned)x.w[w], k2, P.Lo2[w]);
      const unsigned d2 = __viaddmax_s16x2(u, P.nE2[w], 0xff82ff82u);
      mul2(tq[2 * w], tq[2 * w + 1], x.m[2 * w], x.m[2 * w + 1], __uint_as_float(kb + (d2 << 23)),
           __uint_as_float(kb + MMF_HI23(d2)));
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int d = max(x.e(c) + ke + P.nE[c], -126);
      tq[c] = x.m[c] * __uint_as_float(kb + ((unsigned)d << 23));
    }
  }
}
template <int CPT>
__device__ __forceinline__ void xacc(const Row<TrF32, CPT>& x, unsigned kb, unsigned k2, int ke, const XPre<CPT>& P,
                                     float* acc) {
  if constexpr (CPT % 2 == 0) {
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) {
      const unsigned u = __viaddmax_s16x2((unsigned)x.w[w], k2, P.Lo2[w]);
      const unsigned d2 = __viaddmax_s16x2(u, P.nE2[w], 0xff82ff82u);
      fma2(acc[2 * w], acc[2 * w + 1], x.m[2 * w], x.m[2 * w + 1], __uint_as_float(kb + (d2 << 23)),
           __uint_as_float(kb + MMF_HI23(d2)));
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int d = max(x.e(c) + ke + P.nE[c], -126);
      acc[c] = fmaf(x.m[c], __uint_as_float(kb + ((unsigned)d << 23)), acc[c]);
    }
  }
}
__device__ __forceinline__ int k2_to_ke(unsigned k2) { return (int)(short)(k2 & 0xffffu); }
__device__ __forceinline__ unsigned pack_e2(int lo, int hi) { return ((unsigned)lo & 0xffffu) | ((unsigned)hi << 16); }

// flow term of one lane, fp32 mode, commodity pairs: sum_c a_c b_c K W with the same flush as flow_terms (scale
// 2^es, es = a.e + b.e + ke clamped to -127 -> exactly 0).  The exponent sum takes two 16x2 max-plus operations:
// a.e + b.e (>= -32768: no wrap) is first clamped to -16200 (below it es < -127 for any |ke| <= 16000, so the
// flush is unchanged), then ke is added and the result clamped to -127.
template <int CPT>
__device__ __forceinline__ float flow_terms_f2(const float* am, const unsigned* aw, const Row<TrF32, CPT>& b, float kwm,
                                               int kwe) {
  const unsigned k2 = pack2(kwe);
  float f0 = 0.f, f1 = 0.f;
#pragma unroll
  for (int k = 0; k < CPT / 2; ++k) {
    const unsigned u2 = __viaddmax_s16x2(aw[k], (unsigned)b.w[k], 0xc0b8c0b8u);  // max(a.e + b.e, -16200)
    const unsigned es2 = __viaddmax_s16x2(u2, k2, 0xff81ff81u);                  // max(. + ke, -127)
    const float s0 = __uint_as_float((es2 << 23) + 0x3f800000u);                // 2^es (0 at es = -127)
    const float s1 = __uint_as_float(MMF_HI23(es2) + 0x3f800000u);
    float p0, p1;
    mul2(p0, p1, am[2 * k], am[2 * k + 1], kwm, kwm);
    mul2(p0, p1, p0, p1, b.m[2 * k], b.m[2 * k + 1]);
    fma2(f0, f1, p0, p1, s0, s1);
  }
  return f0 + f1;
}

}  // namespace mmf
