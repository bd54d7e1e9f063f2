// xf.cuh — extended-range ("XF") numbers for the Sinkhorn messages.
//
// A message element is  value = m * 2^e  with m in [1, 2) (or m == 0, e == EZERO) held in two
// planes: a significand plane of type M (float | double) and an exponent plane of type E
// (int16 | int32).  Arc factors K, W use the same pair with an int32 exponent.  The significand
// keeps the native relative precision at any magnitude; the exponent covers the e^{±thousands}
// spans of long horizons and small eps (SURVEY §8(d) dynamic-range table).
#pragma once
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

namespace mmf {

template <class M> struct FPB;
template <> struct FPB<float> {
  typedef uint32_t U;
  static constexpr int MB = 23, BIAS = 127, EMAXB = 254;
  static __device__ __forceinline__ U bits(float x) { return __float_as_uint(x); }
  static __device__ __forceinline__ float from(U u) { return __uint_as_float(u); }
};
template <> struct FPB<double> {
  typedef uint64_t U;
  static constexpr int MB = 52, BIAS = 1023, EMAXB = 2046;
  static __device__ __forceinline__ U bits(double x) { return (U)__double_as_longlong(x); }
  static __device__ __forceinline__ double from(U u) { return __longlong_as_double((long long)u); }
};

// exponent of an exact zero.  Stored message exponents lie in [-ELIM, ELIM] or equal EZERO, and arc
// exponents used by the packed fp32 path are clamped to [-ELIM, ELIM], so a message exponent plus an
// arc exponent always fits in int16 (the sm_100a 16x2 SIMD max-plus VIADDMNMX.S16x2 relies on it).
constexpr int EZERO = -16384;
// largest |e| a stored message may carry before MMF_ERANGE (int16 plane: +-16000)
constexpr int ELIM = 16000;

// error bits of the sticky device error word
constexpr unsigned ERR_INFEASIBLE = 1u, ERR_RANGE = 2u, ERR_NAN = 4u;

// device-side checks of the debug build (-DMMF_DEBUG, libmmf_debug.so: the memory-safety net in place of
// compute-sanitizer, which this pool does not offer): ring slots, CSR / ELL indices, message exponents; a failed
// check prints its location and traps (the launch fails with cudaErrorIllegalInstruction -> MMF_ECUDA)
#ifdef MMF_DEBUG
#define MMF_DASSERT(c)                                                                          \
  do {                                                                                          \
    if (!(c)) {                                                                                 \
      printf("MMF_DEBUG check failed: %s at %s:%d (block %d thread %d)\n", #c, __FILE__, __LINE__, \
             (int)blockIdx.x, (int)threadIdx.x);                                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define MMF_DASSERT(c) \
  do {                 \
  } while (0)
#endif

// 2^d as M for d <= 0 (0 once below the normal range)
template <class M> __device__ __forceinline__ M pow2_nonpos(int d) {
  typedef FPB<M> B;
  int x = d + B::BIAS;
  return x > 0 ? B::from((typename B::U)x << B::MB) : M(0);
}

// linear value of m * 2^e for m >= 0 finite (any size of m); flush below the normal range,
// +inf above it
template <class M> __device__ __forceinline__ M xf_to_lin(M m, int e) {
  typedef FPB<M> B;
  typename B::U u = B::bits(m);
  int be = (int)(u >> B::MB);            // m >= 0: no sign bit
  if (m == M(0)) return M(0);
  int nb = be + e;
  if (nb <= 0) return M(0);
  if (nb > B::EMAXB) return B::from((typename B::U)(B::EMAXB + 1) << B::MB);  // +inf
  return B::from(u + ((typename B::U)(int64_t)e << B::MB));
}

// normalise x = s * 2^E (s >= 0 finite, normal or zero) into (m in [1,2), e)
template <class M> __device__ __forceinline__ void xf_norm(M s, int E, M& m, int& e) {
  typedef FPB<M> B;
  if (!(s > M(0))) {
    m = M(0);
    e = EZERO;
    return;
  }
  typename B::U u = B::bits(s);
  int be = (int)(u >> B::MB);
  if (be == 0) {  // subnormal: scale up
    s = s * B::from((typename B::U)(B::BIAS + B::MB) << B::MB);
    u = B::bits(s);
    be = (int)(u >> B::MB) - B::MB;
  }
  m = B::from((u & ((((typename B::U)1) << B::MB) - 1)) | ((typename B::U)B::BIAS << B::MB));
  e = E + be - B::BIAS;
}

// running sum of terms m_k * 2^{e_k} (m_k >= 0 finite, < 2^8): s * 2^E with E = max exponent so far
template <class M> struct XAcc {
  M s;
  int E;
  __device__ __forceinline__ XAcc() : s(M(0)), E(EZERO - 4096) {}
  __device__ __forceinline__ void add(M m, int e) {
    int nE = max(E, e);
    s = s * pow2_nonpos<M>(E - nE) + m * pow2_nonpos<M>(e - nE);
    E = nE;
  }
};

}  // namespace mmf
