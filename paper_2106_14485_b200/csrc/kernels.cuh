// kernels.cuh — sm_100a kernels of one Gauss-Seidel Sinkhorn sweep.
//
// Layouts: messages [slot][N][Lp] with commodities innermost (Lp = L padded to the
// group width; padded commodities carry exact zeros), significand and exponent in separate planes;
// arc arrays in internal arc order = sorted by (head, tail) (in-CSR), out-CSR by (tail, head) with
// an indirection to the internal arc.  Grid: blockIdx.x = node, blockIdx.y = commodity group of
// blockDim.x commodities (one thread per commodity).
#pragma once
#include "xf.cuh"

namespace mmf {

template <class M_, class E_> struct Tr {
  typedef M_ M;
  typedef E_ E;
};
typedef Tr<float, int16_t> TrF32;
typedef Tr<double, int32_t> TrF64;

struct DevPtrs {
  int N, Lp, L, A, T, TK, TC, G, maxdeg_in;
  const int* tail;      // [A] internal order
  const int* in_ptr;    // [N+1]
  const int* out_ptr;   // [N+1]
  const int* out_arc;   // [A] out-CSR position -> internal arc
  const int* out_head;  // [A] head of that arc
  const void* Km;       // [TK][A] significand of K
  const int* Ke;        // [TK][A] exponent of K
  const void* dcap;     // [TC][A] capacity (M), +inf free, 0 closed
  void* Wm;             // [T][A]
  int* We;              // [T][A]
  void* am;             // alpha [2][N][Lp]
  void* ae;
  void* bm;             // beta [T+1][N][Lp]
  void* be;
  void* u0m;            // U0 [N][Lp]
  void* u0e;
  const void* mu0m;     // dense marginals [N][Lp] (or null)
  const void* mu0e;
  const void* muTm;
  const void* muTe;
  const int* psrc;      // point marginals [L] (or null)
  const int* pdst;
  const double* pmass;
  void* part;           // [G][A] partial flows (M)
  void* Fsum;           // [Ecap] the multi-GPU exchange buffer: flows of the capacitated arcs only (M)
  const int* fpos;      // [A] internal arc -> its position in Fsum (-1: uncapacitated at every step)
  int Ecap;             // capacitated arcs (Fsum length; the all-reduce moves Ecap values, not A)
  void* Fout;           // [T][A] readout flows (M)
  unsigned* err;        // sticky error word
  unsigned long long* errloc;  // first error (commodity << 32 | node)
  double* stats;        // [8] accumulators
  void* inrec;          // [T][A] ArcKW<M> per internal (in-CSR) arc: tail, K_t W_t      (or null)
  void* outrec;         // [T][A] ArcKW<M> per out-CSR position: head, K_t W_t, arc id    (or null)
  const int* opos;      // [A] internal arc -> out-CSR position
  // ELL copies of the records for the pipelined kernels (or null): [T][N][D] per node, unused slots node = -1
  void* ell_in;         // in-arcs of each head: node = tail, aux = arc id | uncapacitated bit
  void* ell_ops;        // [T][N][Din] ArcOps of the in-arcs (dual-update operands), same slots as ell_in (or null)
  void* ell_out;        // out-arcs of each tail: node = head
  const int* ell_ipos;  // [A] internal arc -> slot in ell_in (head * Din + k)
  const int* ell_opos;  // [A] internal arc -> slot in ell_out (tail * Dout + k)
  int Din, Dout;
  // commodity node factors D = exp(-c / eps) [N][Lp], applied by the message epilogues
  // (norm_lane, store_msg) of launches whose output layer is intermediate (1..T-1); null otherwise
  const void* dnm;
  const void* dne;
  int akeep;  // 1: the alpha store keeps every layer (slot t; symmetric GS), 0: double buffer (slot t & 1)
  // node (state) capacities: d [TN][N] (M), the duals u [T+1][N] (M significand + int exponent),
  // and per launch the layer's u applied by the message epilogues (unlm / unle, null when not applied)
  const void* dnc;
  int dnc_tv;
  void* unm;
  int* une;
  const void* unlm;
  const int* unle;
  int diag;  // diagnostics of the pipelined forward (option "dry" >= 2; results invalid), else 0
  int l2hint;  // 1: the pipelined kernels gather message rows with an L2 evict_last policy (option "l2hint")
  float theta;  // Jacobi schedule damping: W <- W^(1 - theta) min(W d / F, 1)^theta
};

// per-step arc record: gathered node, arc factor K_t W_t as XF (km = 0: zero factor), aux word
// (outrec: arc id, bit 31 set when the arc is uncapacitated at step t)
template <class M> struct ArcKW;
template <> struct __align__(16) ArcKW<float> {
  int node;
  int ke;
  int aux;
  float km;
};
template <> struct __align__(8) ArcKW<double> {
  int node;
  int ke;
  int aux;
  int pad;
  double km;
};

// dual-update operands of an arc at step t, kept next to its in-record (fp32 mode, pipelined forward):
// capacity, current W (significand, exponent), K (significand, exponent), and the arc's slots in the ELL
// and CSR out-records
struct __align__(16) ArcOps {
  float d;
  float wm;
  int we;
  float Km;
  int Ke;
  int eopos;
  int copos;
  int pad;
};

template <class T_> struct View {
  typedef typename T_::M M;
  typedef typename T_::E E;
  const DevPtrs& p;
  __device__ __forceinline__ View(const DevPtrs& pp) : p(pp) {}
  __device__ __forceinline__ const M* Km(int t) const { return (const M*)p.Km + (size_t)(p.TK > 1 ? t : 0) * p.A; }
  __device__ __forceinline__ const int* Ke(int t) const { return p.Ke + (size_t)(p.TK > 1 ? t : 0) * p.A; }
  __device__ __forceinline__ const M* dcap(int t) const { return (const M*)p.dcap + (size_t)(p.TC > 1 ? t : 0) * p.A; }
  __device__ __forceinline__ M* Wm(int t) const { return (M*)p.Wm + (size_t)t * p.A; }
  __device__ __forceinline__ int* We(int t) const { return p.We + (size_t)t * p.A; }
  __device__ __forceinline__ size_t slot(int s) const { return (size_t)s * p.N * p.Lp; }
  __device__ __forceinline__ M* am(int t) const { return (M*)p.am + slot(p.akeep ? t : (t & 1)); }
  __device__ __forceinline__ E* ae(int t) const { return (E*)p.ae + slot(p.akeep ? t : (t & 1)); }
  __device__ __forceinline__ M* bm(int t) const { return (M*)p.bm + slot(t); }
  __device__ __forceinline__ E* be(int t) const { return (E*)p.be + slot(t); }
};

__device__ __forceinline__ void set_error(const DevPtrs& p, unsigned bit, int commodity, int node) {
  unsigned old = atomicOr(p.err, bit);
  if (old == 0u)
    atomicCAS(p.errloc, 0ull, ((unsigned long long)(unsigned)commodity << 32) | (unsigned)node | (1ull << 63));
}

template <class T_>
__device__ __forceinline__ void store_msg(const DevPtrs& p, typename T_::M* pm, typename T_::E* pe, size_t idx,
                                          typename T_::M s, int E, int l, int node) {
  typedef typename T_::M M;
  M m;
  int e;
  xf_norm<M>(s, E, m, e);
  if (p.dnm && m != M(0)) {  // commodity node factor of this layer (NEXT-2)
    m *= ((const M*)p.dnm)[idx];
    e += (int)((const typename T_::E*)p.dne)[idx];
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
  if (m != M(0) && (e > ELIM || e < -ELIM)) {
    set_error(p, ERR_RANGE, l, node);
    e = e > 0 ? ELIM : -ELIM;
  }
  pm[idx] = m;
  pe[idx] = (typename T_::E)e;
}

// ---------------------------------------------------------------------------------------------
// a5 backward step: beta_t[i,l] = sum_{a: i_a = i} K_t[a] W_t[a] beta_{t+1}[j_a, l]  (eq:psi)
template <class T_> __global__ void k_bwd(DevPtrs p, int t) {
  typedef typename T_::M M;
  View<T_> v(p);
  const int i = blockIdx.x;
  const int l = blockIdx.y * blockDim.x + threadIdx.x;
  const M* bm1 = v.bm(t + 1);
  const typename T_::E* be1 = v.be(t + 1);
  const M* Km = v.Km(t);
  const int* Ke = v.Ke(t);
  const M* Wm = v.Wm(t);
  const int* We = v.We(t);
  XAcc<M> acc;
  const int k0 = p.out_ptr[i], k1 = p.out_ptr[i + 1];
  for (int k = k0; k < k1; ++k) {
    const int a = p.out_arc[k];
    const int j = p.out_head[k];
    const M mkw = Km[a] * Wm[a];
    const int ekw = Ke[a] + We[a];
    const size_t idx = (size_t)j * p.Lp + l;
    acc.add(mkw * bm1[idx], ekw + (int)be1[idx]);
  }
  store_msg<T_>(p, v.bm(t), v.be(t), (size_t)i * p.Lp + l, acc.s, acc.E, l, i);
}

// block sum of one value per thread; result valid in thread 0
template <class M> __device__ __forceinline__ M block_sum(M x, M* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nw = blockDim.x >> 5;
  if (nw == 1) return x;
  __syncthreads();
  if (lane == 0) red[w] = x;
  __syncthreads();
  M s = M(0);
  if (threadIdx.x == 0)
    for (int k = 0; k < nw; ++k) s += red[k];
  return s;
}

// a3(i) edge flows, partial over this commodity group:
//   part[g][a] = sum_{l in g} alpha_t[i_a,l] K_t[a] W_t[a] beta_{t+1}[j_a,l]       (cor:proj P:1078)
// capped_only: skip uncapacitated arcs (the sweep needs F only where d < inf).
template <class T_> __global__ void k_flow(DevPtrs p, int t, int capped_only) {
  typedef typename T_::M M;
  __shared__ M red[32];
  View<T_> v(p);
  const int j = blockIdx.x;
  const int l = blockIdx.y * blockDim.x + threadIdx.x;
  const size_t jdx = (size_t)j * p.Lp + l;
  const M mb = v.bm(t + 1)[jdx];
  const int eb = (int)v.be(t + 1)[jdx];
  const M* am = v.am(t);
  const typename T_::E* ae = v.ae(t);
  const M* Km = v.Km(t);
  const int* Ke = v.Ke(t);
  const M* Wm = v.Wm(t);
  const int* We = v.We(t);
  const M* dc = v.dcap(t);
  M* part = (M*)p.part + (size_t)blockIdx.y * p.A;
  for (int a = p.in_ptr[j]; a < p.in_ptr[j + 1]; ++a) {
    if (capped_only && isinf(dc[a])) continue;
    const int i = p.tail[a];
    const size_t idx = (size_t)i * p.Lp + l;
    const M f = xf_to_lin<M>(am[idx] * mb * (Km[a] * Wm[a]), (int)ae[idx] + eb + Ke[a] + We[a]);
    const M s = block_sum<M>(f, red);
    if (threadIdx.x == 0) part[a] = s;
  }
}

// capacity-dual update of one arc (eq:sinkhorn_graph_Vineq):
//   W_t[a] <- min(W_t[a] d_t[a] / F_t[a], 1);  d = inf -> unchanged (= 1); d = 0 -> 0; F = 0 -> 1
// computed in fp64 (one value per arc), stored as XF.
// refresh the records of arc a at step t from K_t and the given W_t = (wm, we)
template <class T_>
__device__ __forceinline__ void write_recs(const DevPtrs& p, int t, int a, typename T_::M wm, int we) {
  typedef typename T_::M M;
  View<T_> v(p);
  M m = v.Km(t)[a] * wm;
  int e = v.Ke(t)[a] + we;
  if (!(m > M(0)) || e < -ELIM) {
    m = M(0);
    e = -ELIM;
  }
  if (e > ELIM) e = ELIM;
  ArcKW<M>* ir = (ArcKW<M>*)p.inrec + (size_t)t * p.A;
  ArcKW<M>* orr = (ArcKW<M>*)p.outrec + (size_t)t * p.A;
  const int q = p.opos[a];
  ArcKW<M> r;
  r.node = p.tail[a];
  r.ke = e;
  r.km = m;
  if constexpr (sizeof(M) == 8) r.pad = 0;
  const int uncap = isinf(v.dcap(t)[a]) ? (int)0x80000000u : 0;  // bit 31: uncapacitated at step t
  r.aux = uncap;
  ir[a] = r;
  if (p.ell_in) {
    r.aux = a | uncap;
    ((ArcKW<M>*)p.ell_in)[(size_t)t * p.N * p.Din + p.ell_ipos[a]] = r;
    if constexpr (sizeof(M) == 4) {
      if (p.ell_ops) {
        ArcOps o;
        o.d = v.dcap(t)[a];
        o.wm = wm;
        o.we = we;
        o.Km = v.Km(t)[a];
        o.Ke = v.Ke(t)[a];
        o.eopos = p.ell_opos[a];
        o.copos = q;
        o.pad = 0;
        ((ArcOps*)p.ell_ops)[(size_t)t * p.N * p.Din + p.ell_ipos[a]] = o;
      }
    }
  }
  r.node = p.out_head[q];
  r.aux = a | uncap;
  orr[q] = r;
  if (p.ell_out) ((ArcKW<M>*)p.ell_out)[(size_t)t * p.N * p.Dout + p.ell_opos[a]] = r;
}

template <class T_> __global__ void k_init_recs(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const size_t n = (size_t)p.T * p.A;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(idx / p.A), a = (int)(idx % p.A);
    write_recs<T_>(p, t, a, v.Wm(t)[a], v.We(t)[a]);
  }
}

template <class T_> __device__ __forceinline__ void dual_update(const DevPtrs& p, int t, int a, double F) {
  typedef typename T_::M M;
  View<T_> v(p);
  const M d = v.dcap(t)[a];
  if (isinf(d)) return;
  M* Wm = v.Wm(t);
  int* We = v.We(t);
  M wm;
  int we;
  if (d == M(0)) {
    wm = M(0);
    we = EZERO;
  } else if (!(F > 0.0)) {
    wm = M(1);
    we = 0;
  } else {
    double m;
    int e;
    const double x = (double)Wm[a] * ((double)d / F);
    xf_norm<double>(x, We[a], m, e);
    if (isinf(x)) e = 0;
    wm = (M)m;
    if (wm >= M(2)) {  // significand rounded up to 2 in fp32
      wm = M(1);
      e += 1;
    }
    we = e;
    if (e >= 0) {  // W d / F >= 1
      wm = M(1);
      we = 0;
    }
  }
  Wm[a] = wm;
  We[a] = we;
  if (p.inrec) write_recs<T_>(p, t, a, wm, we);
}

// sum the group partials of every arc: F[a] = sum_g part[g][a]
//   mode 0: out[a] = F for all arcs (readout);  mode 1: out[a] = F for capacitated arcs (before the
//   multi-GPU all-reduce);  mode 2: capacity-dual update in place (single GPU)
template <class T_> __global__ void k_reduce(DevPtrs p, int t, typename T_::M* out, int mode) {
  typedef typename T_::M M;
  View<T_> v(p);
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= p.A) return;
  if (mode != 0 && isinf(v.dcap(t)[a])) return;
  const M* part = (const M*)p.part;
  M s = M(0);
  for (int g = 0; g < p.G; ++g) s += part[(size_t)g * p.A + a];
  if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, a);
  if (mode == 2)
    dual_update<T_>(p, t, a, (double)s);
  else if (mode == 1)
    out[p.fpos[a]] = s;  // (finite capacity at t: fpos >= 0)
  else
    out[a] = s;
}

// capacity-dual update from the all-reduced flows (multi-GPU path)
// NEXT-3 node-capacity block of layer t (Algorithm 2's u_t, on the states): one CTA per node j,
//   P = sum_l alpha_t[j,l] beta-hat_t[j,l] / (D[l,j] u_old[j])   (alpha_t written without u_t; beta-hat_t carries the
//       previous u_t and D: P is the marginal of the current tensor up to u_t),
//   u_t[j] = min(d_t[j] / P, 1)  (d = inf: 1, d = 0: 0, P = 0: 1), then alpha_t[j, :] *= u_t[j].
template <class T_> __global__ void __launch_bounds__(256) k_node_cap(DevPtrs p, int t) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  View<T_> v(p);
  const int j = blockIdx.x;
  const M d = ((const M*)p.dnc)[(size_t)(p.dnc_tv ? t : 0) * p.N + j];
  if (isinf(d)) return;
  M* um = (M*)p.unm + (size_t)t * p.N;
  int* ue = p.une + (size_t)t * p.N;
  M* am = v.am(t) + (size_t)j * p.Lp;
  E* ae = v.ae(t) + (size_t)j * p.Lp;
  double nm;
  int ne;
  if (d == M(0)) {
    nm = 0.0;
    ne = EZERO;
  } else {
    const M* bm = v.bm(t) + (size_t)j * p.Lp;
    const E* be = v.be(t) + (size_t)j * p.Lp;
    XAcc<double> acc;
    for (int l = threadIdx.x; l < p.L; l += blockDim.x) {
      double m = (double)am[l] * (double)bm[l];
      int e = (int)ae[l] + (int)be[l];
      if (p.dnm) {
        m /= (double)((const M*)p.dnm)[(size_t)j * p.Lp + l];
        e -= (int)((const E*)p.dne)[(size_t)j * p.Lp + l];
      }
      if (m > 0.0) acc.add(m, e);
    }
    // block reduction of (s, E)
    __shared__ double ss[256];
    __shared__ int se[256];
    ss[threadIdx.x] = acc.s;
    se[threadIdx.x] = acc.E;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) {
        const int E1 = se[threadIdx.x], E2 = se[threadIdx.x + o], Em = max(E1, E2);
        ss[threadIdx.x] = ss[threadIdx.x] * pow2_nonpos<double>(E1 - Em) + ss[threadIdx.x + o] * pow2_nonpos<double>(E2 - Em);
        se[threadIdx.x] = Em;
      }
      __syncthreads();
    }
    const double s = ss[0];
    const int E_ = se[0];
    const double uo = (double)um[j];
    const int uoe = ue[j];
    if (!(s > 0.0) || !(uo > 0.0)) {
      nm = 1.0;
      ne = 0;
    } else {
      // x = d / P = d u_old / (s 2^E)
      xf_norm<double>((double)d * uo / s, uoe - E_, nm, ne);
      if (ne >= 0) {
        nm = 1.0;
        ne = 0;
      }
    }
  }
  __syncthreads();
  MMF_DASSERT(nm == 0.0 || (nm >= 1.0 && nm < 2.0 && ne <= 0));  // (u in [0, 1])
  if (threadIdx.x == 0) {
    um[j] = (M)nm;
    ue[j] = ne;
  }
  for (int l = threadIdx.x; l < p.Lp; l += blockDim.x) {
    double m = (double)am[l] * nm;
    int e = (int)ae[l] + ne;
    M mm;
    int ee;
    xf_norm<M>((M)m, e, mm, ee);
    if (mm == M(0)) ee = EZERO;
    am[l] = mm;
    ae[l] = (E)ee;
  }
}

// compact = 1: F from the exchange buffer Fsum[fpos[a]]; 0: from an arc-indexed array (Fsum = a step of Fout)
template <class T_> __global__ void k_dual(DevPtrs p, int t, int compact) {
  const int a = blockIdx.x * blockDim.x + threadIdx.x;
  if (a >= p.A) return;
  typedef typename T_::M M;
  if (compact) {
    const int f = p.fpos[a];
    if (f >= 0) dual_update<T_>(p, t, a, (double)((const M*)p.Fsum)[f]);  // (uncapacitated: nothing to update)
  } else {
    dual_update<T_>(p, t, a, (double)((const M*)p.Fsum)[a]);
  }
}

// a3(iv) SpMM^T: alpha_{t+1}[j,l] = sum_{a -> j} alpha_t[i_a,l] K_t[a] W_t[a]   (eq:psi_hat P:1031-1036)
template <class T_> __global__ void k_spmm_fwd(DevPtrs p, int t) {
  typedef typename T_::M M;
  View<T_> v(p);
  const int j = blockIdx.x;
  const int l = blockIdx.y * blockDim.x + threadIdx.x;
  const M* Km = v.Km(t);
  const int* Ke = v.Ke(t);
  const M* Wm = v.Wm(t);
  const int* We = v.We(t);
  const M* am = v.am(t);
  const typename T_::E* ae = v.ae(t);
  XAcc<M> acc;
  for (int a = p.in_ptr[j]; a < p.in_ptr[j + 1]; ++a) {
    const int i = p.tail[a];
    const size_t idx = (size_t)i * p.Lp + l;
    acc.add(am[idx] * (Km[a] * Wm[a]), (int)ae[idx] + Ke[a] + We[a]);
  }
  store_msg<T_>(p, v.am(t + 1), v.ae(t + 1), (size_t)j * p.Lp + l, acc.s, acc.E, l, j);
}

// XF division x / y (both normalised or zero)
template <class M> __device__ __forceinline__ void xf_div(M xm, int xe, M ym, int ye, M& m, int& e) {
  xf_norm<M>(xm / ym, xe - ye, m, e);
}

// a2 / a4 boundary scalings, dense marginals:
//   which = 0: U0 = mu0 ./ beta_0 -> alpha_0 and the U0 plane
//   which = 1: UT = muT ./ alpha_T -> beta_T
// 0/0 := 0; x/0 with x > 0 -> ERR_INFEASIBLE
template <class T_> __global__ void k_boundary_dense(DevPtrs p, int which) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  View<T_> v(p);
  const size_t n = (size_t)p.N * p.Lp;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const M* mum = (const M*)(which == 0 ? p.mu0m : p.muTm);
    const E* mue = (const E*)(which == 0 ? p.mu0e : p.muTe);
    const M* xm = which == 0 ? v.bm(0) : v.am(p.T);
    const E* xe = which == 0 ? v.be(0) : v.ae(p.T);
    M m = M(0);
    int e = EZERO;
    const M mu = mum[idx];
    if (mu > M(0)) {
      const M x = xm[idx];
      if (x > M(0)) {
        xf_div<M>(mu, (int)mue[idx], x, (int)xe[idx], m, e);
      } else {
        set_error(p, ERR_INFEASIBLE, (int)(idx % p.Lp), (int)(idx / p.Lp));
      }
    }
    if (m != M(0) && (e > ELIM || e < -ELIM)) {
      set_error(p, ERR_RANGE, (int)(idx % p.Lp), (int)(idx / p.Lp));
      e = e > 0 ? ELIM : -ELIM;
    }
    if (which == 0) {
      v.am(0)[idx] = m;
      v.ae(0)[idx] = (E)e;
      ((M*)p.u0m)[idx] = m;
      ((E*)p.u0e)[idx] = (E)e;
    } else {
      v.bm(p.T)[idx] = m;
      v.be(p.T)[idx] = (E)e;
    }
  }
}

// zero-fill a message slot (exact zero = (0, EZERO))
template <class T_> __global__ void k_zero(typename T_::M* pm, typename T_::E* pe, size_t n) {
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    pm[idx] = typename T_::M(0);
    pe[idx] = (typename T_::E)EZERO;
  }
}

// point-mass boundary: one thread per commodity (slot already zero-filled)
template <class T_> __global__ void k_boundary_point(DevPtrs p, int which) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  View<T_> v(p);
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= p.L) return;
  const int node = which == 0 ? p.psrc[l] : p.pdst[l];
  const size_t idx = (size_t)node * p.Lp + l;
  const M* xm = which == 0 ? v.bm(0) : v.am(p.T);
  const E* xe = which == 0 ? v.be(0) : v.ae(p.T);
  const M x = xm[idx];
  M m = M(0);
  int e = EZERO;
  if (x > M(0)) {
    int mexp;
    const double fr = frexp(p.pmass[l], &mexp);  // mass = fr * 2^mexp, fr in [0.5, 1)
    xf_div<M>((M)(fr * 2.0), mexp - 1, x, (int)xe[idx], m, e);
  } else {
    set_error(p, ERR_INFEASIBLE, l, node);
  }
  if (m != M(0) && (e > ELIM || e < -ELIM)) {
    set_error(p, ERR_RANGE, l, node);
    e = e > 0 ? ELIM : -ELIM;
  }
  if (which == 0) {
    v.am(0)[idx] = m;
    v.ae(0)[idx] = (E)e;
    ((M*)p.u0m)[idx] = m;
    ((E*)p.u0e)[idx] = (E)e;
  } else {
    v.bm(p.T)[idx] = m;
    v.be(p.T)[idx] = (E)e;
  }
}

template <class T_> __global__ void k_init_w(DevPtrs p) {
  typedef typename T_::M M;
  const size_t n = (size_t)p.T * p.A;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    ((M*)p.Wm)[idx] = M(1);
    p.We[idx] = 0;
  }
}

// UT = 1 on supp(muT) (Q7) -> beta_T
template <class T_> __global__ void k_init_ut_dense(DevPtrs p) {
  typedef typename T_::M M;
  typedef typename T_::E E;
  View<T_> v(p);
  const size_t n = (size_t)p.N * p.Lp;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const bool on = ((const M*)p.muTm)[idx] > M(0);
    v.bm(p.T)[idx] = on ? M(1) : M(0);
    v.be(p.T)[idx] = on ? (E)0 : (E)EZERO;
  }
}
template <class T_> __global__ void k_init_ut_point(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= p.L) return;
  const size_t idx = (size_t)p.pdst[l] * p.Lp + l;
  v.bm(p.T)[idx] = M(1);
  v.be(p.T)[idx] = 0;
}

// log of an XF value (m > 0)
template <class M> __device__ __forceinline__ double xf_log(M m, int e) {
  return log((double)m) + (double)e * 0.69314718055994530942;
}

// statistics of the end-of-sweep state (mmf_stats): block partials -> double atomics
//   stats[0] mass = sum alpha_T beta_T; [1] sum|U0 beta_0 - mu0|; [2] sum|alpha_T beta_T - muT|;
//   [3] sum mu0 log U0; [4] sum muT log UT
template <class T_> __global__ void k_stats_nodes(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const size_t n = (size_t)p.N * p.Lp;
  double acc[5] = {0, 0, 0, 0, 0};
  const bool point = p.psrc != nullptr;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const int l = (int)(idx % p.Lp);
    const int node = (int)(idx / p.Lp);
    if (l >= p.L) continue;
    double mu0, muT;
    if (point) {
      mu0 = p.psrc[l] == node ? p.pmass[l] : 0.0;
      muT = p.pdst[l] == node ? p.pmass[l] : 0.0;
    } else {
      mu0 = (double)xf_to_lin<double>((double)((const M*)p.mu0m)[idx], (int)((const typename T_::E*)p.mu0e)[idx]);
      muT = (double)xf_to_lin<double>((double)((const M*)p.muTm)[idx], (int)((const typename T_::E*)p.muTe)[idx]);
    }
    const M um = ((const M*)p.u0m)[idx];
    const int ue = (int)((const typename T_::E*)p.u0e)[idx];
    const M b0m = v.bm(0)[idx];
    const int b0e = (int)v.be(0)[idx];
    const M aTm = v.am(p.T)[idx];
    const int aTe = (int)v.ae(p.T)[idx];
    const M bTm = v.bm(p.T)[idx];
    const int bTe = (int)v.be(p.T)[idx];
    const double P0 = xf_to_lin<double>((double)um * (double)b0m, ue + b0e);
    const double PT = xf_to_lin<double>((double)aTm * (double)bTm, aTe + bTe);
    acc[0] += PT;
    acc[1] += fabs(P0 - mu0);
    acc[2] += fabs(PT - muT);
    if (mu0 > 0 && um > M(0)) acc[3] += mu0 * xf_log<M>(um, ue);
    if (muT > 0 && bTm > M(0)) acc[4] += muT * xf_log<M>(bTm, bTe);
  }
  for (int k = 0; k < 5; ++k) {
    double x = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(&p.stats[k], x);
  }
}

// stats[5] = sum over capacitated arcs with 0 < d < inf of d * log W  (0 * -inf = 0)
template <class T_> __global__ void k_stats_arcs(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const size_t n = (size_t)p.T * p.A;
  double acc = 0;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(idx / p.A), a = (int)(idx % p.A);
    const double d = (double)v.dcap(t)[a];
    const M wm = v.Wm(t)[a];
    if (d > 0 && !isinf(d) && wm > M(0)) acc += d * xf_log<M>(wm, v.We(t)[a]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&p.stats[5], acc);
}

// bulk-coupled (Jacobi) capacity-dual update of every step from the flows of one forward pass
// (Fout, already summed over all commodities / ranks):  W <- W^(1 - theta) min(W d / F, 1)^theta  in fp64
template <class T_> __global__ void k_jacobi_update(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const size_t n = (size_t)p.T * p.A;
  const double theta = (double)p.theta;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(idx / p.A), a = (int)(idx % p.A);
    const M d = v.dcap(t)[a];
    if (isinf(d)) continue;
    M* Wm = v.Wm(t);
    int* We = v.We(t);
    const M wm0 = Wm[a];
    const int we0 = We[a];
    const double F = (double)((const M*)p.Fout)[idx];
    M wm;
    int we;
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
    if (theta != 1.0) {  // damping in logs: log W = (1 - theta) log W_old + theta log W_full; zero stays zero
      if (wm0 > M(0) && wm > M(0)) {
        const double L = (1.0 - theta) * ((double)we0 + log2((double)wm0)) + theta * ((double)we + log2((double)wm));
        int ne = (int)floor(L);
        M m = (M)exp2(L - (double)ne);
        if (m >= M(2)) {
          m *= M(0.5);
          ++ne;
        }
        wm = m;
        we = ne;
      } else {
        wm = M(0);
        we = EZERO;
      }
    }
    Wm[a] = wm;
    We[a] = we;
    if (p.inrec) write_recs<T_>(p, t, a, wm, we);
  }
}

// per-commodity arc flows of step t (cor:proj P:1078 in node form): out[a_user][l] = alpha_t[i_a, l] K_t W_t[a]
// beta_{t+1}[j_a, l] in fp64 (alpha_t of the end-of-sweep tensor is in its slot)
template <class T_>
__global__ void k_commodity_flows(DevPtrs p, const int* __restrict__ ioa, int t, double* __restrict__ out) {
  typedef typename T_::M M;
  View<T_> v(p);
  const int64_t n = (int64_t)p.A * p.L;
  for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < n; k += (int64_t)gridDim.x * blockDim.x) {
    const int64_t au = k / p.L;
    const int l = (int)(k - au * p.L);
    const int a = ioa[au];
    const int i = p.tail[a], j = p.out_head[p.opos[a]];
    const size_t gi = (size_t)i * p.Lp + l, gj = (size_t)j * p.Lp + l;
    const double m = (double)v.am(t)[gi] * (double)v.bm(t + 1)[gj] * (double)v.Km(t)[a] * (double)v.Wm(t)[a];
    const int e = (int)v.ae(t)[gi] + (int)v.be(t + 1)[gj] + v.Ke(t)[a] + v.We(t)[a];
    out[k] = m == 0.0 ? 0.0 : ldexp(m, e);
  }
}

// capacity excess of the readout flows: sum over capacitated (t, a) of (F_t[a] - d_t[a])_+ -> stats[6]
// (solve-to-tolerance; the flows are already summed over all commodities / ranks)
template <class T_> __global__ void k_stats_excess(DevPtrs p) {
  typedef typename T_::M M;
  View<T_> v(p);
  const size_t n = (size_t)p.T * p.A;
  double acc = 0;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < n; idx += (size_t)gridDim.x * blockDim.x) {
    const int t = (int)(idx / p.A), a = (int)(idx % p.A);
    const double d = (double)v.dcap(t)[a];
    const double F = (double)((const M*)p.Fout)[idx];
    if (!isinf(d) && F > d) acc += F - d;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_down_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(&p.stats[6], acc);
}

}  // namespace mmf
