// pipefwd.cuh — TMA-pipelined persistent forward step (option kernels = 5, fp32, one slice per node).
//
// Forward kernel of step t (1 <= t <= T), one item per node j (all Lp commodities), the head-flow order of
// headflow.cuh (Algorithm 2's Gauss-Seidel order):
//   (i)   F_{t-1}[a] = K W_{t-1}[a] sum_l alpha_{t-1}[i_a,l] beta_t[j,l] for the in-arcs a -> j  (cor:proj P:1078)
//   (ii)  W_{t-1}[a] <- min(W_{t-1}[a] d[a] / F_{t-1}[a], 1)                         (eq:sinkhorn_graph_Vineq P:861)
//   (iii) alpha_t[j] = sum_{a -> j} alpha_{t-1}[i_a] K W_{t-1}[a] with the updated W    (eq:psi_hat P:1031-1036)
// The producer warp stages, per item: the compacted rows alpha_{t-1}[i_a] (nonzero factor) and the node's
// own row beta_t[j] (cp.async.bulk), the arc records (cp.async ring, prefetched), and the dual-update
// operands d, W, K of every in-arc (4-byte cp.async into the item descriptor, tracked by the same
// mbarrier through cp.async.mbarrier.arrive.noinc).
//
// Consumers (a group of 8 warps per item, 2 groups alternating items) compute the per-row terms
//   t_q[c] = alpha_q[c] K W_q 2^-E[c]     (E[c] = max_q exponent of alpha_q[c] K W_q, extended range)
// once, in registers.  Then
//   flows:  F_q = sum_c t_q[c] * beta_lin[c],   beta_lin[c] = beta[j,c] 2^E[c]  (one FMA per element),
//           reduced over the lanes (shuffles) and the group's warps (shared memory, fixed order);
//   update: one lane per arc applies (ii) and publishes the ratio r_q = W_new / W_old;
//   alpha:  alpha_t[j,c] = 2^E[c] sum_q r_q t_q[c]   (one FMA per element)
// — valid while every |log2 r_q| <= 40 (the dropped terms, below 2^-126 of the old maximum, stay below
// 2^-46 of the new one); otherwise the item is recomputed from shared memory with the new factors.
#pragma once
#include "pipe.cuh"

namespace mmf {

struct FwdHdr {
  float km[32];  // rows (compacted, nonzero factor): K W significand
  int ke[32];    //   ... exponent
  int rarc[32];  //   ... arc position q of the row
  int rowof[32]; // arcs (all in-arcs, q < na): row index or -1
  int aux[32];   //   ... arc id | bit 31 uncapacitated
  float d[32];   //   ... dual-update operands (cp.async)
  float wm[32];
  int we[32];
  float Km[32];
  int Ke[32];
  int eopos[32]; //   ... slot of the arc in the ELL out-records (cp.async)
  int rtail[32]; //   ... tail node
  int nr, na, start, end;
};

// per consumer group scratch
struct FwdGrp {
  float fpart[32][PIPE_NWC];  // flow partials (row, warp)
  float rq[32];               // ratio W_new / W_old per arc position (linear)
  float nkm[32];              // new K W per row (slow path)
  int nke[32];
  int slow;
  int pad[3];
};

struct PFwdSmem {
  size_t off_full, off_empty, off_ring, off_hdr, off_grp, off_sig, off_exp, total;
};

__host__ __device__ inline PFwdSmem pfwd_smem(int R, int D, int SW) {
  PFwdSmem m;
  size_t o = 0;
  m.off_full = o;
  o += 8 * (size_t)PIPE_SD;
  m.off_empty = o;
  o += 8 * (size_t)PIPE_SD;
  o = (o + 15) / 16 * 16;
  m.off_ring = o;
  o += (size_t)PIPE_RP * D * 16;
  m.off_hdr = o;
  o += (size_t)PIPE_SD * sizeof(FwdHdr);
  o = (o + 15) / 16 * 16;
  m.off_grp = o;
  o += (size_t)PIPE_NG * sizeof(FwdGrp);
  o = (o + 127) / 128 * 128;
  m.off_sig = o;
  o += (size_t)R * SW * 4;
  m.off_exp = o;
  o += (size_t)R * SW * 2;
  m.total = o;
  return m;
}

__device__ __forceinline__ void cp_async4(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(smem_u32(smem_dst)), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_mbar_arrive_noinc(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(nthreads) : "memory");
}

template <int CPT> struct FwdNR;
template <> struct FwdNR<4> { static constexpr int v = 8; };
template <> struct FwdNR<2> { static constexpr int v = 12; };
template <> struct FwdNR<1> { static constexpr int v = 16; };

// per-row terms of a lane: t[c] = x.m[c] * KW * 2^(x.e[c] + ke - E[c]), clamped below 2^-126
template <int CPT>
__device__ __forceinline__ void row_terms(const Row<TrF32, CPT>& x, float km, int ke, const unsigned* nE2,
                                          const unsigned* Lo2, const int* nE, float* tq) {
  const unsigned kb = __float_as_uint(km);
  if constexpr (Row<TrF32, CPT>::PACKED) {
    const unsigned k2 = pack2(ke);
#pragma unroll
    for (int w = 0; w < CPT / 2; ++w) {
      const unsigned u = __viaddmax_s16x2((unsigned)x.w[w], k2, Lo2[w]);
      const unsigned d2 = __viaddmax_s16x2(u, nE2[w], 0xff82ff82u);
      tq[2 * w] = x.m[2 * w] * __uint_as_float(kb + (d2 << 23));
      tq[2 * w + 1] = x.m[2 * w + 1] * __uint_as_float(kb + ((d2 & 0xffff0000u) << 7));
    }
  } else {
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int d = max(x.e(c) + ke + nE[c], -126);
      tq[c] = x.m[c] * __uint_as_float(kb + ((unsigned)d << 23));
    }
  }
}

template <int CPT, int MODE>
__global__ void __launch_bounds__(PIPE_THREADS, 1) k_fwd_pipe(DevPtrs p, PipeCfg5 pc, int t) {
  typedef float M;
  typedef int16_t E;
  typedef Row<TrF32, CPT> R_;
  constexpr int NR = FwdNR<CPT>::v;
  extern __shared__ __align__(16) unsigned char smem[];
  const PFwdSmem L = pfwd_smem(pc.R, pc.D, pc.SW);
  unsigned long long* full = (unsigned long long*)(smem + L.off_full);
  unsigned long long* empty = (unsigned long long*)(smem + L.off_empty);
  ArcKW<M>* ring = (ArcKW<M>*)(smem + L.off_ring);
  FwdHdr* hdr = (FwdHdr*)(smem + L.off_hdr);
  FwdGrp* grps = (FwdGrp*)(smem + L.off_grp);
  M* sig = (M*)(smem + L.off_sig);
  E* sex = (E*)(smem + L.off_exp);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int D = pc.D, SW = pc.SW, R = pc.R;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PIPE_SD; ++s) {
      mbar_init(&full[s], 1 + 32);     // expect_tx arrive + one cp.async (noinc) arrive per producer lane
      mbar_init(&empty[s], PIPE_NWC);  // one consumer group per item
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);

  if (warp == PIPE_NWC * PIPE_NG) {  // ---------------- producer
    const ArcKW<M>* ell = (const ArcKW<M>*)p.ell_in + (size_t)(t - 1) * p.N * D;
    const M* gm = v.am(t - 1);
    const E* ge = v.ae(t - 1);
    const M* bm = v.bm(t);
    const E* be = v.be(t);
    const M* dc = v.dcap(t - 1);
    const M* Wm = v.Wm(t - 1);
    const int* We = v.We(t - 1);
    const M* Km = v.Km(t - 1);
    const int* Ke = v.Ke(t - 1);
    int pnode = blockIdx.x, pslot = 0;
    auto prefetch = [&]() {
      if (pnode < p.N && lane < D) cp_async16(&ring[pslot * D + lane], ell + (size_t)pnode * D + lane);
      cp_async_commit();
      pnode += gridDim.x;
      pslot = pslot + 1 == PIPE_RP ? 0 : pslot + 1;
    };
#pragma unroll 1
    for (int k = 0; k < PIPE_P; ++k) prefetch();
    unsigned head = 0, tail = 0;
    int rpos = 0, kold = 0, cslot = 0;
    auto release = [&]() {
      const int ds = kold & (PIPE_SD - 1);
      mbar_wait(&empty[ds], (kold / PIPE_SD) & 1);
      tail = (unsigned)hdr[ds].end;
      ++kold;
    };
    int k = 0;
    for (int j = blockIdx.x; j < p.N; j += gridDim.x, ++k) {
      cp_async_wait<PIPE_P - 1>();
      __syncwarp();
      ArcKW<M> r;
      r.node = -1;
      r.km = M(0);
      r.ke = 0;
      r.aux = 0;
      if (lane < D) r = ring[cslot * D + lane];
      cslot = cslot + 1 == PIPE_RP ? 0 : cslot + 1;
      __syncwarp();
      const bool valid = lane < D && r.node >= 0;
      const bool ok = valid && r.km > M(0);
      const unsigned vbal = __ballot_sync(0xffffffffu, valid);
      const unsigned obal = __ballot_sync(0xffffffffu, ok);
      const int na = __popc(vbal), nr = __popc(obal);
      while (kold <= k - PIPE_SD) release();
      while (head + (unsigned)(nr + 1) - tail > (unsigned)R) release();
      const int ds = k & (PIPE_SD - 1);
      FwdHdr& h = hdr[ds];
      const int rs = __popc(obal & ((1u << lane) - 1u));
      if (ok) {
        h.km[rs] = r.km;
        h.ke[rs] = r.ke;
        h.rarc[rs] = lane;
      }
      if (valid) {
        h.rowof[lane] = ok ? rs : -1;
        h.aux[lane] = r.aux;
        h.rtail[lane] = r.node;
        if (r.aux >= 0) {  // capacitated: dual-update operands
          const int a = r.aux;
          cp_async4(&h.eopos[lane], p.ell_opos + a);
          cp_async4(&h.d[lane], dc + a);
          cp_async4(&h.wm[lane], Wm + a);
          cp_async4(&h.we[lane], We + a);
          cp_async4(&h.Km[lane], Km + a);
          cp_async4(&h.Ke[lane], Ke + a);
        }
      }
      if (lane == 0) {
        h.nr = nr;
        h.na = na;
        h.start = rpos;
        h.end = (int)(head + (unsigned)(nr + 1));
      }
      cp_async_mbar_arrive_noinc(&full[ds]);
      prefetch();
      __syncwarp();
      if (lane == 0) mbar_arrive_expect_tx(&full[ds], (unsigned)(nr + 1) * (unsigned)SW * 6u);
      __syncwarp();
      if (ok) {
        const size_t g = (size_t)r.node * p.Lp;
        int q = rpos + rs;
        if (q >= R) q -= R;
        bulk_g2s(sig + q * SW, gm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, ge + g, SW * 2, &full[ds]);
      }
      if (lane == 31) {  // the node's own beta_t row -> slot nr
        const size_t g = (size_t)j * p.Lp;
        int q = rpos + nr;
        if (q >= R) q -= R;
        bulk_g2s(sig + q * SW, bm + g, SW * 4, &full[ds]);
        bulk_g2s(sex + q * SW, be + g, SW * 2, &full[ds]);
      }
      head += (unsigned)(nr + 1);
      rpos += nr + 1;
      if (rpos >= R) rpos -= R;
    }
    cp_async_wait<0>();
    return;
  }

  // ---------------- consumers
  const int grp = warp / PIPE_NWC, wg = warp % PIPE_NWC;
  FwdGrp& G = grps[grp];
  const int col = wg * 32 * CPT + lane * CPT;
  const int bar_id = 1 + grp;
  constexpr int BAR_N = PIPE_NWC * 32;
  int k = grp;
  for (int j = blockIdx.x + grp * gridDim.x; j < p.N; j += PIPE_NG * gridDim.x, k += PIPE_NG) {
    const int ds = k & (PIPE_SD - 1);
    mbar_wait(&full[ds], (k / PIPE_SD) & 1);
    const FwdHdr& h = hdr[ds];
    const int nr = h.nr, na = h.na, start = h.start;
    auto slot = [&](int q) {
      const int r = start + q;
      return (r >= R ? r - R : r) * SW + col;
    };
    // own row beta_t[j] and the per-commodity maximum exponent E over the rows
    R_ b;
    lds_row<CPT>(sig + slot(nr), sex + slot(nr), b);
    unsigned E2[R_::NW];
#pragma unroll
    for (int w = 0; w < R_::NW; ++w) E2[w] = R_::PACKED ? 0x80008000u : (unsigned)(EZERO - 4 * ELIM);
    for (int q = 0; q < nr; ++q) {
      R_ x;
      lds_row<CPT>(sig + slot(q), sex + slot(q), x);
      if constexpr (R_::PACKED) {
        const unsigned k2 = pack2(h.ke[q]);
#pragma unroll
        for (int w = 0; w < R_::NW; ++w) E2[w] = __viaddmax_s16x2((unsigned)x.w[w], k2, E2[w]);
      } else {
#pragma unroll
        for (int c = 0; c < CPT; ++c) E2[c] = (unsigned)max((int)E2[c], x.e(c) + h.ke[q]);
      }
    }
    int Ex[CPT], nE[CPT];
    unsigned nE2[R_::NW], Lo2[R_::NW];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      Ex[c] = R_::PACKED ? ((c & 1) ? ((int)E2[c >> 1] >> 16) : (int)(short)(E2[c >> 1] & 0xffffu)) : (int)E2[c];
      nE[c] = -Ex[c];
    }
    if constexpr (R_::PACKED) {
#pragma unroll
      for (int w = 0; w < R_::NW; ++w) {
        nE2[w] = __vneg2(E2[w]);
        Lo2[w] = __vsubss2(E2[w], 0x7f007f00u);
      }
    }
    // beta_lin[c] = beta[j,c] 2^E[c] (flows are bounded by the mass: exponent clamped to the normal range)
    float bl[CPT];
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
      const int es = b.e(c) + Ex[c];
      bl[c] = (es < -126 || !(b.m[c] > 0.f)) ? 0.f : b.m[c] * __uint_as_float((unsigned)(min(es, 127) + 127) << 23);
    }
    const bool fast = nr <= NR;
    float tq[NR][CPT];
    // ---- flows (old factors)
    if (fast) {
#pragma unroll
      for (int q = 0; q < NR; ++q)
        if (q < nr) {
          R_ x;
          lds_row<CPT>(sig + slot(q), sex + slot(q), x);
          row_terms<CPT>(x, h.km[q], h.ke[q], nE2, Lo2, nE, tq[q]);
          if (h.aux[h.rarc[q]] >= 0) {
            float f = 0.f;
#pragma unroll
            for (int c = 0; c < CPT; ++c) f = fmaf(tq[q][c], bl[c], f);
            f = warp_sum<float>(f);
            if (lane == 0) G.fpart[q][wg] = f;
          }
        }
    } else {
      for (int q = 0; q < nr; ++q) {
        if (h.aux[h.rarc[q]] < 0) continue;
        R_ x;
        lds_row<CPT>(sig + slot(q), sex + slot(q), x);
        float tt[CPT];
        row_terms<CPT>(x, h.km[q], h.ke[q], nE2, Lo2, nE, tt);
        float f = 0.f;
#pragma unroll
        for (int c = 0; c < CPT; ++c) f = fmaf(tt[c], bl[c], f);
        f = warp_sum<float>(f);
        if (lane == 0) G.fpart[q][wg] = f;
      }
    }
    named_bar(bar_id, BAR_N);
    // ---- capacity-dual update: warp 0 of the group, one lane per in-arc
    if (wg == 0) {
      bool big = false;
      if (lane < na) {
        const int aux = h.aux[lane];
        float rq = 1.f;
        if (aux >= 0) {
          const int a = aux;
          const int row = h.rowof[lane];
          float s = 0.f;
          if (row >= 0)
            for (int w = 0; w < PIPE_NWC; ++w) s += G.fpart[row][w];
          if (!(s == s) || isinf(s)) set_error(p, ERR_NAN, -1, a);
          const float d = h.d[lane], w0 = h.wm[lane];
          const int e0 = h.we[lane];
          float wm;
          int we;
          w_new<TrF32>(d, w0, e0, (double)s, wm, we);
          v.Wm(t - 1)[a] = wm;
          v.We(t - 1)[a] = we;
          {  // refresh the step's ELL records (in: this node's slot; out: the tail's slot); the CSR record
             // copies used by the readout kernels are rebuilt from W before a readout (mmf.cu)
            ArcKW<M> rr;
            kw_clamp<TrF32>(h.Km[lane], h.Ke[lane], wm, we, rr.km, rr.ke);
            rr.aux = aux;
            rr.node = h.rtail[lane];
            ((ArcKW<M>*)p.ell_in)[(size_t)(t - 1) * p.N * D + (size_t)j * D + lane] = rr;
            rr.node = j;
            ((ArcKW<M>*)p.ell_out)[(size_t)(t - 1) * p.N * p.Dout + h.eopos[lane]] = rr;
          }
          // ratio W_new / W_old (linear) and the new factor for the slow path
          if (w0 > 0.f && wm > 0.f) {
            const int de = we - e0;
            big = de > 40 || de < -40;
            rq = big ? 0.f : (wm / w0) * __uint_as_float((unsigned)(de + 127) << 23);
          } else {
            big = true;  // W changed from / to exact zero
            rq = 0.f;
          }
          if (row >= 0) {
            float m;
            int e;
            kw_clamp<TrF32>(h.Km[lane], h.Ke[lane], wm, we, m, e);
            G.nkm[row] = m;
            G.nke[row] = e;
          }
        } else if (h.rowof[lane] >= 0) {
          G.nkm[h.rowof[lane]] = h.km[h.rowof[lane]];
          G.nke[h.rowof[lane]] = h.ke[h.rowof[lane]];
        }
        G.rq[lane] = rq;
      }
      const unsigned anyb = __ballot_sync(0xffffffffu, big);
      if (lane == 0) G.slow = anyb != 0u;
    }
    named_bar(bar_id, BAR_N);
    // ---- alpha_t[j]
    float s[CPT];
    if (fast && !G.slow) {
#pragma unroll
      for (int c = 0; c < CPT; ++c) s[c] = 0.f;
#pragma unroll
      for (int q = 0; q < NR; ++q)
        if (q < nr) {
          const float r = G.rq[h.rarc[q]];
#pragma unroll
          for (int c = 0; c < CPT; ++c) s[c] = fmaf(r, tq[q][c], s[c]);
        }
    } else {  // recompute with the new factors from shared memory
      unsigned F2[R_::NW];
#pragma unroll
      for (int w = 0; w < R_::NW; ++w) F2[w] = R_::PACKED ? 0x80008000u : (unsigned)(EZERO - 4 * ELIM);
      for (int q = 0; q < nr; ++q) {
        if (!(G.nkm[q] > 0.f)) continue;
        R_ x;
        lds_row<CPT>(sig + slot(q), sex + slot(q), x);
        if constexpr (R_::PACKED) {
          const unsigned k2 = pack2(G.nke[q]);
#pragma unroll
          for (int w = 0; w < R_::NW; ++w) F2[w] = __viaddmax_s16x2((unsigned)x.w[w], k2, F2[w]);
        } else {
#pragma unroll
          for (int c = 0; c < CPT; ++c) F2[c] = (unsigned)max((int)F2[c], x.e(c) + G.nke[q]);
        }
      }
#pragma unroll
      for (int c = 0; c < CPT; ++c) {
        Ex[c] = R_::PACKED ? ((c & 1) ? ((int)F2[c >> 1] >> 16) : (int)(short)(F2[c >> 1] & 0xffffu)) : (int)F2[c];
        nE[c] = -Ex[c];
        s[c] = 0.f;
      }
      if constexpr (R_::PACKED) {
#pragma unroll
        for (int w = 0; w < R_::NW; ++w) {
          nE2[w] = __vneg2(F2[w]);
          Lo2[w] = __vsubss2(F2[w], 0x7f007f00u);
        }
      }
      for (int q = 0; q < nr; ++q) {
        if (!(G.nkm[q] > 0.f)) continue;
        R_ x;
        lds_row<CPT>(sig + slot(q), sex + slot(q), x);
        float tt[CPT];
        row_terms<CPT>(x, G.nkm[q], G.nke[q], nE2, Lo2, nE, tt);
#pragma unroll
        for (int c = 0; c < CPT; ++c) s[c] += tt[c];
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[ds]);
    Lane<M, E, CPT> a;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {  // s may lie anywhere in the normal range (ratios): general normalisation
      M m;
      int e;
      xf_norm<M>(s[c], Ex[c], m, e);
      if (e > ELIM || (m != M(0) && e < -ELIM)) {
        set_error(p, ERR_RANGE, col + c, j);
        e = e > 0 ? ELIM : -ELIM;
      }
      a.m[c] = m;
      a.e[c] = (E)e;
    }
    const size_t g = (size_t)j * p.Lp + col;
    a.store(v.am(t) + g, v.ae(t) + g);
    if (MODE == 2) {  // a4: UT = muT ./ alpha_T -> beta_T
      Lane<M, E, CPT> ut;
      boundary_lane<TrF32, CPT>(p, 1, j, col, g, a, ut);
      ut.store(v.bm(p.T) + g, v.be(p.T) + g);
    }
    // the group scratch is rewritten by the next item of this group only after its first named barrier
  }
}

}  // namespace mmf
