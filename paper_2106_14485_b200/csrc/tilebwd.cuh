// tilebwd.cuh — node-tile backward step with staged halos (option tbwd, fp32 mode; the default for fp32, L >= 256
// and mean degree >= 7: BJ [3], [5]) and the node-tile forward step on the same tiles (option tfwd, opt-in: measured
// slower than the wide-lane forward on [5], 77.5 vs 67.2 ms per sweep; kept parity-tested for the record).
//
// Backward step (eq:psi):  beta_t[i, :] = sum_{a: i_a = i} K_t W_t[a] beta_{t+1}[j_a, :].
//
// Why: the pipelined backward gathers every out-neighbour row once per arc (|A|/N rows per node: 4.8 on [4],
// 10.3 on [5]) from L2.  Here nodes are grouped into compact tiles (BFS-grown blobs, host side, make_tiles) and a
// work item is (tile, commodity chunk of SW = 32 CPT): the producer warp stages the tile's out-halo rows (the
// distinct heads of its out-arcs, bounded by the host) for the chunk into a ring stage with cp.async.bulk (TMA,
// one copy per row plane, completion by mbarrier transaction count), and the TB_NWC consumer warps compute the
// tile's nodes from shared memory — a gathered row crosses L2 -> SM once per (tile, chunk) instead of once per
// arc (halo / tile instead of the mean degree).  Items are visited in grid-stride order, tile-major: the chunks
// of one tile are staged by neighbouring CTAs at the same time.
//
// The producer also stages the tile's arc metadata of the step (K W from the out-CSR records, the head's halo index;
// the tile's nodes are contiguous, so are their out-arcs) next to the rows.  Per node (one warp, CPT commodities per
// lane): pass 1 takes the per-commodity maximum exponent (16x2 max-plus), pass 2 accumulates x K W 2^(e - E) (xacc:
// two 16x2 max-plus for the scale, FFMA2); zero-factor arcs are skipped.
#pragma once
#include "pipefwd.cuh"

namespace mmf {

#ifndef MMF_TB_NWC
#define MMF_TB_NWC 16
#endif
constexpr int TB_NWC = MMF_TB_NWC;             // consumer warps per CTA
constexpr int TB_THREADS = (TB_NWC + 1) * 32;  // + one producer warp

struct TileCfg {
  int nst;     // ring stages
  int H;       // rows per stage (the largest out-halo)
  int MA;      // arc record slots per stage (the largest per-tile out-arc count)
  int MB;      // static metadata ints per stage (the largest per-tile block)
  int nch;     // commodity chunks of SW per node row
  int nitems;  // ntiles * nch
  const int* tile_ptr;   // [ntiles + 1] node ranges (internal ids)
  const int* hout_ptr;   // [ntiles + 1]
  const int* hout_node;  // out-halo nodes of each tile (sorted)
  const int* out_hidx;   // [A] out-CSR position -> index of its head in the tail tile's out-halo
  const int* desc;       // [ntiles][8] {v0, nv, q0, na, h0, nh, meta offset, meta ints}
  const int* meta;       // per tile: nv + 1 local out-CSR offsets, pad to 4, na halo indices, pad to 4
};

// per stage: H rows of SW significands + exponents, the tile's out-arc records of the step (ArcKW, 16 B), its static
// metadata block
__host__ __device__ inline size_t tb_smem(int nst, int H, int SW, int MA, int MB) {
  return 128 + (size_t)nst * H * SW * 6 + (size_t)nst * MA * 16 + (size_t)nst * MB * 4;
}

template <int CPT>
__global__ void __launch_bounds__(TB_THREADS, 1) k_bwd_tile2(DevPtrs p, TileCfg tc, int t) {
  constexpr int SW = 32 * CPT;
  extern __shared__ __align__(128) unsigned char smem_tb[];
  unsigned long long* full = (unsigned long long*)smem_tb;
  unsigned long long* empty = full + tc.nst;
  float* sig = (float*)(smem_tb + 128);
  int16_t* sex = (int16_t*)(sig + (size_t)tc.nst * tc.H * SW);
  ArcKW<float>* sarc = (ArcKW<float>*)(sex + (size_t)tc.nst * tc.H * SW);
  int* smeta = (int*)(sarc + (size_t)tc.nst * tc.MA);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < tc.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TB_NWC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);
  const float* gm = v.bm(t + 1);
  const int16_t* ge = v.be(t + 1);

  const ArcKW<float>* rec = (const ArcKW<float>*)p.outrec + (size_t)t * p.A;
  if (warp == TB_NWC) {  // ---------------- producer
    int k = 0;
    for (int it = blockIdx.x; it < tc.nitems; it += gridDim.x, ++k) {
      const int s = k % tc.nst;
      if (k >= tc.nst) mbar_wait(&empty[s], ((k / tc.nst) - 1) & 1);
      const int tile = it / tc.nch, ch = it - tile * tc.nch;
      const int4 d0 = *reinterpret_cast<const int4*>(tc.desc + (size_t)tile * 8);
      const int4 d1 = *reinterpret_cast<const int4*>(tc.desc + (size_t)tile * 8 + 4);
      const int q0 = d0.z, na = d0.w, h0 = d1.x, nh = d1.y, moff = d1.z, mn = d1.w;
      MMF_DASSERT(nh >= 0 && nh <= tc.H && na <= tc.MA && mn <= tc.MB);
      if (lane == 0)
        mbar_arrive_expect_tx(&full[s], (unsigned)nh * (unsigned)SW * 6u + (unsigned)na * 16u + (unsigned)mn * 4u);
      __syncwarp();
      if (lane == 0 && na > 0) bulk_g2s(sarc + (size_t)s * tc.MA, rec + q0, (unsigned)na * 16u, &full[s]);
      if (lane == 1 && mn > 0) bulk_g2s(smeta + (size_t)s * tc.MB, tc.meta + moff, (unsigned)mn * 4u, &full[s]);
      float* ds = sig + (size_t)s * tc.H * SW;
      int16_t* de = sex + (size_t)s * tc.H * SW;
      for (int r = lane; r < nh; r += 32) {
        const int node = tc.hout_node[h0 + r];
        MMF_DASSERT(node >= 0 && node < p.N);
        const size_t g = (size_t)node * p.Lp + (size_t)ch * SW;
        bulk_g2s(ds + (size_t)r * SW, gm + g, SW * 4, &full[s]);
        bulk_g2s(de + (size_t)r * SW, ge + g, SW * 2, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers
  float* const bmt = v.bm(t);
  int16_t* const bet = v.be(t);
  int k = 0;
  for (int it = blockIdx.x; it < tc.nitems; it += gridDim.x, ++k) {
    const int s = k % tc.nst;
    const int tile = it / tc.nch, ch = it - tile * tc.nch;
    const int2 dv = *reinterpret_cast<const int2*>(tc.desc + (size_t)tile * 8);  // (v0, nv)
    mbar_wait(&full[s], (k / tc.nst) & 1);
    const float* ss = sig + (size_t)s * tc.H * SW + lane * CPT;
    const int16_t* se = sex + (size_t)s * tc.H * SW + lane * CPT;
    const ArcKW<float>* sa = sarc + (size_t)s * tc.MA;
    const int* sm = smeta + (size_t)s * tc.MB;
    const int* shx = sm + ((dv.y + 1 + 3) & ~3);  // (halo indices after the padded offsets)
    for (int li = warp; li < dv.y; li += TB_NWC) {
      const int i = dv.x + li;
      const int a0 = sm[li], a1 = sm[li + 1];
      // pass 1: maximum exponent of x K W per commodity
      unsigned E2[CPT / 2];
      xmax_init<CPT>(E2);
      for (int q = a0; q < a1; ++q) {
        const float km = sa[q].km;
        if (!(km > 0.f)) continue;
        const unsigned k2 = pack2(sa[q].ke);
        int w[CPT / 2];
        load_exps<CPT>(se + (size_t)shx[q] * SW, w);
#pragma unroll
        for (int jj = 0; jj < CPT / 2; ++jj) E2[jj] = __viaddmax_s16x2((unsigned)w[jj], k2, E2[jj]);
      }
      XPre<CPT> P;
      P.set(E2);
      float acc[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
      // pass 2: acc += x K W 2^(e + ke - E)
      for (int q = a0; q < a1; ++q) {
        const float km = sa[q].km;
        if (!(km > 0.f)) continue;
        const int ke = sa[q].ke;
        const int h = shx[q];
        Row<TrF32, CPT> r;
        r.load(ss + (size_t)h * SW, se + (size_t)h * SW);
        xacc<CPT>(r, __float_as_uint(km), pack2(ke), ke, P, acc);
      }
      const int col = ch * SW + lane * CPT;
      const size_t g = (size_t)i * p.Lp + col;
      Lane<float, int16_t, CPT> out;
      norm_lane<TrF32, CPT, false>(p, acc, P.E, out, col, i);
      out.store(bmt + g, bet + g);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

}  // namespace mmf

namespace mmf {

// ------------------------------------------------------------------------------------------------
// Node-tile forward step (option tfwd; the forward of commodity-sliced nodes, BJ [5]), launch t = 1..T:
//   alpha_t[i] = sum_{a -> i} alpha_{t-1}[i_a] K_{t-1} W_{t-1}[a]            (eq:psi_hat P:1031-1036; W_{t-1} final)
//   then, t < T, the chunk's flow partials of i's out-arcs a = (i -> j):
//     part[ch][q] = sum_{l in chunk} alpha_t[i,l] K_t W_t[a] beta_{t+1}[j,l]  (cor:proj P:1078)
//   (t = T: UT = muT ./ alpha_T -> beta_T, a4), and k_tile_dual sums the partials over the chunks in a fixed
//   order and applies the capacity-dual update of step t (eq:sinkhorn_graph_Vineq P:861) before launch t + 1.
// Work item = (tile, chunk): the producer stages the tile's in-halo rows of alpha_{t-1}, its out-halo rows of
// beta_{t+1}, its in- and out-arc records of the steps t - 1 and t and its static metadata; a consumer warp computes
// alpha_t of a node into registers, stores it, and forms the flows of the node's out-arcs from the staged rows.
struct TileCfgF {
  int nst, Hin, Hout, MAi, MAo, MM, nch, nitems;
  const int* desc;  // [ntiles][16] {v0, nv, qi0, nai, qo0, nao, hin0, nhin, hout0, nhout, moff, mn, o_inidx,
                    //                o_outptr, o_outidx, 0}
  const int* meta;  // per tile: [nv + 1 in offsets | in-halo indices | nv + 1 out offsets | out-halo indices], each
                    // part padded to 4 ints
  const int* hin_node;
  const int* hout_node;
  float* part;      // [nch][A] flow partials (out-CSR positions)
};
__host__ __device__ inline size_t tf_stage(int Hin, int Hout, int SW, int MAi, int MAo, int MM) {
  return (size_t)(Hin + Hout) * SW * 6 + (size_t)(MAi + MAo) * 16 + (size_t)MM * 4;
}
__host__ __device__ inline size_t tf_smem(int nst, int Hin, int Hout, int SW, int MAi, int MAo, int MM) {
  return 128 + (size_t)nst * tf_stage(Hin, Hout, SW, MAi, MAo, MM);
}

template <int CPT>
__global__ void __launch_bounds__(TB_THREADS, 1) k_fwd_tile2(DevPtrs p, TileCfgF tc, int t) {
  constexpr int SW = 32 * CPT;
  extern __shared__ __align__(128) unsigned char smem_tf[];
  unsigned long long* full = (unsigned long long*)smem_tf;
  unsigned long long* empty = full + tc.nst;
  const size_t stage = tf_stage(tc.Hin, tc.Hout, SW, tc.MAi, tc.MAo, tc.MM);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < tc.nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], TB_NWC);
    }
    mbar_fence_init();
  }
  __syncthreads();
  View<TrF32> v(p);
  const bool flows = t < p.T;
  // stage layout: in rows (sig, exp), out rows (sig, exp), in records, out records, metadata
  auto base = [&](int s) { return smem_tf + 128 + (size_t)s * stage; };
  auto in_sig = [&](int s) { return (float*)base(s); };
  auto in_exp = [&](int s) { return (int16_t*)(base(s) + (size_t)tc.Hin * SW * 4); };
  auto out_sig = [&](int s) { return (float*)(base(s) + (size_t)tc.Hin * SW * 6); };
  auto out_exp = [&](int s) { return (int16_t*)(base(s) + (size_t)tc.Hin * SW * 6 + (size_t)tc.Hout * SW * 4); };
  auto in_rec = [&](int s) { return (ArcKW<float>*)(base(s) + (size_t)(tc.Hin + tc.Hout) * SW * 6); };
  auto out_rec = [&](int s) { return in_rec(s) + tc.MAi; };
  auto meta = [&](int s) { return (int*)(out_rec(s) + tc.MAo); };

  if (warp == TB_NWC) {  // ---------------- producer
    const ArcKW<float>* irec = (const ArcKW<float>*)p.inrec + (size_t)(t - 1) * p.A;
    const ArcKW<float>* orec = (const ArcKW<float>*)p.outrec + (size_t)t * p.A;
    const float* am = v.am(t - 1);
    const int16_t* ae = v.ae(t - 1);
    const float* bm = flows ? v.bm(t + 1) : nullptr;
    const int16_t* be = flows ? v.be(t + 1) : nullptr;
    int k = 0;
    for (int it = blockIdx.x; it < tc.nitems; it += gridDim.x, ++k) {
      const int s = k % tc.nst;
      if (k >= tc.nst) mbar_wait(&empty[s], ((k / tc.nst) - 1) & 1);
      const int tile = it / tc.nch, ch = it - tile * tc.nch;
      const int4* dp = reinterpret_cast<const int4*>(tc.desc + (size_t)tile * 16);
      const int4 d0 = dp[0], d1 = dp[1], d2 = dp[2];
      const int qi0 = d0.z, nai = d0.w, qo0 = d1.x, nao = flows ? d1.y : 0;
      const int hin0 = d1.z, nhin = d1.w, hout0 = d2.x, nhout = flows ? d2.y : 0, moff = d2.z, mn = d2.w;
      MMF_DASSERT(nhin <= tc.Hin && nhout <= tc.Hout && nai <= tc.MAi && nao <= tc.MAo && mn <= tc.MM);
      if (lane == 0)
        mbar_arrive_expect_tx(&full[s], (unsigned)(nhin + nhout) * (unsigned)SW * 6u + (unsigned)(nai + nao) * 16u +
                                            (unsigned)mn * 4u);
      __syncwarp();
      if (lane == 0 && nai > 0) bulk_g2s(in_rec(s), irec + qi0, (unsigned)nai * 16u, &full[s]);
      if (lane == 1 && nao > 0) bulk_g2s(out_rec(s), orec + qo0, (unsigned)nao * 16u, &full[s]);
      if (lane == 2 && mn > 0) bulk_g2s(meta(s), tc.meta + moff, (unsigned)mn * 4u, &full[s]);
      for (int r = lane; r < nhin; r += 32) {
        const size_t g = (size_t)tc.hin_node[hin0 + r] * p.Lp + (size_t)ch * SW;
        bulk_g2s(in_sig(s) + (size_t)r * SW, am + g, SW * 4, &full[s]);
        bulk_g2s(in_exp(s) + (size_t)r * SW, ae + g, SW * 2, &full[s]);
      }
      for (int r = lane; r < nhout; r += 32) {
        const size_t g = (size_t)tc.hout_node[hout0 + r] * p.Lp + (size_t)ch * SW;
        bulk_g2s(out_sig(s) + (size_t)r * SW, bm + g, SW * 4, &full[s]);
        bulk_g2s(out_exp(s) + (size_t)r * SW, be + g, SW * 2, &full[s]);
      }
    }
    return;
  }

  // ---------------- consumers
  int k = 0;
  for (int it = blockIdx.x; it < tc.nitems; it += gridDim.x, ++k) {
    const int s = k % tc.nst;
    const int tile = it / tc.nch, ch = it - tile * tc.nch;
    const int4 d0 = *reinterpret_cast<const int4*>(tc.desc + (size_t)tile * 16);
    const int4 d3 = *reinterpret_cast<const int4*>(tc.desc + (size_t)tile * 16 + 12);  // (o_outidx, 0, ..)
    const int2 dm = *reinterpret_cast<const int2*>(tc.desc + (size_t)tile * 16 + 12);    // (o_inidx, o_outptr)
    const int v0 = d0.x, nv = d0.y;
    const int o_inidx = dm.x, o_outptr = dm.y, o_outidx = d3.z;
    mbar_wait(&full[s], (k / tc.nst) & 1);
    const float* is = in_sig(s) + lane * CPT;
    const int16_t* ie = in_exp(s) + lane * CPT;
    const float* os = out_sig(s) + lane * CPT;
    const int16_t* oe = out_exp(s) + lane * CPT;
    const ArcKW<float>* ir = in_rec(s);
    const ArcKW<float>* orr = out_rec(s);
    const int* mt = meta(s);
    for (int li = warp; li < nv; li += TB_NWC) {
      const int i = v0 + li;
      const int col = ch * SW + lane * CPT;
      const size_t g = (size_t)i * p.Lp + col;
      // alpha_t[i]: two passes over the in-arcs (rows of alpha_{t-1} in the in-halo)
      const int a0 = mt[li], a1 = mt[li + 1];
      unsigned E2[CPT / 2];
      xmax_init<CPT>(E2);
      for (int q = a0; q < a1; ++q) {
        const float km = ir[q].km;
        if (!(km > 0.f)) continue;
        const unsigned k2 = pack2(ir[q].ke);
        int w[CPT / 2];
        load_exps<CPT>(ie + (size_t)mt[o_inidx + q] * SW, w);
#pragma unroll
        for (int jj = 0; jj < CPT / 2; ++jj) E2[jj] = __viaddmax_s16x2((unsigned)w[jj], k2, E2[jj]);
      }
      XPre<CPT> P;
      P.set(E2);
      float acc[CPT];
#pragma unroll
      for (int c = 0; c < CPT; ++c) acc[c] = 0.f;
      for (int q = a0; q < a1; ++q) {
        const float km = ir[q].km;
        if (!(km > 0.f)) continue;
        const int ke = ir[q].ke;
        const int h = mt[o_inidx + q];
        Row<TrF32, CPT> r;
        r.load(is + (size_t)h * SW, ie + (size_t)h * SW);
        xacc<CPT>(r, __float_as_uint(km), pack2(ke), ke, P, acc);
      }
      Lane<float, int16_t, CPT> a;
      norm_lane<TrF32, CPT, true>(p, acc, P.E, a, col, i);  // (with the layer's node factors: the flows use them)
      a.store(v.am(t) + g, v.ae(t) + g);
      if (!flows) {  // a4: UT = muT ./ alpha_T -> beta_T
        Lane<float, int16_t, CPT> ut;
        boundary_lane<TrF32, CPT>(p, 1, i, col, g, a, ut);
        ut.store(v.bm(p.T) + g, v.be(p.T) + g);
        continue;
      }
      // flow partials of the out-arcs of i over this chunk
      unsigned aw[CPT / 2];
#pragma unroll
      for (int kk = 0; kk < CPT / 2; ++kk) aw[kk] = pack_e2((int)a.e[2 * kk], (int)a.e[2 * kk + 1]);
      const int b0 = mt[o_outptr + li], b1 = mt[o_outptr + li + 1];
      const int qo0 = p.out_ptr[v0];
      // batches of 8 out-arcs: the lane sums of 8 flows reduced together by a transposed butterfly (9 shuffles
      // instead of 8 x 5 dependent ones); uncapacitated arcs (no update) and zero factors contribute 0
      for (int bq = b0; bq < b1; bq += 8) {
        float f[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          f[u] = 0.f;
          const int q = bq + u;
          if (q < b1) {
            const ArcKW<float> rr = orr[q];
            if (rr.aux >= 0 && rr.km > 0.f) {
              const int h = mt[o_outidx + q];
              Row<TrF32, CPT> b;
              b.load(os + (size_t)h * SW, oe + (size_t)h * SW);
              f[u] = flow_terms_f2<CPT>(a.m, aw, b, rr.km, rr.ke);
            }
          }
        }
        const float r = bfly8(f, lane);
        const int q = bq + bfly_row(lane);
        if ((lane & 3) == 0 && q < b1 && orr[q].aux >= 0) tc.part[(size_t)ch * p.A + qo0 + q] = r;
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }
}

// the capacity-dual update of step t from the chunk partials (fixed-order sum), per out-CSR position
__global__ void k_tile_dual(DevPtrs p, const float* __restrict__ part, int nch, int t) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= p.A) return;
  const int a = p.out_arc[q];
  View<TrF32> v(p);
  if (isinf(v.dcap(t)[a])) return;
  float F = 0.f;
  for (int c = 0; c < nch; ++c) F += part[(size_t)c * p.A + q];
  if (!(F == F) || isinf(F)) set_error(p, ERR_NAN, -1, a);
  dual_update<TrF32>(p, t, a, (double)F);
}

}  // namespace mmf
