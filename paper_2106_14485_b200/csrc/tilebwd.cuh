// tilebwd.cuh — node-tile backward step with staged halos (option tbwd = 1, fp32 mode).
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

constexpr int TB_NWC = 16;                     // consumer warps per CTA
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
