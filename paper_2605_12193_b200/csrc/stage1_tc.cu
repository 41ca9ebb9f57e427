// stage1_tc.cu — fast Stage-1 block scores on the tensor cores, certified against the canonical order.
//
// The canonical fp32 chain of DESIGN.md §4 fixes the mask bit for bit.  Tensor cores reach the same
// dot products in a different (undocumented) accumulation order, so their scores S_f differ from the
// canonical S_c by a small amount.  This file computes
//   (1) group norms  ||Phi(Q)[p,i,u]||, ||Phi(K)[h,j,v]||  (max over the groups of each block), and
//   (2) S_f[p,i,j] = max_{u,v} Phi(Q)[p,i,u] . Phi(K)[h,j,v]  with tcgen05 (bf16 x bf16 -> fp32, TMEM
//       accumulator, TMA-fed), Eq. 9-10;
// the selector (stage1_select.cu) then accepts a row's decision only if it is provably the same for
// every score within |S_f - S_c| <= tau * ||x|| ||y|| (Cauchy-Schwarz bounds sum |x_k y_k|), and the
// rows it cannot certify are recomputed here in the canonical order (k_s1_recompute_rows).
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {

constexpr int TM = 128;   // query groups per tile (MMA M)
constexpr int TN = kTcTileN;  // key groups per tile (MMA N = 256)
constexpr int TK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int ST = 4;     // pipeline stages (48 KB each)
constexpr int kBBox = kTcBBox;  // B rows per TMA box (at csz > 2 some cluster CTAs fetch none)
constexpr int ABYTES = TM * TK * 2;
constexpr int BBYTES = TN * TK * 2;
constexpr int SMEM = ST * (ABYTES + BBYTES) + 2 * ST * 8 + 8 + 16 + 1024;  // + barriers, TMEM slot, ticket

// ---- group norms: one CTA per (request, head, block) of Q (first) or K.  All eight warps stream:
// warp w takes group w % G and the (w / G)-th of 8 / G contiguous token slices of it (G <= 8), each lane
// keeps eight 16-byte loads in flight; slices combine through smem, the block keeps the max over its
// groups.  Rounded up by a relative 2^-10 so it bounds the exact norm despite fp32 rounding.  HBM-bound
// (reads Q and K once); it runs on a side stream next to the tensor-core scores.
__global__ void __launch_bounds__(256) k_s1_block_norms(Geom g, const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k, float* __restrict__ qn,
                                                        float* __restrict__ kn, int with_q) {
  __shared__ float part[8];
  const long long u = blockIdx.x + (with_q ? 0 : (long long)g.B * g.Hq * g.Lq);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nq = (long long)g.B * g.Hq * g.Lq;
  const bool isq = u < nq;
  const long long w = isq ? u : u - nq;
  const int L = isq ? g.Lq : g.Lkv, H = isq ? g.Hq : g.Hkv;
  const int blk = (int)(w % L), hh = (int)((w / L) % H), r = (int)(w / ((long long)L * H));
  const Req R = req_of(g, r);
  const int N = isq ? R.Nq : R.Nkv;
  const int vec_per_tok = g.D / 8;  // 16 or 32 (head_dim 128 / 256)
  const int vsh = vec_per_tok == 16 ? 4 : 5;
  const int G = g.G <= 8 ? g.G : 8, parts = 8 / G;
  float acc = 0.f;
  for (int grp = warp % G; grp < g.G; grp += G) {  // G > 8 (not built for FLATTEN) stays correct
    const int t0 = blk * g.b + grp * g.g;
    const int ntok = min(g.g, N - t0);
    if (ntok <= 0) continue;
    const int per = (ntok + parts - 1) / parts;
    const int ta = t0 + (warp / G) * per, tb = min(t0 + ntok, ta + per);
    if (ta >= tb) continue;
    const int nvec = (tb - ta) * vec_per_tok;
    const __nv_bfloat16* base = isq ? q + (long long)r * g.qs0 + (long long)hh * g.qs1
                                    : k + (long long)r * g.kvs0 + (long long)(hh / g.kvdiv) * g.kvs1;
    const long long ts = isq ? g.qs2 : g.kvs2;
    float a8[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) a8[e] = 0.f;
    for (int x0 = lane; x0 < nvec; x0 += 8 * 32) {
      uint4 raw[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const int x = x0 + e * 32;
        raw[e] = make_uint4(0, 0, 0, 0);
        if (x < nvec) {
          const int t = ta + (x >> vsh), c = (x & (vec_per_tok - 1)) * 8;
          raw[e] = __ldg(reinterpret_cast<const uint4*>(base + (long long)t * ts + c));
        }
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const uint32_t w4[4] = {raw[e].x, raw[e].y, raw[e].z, raw[e].w};
#pragma unroll
        for (int f = 0; f < 4; ++f) {
          const float a = __uint_as_float(w4[f] << 16), b2 = __uint_as_float(w4[f] & 0xffff0000u);
          a8[e] = fmaf(a, a, fmaf(b2, b2, a8[e]));
        }
      }
    }
    float s = ((a8[0] + a8[1]) + (a8[2] + a8[3])) + ((a8[4] + a8[5]) + (a8[6] + a8[7]));
#pragma unroll
    for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    acc = fmaxf(acc, s);  // G > 8: several whole groups per warp (parts = 1), max over them
  }
  if (lane == 0) part[warp] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int gi = 0; gi < G; ++gi) {  // group gi's slices sit in warps gi, gi + G, ...
      float s = 0.f;
      for (int pi = 0; pi < parts; ++pi) s += part[gi + pi * G];
      m = fmaxf(m, s);
    }
    (isq ? qn : kn)[w] = sqrtf(m) * (1.0f + 0x1p-10f) + 1e-30f;  // fp32 sum slack
  }
}

// ---- tcgen05 scores: one CTA per (request, query head, M tile of 128 query groups, N tile of 256 key
// groups, K split); causally dead tiles exit.  Warp 0: TMA producer; warp 1: MMA issuer; warp 2: TMEM
// alloc; warps 4-7: epilogue (thread = query group row): max over the G key groups of each KV block in
// registers, max over the G query groups of each query block by shuffles (Eq. 10).
//
// Query-group norms for the certification come out of the same kernel: in the CTAs of
// the first N tile (nt = 0, every query group) the idle epilogue warps read each A stage as it lands
// (thread = its query-group row, 64 bf16 per stage, no extra bytes from L2) and accumulate the sum of
// squares in fp32 (per stage a 64-long FMA chain, then one add: relative error <= gamma_192, far inside
// the 2^-10 slack); they release the stage on its `empty` barrier next to the MMA commit.  Only the K
// norms remain for k_s1_block_norms.
//
// Split-K (splits > 1, few tiles: short prompts and the 1.3-wave grid at 32K): the CTAs of a tile
// take a ticket when their accumulators are ready; all but the last write their raw fp32 partials,
// column-major [col][row], to `part` (query-norm partials to `qpart`) and count themselves done; the
// last waits for them (they hold tickets, so they are resident) and adds the splits in ascending order
// — the same sum whichever CTA finishes last — then runs the max-pool epilogue and resets the tile's
// counters.  The certification bound counts the extra additions (api.cu certify_tau).
__host__ __device__ __forceinline__ bool tc_tile_live(const Geom& g, const Req& R, int mt, int nt, int* nlive) {
  const int BQ = TM / g.G, BK = TN / g.G;  // blocks per tile
  long long e_last = (long long)R.Nc + (long long)((mt + 1) * BQ) * g.b - 1;
  if (e_last > R.Nkv - 1) e_last = R.Nkv - 1;
  if ((long long)nt * BK * g.b > e_last || mt * BQ >= R.Lq) return false;
  *nlive = ((long long)(nt * BK + BK / 2) * g.b > e_last) ? TN / 2 : TN;
  return true;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Epilogue of a score tile (epilogue warps, thread = query-group row of the tile): split-K bookkeeping
// (ticket / partials), query-group norm bounds (qduty) and the G x G max-pool into S.
__device__ __forceinline__ void tc_score_epilogue(const Geom& g, const Req& R, float* __restrict__ S,
                                                  float* __restrict__ qn, int splits, float* __restrict__ part,
                                                  float* __restrict__ qpart, int* __restrict__ tick, int* ticket,
                                                  long long tile, int rp, int p, int r, int mt, int nt, int n_mt,
                                                  int split, int nlive, uint32_t tmem, int lg, int lane, int row,
                                                  float sq, bool qduty) {
  bool last = true;
  if (splits > 1) {
    // tick == nullptr: every split publishes its partials and k_s1_tc_reduce finishes the tile
    if (threadIdx.x == 128) *ticket = tick ? atomicAdd(tick + 2 * tile, 1) : 0;
    epi_bar();
    last = tick && *ticket == splits - 1;
    if (!last) {  // publish the raw partials, count this split done
      if (qduty) qpart[(((long long)rp * n_mt + mt) * splits + split) * TM + row] = sq;
      float* pp = part + (tile * splits + split) * (long long)(TN * TM);
      for (int c0 = 0; c0 < nlive; c0 += 32) {
        float v[32];
        tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + c0, v);
        tmem_wait_ld();
#pragma unroll
        for (int e = 0; e < 32; ++e) __stcg(pp + (c0 + e) * TM + row, v[e]);  // lanes = consecutive rows
      }
      if (tick) {
        __threadfence();
        epi_bar();
        if (threadIdx.x == 128) atomicAdd(tick + 2 * tile + 1, 1);
      }
    } else {  // the others hold tickets: they are resident and finish their stores
      if (threadIdx.x == 128) {
        while (atomicAdd(tick + 2 * tile + 1, 0) < splits - 1) {
        }
        __threadfence();
      }
      epi_bar();
      if (qduty) {
        float a = 0.f;
        for (int sp = 0; sp < splits; ++sp)
          a = __fadd_rn(a, sp == split ? sq : __ldcg(qpart + (((long long)rp * n_mt + mt) * splits + sp) * TM + row));
        sq = a;
      }
    }
  }
  if (last) {
    const int grow = mt * TM + row;  // global query group of head p
    const int ib = grow / g.G, u = grow % g.G;
    if (qduty) {
      // full groups only: a partial group's row holds padding (zero-filled or another request's
      // bytes); its scores come from k_s1_ragged_fixup in the canonical order (exact, no bound needed)
      const bool ufull = (long long)(grow + 1) * g.g <= R.Nq;
      float mx = ufull ? sqrtf(fmaxf(sq, 0.f)) : 0.f;
      for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      if (u == 0 && ib < R.Lq) qn[((long long)r * g.Hq + p) * g.Lq + ib] = mx * (1.0f + 0x1p-10f) + 1e-30f;
    }
    // padding-only groups never take the max (R3); partial groups (ragged N, varlen) are left to the
    // canonical fixup, which rewrites every block score they take part in
    const bool uvalid = (long long)(grow + 1) * g.g <= R.Nq;
    long long e_i = (long long)R.Nc + (long long)(ib + 1) * g.b - 1;
    if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
    float* srow = S + (((long long)r * g.Hq + p) * g.Lq + ib) * g.Lkv;
    const float* pp = part + tile * splits * (long long)(TN * TM) + row;
    for (int c0 = 0; c0 < nlive; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + c0, v);
      tmem_wait_ld();
      if (splits > 1) {  // ascending split order: the same sum whichever split finished last
        float a[32];
#pragma unroll
        for (int e = 0; e < 32; ++e) a[e] = split == 0 ? v[e] : __ldcg(pp + (c0 + e) * TM);
        for (int sp = 1; sp < splits; ++sp) {
          const float* ps = pp + (long long)sp * TN * TM + c0 * TM;
          float b[32];
#pragma unroll
          for (int e = 0; e < 32; ++e) b[e] = sp == split ? v[e] : __ldcg(ps + e * TM);  // 32 loads in flight
#pragma unroll
          for (int e = 0; e < 32; ++e) a[e] = __fadd_rn(a[e], b[e]);
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = a[e];
      }
      for (int jb0 = 0; jb0 < 32; jb0 += g.G) {
        const int gcol = nt * TN + c0 + jb0;  // first key group of this KV block
        float mx = -INFINITY;
        for (int vv = 0; vv < g.G; ++vv)
          if ((long long)(gcol + vv + 1) * g.g <= R.Nkv) mx = fmaxf(mx, v[jb0 + vv]);  // full key groups
        if (!uvalid) mx = -INFINITY;
        for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int jb = gcol / g.G;
        if (u == 0 && ib < R.Lq && jb < R.Lkv && (long long)jb * g.b <= e_i) srow[jb] = mx;
      }
    }
    if (splits > 1 && threadIdx.x == 128) {  // every split has counted itself: reset for the next call
      tick[2 * tile] = 0;
      tick[2 * tile + 1] = 0;
    }
  }
}

__global__ void __launch_bounds__(256, 1) k_s1_tc_scores(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, Geom g,
                                                         float* __restrict__ S, int n_mt, int n_nt,
                                                         float* __restrict__ qn, int splits,
                                                         float* __restrict__ part, float* __restrict__ qpart,
                                                         int* __restrict__ tick, int csz) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * (ABYTES + BBYTES));
  uint64_t* empty = full + ST;
  uint64_t* done = empty + ST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  int* ticket = reinterpret_cast<int*>(tslot + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // grid order: (head group of csz heads of one KV group, mt, nt, split, cluster rank); the csz CTAs of
  // a cluster are the same tile of csz query heads that share the KV head, so they share every B stage
  const int crank = csz > 1 ? (int)cluster_ctarank() : 0;
  int t = blockIdx.x / csz;
  const int split = t % splits;
  t /= splits;
  const int nt = t % n_nt;
  t /= n_nt;
  const int mt = t % n_mt;
  const int rp = (t / n_mt) * csz + crank;  // r * Hq + p
  const long long tile = ((long long)rp * n_mt + mt) * n_nt + nt;
  const int p = rp % g.Hq, r = rp / g.Hq, h = p / g.m;
  const Req R = req_of(g, r);  // this request's logical dims (varlen); g.* is the buffer layout
  // key-group columns with any causal block for this M tile: 256, or 128 when the tile's second half
  // lies entirely past the causal frontier (diagonal tiles); causally dead tiles exit (Eq. 11-13)
  int nlive = TN;
  if (!tc_tile_live(g, R, mt, nt, &nlive)) return;
  const bool qduty = qn != nullptr && nt == 0;  // uniform over the CTA
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, csz + (qduty ? 4 : 0));  // every cluster CTA's MMA commit (+ norm warps)
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TN>(tslot);
  tc_fence_before();
  __syncthreads();
  if (csz > 1) cluster_sync_all();  // peers' barriers initialised before any multicast lands
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nk = g.g * g.D / TK;
  const int k0 = (int)((long long)nk * split / splits), k1 = (int)((long long)nk * (split + 1) / splits);
  if (warp == 0 && lane == 0) {
    for (int kk = k0; kk < k1; ++kk) {
      const int s = (kk - k0) % ST;
      mbar_wait(empty + s, (((kk - k0) / ST) & 1) ^ 1);
      mbar_arrive_expect_tx(full + s, ABYTES + nlive * TK * 2);  // own A + the whole live B
      unsigned char* a = smem + s * (ABYTES + BBYTES);
      tma_load_4d(a, &tmA, full + s, kk * TK, mt * TM, p, r);
      // B in 64-row boxes; with a cluster each CTA fetches every csz-th box once and multicasts it
      for (int q = crank; q < nlive / kBBox; q += csz) {
        if (csz > 1)
          tma_load_4d_mc(a + ABYTES + q * kBBox * 128, &tmB, full + s, kk * TK, nt * TN + q * kBBox, h / g.kvdiv, r,
                         (uint16_t)((1u << csz) - 1u));
        else
          tma_load_4d(a + ABYTES + q * kBBox * 128, &tmB, full + s, kk * TK, nt * TN + q * kBBox, h / g.kvdiv, r);
      }
    }
  } else if (warp == 1) {  // converged warp, one elected lane issues (see umma_f16_ss_warp)
    const uint32_t idesc = nlive == TN ? idesc_bf16(TM, TN, 0, 0) : idesc_bf16(TM, TN / 2, 0, 0);
    const uint64_t d0 = sdesc_sw128(smem_u32(smem), 16, 1024);
    for (int kk = k0; kk < k1; ++kk) {
      const int s = (kk - k0) % ST;
      mbar_wait(full + s, ((kk - k0) / ST) & 1);
      tc_fence_after();
      const uint64_t a = d0 + (uint64_t)((s * (ABYTES + BBYTES)) >> 4), b = a + (uint64_t)(ABYTES >> 4);
#pragma unroll
      for (int k16 = 0; k16 < TK / 16; ++k16)
        umma_f16_ss_warp(tmem, a + (uint64_t)(k16 * 2), b + (uint64_t)(k16 * 2), idesc, (kk > k0 || k16) ? 1u : 0u);
      if (csz > 1) umma_commit_mc_warp(empty + s, (uint16_t)((1u << csz) - 1u));  // B slots are shared
      else umma_commit_warp(empty + s);
    }
    umma_commit_warp(done);
  } else if (warp >= 4) {
    const int lg = warp & 3;
    const int row = lg * 32 + lane;  // query group within the tile
    float sq = 0.f;                  // ||x_row||^2 over this split's k-range (qduty)
    if (qduty) {
      // the row's 128 bytes of each A stage (SWIZZLE_128B permutes its eight 16-byte chunks within the
      // row; a sum of squares does not care).  Chunk (c + lane) & 7: the eight rows of a quarter warp
      // hit eight distinct chunk positions, so every LDS.128 wavefront covers all 32 banks once.
      for (int kk = k0; kk < k1; ++kk) {
        const int s = (kk - k0) % ST;
        mbar_wait(full + s, ((kk - k0) / ST) & 1);
        const uint32_t arow = smem_u32(smem + s * (ABYTES + BBYTES) + row * 128);
        float a8[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t w4[4];
          ld_shared_v4(arow + (((c + lane) & 7) << 4), w4);
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            const float lo = __uint_as_float(w4[f] << 16), hi = __uint_as_float(w4[f] & 0xffff0000u);
            a8[f] = __fmaf_rn(hi, hi, __fmaf_rn(lo, lo, a8[f]));
          }
        }
        const float part_sq = __fadd_rn(__fadd_rn(a8[0], a8[1]), __fadd_rn(a8[2], a8[3]));
        // release the stage to the next TMA fill (async proxy) only after this warp's shared-memory
        // reads are performed: proxy fence, then the arrive (a generic load still in flight when the
        // arrive landed let the next fill race it — the bug of an earlier two-heads variant)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        sq = __fadd_rn(sq, part_sq);
      }
    }
    mbar_wait(done, 0);
    tc_fence_after();
    tc_score_epilogue(g, R, S, qn, splits, part, qpart, tick, ticket, tile, rp, p, r, mt, nt, n_mt, split, nlive,
                      tmem, lg, lane, row, sq, qduty);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TN>(tmem);
  }
  if (csz > 1) cluster_sync_all();  // no CTA leaves while a peer's multicast or commit may target it
}

// ---- CTA-pair variant (cta_group::2): the two query heads of a cluster form ONE M = 256 MMA.  Each CTA
// stages its own 128 A rows and HALF of the B tile (N/2 key groups), so a stage is 32 KB instead of 48 and
// six stages fit (1.5x the bytes in flight per k-step of latency); the leader CTA issues the pair MMAs,
// whose D rows 0-127 land in its TMEM and 128-255 in the peer's; both CTAs' TMA loads signal the
// leader's `full` barrier (the peer's own A rows signal the peer's barrier, so its norm warps can read
// them, and a forwarding warp then arrives on the leader's), the leader's commits release `empty` (and
// `done`) in both CTAs.  Epilogue,
// split-K and the query norms (epilogue warps on each CTA's own A rows) are the single-CTA kernel's.
#ifndef BFLA_S1_PST
#define BFLA_S1_PST 6
#endif
constexpr int PST = BFLA_S1_PST;        // pair stages
constexpr int PBB = (TN / 2) * TK * 2;  // B half per CTA and stage (16 KB)
constexpr int PSTAGE = ABYTES + PBB;    // 32 KB
constexpr int PSMEM = PST * PSTAGE + 2 * PST * 8 + 8 + 16 + 1024;

__global__ void __launch_bounds__(256, 1) k_s1_tc_scores_pair(const __grid_constant__ CUtensorMap tmA,
                                                              const __grid_constant__ CUtensorMap tmB,
                                                              const __grid_constant__ CUtensorMap tmB64, Geom g,
                                                              float* __restrict__ S, int n_mt, int n_nt,
                                                              float* __restrict__ qn, int splits,
                                                              float* __restrict__ part, float* __restrict__ qpart,
                                                              int* __restrict__ tick) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + PST * PSTAGE);
  uint64_t* empty = full + PST;
  uint64_t* done = empty + PST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  int* ticket = reinterpret_cast<int*>(tslot + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int crank = (int)cluster_ctarank();
  const bool leader = crank == 0;
  int t = blockIdx.x / 2;
  const int split = t % splits;
  t /= splits;
  const int nt = t % n_nt;
  t /= n_nt;
  const int mt = t % n_mt;
  const int rp = (t / n_mt) * 2 + crank;  // r * Hq + p
  const long long tile = ((long long)rp * n_mt + mt) * n_nt + nt;
  const int p = rp % g.Hq, r = rp / g.Hq, h = p / g.m;
  const Req R = req_of(g, r);
  int nlive = TN;
  if (!tc_tile_live(g, R, mt, nt, &nlive)) return;  // uniform over the pair (same mt, nt, request)
  const bool qduty = qn != nullptr && nt == 0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < PST; ++s) {
      mbar_init(full + s, leader ? 2 : 1);  // leader: own producer + the peer's forward; peer: own producer
      mbar_init(empty + s, 1 + (qduty ? 4 : 0));  // the leader's pair commit (+ this CTA's norm warps)
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc_pair<TN>(tslot);
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // both CTAs' barriers and TMEM exist before any load or MMA targets them
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nk = g.g * g.D / TK;
  const int k0 = (int)((long long)nk * split / splits), k1 = (int)((long long)nk * (split + 1) / splits);
  const int hb = nlive / 2;  // B rows per CTA
  if (warp == 0 && lane == 0) {
    for (int kk = k0; kk < k1; ++kk) {
      const int s = (kk - k0) % PST;
      mbar_wait(empty + s, (((kk - k0) / PST) & 1) ^ 1);
      // leader: own A + both B halves; peer: its own A (its B half counts at the leader)
      mbar_arrive_expect_tx(full + s, leader ? ABYTES + 2 * hb * TK * 2 : ABYTES);
      unsigned char* a = smem + s * PSTAGE;
      tma_load_4d(a, &tmA, full + s, kk * TK, mt * TM, p, r);
      if (hb == TN / 2)
        tma_load_4d_pair(a + ABYTES, &tmB, full + s, kk * TK, nt * TN + crank * (TN / 2), h / g.kvdiv, r);
      else
        tma_load_4d_pair(a + ABYTES, &tmB64, full + s, kk * TK, nt * TN + crank * (TN / 4), h / g.kvdiv, r);
    }
  } else if (warp == 1 && leader) {
    const uint32_t idesc = idesc_bf16(2 * TM, nlive, 0, 0);
    const uint64_t d0 = sdesc_sw128(smem_u32(smem), 16, 1024);
    for (int kk = k0; kk < k1; ++kk) {
      const int s = (kk - k0) % PST;
      mbar_wait(full + s, ((kk - k0) / PST) & 1);
      tc_fence_after();
      const uint64_t a = d0 + (uint64_t)((s * PSTAGE) >> 4), b = a + (uint64_t)(ABYTES >> 4);
#pragma unroll
      for (int k16 = 0; k16 < TK / 16; ++k16)
        umma_f16_ss_pair_warp(tmem, a + (uint64_t)(k16 * 2), b + (uint64_t)(k16 * 2), idesc,
                              (kk > k0 || k16) ? 1u : 0u);
      umma_commit_pair_warp(empty + s, (uint16_t)3u);
    }
    umma_commit_pair_warp(done, (uint16_t)3u);
  } else if (warp == 3 && !leader) {  // forward "the peer's A rows have landed" to the leader's barrier
    for (int kk = k0; kk < k1; ++kk) {
      const int s = (kk - k0) % PST;
      mbar_wait(full + s, ((kk - k0) / PST) & 1);
      if (lane == 0) mbar_arrive_remote(full + s, 0);
      __syncwarp();
    }
  } else if (warp >= 4) {
    const int lg = warp & 3;
    const int row = lg * 32 + lane;
    float sq = 0.f;
    if (qduty) {
      for (int kk = k0; kk < k1; ++kk) {
        const int s = (kk - k0) % PST;
        mbar_wait(full + s, ((kk - k0) / PST) & 1);
        const uint32_t arow = smem_u32(smem + s * PSTAGE + row * 128);
        float a8[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          uint32_t w4[4];
          ld_shared_v4(arow + (((c + lane) & 7) << 4), w4);
#pragma unroll
          for (int f = 0; f < 4; ++f) {
            const float lo = __uint_as_float(w4[f] << 16), hi = __uint_as_float(w4[f] & 0xffff0000u);
            a8[f] = __fmaf_rn(hi, hi, __fmaf_rn(lo, lo, a8[f]));
          }
        }
        const float part_sq = __fadd_rn(__fadd_rn(a8[0], a8[1]), __fadd_rn(a8[2], a8[3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(empty + s);
        sq = __fadd_rn(sq, part_sq);
      }
    }
    mbar_wait(done, 0);
    tc_fence_after();
    tc_score_epilogue(g, R, S, qn, splits, part, qpart, tick, ticket, tile, rp, p, r, mt, nt, n_mt, split, nlive,
                      tmem, lg, lane, row, sq, qduty);
  }
  tc_fence_before();
  __syncthreads();
  cluster_sync_all();  // the peer's epilogue has read its TMEM; no load or commit still targets either CTA
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc_pair<TN>(tmem);
  }
}

// Split-K finish: TN / kRedCols CTAs (128 threads, thread = query-group row) per tile, one per
// kRedCols-column group; sums the splits in ascending order, then the epilogue of k_s1_tc_scores
// (query-norm partials -> query norms; G x G max).  Loads are column-major partials: a warp reads 128
// contiguous bytes, and every load of the CTA's columns and splits is in flight together.
#ifndef BFLA_RED_COLS
#define BFLA_RED_COLS 16  // A/B (profiles/r3_s1_reduce_cols.txt): 64 -> 16 cols: 32K 0.198 -> 0.194, 16K 0.169 -> 0.132 ms
#endif
#if BFLA_RED_COLS % 16
#error "BFLA_RED_COLS must be a multiple of 16 (the G <= 16 max pyramid)"
#endif
constexpr int kRedCols = BFLA_RED_COLS;  // key-group columns per reduce CTA
__global__ void __launch_bounds__(128) k_s1_tc_reduce(Geom g, float* __restrict__ S, int n_mt, int n_nt,
                                                      float* __restrict__ qn, int splits,
                                                      const float* __restrict__ part,
                                                      const float* __restrict__ qpart) {
  const int cg = blockIdx.x % (TN / kRedCols);
  int t = blockIdx.x / (TN / kRedCols);
  const long long tile = t;
  const int nt = t % n_nt;
  t /= n_nt;
  const int mt = t % n_mt;
  const int rp = t / n_mt;
  const int p = rp % g.Hq, r = rp / g.Hq;
  const Req R = req_of(g, r);
  int nlive;
  if (!tc_tile_live(g, R, mt, nt, &nlive)) return;
  const int row = threadIdx.x;
  const int grow = mt * TM + row;
  const int ib = grow / g.G, u = grow % g.G;
  if (qn != nullptr && nt == 0 && cg == 0) {
    float sq = 0.f;
    for (int sp = 0; sp < splits; ++sp) sq += qpart[(((long long)rp * n_mt + mt) * splits + sp) * TM + row];
    float mx = (long long)(grow + 1) * g.g <= R.Nq ? sqrtf(fmaxf(sq, 0.f)) : 0.f;  // full groups only
    for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (u == 0 && ib < R.Lq) qn[((long long)r * g.Hq + p) * g.Lq + ib] = mx * (1.0f + 0x1p-10f) + 1e-30f;
  }
  const bool uvalid = (long long)(grow + 1) * g.g <= R.Nq;  // full groups (partial: k_s1_ragged_fixup)
  long long e_i = (long long)R.Nc + (long long)(ib + 1) * g.b - 1;
  if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
  float* srow = S + (((long long)r * g.Hq + p) * g.Lq + ib) * g.Lkv;
  const float* pp = part + tile * splits * (long long)(TN * TM) + row;
  const int c0 = cg * kRedCols;
  if (c0 >= nlive) return;
  // all kRedCols columns of every split in flight at once (fully unrolled, static register indexing)
  float a[kRedCols];
#pragma unroll
  for (int c = 0; c < kRedCols; ++c) a[c] = __ldg(pp + (long long)(c0 + c) * TM);
  for (int sp = 1; sp < splits; ++sp) {  // ascending split order
    float b[kRedCols];
#pragma unroll
    for (int c = 0; c < kRedCols; ++c) b[c] = __ldg(pp + ((long long)sp * TN + c0 + c) * TM);
#pragma unroll
    for (int c = 0; c < kRedCols; ++c) a[c] += b[c];
  }
#pragma unroll
  for (int c = 0; c < kRedCols; ++c)  // full, live key groups only
    if (c0 + c >= nlive || (long long)(nt * TN + c0 + c + 1) * g.g > R.Nkv) a[c] = -INFINITY;
  // max over each block's G key groups: a pyramid of pairwise maxima, read at the level of G
  float m2[kRedCols / 2], m4[kRedCols / 4], m8[kRedCols / 8], m16[kRedCols / 16];
#pragma unroll
  for (int c = 0; c < kRedCols / 2; ++c) m2[c] = fmaxf(a[2 * c], a[2 * c + 1]);
#pragma unroll
  for (int c = 0; c < kRedCols / 4; ++c) m4[c] = fmaxf(m2[2 * c], m2[2 * c + 1]);
#pragma unroll
  for (int c = 0; c < kRedCols / 8; ++c) m8[c] = fmaxf(m4[2 * c], m4[2 * c + 1]);
#pragma unroll
  for (int c = 0; c < kRedCols / 16; ++c) m16[c] = fmaxf(m8[2 * c], m8[2 * c + 1]);
#pragma unroll
  for (int k = 0; k < kRedCols; ++k) {
    if (k >= kRedCols / g.G) break;  // G uniform over the grid
    float mx = g.G == 1 ? a[k] : g.G == 2 ? m2[k % (kRedCols / 2)] : g.G == 4 ? m4[k % (kRedCols / 4)]
             : g.G == 8 ? m8[k % (kRedCols / 8)] : m16[k % (kRedCols / 16)];
    if (!uvalid) mx = -INFINITY;
    for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const int jb = (nt * TN + c0) / g.G + k;
    if (u == 0 && ib < R.Lq && jb < R.Lkv && (long long)jb * g.b <= e_i) srow[jb] = mx;
  }
}

// ---- canonical recompute of flagged head rows (DESIGN.md §4 item 2 order).  Work unit = (flagged head
// row (r,p,i), KV block j) for every causal j whose score can still carry canonical probability
// (S_f inside the row's band, listed by k_s1_select: MASS — below it 2^t underflows to an exact 0
// whatever the rounding; RATIO — outside it the rank against the canonical k-th score is certain).  The unit's G x G
// group dots are G*G*g independent token-pair chains (C-long fp32 FMA chains, channel ascending): a
// thread runs four of them side by side straight from global memory (16-byte loads, L1/L2-resident
// rows), the token dots land in smem, and G*G threads add them in ascending token order — the
// oracle's order exactly.  Units are short (one C-long chain plus a g-long sum), so the flagged set
// spreads over every SM and finishes in a few microseconds.
constexpr int kRecThreads = 256;

__device__ __forceinline__ void bf16x8_f32(const uint4& u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
  }
}

// Canonical S[r, p, i, j] by one CTA (all threads call it): the block pair's G x G group dots as
// G*G*g token-pair chains (C-long fp32 FMA chains, channel ascending), four per thread side by side
// straight from global memory (16-byte loads, L1/L2-resident rows); the token dots land in smem and
// G*G threads add them in ascending token order — the oracle's order exactly; Eq. 10 max over pairs.
// tokdot: [G*G*g + G*G] floats of shared memory.
template <int D>
__device__ void canon_block_score(const Geom& g, const Req& R, const __nv_bfloat16* __restrict__ q,
                                  const __nv_bfloat16* __restrict__ k, int r, int p, int i, int j,
                                  float* tokdot, float* __restrict__ S) {
  const int G = g.G, gg = g.g, nch = G * G * gg;
  const int h = p / g.m;
  float* srow = S + (((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv;
  const __nv_bfloat16* qb = q + (long long)r * g.qs0 + (long long)p * g.qs1;
  const __nv_bfloat16* kb = k + (long long)r * g.kvs0 + (long long)(h / g.kvdiv) * g.kvs1;
  // chains c = (u, v, t), t fastest: four per thread per pass
  for (int c0 = threadIdx.x * 4; c0 < nch; c0 += kRecThreads * 4) {
    const __nv_bfloat16* xs[4];
    const __nv_bfloat16* ys[4];
    bool ok[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int c = c0 + e;
      const int t = c % gg, uv = c / gg, u = uv / G, v = uv % G;
      const int tq = i * g.b + u * gg + t, tk = j * g.b + v * gg + t;
      ok[e] = c < nch && tq < R.Nq && tk < R.Nkv;  // padding tokens are exact zeros: dot 0
      xs[e] = qb + (long long)(ok[e] ? tq : 0) * g.qs2;
      ys[e] = kb + (long long)(ok[e] ? tk : 0) * g.kvs2;
    }
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 2
    for (int cc = 0; cc < D; cc += 8) {
      float xf[4][8], yf[4][8];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        bf16x8_f32(__ldg(reinterpret_cast<const uint4*>(xs[e] + cc)), xf[e]);
        bf16x8_f32(__ldg(reinterpret_cast<const uint4*>(ys[e] + cc)), yf[e]);
      }
#pragma unroll
      for (int x = 0; x < 8; ++x)
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = __fmaf_rn(xf[e][x], yf[e][x], acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (c0 + e < nch) tokdot[c0 + e] = ok[e] ? acc[e] : 0.0f;
  }
  __syncthreads();
  float* pairtot = tokdot + nch;
  if (threadIdx.x < G * G) {
    // thread (u, v): the g token dots added in ascending t (the oracle's order)
    const int uv = threadIdx.x, u = uv / G, v = uv % G;
    float a = 0.0f;
    for (int t = 0; t < gg; ++t) a = __fadd_rn(a, tokdot[uv * gg + t]);
    const bool valid = i * g.b + u * gg < R.Nq && j * g.b + v * gg < R.Nkv;  // padding-only groups (R3)
    pairtot[uv] = valid ? a : -INFINITY;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float mx = -INFINITY;  // Eq. 10: max over the group pairs (exact, order-free)
    for (int uv = 0; uv < G * G; ++uv) mx = fmaxf(mx, pairtot[uv]);
    srow[j] = mx;
  }
  __syncthreads();  // tokdot is reused by the caller's next unit
}

template <int D>
__global__ void __launch_bounds__(kRecThreads) k_s1_recompute_rows(Geom g, const __nv_bfloat16* __restrict__ q,
                                                                   const __nv_bfloat16* __restrict__ k,
                                                                   const int32_t* __restrict__ flagged,
                                                                   const int32_t* __restrict__ n_flagged,
                                                                   const int32_t* __restrict__ ulist,
                                                                   const int32_t* __restrict__ n_units,
                                                                   float* __restrict__ S) {
  extern __shared__ float tokdot[];  // [G*G][g] token dots of the current unit
  (void)n_flagged;
  const int nunits = *n_units;
  for (int uidx = blockIdx.x; uidx < nunits; uidx += gridDim.x) {
    const int unit = ulist[uidx];  // fidx * Lkv + j (k_s1_select: the row's recompute band)
    const int j = unit % g.Lkv;
    const int fidx = unit / g.Lkv;
    const int row = flagged[fidx];  // (r * Hq + p) * Lq + i
    const int i = row % g.Lq, p = (row / g.Lq) % g.Hq, r = row / (g.Lq * g.Hq);
    const Req R = req_of(g, r);
    long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
    if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
    if ((long long)j * g.b > e_i || j >= R.Lkv) continue;  // non-causal (uniform over the CTA)
    canon_block_score<D>(g, R, q, k, r, p, i, j, tokdot, S);
  }
}

// Ragged tails and varlen requests on the tensor-core path (§8 f1): the scores kernel max-pools full
// groups only (a partial group's TMA row would read padding), so every block pair a partial group
// takes part in — row i = L_q,r - 1 when n_q,r mod g != 0, column j = L_kv,r - 1 when n_kv,r mod g != 0 —
// is finished here: the group pairs that involve a partial group, (u_p, v) and (u, v_p), are computed
// in the canonical order (token chains of C fp32 FMAs, token dots added in ascending t) and max-ed into
// the tensor-core score of the full pairs.  Those pairs are exact, so |S_f - S_c| <= tau ||x|| ||y|| (norms
// over the full groups) still bounds the block score: the certification stays a proof.  CTA per
// (r, h, unit) over the m query heads of mask group h (so a KV block is read from L2 once and re-read
// from L1 by the other heads): units [0, L_kv) walk the partial row, [L_kv, L_kv + L_q) the partial column.
template <int D, bool STAGE>
__global__ void __launch_bounds__(kRecThreads) k_s1_ragged_fixup(Geom g, const __nv_bfloat16* __restrict__ q,
                                                                 const __nv_bfloat16* __restrict__ k,
                                                                 float* __restrict__ S) {
  constexpr int PITCH = D * 2 + 16;  // staged key row (bytes), padded: lanes (consecutive tokens) hit distinct banks
  extern __shared__ __align__(16) unsigned char fx[];  // [b][PITCH] key block, then token dots + pair totals
  // (STAGE = false, blocks too large for smem: keys are read from global memory / L1 instead)
  float* tokdot = reinterpret_cast<float*>(fx + (STAGE ? (size_t)g.b * PITCH : 0));  // [2G - 1][g], then [2G - 1]
  const int per = g.Lkv + g.Lq;
  // grid-stride over every (r, h, unit): most units of a varlen batch are dead (no partial group, not
  // causal) and skipping them in a loop costs far less than launching a CTA for each
  const long long total = (long long)g.B * g.Hkv * per;
  for (long long unit = blockIdx.x; unit < total; unit += gridDim.x) {
  const int idx = (int)(unit % per), rh = (int)(unit / per);
  const int h = rh % g.Hkv, r = rh / g.Hkv;
  const Req R = req_of(g, r);
  const bool qrag = R.Nq % g.g != 0, krag = R.Nkv % g.g != 0;
  int i, j;
  if (idx < g.Lkv) {
    if (!qrag) continue;
    i = R.Lq - 1;
    j = idx;
  } else {
    if (!krag) continue;
    i = idx - g.Lkv;
    j = R.Lkv - 1;
    if (qrag && i == R.Lq - 1) continue;  // the row units cover it
  }
  if (i >= R.Lq || j >= R.Lkv) continue;
  long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
  if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
  if ((long long)j * g.b > e_i) continue;  // Eq. 11-13: not causal
  const int G = g.G, gg = g.g;
  // partial groups of this unit: u_p = full groups before the tail of the last query block (-1: none)
  const int up = (qrag && i == R.Lq - 1) ? (R.Nq - i * g.b) / gg : -1;
  const int vp = (krag && j == R.Lkv - 1) ? (R.Nkv - j * g.b) / gg : -1;
  const int nrow = up >= 0 ? G : 0;                 // pairs (u_p, v), v = 0..G-1
  const int npair = nrow + (vp >= 0 ? (up >= 0 ? G - 1 : G) : 0);  // + pairs (u, v_p), u != u_p
  auto pair_uv = [&](int pi, int& u, int& v) {
    if (pi < nrow) {
      u = up;
      v = pi;
    } else {
      const int kx = pi - nrow;
      u = (up >= 0 && kx >= up) ? kx + 1 : kx;
      v = vp;
    }
  };
  const __nv_bfloat16* kb = k + (long long)r * g.kvs0 + (long long)(h / g.kvdiv) * g.kvs1;
  // the unit's key block, staged once with coalesced 16-byte copies (shared by every chain and head)
  const int kt0 = j * g.b, nkt = min(g.b, R.Nkv - kt0);
  for (int x = threadIdx.x; STAGE && x < nkt * (D / 8); x += kRecThreads) {
    const int tr = x / (D / 8), c8 = x % (D / 8);
    *reinterpret_cast<uint4*>(fx + (size_t)tr * PITCH + c8 * 16) =
        __ldg(reinterpret_cast<const uint4*>(kb + (long long)(kt0 + tr) * g.kvs2) + c8);
  }
  __syncthreads();
  for (int p = h * g.m; p < (h + 1) * g.m; ++p) {
  const __nv_bfloat16* qb = q + (long long)r * g.qs0 + (long long)p * g.qs1;
  for (int c = threadIdx.x; c < npair * gg; c += kRecThreads) {  // chain (pair, t), t fastest
    int u, v;
    pair_uv(c / gg, u, v);
    const int t = c % gg;
    const int tq = i * g.b + u * gg + t, tk = j * g.b + v * gg + t;
    float acc = 0.f;
    if (tq < R.Nq && tk < R.Nkv) {  // padding tokens are exact zeros: dot 0
      const __nv_bfloat16* x = qb + (long long)tq * g.qs2;
      const unsigned char* y = fx + (size_t)(tk - kt0) * PITCH;
      const __nv_bfloat16* yg = kb + (long long)tk * g.kvs2;
#pragma unroll 4
      for (int cc = 0; cc < D; cc += 8) {
        float xf[8], yf[8];
        bf16x8_f32(__ldg(reinterpret_cast<const uint4*>(x + cc)), xf);
        bf16x8_f32(STAGE ? *reinterpret_cast<const uint4*>(y + cc * 2) : __ldg(reinterpret_cast<const uint4*>(yg + cc)), yf);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = __fmaf_rn(xf[e], yf[e], acc);
      }
    }
    tokdot[c] = acc;
  }
  __syncthreads();
  float* pairtot = tokdot + npair * gg;
  for (int pi = threadIdx.x; pi < npair; pi += kRecThreads) {
    int u, v;
    pair_uv(pi, u, v);
    float a = 0.0f;
    for (int t = 0; t < gg; ++t) a = __fadd_rn(a, tokdot[pi * gg + t]);  // ascending t (§4 item 2)
    const bool valid = i * g.b + u * gg < R.Nq && j * g.b + v * gg < R.Nkv;  // padding-only groups (R3)
    pairtot[pi] = valid ? a : -INFINITY;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float* s = S + (((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j;
    float mx = *s;  // the tensor-core max over the full pairs (-inf if there are none)
    for (int pi = 0; pi < npair; ++pi) mx = fmaxf(mx, pairtot[pi]);  // Eq. 10
    *s = mx;
  }
  __syncthreads();  // tokdot / pairtot reused by the next query head (and the key block by the next unit)
  }
  }
}

// Same units and the same arithmetic order, operands staged in shared memory: the unit's K block and
// its query groups (double-buffered, one group per phase) arrive by bulk copies (one per token row,
// rows padded by 16 bytes so the 32 lanes of a warp — consecutive tokens — read distinct banks);
// thread = token-pair chain (v, t) of the current query group u.  Used when the block fits in smem.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

template <int D>
__global__ void __launch_bounds__(kRecThreads) k_s1_recompute_smem(Geom g, const __nv_bfloat16* __restrict__ q,
                                                                   const __nv_bfloat16* __restrict__ k,
                                                                   const int32_t* __restrict__ flagged,
                                                                   const int32_t* __restrict__ n_flagged,
                                                                   const int32_t* __restrict__ ulist,
                                                                   const int32_t* __restrict__ n_units,
                                                                   float* __restrict__ S) {
  constexpr int PITCH = D * 2 + 16;  // bytes per staged token row
  extern __shared__ __align__(16) unsigned char rs[];
  const int G = g.G, gg = g.g, b = g.b;
  unsigned char* kb_s = rs;                                  // [b][PITCH]
  unsigned char* qg_s = rs + (size_t)b * PITCH;              // [2][g][PITCH]
  float* tokdot = reinterpret_cast<float*>(qg_s + (size_t)2 * gg * PITCH);  // [G*G][g]
  float* pairtot = tokdot + G * G * gg;                      // [G*G]
  __shared__ __align__(8) uint64_t bar[3];                   // K block, query group buffers 0 / 1
  if (threadIdx.x == 0) {
    for (int e = 0; e < 3; ++e) mbar_init(bar + e, 1);
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t ph[3] = {0, 0, 0};
  (void)n_flagged;
  const int nunits = *n_units;
  for (int uidx = blockIdx.x; uidx < nunits; uidx += gridDim.x) {
    const int unit = ulist[uidx];  // fidx * Lkv + j (k_s1_select: the row's recompute band)
    const int j = unit % g.Lkv;
    const int fidx = unit / g.Lkv;
    const int row = flagged[fidx];  // (r * Hq + p) * Lq + i
    const int i = row % g.Lq, p = (row / g.Lq) % g.Hq, r = row / (g.Lq * g.Hq);
    const int h = p / g.m;
    const Req R = req_of(g, r);
    long long e_i = (long long)R.Nc + (long long)(i + 1) * b - 1;
    if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
    if ((long long)j * b > e_i || j >= R.Lkv) continue;  // non-causal (uniform over the CTA)
    float* srow = S + (((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv;
    const __nv_bfloat16* qb = q + (long long)r * g.qs0 + (long long)p * g.qs1;
    const __nv_bfloat16* kb = k + (long long)r * g.kvs0 + (long long)(h / g.kvdiv) * g.kvs1;
    const int kt0 = j * b, nkt = min(b, R.Nkv - kt0);  // valid key tokens of the block
    auto stage_q = [&](int u, int buf) {  // warp 0: query group u -> buffer buf
      const int qt0 = i * b + u * gg, nqt = max(0, min(gg, R.Nq - qt0));
      if (threadIdx.x == 0) mbar_arrive_expect_tx(bar + 1 + buf, (uint32_t)(nqt * D * 2));
      __syncwarp();
      for (int t = threadIdx.x; t < nqt; t += 32)
        bulk_g2s(qg_s + ((size_t)buf * gg + t) * PITCH, qb + (long long)(qt0 + t) * g.qs2, D * 2, bar + 1 + buf);
    };
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, (uint32_t)(nkt * D * 2));
      __syncwarp();
      for (int t = threadIdx.x; t < nkt; t += 32)
        bulk_g2s(kb_s + (size_t)t * PITCH, kb + (long long)(kt0 + t) * g.kvs2, D * 2, bar);
      stage_q(0, 0);
    }
    mbar_wait(bar, ph[0]);
    ph[0] ^= 1;
    for (int u = 0; u < G; ++u) {
      const int buf = u & 1;
      if (u + 1 < G && threadIdx.x < 32) stage_q(u + 1, buf ^ 1);  // buffer buf^1 was released at u-1
      mbar_wait(bar + 1 + buf, ph[1 + buf]);
      ph[1 + buf] ^= 1;
      const int qt0 = i * b + u * gg;
      for (int c = threadIdx.x; c < G * gg; c += kRecThreads) {  // chain (v, t), t fastest
        const int t = c % gg, v = c / gg;
        const bool ok = qt0 + t < R.Nq && v * gg + t < nkt;  // padding tokens: exact zero dot
        float acc = 0.f;
        if (ok) {
          const unsigned char* xr = qg_s + ((size_t)buf * gg + t) * PITCH;
          const unsigned char* yr = kb_s + (size_t)(v * gg + t) * PITCH;
#pragma unroll 4
          for (int cc = 0; cc < D; cc += 8) {
            float xf[8], yf[8];
            bf16x8_f32(*reinterpret_cast<const uint4*>(xr + cc * 2), xf);
            bf16x8_f32(*reinterpret_cast<const uint4*>(yr + cc * 2), yf);
#pragma unroll
            for (int e = 0; e < 8; ++e) acc = __fmaf_rn(xf[e], yf[e], acc);
          }
        }
        tokdot[(u * G + v) * gg + t] = acc;
      }
      __syncthreads();  // query buffer buf is free again; after the last u tokdot is complete
    }
    if (threadIdx.x < G * G) {
      const int uv = threadIdx.x, u = uv / G, v = uv % G;
      float a = 0.0f;
      for (int t = 0; t < gg; ++t) a = __fadd_rn(a, tokdot[uv * gg + t]);  // ascending t
      const bool valid = i * b + u * gg < R.Nq && j * b + v * gg < R.Nkv;  // padding-only groups (R3)
      pairtot[uv] = valid ? a : -INFINITY;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mx = -INFINITY;  // Eq. 10
      for (int uv = 0; uv < G * G; ++uv) mx = fmaxf(mx, pairtot[uv]);
      srow[j] = mx;
    }
    __syncthreads();  // smem reused by the next unit
  }
}

// TMA-staged variant (head_dim 128): each CTA walks a contiguous range of units (flagged row, KV
// block), so consecutive units share the row's query block, which is loaded once; the KV blocks are
// double-buffered (the next live unit's block loads while the current one is computed).  Blocks arrive
// as 64-token x 64-column SW128 boxes through the same kind of tensor maps as the attention, so a
// warp's lanes — consecutive tokens — read distinct banks.  Thread = (query group u, token t); it
// runs the G chains (u, v, t), v = 0..G-1, side by side (the query token is shared).
template <int D>
__global__ void __launch_bounds__(kRecThreads) k_s1_recompute_tma(const __grid_constant__ CUtensorMap tmQ,
                                                                  const __grid_constant__ CUtensorMap tmK, Geom g,
                                                                  const int32_t* __restrict__ flagged,
                                                                  const int32_t* __restrict__ n_flagged,
                                                                  const int32_t* __restrict__ ulist,
                                                                  const int32_t* __restrict__ n_units,
                                                                  float* __restrict__ S) {
  constexpr int NCH = D / 64;  // 64-column chunks per token row
  extern __shared__ __align__(1024) unsigned char rs_raw[];
  unsigned char* rs = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(rs_raw) + 1023) & ~uintptr_t(1023));
  const int G = g.G, gg = g.g, b = g.b, nrt = b / 64;  // 64-token row tiles per block
  const int blk_bytes = b * D * 2;
  unsigned char* qs = rs;                                      // query block
  unsigned char* ks[2] = {rs + blk_bytes, rs + 2 * blk_bytes};  // KV blocks (double buffer)
  float* tokdot = reinterpret_cast<float*>(rs + 3 * blk_bytes);  // [G*G][g]
  float* pairtot = tokdot + G * G * gg;
  __shared__ __align__(8) uint64_t bar[3];  // query block, KV buffers 0 / 1
  if (threadIdx.x == 0) {
    for (int e = 0; e < 3; ++e) mbar_init(bar + e, 1);
    fence_barrier_init();
  }
  __syncthreads();
  // the units (flagged row, KV block) of every row's recompute band, listed row by row by k_s1_select:
  // an even contiguous share per CTA, no scanning of dead units
  const long long units = *n_units;
  const long long per = (units + gridDim.x - 1) / gridDim.x;
  const long long u0 = (long long)blockIdx.x * per, u1 = min(units, u0 + per);
  auto next_live = [&](long long from) -> long long { return from; };
  auto load_block = [&](unsigned char* dst, const CUtensorMap* map, uint64_t* br, int t0, int hh, int r) {
    mbar_arrive_expect_tx(br, (uint32_t)blk_bytes);
    for (int rt = 0; rt < nrt; ++rt)
      for (int cc = 0; cc < NCH; ++cc)
        tma_load_4d(dst + (rt * NCH + cc) * 8192, map, br, cc * 64, t0 + rt * 64, hh, r);
  };
  auto decode = [&](long long uidx, int& j, int& i, int& p, int& r, int& fidx) {
    const int unit = ulist[uidx];
    j = unit % g.Lkv;
    fidx = unit / g.Lkv;
    const int row = flagged[fidx];
    i = row % g.Lq;
    p = (row / g.Lq) % g.Hq;
    r = row / (g.Lq * g.Hq);
  };
  uint32_t qph = 0, kph[2] = {0, 0};
  long long cu = next_live(u0);
  int buf = 0, qrow = -1;
  if (cu < u1 && threadIdx.x == 0) {
    int j, i, p, r, f;
    decode(cu, j, i, p, r, f);
    load_block(qs, &tmQ, bar, i * b, p, r);
    load_block(ks[0], &tmK, bar + 1, j * b, p / g.m / g.kvdiv, r);
  }
  while (cu < u1) {
    int j, i, p, r, fidx;
    decode(cu, j, i, p, r, fidx);
    const long long nu = next_live(cu + 1);
    int nj = 0, ni = 0, np = 0, nr = 0, nfi = 0;
    if (nu < u1) decode(nu, nj, ni, np, nr, nfi);
    const bool new_q = nu < u1 && (ni != i || np != p || nr != r);
    if (nu < u1 && threadIdx.x == 0) load_block(ks[buf ^ 1], &tmK, bar + 1 + (buf ^ 1), nj * b, np / g.m / g.kvdiv, nr);
    if (qrow != fidx) {  // this unit's query block (loaded at the previous unit's end, or first)
      mbar_wait(bar, qph);
      qph ^= 1;
      qrow = fidx;
    }
    mbar_wait(bar + 1 + buf, kph[buf]);
    kph[buf] ^= 1;
    const Req R = req_of(g, r);
    const int kt0 = j * b;
    const unsigned char* kbuf = ks[buf];
    auto elem16 = [&](const unsigned char* base, int tok, int cc, int k16) -> uint4 {
      const int rt = tok >> 6, row = tok & 63;
      return *reinterpret_cast<const uint4*>(base + (rt * NCH + cc) * 8192 + row * 128 + ((k16 ^ (row & 7)) << 4));
    };
    for (int idx = threadIdx.x; idx < G * gg; idx += kRecThreads) {
      const int t = idx % gg, u = idx / gg;
      const int qtok = u * gg + t;
      float acc[16];  // G <= 16 chains side by side
#pragma unroll
      for (int v = 0; v < 16; ++v) acc[v] = 0.f;
      const bool qok = i * b + qtok < R.Nq;
      if (qok) {
        for (int cc = 0; cc < NCH; ++cc) {
#pragma unroll 2
          for (int k16 = 0; k16 < 8; ++k16) {
            float xf[8];
            bf16x8_f32(elem16(qs, qtok, cc, k16), xf);
#pragma unroll
            for (int v = 0; v < 16; ++v) {
              if (v >= G) break;
              float yf[8];
              bf16x8_f32(elem16(kbuf, v * gg + t, cc, k16), yf);
#pragma unroll
              for (int e = 0; e < 8; ++e) acc[v] = __fmaf_rn(xf[e], yf[e], acc[v]);
            }
          }
        }
      }
      for (int v = 0; v < G; ++v) {
        const bool ok = qok && kt0 + v * gg + t < R.Nkv;  // padding tokens: exact zero dot
        tokdot[(u * G + v) * gg + t] = ok ? acc[v] : 0.0f;
      }
    }
    __syncthreads();  // tokdot complete; buffer buf and the query block are free again
    if (new_q && threadIdx.x == 0) load_block(qs, &tmQ, bar, ni * b, np, nr);
    if (threadIdx.x < G * G) {
      const int uv = threadIdx.x, u = uv / G, v = uv % G;
      float a = 0.0f;
      for (int t = 0; t < gg; ++t) a = __fadd_rn(a, tokdot[uv * gg + t]);  // ascending t
      const bool valid = i * b + u * gg < R.Nq && j * b + v * gg < R.Nkv;  // padding-only groups (R3)
      pairtot[uv] = valid ? a : -INFINITY;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      float mx = -INFINITY;  // Eq. 10
      for (int uv = 0; uv < G * G; ++uv) mx = fmaxf(mx, pairtot[uv]);
      S[(((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j] = mx;
    }
    __syncthreads();  // tokdot / pairtot reused by the next unit
    buf ^= 1;
    cu = nu;
  }
}

// D = 256 variant of k_s1_recompute_tma: the row's query block (b x 256 bf16, 128 KB at b = 256) stays
// resident as before, but K arrives one 64-column chunk per stage (double-buffered, 32 KB at b = 256),
// so a unit takes D/64 stages and each thread's G chains carry their accumulators across them — the
// channel order of every chain is unchanged (chunk ascending, then k16, then element).  Thread =
// (query group u, token t); needs G*g <= the block size.
template <int D>
__global__ void __launch_bounds__(kRecThreads) k_s1_recompute_tma_kc(const __grid_constant__ CUtensorMap tmQ,
                                                                     const __grid_constant__ CUtensorMap tmK, Geom g,
                                                                     const int32_t* __restrict__ flagged,
                                                                     const int32_t* __restrict__ n_flagged,
                                                                     const int32_t* __restrict__ ulist,
                                                                     const int32_t* __restrict__ n_units,
                                                                     float* __restrict__ S) {
  constexpr int NCH = D / 64;
  (void)n_flagged;
  extern __shared__ __align__(1024) unsigned char rk_raw[];
  unsigned char* rs = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(rk_raw) + 1023) & ~uintptr_t(1023));
  const int G = g.G, gg = g.g, b = g.b, nrt = b / 64;
  unsigned char* qs = rs;                                              // query block, all chunks
  unsigned char* kb[2] = {rs + b * D * 2, rs + b * D * 2 + b * 128};  // one K chunk per buffer
  float* tokdot = reinterpret_cast<float*>(rs + b * D * 2 + 2 * b * 128);
  float* pairtot = tokdot + G * G * gg;
  __shared__ __align__(8) uint64_t bar[3];
  if (threadIdx.x == 0) {
    for (int e = 0; e < 3; ++e) mbar_init(bar + e, 1);
    fence_barrier_init();
  }
  __syncthreads();
  const long long units = *n_units;
  const long long per = (units + gridDim.x - 1) / gridDim.x;
  const long long u0 = (long long)blockIdx.x * per, u1 = min(units, u0 + per);
  auto decode = [&](long long uidx, int& j, int& i, int& p, int& r, int& fidx) {
    const int unit = ulist[uidx];
    j = unit % g.Lkv;
    fidx = unit / g.Lkv;
    const int row = flagged[fidx];
    i = row % g.Lq;
    p = (row / g.Lq) % g.Hq;
    r = row / (g.Lq * g.Hq);
  };
  auto load_q = [&](int t0, int p, int r) {
    mbar_arrive_expect_tx(bar, (uint32_t)(b * D * 2));
    for (int rt = 0; rt < nrt; ++rt)
      for (int cc = 0; cc < NCH; ++cc) tma_load_4d(qs + (rt * NCH + cc) * 8192, &tmQ, bar, cc * 64, t0 + rt * 64, p, r);
  };
  auto load_kc = [&](int bi, int t0, int hh, int r, int cc) {
    mbar_arrive_expect_tx(bar + 1 + bi, (uint32_t)(b * 128));
    for (int rt = 0; rt < nrt; ++rt) tma_load_4d(kb[bi] + rt * 8192, &tmK, bar + 1 + bi, cc * 64, t0 + rt * 64, hh, r);
  };
  const long long s0 = u0 * NCH, s1 = u1 * NCH;
  if (s0 < s1 && threadIdx.x == 0) {
    int j, i, p, r, f;
    decode(u0, j, i, p, r, f);
    load_q(i * b, p, r);
    load_kc(0, j * b, p / g.m / g.kvdiv, r, 0);
  }
  uint32_t qph = 0, kph[2] = {0, 0};
  int buf = 0, qrow = -1;
  const int idx = threadIdx.x;
  const bool act = idx < G * gg;
  const int t = act ? idx % gg : 0, u = act ? idx / gg : 0;
  float acc[16];  // G <= 16
  for (long long sg = s0; sg < s1; ++sg) {
    const long long uidx = sg / NCH;
    const int cc = (int)(sg % NCH);
    int j, i, p, r, fidx;
    decode(uidx, j, i, p, r, fidx);
    bool new_q = false;
    int ni = 0, np = 0, nr = 0;
    if (sg + 1 < s1) {
      int nj, nfi;
      decode((sg + 1) / NCH, nj, ni, np, nr, nfi);
      new_q = cc == NCH - 1 && nfi != fidx;
      if (threadIdx.x == 0) load_kc(buf ^ 1, nj * b, np / g.m / g.kvdiv, nr, (int)((sg + 1) % NCH));
    }
    if (qrow != fidx) {
      mbar_wait(bar, qph);
      qph ^= 1;
      qrow = fidx;
    }
    mbar_wait(bar + 1 + buf, kph[buf]);
    kph[buf] ^= 1;
    const Req R = req_of(g, r);
    const int qtok = u * gg + t;
    const bool qok = act && i * b + qtok < R.Nq;
    if (cc == 0) {
#pragma unroll
      for (int v = 0; v < 16; ++v) acc[v] = 0.f;
    }
    if (qok) {
      const unsigned char* kbuf = kb[buf];
#pragma unroll 2
      for (int k16 = 0; k16 < 8; ++k16) {
        float xf[8];
        {
          const int rt = qtok >> 6, row = qtok & 63;
          bf16x8_f32(*reinterpret_cast<const uint4*>(qs + (rt * NCH + cc) * 8192 + row * 128 + ((k16 ^ (row & 7)) << 4)),
                     xf);
        }
#pragma unroll
        for (int v = 0; v < 16; ++v) {
          if (v >= G) break;
          const int ktok = v * gg + t, rt = ktok >> 6, row = ktok & 63;
          float yf[8];
          bf16x8_f32(*reinterpret_cast<const uint4*>(kbuf + rt * 8192 + row * 128 + ((k16 ^ (row & 7)) << 4)), yf);
#pragma unroll
          for (int e = 0; e < 8; ++e) acc[v] = __fmaf_rn(xf[e], yf[e], acc[v]);
        }
      }
    }
    __syncthreads();  // K buffer `buf` (and, after the last chunk, the query block) no longer read
    if (cc == NCH - 1) {
      if (act) {
        const int kt0 = j * b;
        for (int v = 0; v < G; ++v) {
          const bool ok = qok && kt0 + v * gg + t < R.Nkv;  // padding tokens: exact zero dot
          tokdot[(u * G + v) * gg + t] = ok ? acc[v] : 0.0f;
        }
      }
      if (new_q && threadIdx.x == 0) load_q(ni * b, np, nr);
      __syncthreads();
      if (threadIdx.x < G * G) {
        const int uv = threadIdx.x, uu = uv / G, vv = uv % G;
        float a = 0.0f;
        for (int tt = 0; tt < gg; ++tt) a = __fadd_rn(a, tokdot[uv * gg + tt]);  // ascending t
        const bool valid = i * b + uu * gg < R.Nq && j * b + vv * gg < R.Nkv;   // padding-only groups (R3)
        pairtot[uv] = valid ? a : -INFINITY;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        float mx = -INFINITY;  // Eq. 10
        for (int uv = 0; uv < G * G; ++uv) mx = fmaxf(mx, pairtot[uv]);
        S[(((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j] = mx;
      }
      __syncthreads();
    }
    buf ^= 1;
  }
}

// vLLM pages -> contiguous [B][Hkv][Nkv][D] (Stage-1 FLATTEN groups span several pages; the gathered
// copy lets one TMA box cover a whole group row).  One thread per 16 bytes.
__global__ void __launch_bounds__(256) k_paged_gather(Geom g, const uint4* __restrict__ kc, const int32_t* __restrict__ pt,
                                                      uint4* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_tok = g.D / 8;
  const long long total = (long long)g.B * g.Hkv_real * g.Nkv * per_tok;
  if (idx >= total) return;
  const int c = (int)(idx % per_tok);
  long long rest = idx / per_tok;
  const int s = (int)(rest % g.Nkv);
  rest /= g.Nkv;
  const int h = (int)(rest % g.Hkv_real);
  const int r = (int)(rest / g.Hkv_real);
  if (g.lens && s >= __ldg(g.lens + 2 * r + 1)) return;  // past this request's KV (no page mapped)
  const long long page = pt[(long long)r * g.max_pages + s / g.page_size];
  out[idx] = __ldg(kc + ((page * g.page_size + s % g.page_size) * g.Hkv_real + h) * per_tok + c);
}

}  // namespace

void launch_paged_gather(const Geom& g, const void* kcache, const int32_t* pt, void* kout, cudaStream_t st) {
  const long long total = (long long)g.B * g.Hkv_real * g.Nkv * (g.D / 8);
  k_paged_gather<<<(int)((total + 255) / 256), 256, 0, st>>>(g, static_cast<const uint4*>(kcache), pt,
                                                              static_cast<uint4*>(kout));
  count_launch();
}

size_t tc_scores_smem() { return SMEM; }

// Split-K factor from the live (causal) tile count: just under one wave of 148 SMs for small grids, 2
// between one and two waves, else 1; at most 8 and at least 16 k-steps per split; BFLA_TC_SPLITS
// overrides (A/B).  Deterministic in the geometry, so bfla_workspace_size can reserve the partials.
int tc_splits(const Geom& g) {
  const int ngq = (g.Nq + g.g - 1) / g.g, ngk = (g.Nkv + g.g - 1) / g.g;
  const int n_mt = (ngq + TM - 1) / TM, n_nt = (ngk + TN - 1) / TN;
  const int nk = g.g * g.D / TK;
  static const int forced = experiment_knob("BFLA_TC_SPLITS", 0);  // A/B builds only
  int s = forced;
  if (s <= 0) {
    // live (causal) tiles of one (request, head) — buffer dims stand in for varlen requests
    const Req R = make_req(g.Nq, g.Nkv, g.b, g.T);
    long long live = 0;
    int nl;
    for (int mt = 0; mt < n_mt; ++mt)
      for (int nt = 0; nt < n_nt; ++nt) live += tc_tile_live(g, R, mt, nt, &nl) ? 1 : 0;
    live *= (long long)g.B * g.Hq;
    // measured (profiles/r3_s1_splits.txt): a grid just under one wave beats more, shorter splits
    // (8K: 32 live tiles x 4 splits 0.085 ms vs x 8 0.100); between one and two waves of tiles, two
    // splits even out the diagonal half tiles (32K: 192 live tiles, 2 splits 0.194 vs 1 0.214)
    s = live >= 2 * 148 ? 1 : live >= 148 ? 2 : (int)(148 / (live > 0 ? live : 1));
  }
  if (s > 8) s = 8;
  while (s > 1 && nk / s < 16) --s;
  return s < 1 ? 1 : s;
}

// Split-K scratch: raw partials [tile][split][TN][TM] and query-norm partials [rp][mt][split][TM];
// `tick` holds two int counters per tile (ticket, splits done), zero on entry (the caller's memset;
// the last split of each tile also resets its pair).
static long long tc_tiles(const Geom& g, int* n_mt_out = nullptr, int* n_nt_out = nullptr) {
  const int ngq = (g.Nq + g.g - 1) / g.g, ngk = (g.Nkv + g.g - 1) / g.g;
  const int n_mt = (ngq + TM - 1) / TM, n_nt = (ngk + TN - 1) / TN;
  if (n_mt_out) *n_mt_out = n_mt;
  if (n_nt_out) *n_nt_out = n_nt;
  return (long long)g.B * g.Hq * n_mt * n_nt;
}

size_t tc_part_bytes(const Geom& g) {
  const int s = tc_splits(g);
  if (s == 1) return 0;
  int n_mt;
  const long long tiles = tc_tiles(g, &n_mt);
  return (size_t)(tiles * s * TN * TM + (long long)g.B * g.Hq * n_mt * s * TM) * 4;
}

size_t tc_tick_bytes(const Geom& g) { return tc_splits(g) > 1 ? (size_t)tc_tiles(g) * 2 * sizeof(int) : 0; }

// Cluster size for the score kernel: the csz query heads of one KV group that share every K tile run as
// one thread-block cluster and fetch each B stage once (TMA multicast), cutting the L2->SM traffic that
// bounds this kernel.  csz divides m; 1 = no cluster.
static int tc_cluster(const Geom& g) {
  static const int forced = experiment_knob("BFLA_S1_CLUSTER", 0);  // A/B builds only
  int c = forced > 0 ? forced : kTcCluster;
  while (c > 1 && (g.m % c)) c >>= 1;
  return c < 1 ? 1 : c;
}

int launch_tc_scores(const Geom& g, const CUtensorMap& tmA, const CUtensorMap& tmB, float* S, float* qn,
                     cudaStream_t st, float* part, int* tick, const CUtensorMap* tmB64) {
  int n_mt, n_nt;
  const long long ctas = tc_tiles(g, &n_mt, &n_nt);
  const int splits = part ? tc_splits(g) : 1;
  if (ctas <= 0 || ctas * splits > 0x7fffffff) return -1;
  cudaError_t e = cudaFuncSetAttribute(k_s1_tc_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return (int)e;
  float* qpart = part ? part + ctas * splits * (long long)(TN * TM) : nullptr;
  // split-K finish: in the score kernel (the last split of a tile adds the others' partials) for grids
  // of at most about one wave, else by k_s1_tc_reduce over the whole grid
  static const int fused_knob = experiment_knob("BFLA_S1_FUSED_SPLIT", -1);  // A/B builds only
  const bool fused = splits > 1 && (fused_knob >= 0 ? fused_knob == 1 : ctas * splits <= 2 * 148);
  if (fused && !tick) return -1;
  int csz = tc_cluster(g);
  cudaLaunchConfig_t cfg = {};
  cudaLaunchAttribute attr[1];
  cfg.gridDim = dim3((unsigned)(ctas * splits));
  cfg.blockDim = dim3(256);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  if (csz > 1) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = (unsigned)csz;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    // can a cluster of csz one-CTA-per-SM blocks be resident at all (queried once per device and size)
    static thread_local int ok_dev = -1, ok_csz = 0, ok_val = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (ok_dev != dev || ok_csz != csz) {
      int nclusters = 0;
      ok_val = cudaOccupancyMaxActiveClusters(&nclusters, k_s1_tc_scores, &cfg) == cudaSuccess && nclusters >= 1;
      cudaGetLastError();
      ok_dev = dev;
      ok_csz = csz;
    }
    if (!ok_val) {
      csz = 1;
      cfg.attrs = nullptr;
      cfg.numAttrs = 0;
    }
  }
  // CTA-pair MMA variant (cta_group::2) for clusters of two (A/B: BFLA_S1_PAIR)
  static const bool pair_knob = experiment_knob("BFLA_S1_PAIR", kTcPair) == 1;
  if (csz == 2 && pair_knob && tmB64) {
    e = cudaFuncSetAttribute(k_s1_tc_scores_pair, cudaFuncAttributeMaxDynamicSharedMemorySize, PSMEM);
    if (e != cudaSuccess) return (int)e;
    cfg.dynamicSmemBytes = PSMEM;
    e = cudaLaunchKernelEx(&cfg, k_s1_tc_scores_pair, tmA, tmB, *tmB64, g, S, n_mt, n_nt, qn, splits, part, qpart,
                           fused ? tick : nullptr);
  } else {
    e = cudaLaunchKernelEx(&cfg, k_s1_tc_scores, tmA, tmB, g, S, n_mt, n_nt, qn, splits, part, qpart,
                           fused ? tick : nullptr, csz);
  }
  count_launch();
  if (e != cudaSuccess) return (int)e;
  if (splits > 1 && !fused) {
    k_s1_tc_reduce<<<(int)(ctas * (TN / kRedCols)), 128, 0, st>>>(g, S, n_mt, n_nt, qn, splits, part, qpart);
    count_launch();
  }
  return (int)cudaGetLastError();
}

int launch_ragged_fixup(const Geom& g, const void* q, const void* k, float* S, cudaStream_t st) {
  const long long units = (long long)g.B * g.Hkv * (g.Lkv + g.Lq);
  const int dots = ((2 * g.G - 1) * g.g + 2 * g.G) * 4;
  const int staged = g.b * (g.D * 2 + 16) + dots;
  const bool stage = staged <= 200 * 1024;  // else keys from global memory (b = 1024, or d = 256 at b = 512)
  const int smem = stage ? staged : dots;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRecThreads, smem);
    const long long grid = std::min<long long>(units, (long long)148 * (per_sm > 0 ? per_sm : 1));
    kern<<<(int)grid, kRecThreads, smem, st>>>(g, static_cast<const __nv_bfloat16*>(q),
                                               static_cast<const __nv_bfloat16*>(k), S);
  };
  if (g.D == 128) stage ? go(k_s1_ragged_fixup<128, true>) : go(k_s1_ragged_fixup<128, false>);
  else if (g.D == 256) stage ? go(k_s1_ragged_fixup<256, true>) : go(k_s1_ragged_fixup<256, false>);
  else return -1;
  count_launch();
  return (int)cudaGetLastError();
}

void launch_block_norms(const Geom& g, const void* q, const void* k, float* qn, float* kn, cudaStream_t st,
                        bool with_q) {
  const long long ctas = (with_q ? (long long)g.B * g.Hq * g.Lq : 0) + (long long)g.B * g.Hkv * g.Lkv;
  k_s1_block_norms<<<(int)ctas, 256, 0, st>>>(g, static_cast<const __nv_bfloat16*>(q),
                                              static_cast<const __nv_bfloat16*>(k), qn, kn, with_q ? 1 : 0);
  count_launch();
}

int launch_recompute_rows(const Geom& g, const void* q, const void* k, const int32_t* pt, const int32_t* flagged,
                          const int32_t* n_flagged, const int32_t* ulist, const int32_t* n_units, float* S,
                          int num_sms, cudaStream_t st,
                          const CUtensorMap* tmQ, const CUtensorMap* tmK) {
  (void)pt;
  if (g.G * g.G > kRecThreads) return -1;
  auto qq = static_cast<const __nv_bfloat16*>(q);
  auto kk = static_cast<const __nv_bfloat16*>(k);
  // A/B builds only: 0 auto (TMA), 1 global loads, 2 bulk rows
  static const int mode = experiment_knob("BFLA_RECOMPUTE", 0);
  {
    const size_t smem_t = (size_t)3 * g.b * g.D * 2 + ((size_t)g.G * g.G * g.g + g.G * g.G) * 4 + 1024;
    if (mode == 0 && tmQ && tmK && g.D == 128 && g.G <= 16 && g.b % 64 == 0 && smem_t <= 226 * 1024) {
      auto kern = k_s1_recompute_tma<128>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_t);
      kern<<<num_sms, kRecThreads, smem_t, st>>>(*tmQ, *tmK, g, flagged, n_flagged, ulist, n_units, S);
      count_launch();
      return (int)cudaGetLastError();
    }
    const size_t smem_kc = (size_t)g.b * g.D * 2 + (size_t)2 * g.b * 128 + ((size_t)g.G * g.G * g.g + g.G * g.G) * 4 +
                           1024;
    if (mode == 0 && tmQ && tmK && g.D == 256 && g.G <= 16 && g.b % 64 == 0 && g.G * g.g <= kRecThreads &&
        smem_kc <= 226 * 1024) {
      auto kern = k_s1_recompute_tma_kc<256>;
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_kc);
      kern<<<num_sms, kRecThreads, smem_kc, st>>>(*tmQ, *tmK, g, flagged, n_flagged, ulist, n_units, S);
      count_launch();
      return (int)cudaGetLastError();
    }
  }
  // staged variant: K block + two query groups (padded rows) + token dots
  const size_t pitch = (size_t)g.D * 2 + 16;
  const size_t smem_s = ((size_t)g.b + 2 * g.g) * pitch + ((size_t)g.G * g.G * g.g + g.G * g.G) * 4;
  if (mode != 1 && smem_s <= 226 * 1024 && (g.qs2 % 8) == 0 && (g.kvs2 % 8) == 0) {
    auto gs = [&](auto kern) {
      cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_s);
      int per_sm = 1;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kRecThreads, smem_s);
      kern<<<num_sms * (per_sm > 0 ? per_sm : 1), kRecThreads, smem_s, st>>>(g, qq, kk, flagged, n_flagged, ulist, n_units, S);
    };
    if (g.D == 128) gs(k_s1_recompute_smem<128>);
    else if (g.D == 256) gs(k_s1_recompute_smem<256>);
    else return -1;
    count_launch();
    return (int)cudaGetLastError();
  }
  const int smem = (g.G * g.G * g.g + g.G * g.G) * 4;
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    kern<<<num_sms * 4, kRecThreads, smem, st>>>(g, qq, kk, flagged, n_flagged, ulist, n_units, S);
  };
  if (g.D == 128) go(k_s1_recompute_rows<128>);
  else if (g.D == 256) go(k_s1_recompute_rows<256>);
  else return -1;
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace bfla
