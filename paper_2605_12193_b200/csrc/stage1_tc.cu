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

#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {

constexpr int TM = 128;   // query groups per tile (MMA M)
constexpr int TN = kTcTileN;  // key groups per tile (MMA N = 256)
constexpr int TK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int ST = 4;     // pipeline stages (48 KB each)
constexpr int ABYTES = TM * TK * 2;
constexpr int BBYTES = TN * TK * 2;
constexpr int SMEM = ST * (ABYTES + BBYTES) + 2 * ST * 8 + 8 + 16 + 1024;

// ---- group norms: one CTA per (request, head, block) of Q (first) or K; warp w sums the squares of
// group w (16-byte loads, 4 in flight per lane), lanes combine by shuffles, the block keeps the max
// over its groups.  Rounded up by a relative 2^-10 so it bounds the exact norm despite fp32 rounding.
__global__ void __launch_bounds__(256) k_s1_block_norms(Geom g, const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k, float* __restrict__ qn,
                                                        float* __restrict__ kn) {
  __shared__ float wmax[8];
  const long long u = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long nq = (long long)g.B * g.Hq * g.Lq;
  const bool isq = u < nq;
  const long long w = isq ? u : u - nq;
  const int L = isq ? g.Lq : g.Lkv, H = isq ? g.Hq : g.Hkv;
  const int blk = (int)(w % L), hh = (int)((w / L) % H), r = (int)(w / ((long long)L * H));
  const Req R = req_of(g, r);
  const int N = isq ? R.Nq : R.Nkv;
  const int vec_per_tok = g.D / 8;
  float best = 0.f;
  for (int grp = warp; grp < g.G; grp += 8) {
    const int t0 = blk * g.b + grp * g.g;
    const int ntok = min(g.g, N - t0);
    float acc = 0.f;
    if (ntok > 0) {
      const int nvec = ntok * vec_per_tok;
#pragma unroll 4
      for (int x = lane; x < nvec; x += 32) {
        const int t = t0 + x / vec_per_tok, c = (x % vec_per_tok) * 8;
        const __nv_bfloat16* row = isq ? q + (long long)r * g.qs0 + (long long)hh * g.qs1 + (long long)t * g.qs2
                                       : k + (long long)r * g.kvs0 + (long long)hh * g.kvs1 + (long long)t * g.kvs2;
        const uint4 raw = __ldg(reinterpret_cast<const uint4*>(row + c));
        const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float a = __uint_as_float(w4[e] << 16), b2 = __uint_as_float(w4[e] & 0xffff0000u);
          acc = fmaf(a, a, fmaf(b2, b2, acc));
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    best = fmaxf(best, acc);
  }
  if (lane == 0) wmax[warp] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.f;
    for (int e = 0; e < 8; ++e) m = fmaxf(m, wmax[e]);
    (isq ? qn : kn)[w] = sqrtf(m) * (1.0f + 0x1p-10f) + 1e-30f;  // fp32 sum slack
  }
}

// ---- tcgen05 scores: one CTA per (request, query head, M tile of 128 query groups, N tile of 128 key
// groups); causally dead tiles exit.  Warp 0: TMA producer; warp 1: MMA issuer; warp 2: TMEM alloc;
// warps 4-7: epilogue (thread = query group row): max over the G key groups of each KV block in
// registers, max over the G query groups of each query block by shuffles (Eq. 10).
__global__ void __launch_bounds__(256, 1) k_s1_tc_scores(const __grid_constant__ CUtensorMap tmA,
                                                         const __grid_constant__ CUtensorMap tmB, Geom g,
                                                         float* __restrict__ S, int n_mt, int n_nt) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * (ABYTES + BBYTES));
  uint64_t* empty = full + ST;
  uint64_t* done = empty + ST;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  int t = blockIdx.x;
  const int nt = t % n_nt;
  t /= n_nt;
  const int mt = t % n_mt;
  const int rp = t / n_mt;  // r * Hq + p
  const int p = rp % g.Hq, r = rp / g.Hq, h = p / g.m;
  const int BQ = TM / g.G, BK = TN / g.G;  // blocks per tile
  const Req R = req_of(g, r);  // this request's logical dims (varlen); g.* is the buffer layout
  {  // causal skip (Eq. 11-13): smallest j of the N tile vs the largest i of the M tile
    long long e_last = (long long)R.Nc + (long long)((mt + 1) * BQ) * g.b - 1;
    if (e_last > R.Nkv - 1) e_last = R.Nkv - 1;
    if ((long long)nt * BK * g.b > e_last || mt * BQ >= R.Lq) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<TN>(tslot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  const int nk = g.g * g.D / TK;
  if (warp == 0 && lane == 0) {
    for (int kk = 0; kk < nk; ++kk) {
      const int s = kk % ST;
      mbar_wait(empty + s, ((kk / ST) & 1) ^ 1);
      mbar_arrive_expect_tx(full + s, ABYTES + BBYTES);
      unsigned char* a = smem + s * (ABYTES + BBYTES);
      tma_load_4d(a, &tmA, full + s, kk * TK, mt * TM, p, r);
      tma_load_4d(a + ABYTES, &tmB, full + s, kk * TK, nt * TN, h, r);
    }
  } else if (warp == 1) {  // converged warp, one elected lane issues (see umma_f16_ss_warp)
    constexpr uint32_t idesc = idesc_bf16(TM, TN, 0, 0);
    const uint64_t d0 = sdesc_sw128(smem_u32(smem), 16, 1024);
    for (int kk = 0; kk < nk; ++kk) {
      const int s = kk % ST;
      mbar_wait(full + s, (kk / ST) & 1);
      tc_fence_after();
      const uint64_t a = d0 + (uint64_t)((s * (ABYTES + BBYTES)) >> 4), b = a + (uint64_t)(ABYTES >> 4);
#pragma unroll
      for (int k16 = 0; k16 < TK / 16; ++k16)
        umma_f16_ss_warp(tmem, a + (uint64_t)(k16 * 2), b + (uint64_t)(k16 * 2), idesc, (kk | k16) ? 1u : 0u);
      umma_commit_warp(empty + s);
    }
    umma_commit_warp(done);
  } else if (warp >= 4) {
    const int lg = warp & 3;
    const int row = lg * 32 + lane;  // query group within the tile
    mbar_wait(done, 0);
    tc_fence_after();
    const int grow = mt * TM + row;           // global query group of head p
    const int ib = grow / g.G, u = grow % g.G;
    const bool uvalid = (long long)grow * g.g < R.Nq;  // padding-only groups never take the max (R3)
    long long e_i = (long long)R.Nc + (long long)(ib + 1) * g.b - 1;
    if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
    float* srow = S + (((long long)r * g.Hq + p) * g.Lq + ib) * g.Lkv;
    for (int c0 = 0; c0 < TN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + c0, v);
      tmem_wait_ld();
      for (int jb0 = 0; jb0 < 32; jb0 += g.G) {
        const int gcol = nt * TN + c0 + jb0;  // first key group of this KV block
        float mx = -INFINITY;
        for (int vv = 0; vv < g.G; ++vv)
          if ((long long)(gcol + vv) * g.g < R.Nkv) mx = fmaxf(mx, v[jb0 + vv]);
        if (!uvalid) mx = -INFINITY;
        for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int jb = gcol / g.G;
        if (u == 0 && ib < R.Lq && jb < R.Lkv && (long long)jb * g.b <= e_i) srow[jb] = mx;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<TN>(tmem);
  }
}

// ---- canonical recompute of flagged head rows.  Work unit = (flagged head row (r,p,i), chunk of 16 KV
// blocks); thread t owns one dot product (j, u, v).  The G query groups and 16 G key groups stream
// through a 4-stage cp.async ring in k-chunks of 128 elements (bf16, 16-byte copies, padded rows);
// each thread adds its chunk's 128 products in ascending order with single-rounding FMAs, so every
// dot product is exactly the canonical chain (k is the outer loop and ascending).  The G x G max is
// taken through smem.
__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int G>
__global__ void __launch_bounds__(256) k_s1_recompute_rows(Geom g, const __nv_bfloat16* __restrict__ q,
                                                           const __nv_bfloat16* __restrict__ k,
                                                           const int32_t* __restrict__ flagged,
                                                           const int32_t* __restrict__ n_flagged,
                                                           const float* __restrict__ flag_thr,
                                                           float* __restrict__ S) {
  // k-chunk: 256 elements (two tokens at d = 128; rows are contiguous token runs on this path)
  constexpr int KC = G <= 4 ? 256 : 128, JB = 16, NST = 4;
  constexpr int ROWS = G + JB * G, RB = KC * 2 + 16;  // row bytes padded by 16 (bank spread)
  constexpr int NDOT = JB * G * G, PER = (NDOT + 255) / 256;
  extern __shared__ __align__(16) unsigned char rsm[];
  float* part = reinterpret_cast<float*>(rsm + NST * ROWS * RB);
  __shared__ uint32_t live_bits;  // blocks of this chunk whose canonical logit can exceed -127
  const int nf = *n_flagged;
  const int chunks = (g.Lkv + JB - 1) / JB;
  const long long units = (long long)nf * chunks;
  const int gc = g.g * g.D, nk = gc / KC;
  for (long long unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int chunk = (int)(unit % chunks);
    const int row = flagged[unit / chunks];  // (r * Hq + p) * Lq + i
    const int i = row % g.Lq, p = (row / g.Lq) % g.Hq, r = row / (g.Lq * g.Hq);
    const int h = p / g.m;
    const Req R = req_of(g, r);
    long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
    if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
    const int jmax = (int)(e_i / g.b);
    const int j0 = chunk * JB;
    if (j0 > jmax) continue;  // uniform over the CTA
    __syncthreads();          // the previous unit's readers are done with the ring (and live_bits)
    float* srow = S + (((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv;
    if (threadIdx.x < 32) {
      const float thr = flag_thr[unit / chunks];
      const int j = j0 + threadIdx.x;
      const bool live = threadIdx.x < JB && j <= jmax && srow[j] >= thr;
      const uint32_t bal = __ballot_sync(0xffffffffu, live);
      if (threadIdx.x == 0) live_bits = bal;
    }
    __syncthreads();
    const uint32_t live = live_bits;
    if (!live) continue;  // every block of the chunk has an exactly-zero canonical probability
    auto issue = [&](int kc) {
      unsigned char* buf = rsm + (kc % NST) * ROWS * RB;
      const int x0 = kc * KC, tk = x0 / g.D, c0 = x0 % g.D;
      for (int sidx = threadIdx.x; sidx < ROWS * (KC / 8); sidx += blockDim.x) {
        const int rr = sidx / (KC / 8), piece = sidx % (KC / 8);
        const __nv_bfloat16* src = q;
        bool ok = false;
        if (rr < G) {
          const int t = i * g.b + rr * g.g + tk;
          ok = t < R.Nq;
          if (ok) src = q + (long long)r * g.qs0 + (long long)p * g.qs1 + (long long)t * g.qs2 + c0 + piece * 8;
        } else {
          const int bi = rr - G, jl = bi / G, v = bi % G;
          const int s = (j0 + jl) * g.b + v * g.g + tk;
          ok = ((live >> jl) & 1u) && s < R.Nkv;
          if (ok) src = k + (long long)r * g.kvs0 + (long long)h * g.kvs1 + (long long)s * g.kvs2 + c0 + piece * 8;
        }
        cp_async16(buf + rr * RB + piece * 16, src, ok);  // zero-filled when !ok (padding)
      }
      cp_async_commit();
    };
    float acc[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) acc[e] = 0.0f;
    for (int kc = 0; kc < NST - 1; ++kc) {
      if (kc < nk) issue(kc);
      else cp_async_commit();
    }
    for (int kc = 0; kc < nk; ++kc) {
      cp_async_wait<NST - 2>();
      __syncthreads();
      if (kc + NST - 1 < nk) issue(kc + NST - 1);
      else cp_async_commit();
      const unsigned char* buf = rsm + (kc % NST) * ROWS * RB;
#pragma unroll
      for (int e = 0; e < PER; ++e) {
        const int di = threadIdx.x + e * 256;
        if (di < NDOT && ((live >> (di / (G * G))) & 1u)) {
          const int jl = di / (G * G), u = (di / G) % G, v = di % G;
          const uint2* xa = reinterpret_cast<const uint2*>(buf + u * RB);
          const uint2* yb = reinterpret_cast<const uint2*>(buf + (G + jl * G + v) * RB);
          float a = acc[e];
#pragma unroll 8
          for (int q4 = 0; q4 < KC / 4; ++q4) {
            const uint2 xv = xa[q4], yv = yb[q4];
            a = __fmaf_rn(__uint_as_float(xv.x << 16), __uint_as_float(yv.x << 16), a);
            a = __fmaf_rn(__uint_as_float(xv.x & 0xffff0000u), __uint_as_float(yv.x & 0xffff0000u), a);
            a = __fmaf_rn(__uint_as_float(xv.y << 16), __uint_as_float(yv.y << 16), a);
            a = __fmaf_rn(__uint_as_float(xv.y & 0xffff0000u), __uint_as_float(yv.y & 0xffff0000u), a);
          }
          acc[e] = a;
        }
      }
    }
    cp_async_wait<0>();
    __syncthreads();
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int di = threadIdx.x + e * 256;
      if (di < NDOT) part[di] = acc[e];
    }
    __syncthreads();
    if (threadIdx.x < JB) {
      const int jl = threadIdx.x, j = j0 + jl;
      if ((live >> jl) & 1u) {
        float mx = -INFINITY;
        for (int u = 0; u < G; ++u) {
          if (i * g.b + u * g.g >= R.Nq) continue;  // padding-only query group (R3)
          for (int v = 0; v < G; ++v)
            if (j * g.b + v * g.g < R.Nkv) mx = fmaxf(mx, part[(jl * G + u) * G + v]);
        }
        srow[j] = mx;
      }
    }
  }
}

// vLLM pages -> contiguous [B][Hkv][Nkv][D] (Stage-1 FLATTEN groups span several pages; the gathered
// copy lets one TMA box cover a whole group row).  One thread per 16 bytes.
__global__ void __launch_bounds__(256) k_paged_gather(Geom g, const uint4* __restrict__ kc, const int32_t* __restrict__ pt,
                                                      uint4* __restrict__ out) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int per_tok = g.D / 8;
  const long long total = (long long)g.B * g.Hkv * g.Nkv * per_tok;
  if (idx >= total) return;
  const int c = (int)(idx % per_tok);
  long long rest = idx / per_tok;
  const int s = (int)(rest % g.Nkv);
  rest /= g.Nkv;
  const int h = (int)(rest % g.Hkv);
  const int r = (int)(rest / g.Hkv);
  if (g.lens && s >= __ldg(g.lens + 2 * r + 1)) return;  // past this request's KV (no page mapped)
  const long long page = pt[(long long)r * g.max_pages + s / g.page_size];
  out[idx] = __ldg(kc + ((page * g.page_size + s % g.page_size) * g.Hkv + h) * per_tok + c);
}

}  // namespace

void launch_paged_gather(const Geom& g, const void* kcache, const int32_t* pt, void* kout, cudaStream_t st) {
  const long long total = (long long)g.B * g.Hkv * g.Nkv * (g.D / 8);
  k_paged_gather<<<(int)((total + 255) / 256), 256, 0, st>>>(g, static_cast<const uint4*>(kcache), pt,
                                                              static_cast<uint4*>(kout));
  count_launch();
}

size_t tc_scores_smem() { return SMEM; }

int launch_tc_scores(const Geom& g, const CUtensorMap& tmA, const CUtensorMap& tmB, float* S, cudaStream_t st) {
  const int ngq = (g.Nq + g.g - 1) / g.g, ngk = (g.Nkv + g.g - 1) / g.g;
  const int n_mt = (ngq + TM - 1) / TM, n_nt = (ngk + TN - 1) / TN;
  const long long ctas = (long long)g.B * g.Hq * n_mt * n_nt;
  if (ctas <= 0 || ctas > 0x7fffffff) return -1;
  cudaError_t e = cudaFuncSetAttribute(k_s1_tc_scores, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
  if (e != cudaSuccess) return (int)e;
  k_s1_tc_scores<<<(int)ctas, 256, SMEM, st>>>(tmA, tmB, g, S, n_mt, n_nt);
  count_launch();
  return (int)cudaGetLastError();
}

void launch_block_norms(const Geom& g, const void* q, const void* k, float* qn, float* kn, cudaStream_t st) {
  const long long ctas = (long long)g.B * g.Hq * g.Lq + (long long)g.B * g.Hkv * g.Lkv;
  k_s1_block_norms<<<(int)ctas, 256, 0, st>>>(g, static_cast<const __nv_bfloat16*>(q),
                                                                     static_cast<const __nv_bfloat16*>(k), qn, kn);
  count_launch();
}

int launch_recompute_rows(const Geom& g, const void* q, const void* k, const int32_t* pt, const int32_t* flagged,
                          const int32_t* n_flagged, const float* flag_thr, float* S, int num_sms, cudaStream_t st) {
  (void)pt;
  auto qq = static_cast<const __nv_bfloat16*>(q);
  auto kk = static_cast<const __nv_bfloat16*>(k);
  auto go = [&](auto kern, int G) {
    const int KC = G <= 4 ? 256 : 128;
    const size_t smem = (size_t)4 * (G + 16 * G) * (KC * 2 + 16) + (size_t)16 * G * G * 4;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<2 * num_sms, 256, smem, st>>>(g, qq, kk, flagged, n_flagged, flag_thr, S);
  };
  switch (g.G) {
    case 1: go(k_s1_recompute_rows<1>, 1); break;
    case 2: go(k_s1_recompute_rows<2>, 2); break;
    case 4: go(k_s1_recompute_rows<4>, 4); break;
    case 8: go(k_s1_recompute_rows<8>, 8); break;
    default: return -1;
  }
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace bfla
