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
constexpr int TN = 128;   // key groups per tile (MMA N)
constexpr int TK = 64;    // K elements per stage (one 128-byte swizzle row)
constexpr int ST = 6;     // pipeline stages
constexpr int ABYTES = TM * TK * 2;
constexpr int BBYTES = TN * TK * 2;
constexpr int SMEM = ST * (ABYTES + BBYTES) + 2 * ST * 8 + 8 + 16 + 1024;

// ---- group norms: one warp per (request, head, block); each lane sums squares sequentially over a
// strided slice of each group, lanes combine by shuffles, max over the block's groups.  The result is
// rounded up by a relative 2^-20 so it bounds the exact norm despite fp32 rounding.
__global__ void __launch_bounds__(256) k_s1_block_norms(Geom g, const __nv_bfloat16* __restrict__ q,
                                                        const __nv_bfloat16* __restrict__ k, float* __restrict__ qn,
                                                        float* __restrict__ kn) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const long long nq = (long long)g.B * g.Hq * g.Lq, nk = (long long)g.B * g.Hkv * g.Lkv;
  if (w >= nq + nk) return;
  const bool isq = w < nq;
  const long long u = isq ? w : w - nq;
  const int L = isq ? g.Lq : g.Lkv, H = isq ? g.Hq : g.Hkv, N = isq ? g.Nq : g.Nkv;
  const int blk = (int)(u % L), hh = (int)((u / L) % H), r = (int)(u / ((long long)L * H));
  float best = 0.f;
  for (int grp = 0; grp < g.G; ++grp) {
    const int t0 = blk * g.b + grp * g.g;
    float acc = 0.f;
    for (int t = t0; t < t0 + g.g && t < N; ++t) {
      const __nv_bfloat16* row = isq ? q + (long long)r * g.qs0 + (long long)hh * g.qs1 + (long long)t * g.qs2
                                     : k + (long long)r * g.kvs0 + (long long)hh * g.kvs1 + (long long)t * g.kvs2;
      for (int c = lane * 4; c < g.D; c += 128) {
        const uint2 raw = *reinterpret_cast<const uint2*>(row + c);
        const float a = __uint_as_float(raw.x << 16), b2 = __uint_as_float(raw.x & 0xffff0000u);
        const float c3 = __uint_as_float(raw.y << 16), d4 = __uint_as_float(raw.y & 0xffff0000u);
        acc = fmaf(a, a, fmaf(b2, b2, fmaf(c3, c3, fmaf(d4, d4, acc))));
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    best = fmaxf(best, acc);
  }
  if (lane == 0) (isq ? qn : kn)[u] = sqrtf(best) * (1.0f + 0x1p-10f) + 1e-30f;  // fp32 sum slack
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
  {  // causal skip (Eq. 11-13): smallest j of the N tile vs the largest i of the M tile
    long long e_last = (long long)g.Nc + (long long)((mt + 1) * BQ) * g.b - 1;
    if (e_last > g.Nkv - 1) e_last = g.Nkv - 1;
    if ((long long)nt * BK * g.b > e_last) return;
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<128>(tslot);
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
  } else if (warp == 1 && lane == 0) {
    constexpr uint32_t idesc = idesc_bf16(TM, TN, 0, 0);
    const uint32_t base = smem_u32(smem);
    for (int kk = 0; kk < nk; ++kk) {
      const int s = kk % ST;
      mbar_wait(full + s, (kk / ST) & 1);
      tc_fence_after();
      const uint32_t a = base + s * (ABYTES + BBYTES), b = a + ABYTES;
#pragma unroll
      for (int k16 = 0; k16 < TK / 16; ++k16)
        umma_f16_ss(tmem, sdesc_sw128(a + k16 * 32, 16, 1024), sdesc_sw128(b + k16 * 32, 16, 1024), idesc,
                    (kk | k16) ? 1u : 0u);
      umma_commit(empty + s);
    }
    umma_commit(done);
  } else if (warp >= 4) {
    const int lg = warp & 3;
    const int row = lg * 32 + lane;  // query group within the tile
    mbar_wait(done, 0);
    tc_fence_after();
    const int grow = mt * TM + row;           // global query group of head p
    const int ib = grow / g.G, u = grow % g.G;
    const bool uvalid = (long long)grow * g.g < g.Nq;  // padding-only groups never take the max (R3)
    long long e_i = (long long)g.Nc + (long long)(ib + 1) * g.b - 1;
    if (e_i > g.Nkv - 1) e_i = g.Nkv - 1;
    float* srow = S + (((long long)r * g.Hq + p) * g.Lq + ib) * g.Lkv;
    for (int c0 = 0; c0 < TN; c0 += 32) {
      float v[32];
      tmem_ld32(tmem + ((uint32_t)(lg * 32) << 16) + c0, v);
      tmem_wait_ld();
      for (int jb0 = 0; jb0 < 32; jb0 += g.G) {
        const int gcol = nt * TN + c0 + jb0;  // first key group of this KV block
        float mx = -INFINITY;
        for (int vv = 0; vv < g.G; ++vv)
          if ((long long)(gcol + vv) * g.g < g.Nkv) mx = fmaxf(mx, v[jb0 + vv]);
        if (!uvalid) mx = -INFINITY;
        for (int o = 1; o < g.G; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        const int jb = gcol / g.G;
        if (u == 0 && ib < g.Lq && jb < g.Lkv && (long long)jb * g.b <= e_i) srow[jb] = mx;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<128>(tmem);
  }
}

// ---- canonical recompute of flagged rows: for each flagged (request, KV head, query block) and each
// query head p of its group, S[p,i,j] for all causal j in exactly the canonical order (one fp32 FMA
// per element, ascending).  Work unit = (flagged row, head p, chunk of 32 KV blocks); a thread owns one
// (j, u, v) dot product and reads its key group straight from L2; the CTA stages the query groups.
__global__ void __launch_bounds__(256) k_s1_recompute_rows(Geom g, const __nv_bfloat16* __restrict__ q,
                                                           const __nv_bfloat16* __restrict__ k,
                                                           const int32_t* __restrict__ pt,
                                                           const int32_t* __restrict__ flagged,
                                                           const int32_t* __restrict__ n_flagged, float* __restrict__ S) {
  extern __shared__ __align__(16) float sq[];  // [G][g*D] query groups of (p, i) as fp32
  __shared__ float part[256];
  const int nf = *n_flagged;
  const int chunks = (g.Lkv + 31) / 32;
  const long long units = (long long)nf * g.m * chunks;
  const int gc = g.g * g.D;
  for (long long unit = blockIdx.x; unit < units; unit += gridDim.x) {
    const int chunk = (int)(unit % chunks);
    const int pl = (int)((unit / chunks) % g.m);
    const int row = flagged[unit / ((long long)chunks * g.m)];  // (r * Hkv + h) * Lq + i
    const int i = row % g.Lq, h = (row / g.Lq) % g.Hkv, r = row / (g.Lq * g.Hkv);
    const int p = h * g.m + pl;
    long long e_i = (long long)g.Nc + (long long)(i + 1) * g.b - 1;
    if (e_i > g.Nkv - 1) e_i = g.Nkv - 1;
    const int jmax = (int)(e_i / g.b);
    const int j0 = chunk * 32;
    __syncthreads();
    if (j0 > jmax) continue;
    // stage the G query groups (fp32, zero padded)
    for (int x = threadIdx.x; x < g.G * gc; x += blockDim.x) {
      const int u = x / gc, e = x % gc;
      const int t = i * g.b + u * g.g + e / g.D;
      sq[x] = t < g.Nq ? __bfloat162float(q[(long long)r * g.qs0 + (long long)p * g.qs1 + (long long)t * g.qs2 + e % g.D])
                       : 0.0f;
    }
    __syncthreads();
    const int per = 32 * g.G * g.G;  // dot products in this chunk
    for (int d0 = 0; d0 < per; d0 += blockDim.x) {
      const int di = d0 + threadIdx.x;
      float acc = -INFINITY;
      if (di < per) {
        const int jl = di / (g.G * g.G), uv = di % (g.G * g.G), u = uv / g.G, v = uv % g.G;
        const int j = j0 + jl;
        const int s0 = j * g.b + v * g.g;
        if (j <= jmax && i * g.b + u * g.g < g.Nq && s0 < g.Nkv) {
          const float* x = sq + u * gc;
          acc = 0.0f;
          for (int t = 0; t < g.g; ++t) {
            const int s = s0 + t;
            const __nv_bfloat16* kr = nullptr;
            if (s < g.Nkv) {
              if (!g.paged) kr = k + (long long)r * g.kvs0 + (long long)h * g.kvs1 + (long long)s * g.kvs2;
              else kr = k + (((long long)pt[(long long)r * g.max_pages + s / g.page_size] * g.page_size + s % g.page_size) * g.Hkv + h) * g.D;
            }
            for (int c = 0; c < g.D; c += 8) {
              float y[8];
              if (kr) {
                const uint4 raw = __ldg(reinterpret_cast<const uint4*>(kr + c));
                const uint32_t w4[4] = {raw.x, raw.y, raw.z, raw.w};
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                  y[2 * e] = __uint_as_float(w4[e] << 16);
                  y[2 * e + 1] = __uint_as_float(w4[e] & 0xffff0000u);
                }
              } else {
#pragma unroll
                for (int e = 0; e < 8; ++e) y[e] = 0.0f;
              }
#pragma unroll
              for (int e = 0; e < 8; ++e) acc = __fmaf_rn(x[t * g.D + c + e], y[e], acc);
            }
          }
        }
      }
      part[threadIdx.x] = acc;
      __syncthreads();
      // max over the G x G pairs of each block (exact)
      if (threadIdx.x < blockDim.x / (g.G * g.G) && d0 + threadIdx.x * g.G * g.G < per) {
        const int jl = (d0 / (g.G * g.G)) + threadIdx.x;
        float mx = -INFINITY;
        for (int e = 0; e < g.G * g.G; ++e) mx = fmaxf(mx, part[threadIdx.x * g.G * g.G + e]);
        const int j = j0 + jl;
        if (j <= jmax && j < g.Lkv) S[(((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j] = mx;
      }
      __syncthreads();
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
  const long long warps = (long long)g.B * g.Hq * g.Lq + (long long)g.B * g.Hkv * g.Lkv;
  k_s1_block_norms<<<(int)((warps * 32 + 255) / 256), 256, 0, st>>>(g, static_cast<const __nv_bfloat16*>(q),
                                                                     static_cast<const __nv_bfloat16*>(k), qn, kn);
  count_launch();
}

int launch_recompute_rows(const Geom& g, const void* q, const void* k, const int32_t* pt, const int32_t* flagged,
                          const int32_t* n_flagged, float* S, int num_sms, cudaStream_t st) {
  const size_t smem = (size_t)g.G * g.g * g.D * sizeof(float);
  if (smem > 200 * 1024) return -1;
  cudaError_t e = cudaFuncSetAttribute(k_s1_recompute_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return (int)e;
  k_s1_recompute_rows<<<num_sms, 256, smem, st>>>(g, static_cast<const __nv_bfloat16*>(q),
                                                  static_cast<const __nv_bfloat16*>(k), pt, flagged, n_flagged, S);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace bfla
