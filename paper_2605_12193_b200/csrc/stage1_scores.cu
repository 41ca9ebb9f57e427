// stage1_scores.cu — Stage 1 block scores of BFLA (Eq. 4-10, 14).
//
// FLATTEN (the paper's flattening-g pooling, Eq. 6-10): for query head p (KV head h = p/m) the
// block score S[p,i,j] = max over valid group pairs (u,v) of Phi(Q)[p,i,u] . Phi(K)[h,j,v], where a
// group is g consecutive tokens flattened to a g*C vector (a zero-copy view of head-first Q/K).
// The dot products are accumulated in the canonical order (DESIGN.md §4 item 2): per token pair a
// C-long fp32 FMA chain (channel ascending), the g token dots added in ascending token order.  A
// register-blocked SIMT GEMM does exactly that: every thread owns the G x G token-chain accumulators
// and G x G group totals of one (i, j) block pair; k (= t*C + c) ascends, and at every token boundary
// the chains are added into the totals and restarted, so the scores are bit-identical to the
// oracle's and the G x G max-pool (Eq. 10) happens in registers.
//
// MEAN (north_star variant, R1): qbar/kbar = fp32 block means (tokens summed in ascending order,
// 128-bit loads, one half-warp per block), then one canonical C-long dot product per block pair.
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {

constexpr int KC = 32;       // k-chunk (elements of the g*C reduction) staged per iteration
constexpr int KP = KC + 4;   // padded smem row (floats): rows 36 words apart -> conflict-free LDS.128
constexpr int BI = 16;       // query blocks per CTA tile
constexpr int BJ = 16;       // KV blocks per CTA tile

__device__ __forceinline__ const __nv_bfloat16* k_token(const Geom& g, const __nv_bfloat16* k, const int32_t* pt,
                                                        int r, int h, int s) {
  h /= g.kvdiv;  // mask group -> KV head
  if (!g.paged) return k + (long long)r * g.kvs0 + (long long)h * g.kvs1 + (long long)s * g.kvs2;
  const int page = pt[(long long)r * g.max_pages + s / g.page_size];
  return k + (((long long)page * g.page_size + s % g.page_size) * g.Hkv_real + h) * g.D;
}

__device__ __forceinline__ void bf16x8_to_f32(uint4 u, float* f) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    f[2 * e] = __uint_as_float(w[e] << 16);
    f[2 * e + 1] = __uint_as_float(w[e] & 0xffff0000u);
  }
}

// Grid: (ceil(Lkv/16), ceil(Lq/16), B*Hq).  Block: 256 threads = 16 (i) x 16 (j).
template <int G>
__global__ void __launch_bounds__(256) k_s1_flatten_scores(Geom g, const __nv_bfloat16* __restrict__ q,
                                                           const __nv_bfloat16* __restrict__ k,
                                                           const int32_t* __restrict__ pt, float* __restrict__ S) {
  extern __shared__ __align__(16) float smem_f[];
  float* As[2] = {smem_f, smem_f + G * BI * KP};
  float* Bs[2] = {smem_f + 2 * G * BI * KP, smem_f + 2 * G * BI * KP + G * BJ * KP};
  const int tid = threadIdx.x;
  const int ti = tid >> 4, tj = tid & 15;
  const int i0 = blockIdx.y * BI, j0 = blockIdx.x * BJ;
  const int rp = blockIdx.z;
  const int p = rp % g.Hq, r = rp / g.Hq, h = p / g.m;
  const Req R = req_of(g, r);  // this request's logical dims (varlen); g.* is the buffer layout
  // causal skip (Eq. 11-13): the tile's smallest j against the largest i's frontier
  {
    long long e_last = (long long)R.Nc + (long long)(i0 + BI) * g.b - 1;
    if (e_last > R.Nkv - 1) e_last = R.Nkv - 1;
    if ((long long)j0 * g.b > e_last || i0 >= R.Lq) return;
  }
  const int gC = g.g * g.D;
  const int nit = gC / KC;
  // loader mapping: segment = (row, 8-element piece); rows ordered u*16 + local block index
  constexpr int ROWS = G * 16;
  constexpr int SEGS = ROWS * (KC / 8);
  constexpr int PER = (SEGS + 255) / 256;
  uint4 ra[PER], rb[PER];
  auto load = [&](int it) {
    const int x0 = it * KC;  // element index within the group vector: token x0 / C, channel x0 % C
    const int tk = x0 / g.D, c0 = x0 % g.D;
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int sidx = tid + e * 256;
      ra[e] = make_uint4(0, 0, 0, 0);
      rb[e] = make_uint4(0, 0, 0, 0);
      if (sidx < SEGS) {
        const int row = sidx >> 2, piece = sidx & 3;
        const int u = row >> 4, loc = row & 15;
        const int ib = i0 + loc, jb = j0 + loc;
        const int tq = ib * g.b + u * g.g + tk;
        if (ib < R.Lq && tq < R.Nq)
          ra[e] = __ldg(reinterpret_cast<const uint4*>(q + (long long)r * g.qs0 + (long long)p * g.qs1 +
                                                       (long long)tq * g.qs2 + c0 + piece * 8));
        const int sk = jb * g.b + u * g.g + tk;
        if (jb < R.Lkv && sk < R.Nkv)
          rb[e] = __ldg(reinterpret_cast<const uint4*>(k_token(g, k, pt, r, h, sk) + c0 + piece * 8));
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int sidx = tid + e * 256;
      if (sidx < SEGS) {
        const int row = sidx >> 2, piece = sidx & 3;
        float f[8];
        bf16x8_to_f32(ra[e], f);
        float4* da = reinterpret_cast<float4*>(&As[buf][row * KP + piece * 8]);
        da[0] = make_float4(f[0], f[1], f[2], f[3]);
        da[1] = make_float4(f[4], f[5], f[6], f[7]);
        bf16x8_to_f32(rb[e], f);
        float4* db = reinterpret_cast<float4*>(&Bs[buf][row * KP + piece * 8]);
        db[0] = make_float4(f[0], f[1], f[2], f[3]);
        db[1] = make_float4(f[4], f[5], f[6], f[7]);
      }
    }
  };
  float acc[G][G], tot[G][G];
#pragma unroll
  for (int u = 0; u < G; ++u)
#pragma unroll
    for (int v = 0; v < G; ++v) acc[u][v] = tot[u][v] = 0.0f;

  load(0);
  store(0);
  __syncthreads();
  for (int it = 0; it < nit; ++it) {
    if (it + 1 < nit) load(it + 1);
    const float* A = As[it & 1];
    const float* Bm = Bs[it & 1];
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      float4 a[G], bv[G];
#pragma unroll
      for (int u = 0; u < G; ++u) a[u] = *reinterpret_cast<const float4*>(&A[(u * 16 + ti) * KP + kk]);
#pragma unroll
      for (int v = 0; v < G; ++v) bv[v] = *reinterpret_cast<const float4*>(&Bm[(v * 16 + tj) * KP + kk]);
      // canonical order: element kk, kk+1, kk+2, kk+3 — one single-rounding FMA each
#pragma unroll
      for (int u = 0; u < G; ++u)
#pragma unroll
        for (int v = 0; v < G; ++v) {
          acc[u][v] = __fmaf_rn(a[u].x, bv[v].x, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].y, bv[v].y, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].z, bv[v].z, acc[u][v]);
          acc[u][v] = __fmaf_rn(a[u].w, bv[v].w, acc[u][v]);
        }
    }
    if (((it + 1) * KC) % g.D == 0) {  // token boundary: add the token dot, restart the chain
#pragma unroll
      for (int u = 0; u < G; ++u)
#pragma unroll
        for (int v = 0; v < G; ++v) {
          tot[u][v] = __fadd_rn(tot[u][v], acc[u][v]);
          acc[u][v] = 0.0f;
        }
    }
    if (it + 1 < nit) store((it + 1) & 1);
    __syncthreads();
  }
  const int i = i0 + ti, j = j0 + tj;
  if (i >= R.Lq || j >= R.Lkv) return;
  long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
  if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
  if ((long long)j * g.b > e_i) return;  // non-causal: never read (Eq. 14 is applied by the selector)
  float best = -INFINITY;
#pragma unroll
  for (int u = 0; u < G; ++u) {
    if (i * g.b + u * g.g >= R.Nq) continue;  // padding-only query group (R3)
#pragma unroll
    for (int v = 0; v < G; ++v) {
      if (j * g.b + v * g.g >= R.Nkv) continue;  // padding-only key group
      best = fmaxf(best, tot[u][v]);
    }
  }
  S[(((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j] = best;
}

// MEAN pooling: one half-warp per (request, head, block) of Q (first) or K (then); lane l of the
// half-warp owns channels [l*CPL, (l+1)*CPL) and sums tokens sequentially (fp32, ascending t).
template <int CPL>
__global__ void __launch_bounds__(256) k_s1_mean_pool(Geom g, const __nv_bfloat16* __restrict__ q,
                                                      const __nv_bfloat16* __restrict__ k,
                                                      const int32_t* __restrict__ pt, float* __restrict__ qbar,
                                                      float* __restrict__ kbar) {
  const long long unit = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 4;
  const int l = threadIdx.x & 15;
  const long long nq_units = (long long)g.B * g.Hq * g.Lq;
  const long long nk_units = (long long)g.B * g.Hkv * g.Lkv;
  if (unit >= nq_units + nk_units) return;
  const bool isq = unit < nq_units;
  const long long u = isq ? unit : unit - nq_units;
  const int L = isq ? g.Lq : g.Lkv, H = isq ? g.Hq : g.Hkv;
  const int blk = (int)(u % L), hh = (int)((u / L) % H), r = (int)(u / ((long long)L * H));
  const Req R = req_of(g, r);
  const int N = isq ? R.Nq : R.Nkv;
  const int t0 = blk * g.b, t1 = min(N, (blk + 1) * g.b);
  if (t0 >= t1) return;  // padding block of a shorter request (never read)
  float acc[CPL];
#pragma unroll
  for (int c = 0; c < CPL; ++c) acc[c] = 0.0f;
#pragma unroll 4
  for (int t = t0; t < t1; ++t) {
    const __nv_bfloat16* row =
        isq ? q + (long long)r * g.qs0 + (long long)hh * g.qs1 + (long long)t * g.qs2 : k_token(g, k, pt, r, hh, t);
#pragma unroll
    for (int v = 0; v < CPL / 8; ++v) {
      float f[8];
      bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(row + l * CPL + v * 8)), f);
#pragma unroll
      for (int e = 0; e < 8; ++e) acc[v * 8 + e] = __fadd_rn(acc[v * 8 + e], f[e]);
    }
  }
  const float n = (float)(t1 - t0);
  float* out = (isq ? qbar : kbar) + u * g.D + l * CPL;
#pragma unroll
  for (int c = 0; c < CPL; ++c) out[c] = __fdiv_rn(acc[c], n);
}

// One thread per (r, p, i, j): S = canonical dot(qbar, kbar) over channels ascending.
__global__ void __launch_bounds__(256) k_s1_mean_scores(Geom g, const float* __restrict__ qbar,
                                                        const float* __restrict__ kbar, float* __restrict__ S) {
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)g.B * g.Hq * g.Lq * g.Lkv;
  if (idx >= total) return;
  const int j = (int)(idx % g.Lkv);
  const long long row = idx / g.Lkv;  // (r, p, i)
  const int i = (int)(row % g.Lq);
  const int p = (int)((row / g.Lq) % g.Hq);
  const int r = (int)(row / ((long long)g.Lq * g.Hq));
  const Req R = req_of(g, r);
  if (i >= R.Lq) return;
  long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
  if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
  if ((long long)j * g.b > e_i) return;
  const float* a = qbar + row * g.D;
  const float* bb = kbar + (((long long)r * g.Hkv + p / g.m) * g.Lkv + j) * g.D;
  float acc = 0.0f;
  for (int c = 0; c < g.D; c += 4) {
    const float4 x = *reinterpret_cast<const float4*>(a + c);
    const float4 y = *reinterpret_cast<const float4*>(bb + c);
    acc = __fmaf_rn(x.x, y.x, acc);
    acc = __fmaf_rn(x.y, y.y, acc);
    acc = __fmaf_rn(x.z, y.z, acc);
    acc = __fmaf_rn(x.w, y.w, acc);
  }
  S[idx] = acc;
}

// Generic canonical FLATTEN scores for any G = b/g (used for G > 8: the paper's b = 1024, g = 64 row
// of Tab.mask, and g = 1, where Eq. 10 is the exact block max of QK^T).  CTA per (r, p, i, j)
// (non-causal pairs exit, Eq. 11-13); thread = group pair (u, v), running the canonical order of
// DESIGN.md §4 item 2 literally: acc = 0; for t: { d = 0; for c: d = fma(q_t[c], k_t[c], d); acc += d }.
// Padding tokens are skipped (their token dot is an exact +0, and acc + 0 = acc); padding-only groups
// never take the max (R3).  A CTA max-reduces its pairs (Eq. 10, exact).
template <int D>
__global__ void __launch_bounds__(256) k_s1_flatten_scores_any(Geom g, const __nv_bfloat16* __restrict__ q,
                                                               const __nv_bfloat16* __restrict__ k,
                                                               const int32_t* __restrict__ pt, float* __restrict__ S) {
  __shared__ float wmax[8];
  const int j = blockIdx.x, i = blockIdx.y, rp = blockIdx.z;
  const int p = rp % g.Hq, r = rp / g.Hq, h = p / g.m;
  const Req R = req_of(g, r);
  if (i >= R.Lq || j >= R.Lkv) return;
  long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
  if (e_i > R.Nkv - 1) e_i = R.Nkv - 1;
  if ((long long)j * g.b > e_i) return;
  const __nv_bfloat16* qb = q + (long long)r * g.qs0 + (long long)p * g.qs1;
  float best = -INFINITY;
  for (int uv = threadIdx.x; uv < g.G * g.G; uv += 256) {
    const int u = uv / g.G, v = uv % g.G;
    const int tq0 = i * g.b + u * g.g, tk0 = j * g.b + v * g.g;
    if (tq0 >= R.Nq || tk0 >= R.Nkv) continue;  // padding-only group (R3)
    float acc = 0.0f;
    for (int t = 0; t < g.g; ++t) {
      if (tq0 + t >= R.Nq || tk0 + t >= R.Nkv) break;  // the rest of the group is padding
      const __nv_bfloat16* x = qb + (long long)(tq0 + t) * g.qs2;
      const __nv_bfloat16* y = k_token(g, k, pt, r, h, tk0 + t);
      float d = 0.0f;
#pragma unroll 4
      for (int cc = 0; cc < D; cc += 8) {
        float xf[8], yf[8];
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(x + cc)), xf);
        bf16x8_to_f32(__ldg(reinterpret_cast<const uint4*>(y + cc)), yf);
#pragma unroll
        for (int e = 0; e < 8; ++e) d = __fmaf_rn(xf[e], yf[e], d);
      }
      acc = __fadd_rn(acc, d);
    }
    best = fmaxf(best, acc);
  }
  for (int o = 16; o; o >>= 1) best = fmaxf(best, __shfl_xor_sync(0xffffffffu, best, o));
  if ((threadIdx.x & 31) == 0) wmax[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = wmax[0];
    for (int w = 1; w < 8; ++w) m = fmaxf(m, wmax[w]);
    S[(((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv + j] = m;
  }
}

}  // namespace

int launch_flatten_scores(const Geom& g, const void* q, const void* k, const int32_t* pt, float* S,
                          cudaStream_t st) {
  dim3 grid((g.Lkv + BJ - 1) / BJ, (g.Lq + BI - 1) / BI, g.B * g.Hq);
  auto qq = static_cast<const __nv_bfloat16*>(q);
  auto kk = static_cast<const __nv_bfloat16*>(k);
  const size_t smem = (size_t)2 * g.G * (BI + BJ) * KP * sizeof(float);
  auto go = [&](auto kern) {
    if (smem > 48 * 1024) cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    kern<<<grid, 256, smem, st>>>(g, qq, kk, pt, S);
  };
  switch (g.G) {
    case 1: go(k_s1_flatten_scores<1>); break;
    case 2: go(k_s1_flatten_scores<2>); break;
    case 4: go(k_s1_flatten_scores<4>); break;
    case 8: go(k_s1_flatten_scores<8>); break;
    default: {  // any other G (> 8): one CTA per block pair
      if (g.Lq > 65535 || (long long)g.B * g.Hq > 65535) return -1;
      const dim3 ga(g.Lkv, g.Lq, g.B * g.Hq);
      if (g.D == 128) k_s1_flatten_scores_any<128><<<ga, 256, 0, st>>>(g, qq, kk, pt, S);
      else k_s1_flatten_scores_any<256><<<ga, 256, 0, st>>>(g, qq, kk, pt, S);
    }
  }
  count_launch();
  return 0;
}

void launch_mean_scores(const Geom& g, const void* q, const void* k, const int32_t* pt, float* qbar, float* kbar,
                        float* S, cudaStream_t st) {
  const long long units = (long long)g.B * g.Hq * g.Lq + (long long)g.B * g.Hkv * g.Lkv;
  const int blocks = (int)((units * 16 + 255) / 256);
  auto qq = static_cast<const __nv_bfloat16*>(q);
  auto kk = static_cast<const __nv_bfloat16*>(k);
  if (g.D == 128)
    k_s1_mean_pool<8><<<blocks, 256, 0, st>>>(g, qq, kk, pt, qbar, kbar);
  else
    k_s1_mean_pool<16><<<blocks, 256, 0, st>>>(g, qq, kk, pt, qbar, kbar);
  count_launch();
  const long long total = (long long)g.B * g.Hq * g.Lq * g.Lkv;
  k_s1_mean_scores<<<(int)((total + 255) / 256), 256, 0, st>>>(g, qbar, kbar, S);
  count_launch();
}

}  // namespace bfla
