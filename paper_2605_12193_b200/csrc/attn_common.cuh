// attn_common.cuh — helpers shared by the attention kernels (attention.cu, attention2.cu).
#pragma once
#include "common.cuh"

namespace bfla {
namespace attn {

struct Item {
  int r, h, c, i;
};

// split-KV: first index of an ascending kept-tile list (n entries) whose tile is >= x
__device__ __forceinline__ int list_lower_bound(const int32_t* l, int n, int x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(l + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ float max3f(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}

// max of 64 row values: four independent 3-input chains (FMNMX3), then their max
__device__ __forceinline__ float row_max64(const float* v) {
  float mc[4];
#pragma unroll
  for (int k4 = 0; k4 < 4; ++k4) {
    float a = max3f(v[16 * k4], v[16 * k4 + 1], v[16 * k4 + 2]);
#pragma unroll
    for (int c = 3; c < 15; c += 2) a = max3f(a, v[16 * k4 + c], v[16 * k4 + c + 1]);
    mc[k4] = fmaxf(a, v[16 * k4 + 15]);
  }
  return fmaxf(max3f(mc[0], mc[1], mc[2]), mc[3]);
}

// 2^x for a pair on the FMA pipe: x = j + f with j = rint(x) (magic-number rounding, f in [-1/2, 1/2]),
// 2^f by a degree-3 polynomial (relative error 7.7e-5), 2^j folded into the exponent bits.
// x is clamped at -126 so the exponent field cannot wrap: masked entries (-inf) give a denormal ~2^-126.
__device__ __forceinline__ float2 exp2_poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);  // 1.5 * 2^23
  const float2 t = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0x1.c34984p-5f, 0x1.c34984p-5f), f, make_float2(0x1.f0dab6p-3f, 0x1.f0dab6p-3f));
  p = __ffma2_rn(p, f, make_float2(0x1.62f51cp-1f, 0x1.62f51cp-1f));
  p = __ffma2_rn(p, f, make_float2(0x1.fff6aep-1f, 0x1.fff6aep-1f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
// Work slice [row0, row0 + nrows) of the item order (bfla_sparse_prefill_rows): executed in descending i
// with the slice's (r, h) segments interleaved, so the longest rows still go first.  Compiled only into
// the SLICE kernel instances: a runtime branch in the unsliced kernels cost them 1.5 % (measured).
__device__ __forceinline__ Item decode_slice(const Geom& g, int idx, int NC) {
  Item it;
  it.c = idx % NC;
  const int k = idx / NC, Tq = g.Tq;
  const int r0 = g.row0, r1 = g.row0 + g.nrows - 1;
  const int s_lo = r0 / Tq, s_hi = r1 / Tq, nmid = s_hi - s_lo > 1 ? s_hi - s_lo - 1 : 0;
  const int i_start = Tq - 1 - r0 % Tq, i_end = Tq - 1 - r1 % Tq;
  const int lo0 = s_lo == s_hi ? i_end : 0;  // segment s_lo holds i in [lo0, i_start]
  // F(i) = slice rows with query tile >= i
  auto F = [&](int i) {
    int n = max(0, i_start - max(i, lo0) + 1) + nmid * (Tq - i);
    if (s_hi != s_lo) n += Tq - max(i, i_end);
    return n;
  };
  int lo = 0, hi = Tq - 1;  // largest i with F(i) > k
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (F(mid) > k) lo = mid;
    else hi = mid - 1;
  }
  int j = k - (lo + 1 < Tq ? F(lo + 1) : 0);  // rank of the row among the segments holding tile lo
  int seg;
  if (lo >= lo0 && lo <= i_start && j == 0) seg = s_lo;
  else {
    if (lo >= lo0 && lo <= i_start) --j;
    seg = j < nmid ? s_lo + 1 + j : s_hi;
  }
  it.i = lo;
  it.h = seg % g.Hkv;
  it.r = seg / g.Hkv;
  return it;
}

template <bool SLICE>
__device__ __forceinline__ Item decode_item(const Geom& g, int idx, int NC) {
  // order: (r, h) major, query tile descending (longest rows first: LPT proxy), chunk inner
  if constexpr (SLICE) return decode_slice(g, idx, NC);
  Item it;
  it.c = idx % NC;
  int rest = idx / NC;
  it.i = g.Tq - 1 - rest % g.Tq;
  rest /= g.Tq;
  it.h = rest % g.Hkv;
  it.r = rest / g.Hkv;
  return it;
}


__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
#ifdef BFLA_WHATIF_NOSTORE  // timing what-if (A/B builds only): P never written to TMEM
  if (r[0] != 0x12345u) return;
#endif
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
      "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* r) {
#ifdef BFLA_WHATIF_NOSTORE
  if (r[0] != 0x12345u) return;
#endif
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}

// D[tmem] (+)= A[tmem] * B[smem]  (kind::f16, A from tensor memory: row = lane, 2 bf16 per column),
// issued by one elected lane of a converged warp.
__device__ __forceinline__ void umma_f16_ts_warp(uint32_t d_tmem, uint32_t a_tmem, uint64_t b_desc, uint32_t idesc,
                                                 uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b_desc), "r"(idesc), "r"(accumulate)
      : "memory");
}

}  // namespace attn
}  // namespace bfla
