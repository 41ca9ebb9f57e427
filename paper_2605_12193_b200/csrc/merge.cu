// merge.cu — split-KV combination: rows whose kept tiles were split into KV ranges
// (bfla_sparse_prefill_kvrange) are assembled exactly as one online softmax over the union would end:
// with l_k = exp(LSE_k - M), M = max_k LSE_k,  O = sum_k l_k O_k / sum_k l_k  and  LSE = M + log sum_k l_k
// (each O_k is its range's normalised output, Eq. 27 restricted to the range's tiles).
#include <cuda_bf16.h>

#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {

// thread = one 16-byte chunk (8 channels) of one (request, query head, token) row
__global__ void __launch_bounds__(256) k_merge_partials(Geom g, MergeParts mp, __nv_bfloat16* __restrict__ O,
                                                        float* __restrict__ lse) {
  const int per_row = g.D / 8;
  const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long rows = (long long)g.B * g.Hq * g.Nq;
  if (idx >= rows * per_row) return;
  const int c8 = (int)(idx % per_row);
  const long long row = idx / per_row;
  const int t = (int)(row % g.Nq), p = (int)((row / g.Nq) % g.Hq), r = (int)(row / ((long long)g.Nq * g.Hq));
  if (g.lens && t >= __ldg(g.lens + 2 * r)) return;  // varlen padding rows stay untouched
  const long long li = ((long long)r * g.Hq + p) * g.Nq + t;
  const long long oi = (long long)r * g.os0 + (long long)p * g.os1 + (long long)t * g.os2 + c8 * 8;
  float M = -INFINITY;
  for (int k = 0; k < mp.n; ++k) M = fmaxf(M, __ldg(mp.lse[k] + li));
  float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f}, wsum = 0.f;
  if (M > -INFINITY) {
    for (int k = 0; k < mp.n; ++k) {
      const float lk = __ldg(mp.lse[k] + li);
      if (lk == -INFINITY) continue;  // no kept tile of this row in range k
      const float w = __expf(lk - M);
      wsum += w;
      const uint4 u = __ldg(reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(mp.o[k]) + oi));
      const uint32_t ww[4] = {u.x, u.y, u.z, u.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        acc[2 * e] += w * __uint_as_float(ww[e] << 16);
        acc[2 * e + 1] += w * __uint_as_float(ww[e] & 0xffff0000u);
      }
    }
  }
  const float inv = wsum > 0.f ? 1.0f / wsum : 0.f;
  uint32_t out[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) out[e] = pack_bf16x2(acc[2 * e] * inv, acc[2 * e + 1] * inv);
  *reinterpret_cast<uint4*>(O + oi) = make_uint4(out[0], out[1], out[2], out[3]);
  if (lse && c8 == 0) lse[li] = M > -INFINITY ? M + logf(wsum) : -INFINITY;
}

}  // namespace

int launch_merge_partials(const Geom& g, const MergeParts& mp, void* o, float* lse, cudaStream_t st) {
  const long long n = (long long)g.B * g.Hq * g.Nq * (g.D / 8);
  if (n <= 0) return 0;
  k_merge_partials<<<(int)((n + 255) / 256), 256, 0, st>>>(g, mp, static_cast<__nv_bfloat16*>(o), lse);
  count_launch();
  return (int)cudaGetLastError();
}

}  // namespace bfla
