// Check of the tcgen05 A-from-TMEM ("TS") operand layout used by the paired attention kernel:
// P (128 x 128 bf16) is written to TMEM with tcgen05.st as packed bf16x2 (row = lane, column c holds
// elements 2c, 2c+1), V (128 x 128 bf16) sits in SMEM MN-major SW128; D = P V (fp32, TMEM).
// Compares against a host matmul.  Prints max |diff|.
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cuda_bf16.h>
#include "../paper_2605_12193_b200/csrc/common.cuh"
using namespace bfla;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}" ::"r"(d), "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t* r) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
               ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
               "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]) : "memory");
}

__global__ void k(const __nv_bfloat16* P, const __nv_bfloat16* V, float* D) {
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, row = threadIdx.x;
  // V [128 tokens][128 d] -> SMEM MN-major SW128: chunk cc (64 d) at cc*16KB, token row t at t*128 B,
  // 16-byte piece x of the row stored at x ^ (t & 7)
  for (int e = threadIdx.x; e < 128 * 16; e += blockDim.x) {
    const int t = e / 16, x = e % 16, cc = x / 8, xx = x % 8;
    const uint4 v = *reinterpret_cast<const uint4*>(V + t * 128 + x * 8);
    *reinterpret_cast<uint4*>(sm + cc * 16384 + t * 128 + ((xx ^ (t & 7)) << 4)) = v;
  }
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot, lane_addr = (uint32_t)(warp * 32) << 16;
  // P row -> TMEM columns 0..63 (packed pairs)
  for (int c0 = 0; c0 < 64; c0 += 16) {
    uint32_t r[16];
    for (int e = 0; e < 16; ++e) {
      const __nv_bfloat16 lo = P[row * 128 + 2 * (c0 + e)], hi = P[row * 128 + 2 * (c0 + e) + 1];
      r[e] = (uint32_t)__bfloat16_as_ushort(lo) | ((uint32_t)__bfloat16_as_ushort(hi) << 16);
    }
    tmem_st16(tmem + lane_addr + c0, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (threadIdx.x == 0) {
    const uint32_t id = idesc_bf16(128, 128, 0, 1);
    const uint64_t b0 = sdesc_sw128(smem_u32(sm), 16384, 1024);
    for (int kk = 0; kk < 8; ++kk) umma_ts(tmem + 128, tmem + kk * 8, b0 + (uint64_t)((kk * 2048) >> 4), id, kk > 0);
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int c0 = 0; c0 < 128; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + lane_addr + 128 + c0, v);
    tmem_wait_ld();
    for (int e = 0; e < 32; ++e) D[row * 128 + c0 + e] = v[e];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

int main() {
  const int n = 128 * 128;
  __nv_bfloat16 *hP = (__nv_bfloat16*)malloc(n * 2), *hV = (__nv_bfloat16*)malloc(n * 2);
  float* hD = (float*)malloc(n * 4);
  srand(1);
  for (int i = 0; i < n; ++i) { hP[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); hV[i] = __float2bfloat16((rand() % 17 - 8) / 8.0f); }
  __nv_bfloat16 *dP, *dV; float* dD;
  cudaMalloc(&dP, n * 2); cudaMalloc(&dV, n * 2); cudaMalloc(&dD, n * 4);
  cudaMemcpy(dP, hP, n * 2, cudaMemcpyHostToDevice); cudaMemcpy(dV, hV, n * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
  k<<<1, 128, 40000>>>(dP, dV, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(hD, dD, n * 4, cudaMemcpyDeviceToHost);
  double mx = 0;
  for (int i = 0; i < 128; ++i)
    for (int j = 0; j < 128; ++j) {
      double s = 0;
      for (int t = 0; t < 128; ++t) s += (double)__bfloat162float(hP[i * 128 + t]) * __bfloat162float(hV[t * 128 + j]);
      mx = fmax(mx, fabs(s - hD[i * 128 + j]));
    }
  printf("TS MMA (P from TMEM, V MN-major SMEM): max |diff| = %g  (%s)\n", mx, cudaGetErrorString(e));
  return 0;
}
