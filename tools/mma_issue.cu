// mma_issue.cu — how deep is the tcgen05.mma issue queue?  One converged warp issues R MMAs
// (M128 x N128 x K16, SS) back to back; we record the clock when the issue loop returns and when the
// commit barrier fires.  If issue-return ~= completion, the issuing warp is paced by execution.
#include <cstdio>
#include <cuda.h>
#include "../paper_2605_12193_b200/csrc/common.cuh"
using namespace bfla;

__global__ void __launch_bounds__(128, 1) k(long long* out, int reps) {
  extern __shared__ __align__(1024) unsigned char raw[];
  unsigned char* sm = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0x3f803f80u;
  if (threadIdx.x == 0) { mbar_init(&bar, 1); fence_barrier_init(); }
  if (warp == 0) tmem_alloc<256>(&slot);
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t id = idesc_bf16(128, 128, 0, 0);
    const uint64_t ad = sdesc_sw128(a, 16, 1024);
    const uint64_t bd = sdesc_sw128(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) umma_f16_ss_warp(tmem, ad, bd, id, r > 0);
    long long t1 = clock64();
    umma_commit_warp(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    if (threadIdx.x == 32) { out[2 * blockIdx.x] = t1 - t0; out[2 * blockIdx.x + 1] = t2 - t0; }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

int main() {
  long long* d; cudaMalloc(&d, 16 * 148);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  for (int reps : {1, 2, 4, 8, 16, 32, 64, 256}) {
    k<<<148, 128, 70000>>>(d, reps);
    k<<<148, 128, 70000>>>(d, reps);
    cudaDeviceSynchronize();
    long long h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("reps=%4d  issue-return %6lld cyc  complete %6lld cyc  (%.1f cyc/MMA)  %s\n", reps, h[0], h[1],
           (double)h[1] / reps, cudaGetErrorString(cudaGetLastError()));
  }
}
