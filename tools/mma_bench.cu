// Microbenchmark: cycles per tcgen05.mma (kind::f16, cta_group::1, SS operands) for the shapes the
// attention and Stage-1 kernels use.  One CTA per SM, one thread issues `reps` MMAs back to back into
// one TMEM accumulator, commits, waits; reports cycles per MMA.  Operand contents are irrelevant.
#include <cstdio>
#include <cuda.h>
#include "../paper_2605_12193_b200/csrc/common.cuh"
using namespace bfla;

template <int N, int BMN>
__global__ void __launch_bounds__(128, 1) k_bench(long long* out, int reps) {
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
  if (threadIdx.x == 32) {
    const uint32_t a = smem_u32(sm), b = smem_u32(sm + 32768);
    constexpr uint32_t id = idesc_bf16(128, N, 0, BMN);
    const uint64_t ad = sdesc_sw128(a, 16, 1024);
    const uint64_t bd = BMN ? sdesc_sw128(b, 8192, 1024) : sdesc_sw128(b, 16, 1024);
    long long t0 = clock64();
    for (int r = 0; r < reps; ++r) umma_f16_ss(tmem, ad, bd, id, r > 0);
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t1 = clock64();
    out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc<256>(tmem); }
}

template <int N, int BMN>
void run(const char* name, int sms) {
  long long* d; cudaMalloc(&d, sizeof(long long) * sms);
  long long h[256];
  const int reps = 4096;
  cudaFuncSetAttribute(k_bench<N, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
  k_bench<N, BMN><<<sms, 128, 70000>>>(d, reps);
  k_bench<N, BMN><<<sms, 128, 70000>>>(d, reps);
  cudaDeviceSynchronize();
  cudaMemcpy(h, d, sizeof(long long) * sms, cudaMemcpyDeviceToHost);
  double s = 0; for (int i = 0; i < sms; ++i) s += h[i];
  const double cyc = s / sms / reps, ideal = 128.0 * N / 256.0;
  printf("%-28s N=%3d  %7.1f cycles/MMA  (ideal %5.1f, %.0f%%)  err=%s\n", name, N, cyc, ideal, 100 * ideal / cyc,
         cudaGetErrorString(cudaGetLastError()));
  cudaFree(d);
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<64, 0>("S: K-major A,B", sms);
  run<128, 0>("K-major A,B", sms);
  run<256, 0>("K-major A,B", sms);
  run<128, 1>("PV: A K-major, B MN-major", sms);
  run<256, 1>("PV: A K-major, B MN-major", sms);
  run<64, 0>("S (1 SM only)", 1);
  return 0;
}
