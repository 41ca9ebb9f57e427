// pipe_bench.cu — per-SM throughput of the softmax building blocks on B200 (MUFU.EX2, FFMA2, the
// degree-3 exp2 polynomial pair, F2FP pack, FMNMX3).  One CTA per SM, W warps, each warp runs
// independent chains; prints ops per clock per SM.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>

__device__ __forceinline__ float ex2a(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ float2 poly2(float2 x) {
  x.x = fmaxf(x.x, -126.f); x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = __fadd2_rn(x, magic);
  const float2 j = __fadd2_rn(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = __ffma2_rn(j, make_float2(-1.f, -1.f), x);
  float2 p = __ffma2_rn(make_float2(0x1.c34984p-5f, 0x1.c34984p-5f), f, make_float2(0x1.f0dab6p-3f, 0x1.f0dab6p-3f));
  p = __ffma2_rn(p, f, make_float2(0x1.62f51cp-1f, 0x1.62f51cp-1f));
  p = __ffma2_rn(p, f, make_float2(0x1.fff6aep-1f, 0x1.fff6aep-1f));
  return make_float2(__uint_as_float(__float_as_uint(p.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(p.y) + (__float_as_uint(t.y) << 23)));
}
constexpr int CH = 16, IT = 256;
template <int MODE>
__global__ void k(float* out, long long* cyc, float seed) {
  float2 v[CH];
  for (int c = 0; c < CH; ++c) v[c] = make_float2(-0.001f * (threadIdx.x + c), seed - 0.002f * c);
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < IT; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (MODE == 0) { v[c].x = ex2a(v[c].x); v[c].y = ex2a(v[c].y); }            // 2 MUFU
      else if (MODE == 1) v[c] = __ffma2_rn(v[c], make_float2(0.999f, 0.999f), make_float2(-1e-3f, -1e-3f));  // 1 FFMA2
      else if (MODE == 2) { float2 p = poly2(v[c]); v[c] = make_float2(p.x * -1e-3f, p.y * -1e-3f); }
      else if (MODE == 3) { v[c].x = fmaf(v[c].x, 0.999f, -1e-3f); v[c].y = fmaf(v[c].y, 0.999f, -1e-3f); }  // 2 FFMA
      else if (MODE == 4) { uint32_t b; asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(b) : "f"(v[c].y), "f"(v[c].x)); v[c].x = __uint_as_float(b) ; }
      else if (MODE == 5) { float d; asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(v[c].x), "f"(v[c].y), "f"(v[(c+1)%CH].x)); v[c].x = d; }
      else if (MODE == 6) { v[c] = __fadd2_rn(v[c], make_float2(1e-3f, 1e-3f)); }
      else if (MODE == 7) { v[c].x = __uint_as_float(__float_as_uint(v[c].x) + (__float_as_uint(v[c].y) << 23)); }
    }
  }
  long long t1 = clock64();
  float s = 0; for (int c = 0; c < CH; ++c) s += v[c].x + v[c].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(const char* name, int warps, double ops_per_elem_iter) {
  float* o; long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  k<MODE><<<148, warps * 32>>>(o, c, 0.5f);
  k<MODE><<<148, warps * 32>>>(o, c, 0.5f);
  cudaDeviceSynchronize();
  long long h[148]; cudaMemcpy(h, c, sizeof(h), cudaMemcpyDeviceToHost);
  double cy = h[0];
  double ops = (double)warps * 32 * IT * CH * ops_per_elem_iter;
  printf("%-28s warps=%2d  cycles=%8.0f  per-SM ops/clk = %6.2f\n", name, warps, cy, ops / cy);
  cudaFree(o); cudaFree(c);
}
int main() {
  for (int w : {4, 8, 16}) {
    run<0>("MUFU.EX2 (exps)", w, 2);
    run<1>("FFMA2 (fp32 fma)", w, 2);
    run<3>("FFMA scalar (fp32 fma)", w, 2);
    run<2>("poly2 (exps)", w, 2);
    run<4>("F2FP pack (pairs)", w, 1);
    run<5>("FMNMX3", w, 1);
    run<6>("FADD2 (adds)", w, 2);
    run<7>("SHL+IADD", w, 1);
  }
}
