// stage2.cu — Stage 2 of BFLA (Eq. 19-26): expansion of the coarse keep mask to the
// T-tile grid, tile causality, local band, sink, stride and random rescue, final union, and the
// compacted kept-tile lists that drive the sparse prefill kernel.  Integer only.
#include "common.cuh"
#include "kernels.h"

namespace bfla {

// chi / psi of Eq. 24-25 (R15): SplitMix64 finalizer over the packed (i, j) key; psi folds in the
// global KV head index.  Bit-identical definitions are pinned in DESIGN.md §4 item 8.
__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ULL;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebULL;
  x ^= x >> 31;
  return x;
}

// Exact divisibility test chi mod eta == 0 without a 64-bit division (Hacker's Delight 10-17): with
// eta = e0 * 2^k, e0 odd and e0_inv its inverse mod 2^64, x is a multiple of eta iff
// rotr(x * e0_inv, k) <= floor((2^64 - 1) / eta).  (A runtime 64-bit urem is ~100 instructions per
// tile; this is a multiply and a compare.)
struct Div64 {
  uint64_t inv, lim;
  int k;
};
__device__ __forceinline__ bool divisible(uint64_t x, const Div64& d) {
  const uint64_t y = x * d.inv;
  const uint64_t r = d.k ? ((y >> d.k) | (y << (64 - d.k))) : y;
  return r <= d.lim;
}

// One warp per (request r, KV head h, query tile i).  Labels (precedence mass > sink > band >
// stride > random, R13): 1 mass (Eq. 20), 2 sink (Eq. 22), 3 band (Eq. 21), 4 stride (Eq. 24),
// 5 random (Eq. 25); 0 = dropped or non-causal.  The kept list of row (r,h,i) is written in
// ascending j at its closed-form causal offset, so rows need no global scan.
__global__ void __launch_bounds__(256) k_s2_expand_rescue(Geom g, const uint32_t* __restrict__ coarse,
                                                          int n_sink, int n_local, int eta, Div64 deta, double rho,
                                                          uint64_t seed, uint32_t* __restrict__ tile_bits,
                                                          int32_t* __restrict__ list, int32_t* __restrict__ count,
                                                          uint8_t* __restrict__ label,
                                                          unsigned long long* __restrict__ stats) {
  __shared__ unsigned long long bsum[8];  // block sums of stats[0..7] (one atomic per counter and block)
  if (threadIdx.x < 8) bsum[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long row = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const long long nrows = (long long)g.B * g.Hkv * g.Tq;
  auto body = [&]() {
  if (row >= nrows) return;
  const int i = (int)(row % g.Tq);
  const int h = (int)((row / g.Tq) % g.Hkv);
  const int r = (int)(row / ((long long)g.Tq * g.Hkv));
  const Req R = req_of(g, r);  // this request's logical dims (varlen); g.* is the buffer layout
  if (i >= R.Tq) {             // padding row of a shorter request: empty
    for (int w = lane; w < g.Tw; w += 32) tile_bits[row * g.Tw + w] = 0u;
    if (label)
      for (int j = lane; j < g.Tkv; j += 32) label[row * g.Tkv + j] = 0;
    if (lane == 0) count[row] = 0;
    return;
  }
  // Eq. 11-13 at tile size T: causal iff jT <= min(N_c + (i+1)T - 1, N_kv - 1)
  const long long fr = (long long)R.Nc + (long long)(i + 1) * g.T - 1;
  const int jmax = (int)((fr < R.Nkv - 1 ? fr : (long long)R.Nkv - 1) / g.T);
  // R11: band = [max(0, d_i - n_local), d_i], d_i = min(floor(fr / T), Tkv - 1)
  int d_i = (int)(fr / g.T);
  if (d_i > R.Tkv - 1) d_i = R.Tkv - 1;
  const int band_lo = d_i - n_local > 0 ? d_i - n_local : 0;
  const int rbs = __ffs(g.rb) - 1;  // rho_b = b / T is a power of two: j / rho_b = j >> rbs
  const uint32_t* crow = coarse + ((long long)(r * g.Hkv + h) * g.Lq + (i >> rbs)) * g.Lw;
  int32_t* lrow = list + (long long)(r * g.Hkv + h) * g.causal_per_head + req_row_offset(R, g.T, i);
  const uint64_t hglob = (uint64_t)(g.head_offset + h);
  int nk = 0;
  unsigned cnt[6] = {0, 0, 0, 0, 0, 0};
  // the coarse row in registers, one word per lane (Lw <= 32, i.e. up to 1024 blocks), read by shuffle
  const bool creg = g.Lw <= 32;
  const uint32_t cw = (creg && lane < g.Lw) ? __ldg(crow + lane) : 0u;
  // words wholly past the causal frontier are zero: written lane-parallel below, not walked here
  const int jend = label ? g.Tkv : ((jmax >> 5) + 1) << 5;
  for (int w = (jmax >> 5) + 1 + lane; !label && w < g.Tw; w += 32) tile_bits[row * g.Tw + w] = 0u;
  for (int j0 = 0; j0 < jend; j0 += 32) {
    const int j = j0 + lane;
    int lab = 0;
    const int J = j >> rbs;
    const uint32_t word = creg ? __shfl_sync(0xffffffffu, cw, (J >> 5) & 31) : (j <= jmax ? crow[J >> 5] : 0u);
    if (j <= jmax) {
      if ((word >> (J & 31)) & 1u) {
        lab = 1;
      } else if (j < n_sink) {
        lab = 2;
      } else if (j >= band_lo && j <= d_i) {
        lab = 3;
      } else {
        const uint64_t key = ((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)j;
        if (eta > 0 && divisible(mix64(key ^ seed), deta)) {
          lab = 4;
        } else if (rho > 0.0) {
          const uint64_t z = mix64(mix64(key ^ seed ^ 0xD1B54A32D192ED03ULL) ^ (hglob * 0x9E3779B97F4A7C15ULL));
          if ((double)(z >> 11) * 0x1p-53 < rho) lab = 5;
        }
      }
    }
    const uint32_t bal = __ballot_sync(0xffffffffu, lab != 0);
    if (lane == 0) tile_bits[row * g.Tw + (j0 >> 5)] = bal;
    if (lab) lrow[nk + __popc(bal & ((1u << lane) - 1u))] = j;
    nk += __popc(bal);
    if (label && j < g.Tkv) label[row * g.Tkv + j] = (uint8_t)lab;
    cnt[lab]++;
  }
  if (lane == 0) count[row] = nk;
  if (stats) {
#pragma unroll
    for (int l = 1; l < 6; ++l) {
      unsigned v = cnt[l];
      for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if (lane == 0 && v) atomicAdd(&bsum[2 + l], (unsigned long long)v);
    }
    if (lane == 0) {
      atomicAdd(&bsum[0], (unsigned long long)(jmax + 1));  // causal tiles of this row
      atomicAdd(&bsum[1], (unsigned long long)nk);
    }
  }
  };
  body();
  __syncthreads();
  if (stats && threadIdx.x < 8 && bsum[threadIdx.x]) atomicAdd(stats + threadIdx.x, bsum[threadIdx.x]);
}

void launch_expand_rescue(const Geom& g, const uint32_t* coarse, int n_sink, int n_local, int eta, double rho,
                          uint64_t seed, uint32_t* tile_bits, int32_t* list, int32_t* count, uint8_t* label,
                          unsigned long long* stats, cudaStream_t st) {
  const long long rows = (long long)g.B * g.Hkv * g.Tq;
  const int blocks = (int)((rows + 7) / 8);
  Div64 d{1, ~0ull, 0};
  if (eta > 0) {
    uint64_t e0 = (uint64_t)eta;
    d.k = 0;
    while (!(e0 & 1)) {
      e0 >>= 1;
      ++d.k;
    }
    uint64_t inv = e0;  // Newton: each step doubles the correct low bits (e0 * e0 = 1 mod 8 to start)
    for (int it = 0; it < 6; ++it) inv *= 2 - e0 * inv;
    d.inv = inv;
    d.lim = ~0ull / (uint64_t)eta;
  }
  k_s2_expand_rescue<<<blocks, 256, 0, st>>>(g, coarse, n_sink, n_local, eta, d, rho, seed, tile_bits, list,
                                               count, label, stats);
  count_launch();
}

}  // namespace bfla
