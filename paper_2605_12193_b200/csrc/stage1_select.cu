// stage1_select.cu — Stage 1 selection of BFLA (Eq. 13-18 + the GQA union):
// causal block mask, block softmax with alpha = 1/sqrt(C), keep-mass (or keep-ratio) selection,
// OR over each head group H_h.  Canonical fp32 arithmetic: every rounding below
// is an explicit IEEE round-to-nearest intrinsic and this translation unit is compiled with
// -fmad=false, so the device computes exactly the canonical value sequence.
#include "common.cuh"
#include "kernels.h"

namespace bfla {

// Canonical exp2 for t <= 0 (DESIGN.md §4 item 5): n = floor(t), f = t - n, degree-6 Horner
// polynomial (fp32 FMA, coefficients = Chebyshev fit rounded to fp32), scaled by 2^n (exact).
__device__ __forceinline__ float exp2_canon(float t) {
  if (t < -126.0f) return 0.0f;
  const float fl = floorf(t);
  const int n = (int)fl;
  const float f = __fsub_rn(t, fl);
  float p = 0x1.cacdfep-13f;
  p = __fmaf_rn(p, f, 0x1.44bd4cp-10f);
  p = __fmaf_rn(p, f, 0x1.3d5822p-7f);
  p = __fmaf_rn(p, f, 0x1.c67ee4p-5f);
  p = __fmaf_rn(p, f, 0x1.ebfdf8p-3f);
  p = __fmaf_rn(p, f, 0x1.62e428p-1f);
  p = __fmaf_rn(p, f, 0x1p+0f);
  return __fmul_rn(p, __int_as_float((n + 127) << 23));
}

// 64-bit warp max with two redux.sync reductions: the largest high word, then the largest low word
// among the lanes holding it (the same value as a shuffle tree, in 2 instead of 10 shuffles)
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
  const uint32_t hi = (uint32_t)(v >> 32);
  const uint32_t mh = __reduce_max_sync(0xffffffffu, hi);
  const uint32_t ml = __reduce_max_sync(0xffffffffu, hi == mh ? (uint32_t)v : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

// Selection of one head row (r, p, i) by one warp (Eq. 13-18):
//   1. M = max over causal j of S_j (exact);  t_j = (S_j - M) * c_alpha (two roundings);
//      e_j = exp2_canon(t_j);  Z = sum_j e_j sequentially (lane 0, ascending j);  A_j = e_j / Z.
//   2. Repeated extraction of the largest key (A_j bits, ~j): visits the blocks in exactly the order
//      (A desc, j asc) (R6); the prefix P_r is accumulated in that order, one fp32 add per step (R7),
//      until P_r >= gamma (MASS) or r = ceil(ratio n_causal) (RATIO).  gamma >= 1 keeps all causal
//      blocks.  Kept blocks end with keys[j] == 0.
//   3. certify (mode 1 only): with |S_f - S_c| <= delta_j = tau qn kn_j, the decision is provably the
//      canonical one iff
//        order: min over kept (S_f - delta) > max over dropped (S_f + delta), with a margin that keeps
//               the canonical probabilities distinct (no tie can appear at the cut), and the last kept
//               block is far from exp2 underflow;
//        mass : P_r* - gamma and gamma - P_{r*-1} exceed (e^eta - 1)(P(1-P) + 2^-20) + (4n+64) 2^-24,
//               eta = 2 ln2 c_alpha max_j delta_j (a uniform logit shift cancels; the prefix moves by at
//               most P(1-P)(e^eta - 1)), plus the fp32 rounding of either evaluation.
struct RowResult {
  int nsel;
  float P;
  bool tie, certified;
  float M, dmax;  // fast row max and largest score-error bound (mode 1)
  float s_cut;    // RATIO: fast score of the last kept block (mode 1)
  float band_lo, band_hi;  // RATIO, uncertified row: fast-score band that needs canonical scores
};

// Order-preserving uint32 key of a float (larger float -> larger key).
__device__ __forceinline__ uint32_t okey(float x) {
  const uint32_t u = __float_as_uint(x);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float okey_inv(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}
// k-th largest of f(j), j < nc, over a warp (bisection on the order-preserving keys: 32 rounds).
template <class F>
__device__ float warp_kth_largest(int nc, int k, F f) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0u, hi = 0xffffffffu;  // largest key t with #{j : key_j >= t} >= k
  while (lo < hi) {
    const uint32_t mid = lo + (uint32_t)(((unsigned long long)hi - lo + 1ull) >> 1);
    int cnt = 0;
    for (int j = lane; j < nc; j += 32) cnt += okey(f(j)) >= mid;
#pragma unroll
    for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (cnt >= k) lo = mid;
    else hi = mid - 1u;
  }
  return okey_inv(lo);
}

__device__ RowResult select_row(const Geom& g, const float* __restrict__ s, int nc, float c_alpha, int select,
                                float gamma, float keep_ratio, unsigned long long* keys, bool certify, float qnorm,
                                const float* __restrict__ knrow, float tau, bool need_p = true) {
  const int lane = threadIdx.x & 31;
  // the block softmax (Eq. 15) is needed for MASS and for the kept mass; RATIO without it ranks by S
  const bool soft = select == 0 || need_p;
  float M = -INFINITY;
  for (int j = lane; j < nc; j += 32) M = fmaxf(M, s[j]);
#pragma unroll
  for (int o = 16; o; o >>= 1) M = fmaxf(M, __shfl_xor_sync(0xffffffffu, M, o));
  float* e = reinterpret_cast<float*>(keys);  // reuse the key area for e_j (nc floats)
  float Z = 0.0f;
  if (soft) {
    for (int j = lane; j < nc; j += 32) e[j] = exp2_canon(__fmul_rn(__fsub_rn(s[j], M), c_alpha));
    __syncwarp();
    if (lane == 0)
      for (int j = 0; j < nc; ++j) Z = __fadd_rn(Z, e[j]);
    Z = __shfl_sync(0xffffffffu, Z, 0);
    __syncwarp();
  }
  // keys: (A bits << 32) | ~j — larger key = larger A, then smaller j (MASS, R6).  RATIO (R9) ranks
  // by the score instead — the block softmax is monotone in S, so this is the top-k by probability
  // without the ties fp32 underflow of A would create: (order-preserving bits of S << 32) | ~j.
  // Built back to front so the float area (aliasing the low half of the key array) is read before
  // it is overwritten.
  const bool by_score = select == 1;
  for (int j0 = ((nc - 1) / 32) * 32; j0 >= 0; j0 -= 32) {
    const int j = j0 + lane;
    uint32_t hi = 0u;
    if (j < nc) {
      if (by_score) {
        const uint32_t u = __float_as_uint(s[j]);
        hi = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
      } else {
        hi = __float_as_uint(__fdiv_rn(e[j], Z));
      }
    }
    __syncwarp();
    if (j < nc) keys[j] = ((unsigned long long)hi << 32) | (unsigned long long)(~(uint32_t)j);
    __syncwarp();
  }
  int target = nc;
  if (select == 1) {
    double want = ceil((double)keep_ratio * (double)nc);
    target = (int)want;
    if (target < 1) target = 1;
    if (target > nc) target = nc;
  }
  const bool keep_all = (select == 0 && gamma >= 1.0f);
  certify = certify && !keep_all;
  float P = 0.0f, a_last = 0.0f, P_prev = 0.0f, kept_lo = INFINITY, t_last = 0.0f, s_last = 0.0f;
  uint32_t key_last = 0u;
  int nsel = 0;
  bool tie_fast = false, fast = false;
  if (select == 1 && !need_p) {
    // RATIO without the kept mass: the top-k set directly (no extraction loop).  The k-th largest
    // score key by bisection, every block above it, then the smallest-j blocks at that key — the
    // (S desc, j asc) order of the extraction; a block left at that key is the tie at the cut.
    fast = true;
    const float kth = warp_kth_largest(nc, target, [&](int j) { return s[j]; });
    const uint32_t kk = okey(kth);
    int gt = 0, eq = 0;
    for (int j = lane; j < nc; j += 32) {
      const uint32_t kj = okey(s[j]);
      gt += kj > kk;
      eq += kj == kk;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      gt += __shfl_xor_sync(0xffffffffu, gt, o);
      eq += __shfl_xor_sync(0xffffffffu, eq, o);
    }
    int need = target - gt;  // blocks taken at the cut key, smallest j first
    for (int j0 = 0; j0 < nc; j0 += 32) {
      const int j = j0 + lane;
      const uint32_t kj = j < nc ? okey(s[j]) : 0u;
      const uint32_t at = __ballot_sync(0xffffffffu, j < nc && kj == kk);
      const int rank = __popc(at & ((1u << lane) - 1u));
      const bool take = j < nc && (kj > kk || (kj == kk && rank < need));
      need -= __popc(at) < need ? __popc(at) : need;
      if (take) {
        keys[j] = 0ull;
        if (certify) kept_lo = fminf(kept_lo, s[j] - tau * qnorm * knrow[j]);
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) kept_lo = fminf(kept_lo, __shfl_xor_sync(0xffffffffu, kept_lo, o));
    __syncwarp();
    nsel = target;
    key_last = kk;
    tie_fast = eq > target - gt;
    s_last = kth;
  }
  while (!fast && nsel < nc) {
    unsigned long long best = 0ull;
    for (int j = lane; j < nc; j += 32) best = keys[j] > best ? keys[j] : best;
    best = warp_max_u64(best);
    const int jsel = (int)(~(uint32_t)(best & 0xffffffffull));
    // A of the extracted block: the key itself (MASS) or recomputed exactly as above (RATIO)
    a_last = by_score ? __fdiv_rn(exp2_canon(__fmul_rn(__fsub_rn(s[jsel], M), c_alpha)), Z)
                      : __uint_as_float((uint32_t)(best >> 32));
    key_last = (uint32_t)(best >> 32);
    P_prev = P;
    P = __fadd_rn(P, a_last);
    ++nsel;
    if (certify) {
      const float sj = s[jsel];
      kept_lo = fminf(kept_lo, sj - tau * qnorm * knrow[jsel]);
      t_last = (sj - M) * c_alpha;
      s_last = sj;
    }
    if (lane == 0) keys[jsel] = 0ull;
    __syncwarp();
    if (keep_all) continue;
    if (select == 0 ? (P >= gamma) : (nsel >= target)) break;
  }
  RowResult res{nsel, P, false, true, M, 0.f, 0.f, 0.f, 0.f};
  if (fast) {
    res.tie = tie_fast;
  } else if (nsel < nc) {  // a tie at the cut (R6): the next block in order has the same probability
    unsigned long long best = 0ull;
    for (int j = lane; j < nc; j += 32) best = keys[j] > best ? keys[j] : best;
    best = warp_max_u64(best);
    res.tie = (uint32_t)(best >> 32) == key_last;
  }
  if (certify) {
    float drop_hi = -INFINITY, dmax = 0.f;
    for (int j = lane; j < nc; j += 32) {
      const float dj = tau * qnorm * knrow[j];
      dmax = fmaxf(dmax, dj);
      if (keys[j] != 0ull) drop_hi = fmaxf(drop_hi, s[j] + dj);
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      drop_hi = fmaxf(drop_hi, __shfl_xor_sync(0xffffffffu, drop_hi, o));
      dmax = fmaxf(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
    }
    bool ok = true;
    if (select == 1) {
      // RATIO: only the order of the scores at the cut matters (strict separation, with room for the
      // fp32 rounding of S_f -/+ delta)
      if (nsel < nc) ok = kept_lo - drop_hi > 0x1p-22f * (fabsf(kept_lo) + fabsf(drop_hi)) + 1e-30f;
    } else {
      if (nsel < nc) ok = (kept_lo - drop_hi) * c_alpha > 0x1p-18f;  // order of the cut
      if (t_last - 2.0f * c_alpha * dmax < -120.0f) ok = false;     // kept block near exp2 underflow
    }
    if (select == 0) {
      const float eta = 2.0f * 0.6931472f * c_alpha * dmax;
      const float grow = expm1f(eta);
      const float rnd = (4.0f * nc + 64.0f) * 0x1p-24f;
      auto marg = [&](float x) { return grow * (x * (1.0f - x) + 0x1p-20f) + rnd; };
      if (P >= gamma) {
        if (!(P - gamma > marg(P))) ok = false;
        if (!(gamma - P_prev > marg(P_prev))) ok = false;
      } else {  // the prefix never reached gamma: keep-all must also hold canonically
        if (!(gamma - P > marg(P))) ok = false;
      }
    }
    res.certified = ok;
    res.dmax = dmax;
    res.s_cut = s_last;
    if (select == 1 && !ok) {
      // Recompute band of an uncertified RATIO row.  Canonical scores c_j lie in [S_j - d_j, S_j + d_j]
      // (d_j = tau |q| |k_j|), so the canonical k-th score c* lies in [L, U] with L / U the k-th largest
      // of S_j - d_j / S_j + d_j (order statistics are monotone).  With d_b = max d_j over the blocks
      // whose S_j lies in [L - dmax, U + dmax]: S_j > U + d_b implies c_j > c* and S_j < L - d_b implies
      // c_j < c* (a block with d_j > d_b lies outside [L - dmax, U + dmax]), so only [L - d_b, U + d_b]
      // needs canonical scores; outside it the mixed row ranks exactly like the canonical one (c* is
      // attained inside the band, every outside value is strictly above or below it).  The per-block d_j
      // keeps one large-norm block (an attention sink) from widening every row's band.
      const float U = warp_kth_largest(nc, nsel, [&](int j) { return s[j] + tau * qnorm * knrow[j]; });
      const float L = warp_kth_largest(nc, nsel, [&](int j) { return s[j] - tau * qnorm * knrow[j]; });
      float db = 0.f;
      for (int j = lane; j < nc; j += 32)
        if (s[j] >= L - dmax && s[j] <= U + dmax) db = fmaxf(db, tau * qnorm * knrow[j]);
#pragma unroll
      for (int o = 16; o; o >>= 1) db = fmaxf(db, __shfl_xor_sync(0xffffffffu, db, o));
      db *= 1.0f + 0x1p-10f;  // fp32 rounding of S_j -/+ d_j and of the products
      res.band_lo = L - db - 0x1p-20f * fabsf(L);
      res.band_hi = U + db + 0x1p-20f * fabsf(U);
    }
  }
  return res;
}

// OR the kept blocks (keys[j] == 0) of one head row into a coarse row (smem or global).
__device__ __forceinline__ void or_kept(const unsigned long long* keys, int nc, uint32_t* row) {
  const int lane = threadIdx.x & 31;
  for (int j0 = 0; j0 < nc; j0 += 32) {
    const int j = j0 + lane;
    const uint32_t bal = __ballot_sync(0xffffffffu, j < nc && keys[j] == 0ull);
    if (lane == 0 && bal) atomicOr(row + (j0 >> 5), bal);
  }
}

// mode 0: S holds canonical scores; one CTA per (r, h, i), warp w handles query heads p = h m + w,
//         h m + w + nwarps, ...; the OR over H_h (R8) is built in smem and written once.
// mode 1: S holds tensor-core scores; the same, but a head row that fails certification is not OR-ed:
//         its id (r * Hq + p) * Lq + i is appended to `flagged` for the canonical recompute.
// mode 2: grid-stride over the flagged head rows (S now canonical for them); each row's kept bits are
//         OR-ed atomically into the already written coarse row (OR is order independent).
__global__ void __launch_bounds__(128) k_s1_select(Geom g, const float* __restrict__ S, float c_alpha, int select,
                                                   float gamma, float keep_ratio, uint32_t* __restrict__ coarse,
                                                   float* __restrict__ kept_mass,
                                                   unsigned long long* __restrict__ stats, int mode,
                                                   const float* __restrict__ qn, const float* __restrict__ kn,
                                                   float tau, int32_t* __restrict__ flagged,
                                                   int32_t* __restrict__ n_flagged, int32_t* __restrict__ ulist) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int nwarps = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t* row_bits = reinterpret_cast<uint32_t*>(smem);  // [Lw]
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + ((g.Lw * 4 + 15) / 16) * 16) +
                             (size_t)warp * g.Lkv;  // [nwarps][Lkv]
  unsigned rows = 0, ties = 0, kept_sum = 0, unc = 0, recomputed = 0;
  if (mode == 2) {
    const int nf = *n_flagged;
    for (int f = blockIdx.x * nwarps + warp; f < nf; f += gridDim.x * nwarps) {
      const int row = flagged[f];
      const int i = row % g.Lq, p = (row / g.Lq) % g.Hq, r = row / (g.Lq * g.Hq), h = p / g.m;
      const Req R = req_of(g, r);
      const long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
      const int nc = (int)((e_i < R.Nkv - 1 ? e_i : (long long)R.Nkv - 1) / g.b) + 1;
      const float* s = S + (((long long)r * g.Hq + p) * g.Lq + i) * g.Lkv;
      const RowResult res =
          select_row(g, s, nc, c_alpha, select, gamma, keep_ratio, keys, false, 0.f, nullptr, 0.f, false);
      or_kept(keys, nc, coarse + ((long long)(r * g.Hkv + h) * g.Lq + i) * g.Lw);
      rows++, recomputed++;
      ties += res.tie;
      kept_sum += res.nsel;
      __syncwarp();
    }
  } else {
    const int i = blockIdx.x % g.Lq;
    const int h = (blockIdx.x / g.Lq) % g.Hkv;
    const int r = blockIdx.x / (g.Lq * g.Hkv);
    for (int w = threadIdx.x; w < g.Lw; w += blockDim.x) row_bits[w] = 0u;
    __syncthreads();
    const Req R = req_of(g, r);  // this request's logical dims (varlen); g.* is the buffer layout
    const long long e_i = (long long)R.Nc + (long long)(i + 1) * g.b - 1;
    const int nc = (int)((e_i < R.Nkv - 1 ? e_i : (long long)R.Nkv - 1) / g.b) + 1;  // causal blocks
    for (int pl = warp; pl < (i < R.Lq ? g.m : 0); pl += nwarps) {  // padding rows stay empty
      const int p = h * g.m + pl;
      const long long rowid = ((long long)r * g.Hq + p) * g.Lq + i;
      const float* s = S + rowid * g.Lkv;
      const bool cert = mode == 1;
      const RowResult res = select_row(g, s, nc, c_alpha, select, gamma, keep_ratio, keys, cert,
                                       cert ? qn[rowid] : 0.f, cert ? kn + ((long long)r * g.Hkv + h) * g.Lkv : nullptr,
                                       tau,
                                       kept_mass != nullptr);
      if (res.certified) {
        or_kept(keys, nc, row_bits);
        rows++;
        ties += res.tie;
        kept_sum += res.nsel;
        if (kept_mass && lane == 0) kept_mass[rowid] = res.P;
      } else {
        unc++;
        // Recompute band [lo, hi] of fast scores.  MASS: blocks below lo have canonical logit < -127
        // (exact zero probability); every block above matters to the mass, so hi = +inf.  RATIO (top-k
        // by score): the band of select_row — outside it the rank against the canonical k-th score is
        // certain, and the mixed row (fast scores outside, canonical inside) has the same top-k set,
        // k-th key and tie at the cut as the all-canonical row.  (kept_mass, which needs every score
        // canonical, always takes the canonical path: api.cu use_fast_scores.)  The row's band blocks
        // are listed contiguously in ulist as fidx * Lkv + j (n_flagged[1] counts them), so the
        // recompute kernels never scan dead units.
        const float lo = select == 1 ? res.band_lo : res.M - 2.0f * res.dmax - 127.0f / c_alpha;
        const float hi = select == 1 ? res.band_hi : INFINITY;
        int cnt = 0;
        for (int j = lane; j < nc; j += 32) cnt += s[j] >= lo && s[j] <= hi;
#pragma unroll
        for (int o = 16; o; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
        int f = 0, base = 0;
        if (lane == 0) {
          f = atomicAdd(n_flagged, 1);
          base = atomicAdd(n_flagged + 1, cnt);
          flagged[f] = (int32_t)rowid;
        }
        f = __shfl_sync(0xffffffffu, f, 0);
        base = __shfl_sync(0xffffffffu, base, 0);
        for (int j0 = 0; j0 < nc; j0 += 32) {
          const int j = j0 + lane;
          const bool in = j < nc && s[j] >= lo && s[j] <= hi;
          const uint32_t bal = __ballot_sync(0xffffffffu, in);
          if (in) ulist[base + __popc(bal & ((1u << lane) - 1u))] = f * g.Lkv + j;
          base += __popc(bal);
        }
      }
      __syncwarp();
    }
    __syncthreads();
    uint32_t* out = coarse + ((long long)(r * g.Hkv + h) * g.Lq + i) * g.Lw;
    for (int w = threadIdx.x; w < g.Lw; w += blockDim.x) out[w] = row_bits[w];
  }
  if (stats && lane == 0) {
    if (rows) atomicAdd(stats + 8, (unsigned long long)rows);
    if (ties) atomicAdd(stats + 9, (unsigned long long)ties);
    if (kept_sum) atomicAdd(stats + 10, (unsigned long long)kept_sum);
    if (unc) atomicAdd(stats + 11, (unsigned long long)unc);
    if (recomputed) atomicAdd(stats + 12, (unsigned long long)recomputed);
  }
}

size_t select_smem_bytes(const Geom& g, int nwarps) {
  return (size_t)((g.Lw * 4 + 15) / 16) * 16 + (size_t)nwarps * g.Lkv * 8;
}

void launch_select(const Geom& g, const float* S, float c_alpha, int select, float gamma, float keep_ratio,
                   uint32_t* coarse, float* kept_mass, unsigned long long* stats, cudaStream_t st, int mode,
                   const float* qn, const float* kn, float tau, int32_t* flagged, int32_t* n_flagged, int num_sms,
                   int32_t* ulist) {
  const int nwarps = g.m < 4 ? g.m : 4;
  const size_t smem = select_smem_bytes(g, nwarps);
  if (smem > 48 * 1024) cudaFuncSetAttribute(k_s1_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int rows = g.B * g.Hkv * g.Lq;
  const int grid = mode == 2 ? num_sms : rows;
  k_s1_select<<<grid, nwarps * 32, smem, st>>>(g, S, c_alpha, select, gamma, keep_ratio, coarse, kept_mass, stats,
                                               mode, qn, kn, tau, flagged, n_flagged, ulist);
  count_launch();
}

}  // namespace bfla
