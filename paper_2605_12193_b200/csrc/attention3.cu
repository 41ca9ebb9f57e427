// attention3.cu — fused sparse causal prefill (Eq. 27) and dense twin (Eq. 1), head_dim 128:
// ONE 128-row Q tile per work item, S DOUBLE-BUFFERED in TMEM, softmax split over two warpgroups.
//
// Why: in the two-Q-tile kernel (attention2.cu) a tile's next S can only be computed
// after its P was consumed (S, P and O of two tiles fill TMEM), so every step of a tile pays
// softmax + PV + S + the MMA completion latency in series and the tensor pipe idles ~45 % of the time.
// Here TMEM holds S_0, S_1 (2 x 128 columns) and O (128 columns) of one tile: S(s+1) is computed while
// the softmax works on S(s), and the softmax runs its steps back to back.  The step's softmax work is
// split by columns over two warpgroups (half hh owns kept tile hh of the step: its 64 keys, its P, its
// 64 columns of O), so two warps share every TMEM lane group and each carries half the exponentials.
//
// Work item = (request r, KV head h, query tile i, head chunk c): the chunk's query heads (128 / T
// heads of T rows, GQA packing) against the row's kept 64-key tiles, two per step (one 128-key K/V ring
// slot, N = 128 MMAs at full rate); a lone last tile runs as an N = 64 step.  Mask granularity stays T.
//
// Roles (384 threads): warp 0 TMA K (+ item scheduling), warp 1 MMA issue (converged, elect.sync),
// warp 2 TMA Q (+ TMEM allocation), warp 3 TMA V, warps 4-11 softmax / epilogue (warp 4 + 4 hh + lg:
// column half hh, TMEM lane group lg).
#include <cuda_bf16.h>

#include "attn_common.cuh"
#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {
using namespace attn;

constexpr int D = 128;
constexpr int BM = 128;   // MMA M (rows of a Q tile)
constexpr int BN = 64;    // mask tile T
constexpr int RS = 128;   // K/V rows per ring slot (two tiles)
constexpr float kLazy = 24.0f;  // lazy-rescale headroom (log2 units), as in attention2.cu

__device__ __forceinline__ void bar_sync_n(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

struct Cfg3 {
  static constexpr int QS = 2, KS = 3, VS = 2;   // Q ring (the next item's tile loads during this one)
  static constexpr int QBYTES = BM * D * 2;      // 32 KB
  static constexpr int SLOT = RS * D * 2;        // 32 KB (two 64-row tiles)
  static constexpr int HALF = BN * 128;          // bytes of one 64-row half of a 64-column chunk
  static constexpr int CHUNK = RS * 128;         // bytes of one 64-column chunk of a slot
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + QS * QBYTES;
  static constexpr int OFF_V = OFF_K + KS * SLOT;
  static constexpr int OFF_BAR = OFF_V + VS * SLOT;
  // q_full/empty, k_full/empty, v_full/empty, s_full[2], p_full[2], pv_done, o_full, o_free, it ring 2x4
  static constexpr int NBAR = 2 * QS + 2 * KS + 2 * VS + 2 + 2 + 3 + 8;
  static constexpr int OFF_RING = OFF_BAR + NBAR * 8 + 16;   // int2 (item index, kept-tile count) x 4
  static constexpr int OFF_LX = OFF_RING + 4 * 8;             // row sums of the two halves [2][128]
  static constexpr int SMEM_TOTAL = OFF_LX + 2 * 128 * 4;
  static constexpr int THREADS = 128 + 256;
  static constexpr int COL_S = 0;    // S / P buffer b at columns [128 b, 128 b + 128)
  static constexpr int COL_O = 256;  // O at [256, 384)
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
};

template <bool PAGED, bool DENSE, int POLY, bool SLICE = false>
__global__ void __launch_bounds__(Cfg3::THREADS, 1)
    k_attn3(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO, int otma, Geom g,
            const int32_t* __restrict__ list, const int32_t* __restrict__ count, const int32_t* __restrict__ page_table,
            __nv_bfloat16* __restrict__ O, float* __restrict__ lse, int n_items, int hpq, int NC,
            int* __restrict__ sched) {
  using C = Cfg3;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (smem_u32(smem) & 1023) __trap();  // SW128 operands need 1024-byte alignment
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* q_empty = q_full + C::QS;
  uint64_t* k_full = q_empty + C::QS;
  uint64_t* k_empty = k_full + C::KS;
  uint64_t* v_full = k_empty + C::KS;
  uint64_t* v_empty = v_full + C::VS;
  uint64_t* s_full = v_empty + C::VS;  // [2]: S buffer b holds the current step's scores
  uint64_t* p_full = s_full + 2;       // [2]: P of buffer b stored (256 arrivals)
  uint64_t* pv_done = p_full + 2;      // every PV completes one phase (lazy O rescale waits on it)
  uint64_t* o_full = pv_done + 1;      // the item's last PV done
  uint64_t* o_free = o_full + 1;       // epilogue has read O (256 arrivals)
  uint64_t* it_full = o_free + 1;      // [4]: item ring entry published
  uint64_t* it_empty = it_full + 4;    // [4]: entry read by every other role (11 warps)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(it_empty + 4);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_RING);
  float* lx = reinterpret_cast<float*>(smem + C::OFF_LX);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int q = 0; q < C::QS; ++q) {
      mbar_init(q_full + q, 1);
      mbar_init(q_empty + q, 1);
    }
    for (int s = 0; s < C::KS; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < C::VS; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(s_full + b, 1);
      mbar_init(p_full + b, 256);
    }
    mbar_init(pv_done, 1);
    mbar_init(o_full, 1);
    mbar_init(o_free, 256);
    for (int e = 0; e < 4; ++e) {
      mbar_init(it_full + e, 1);
      mbar_init(it_empty + e, 3 + 8);  // warps 1, 2, 3 and the eight softmax warps
    }
    fence_barrier_init();
  }
  if (warp == 2) tmem_alloc<512>(tmem_slot);
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmQ);
    tma_prefetch_desc(&tmK);
    tma_prefetch_desc(&tmV);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  const int TR = g.T / BN;  // 64-key tiles per mask tile (T = 128: a kept tile is two of them)
  auto row_count = [&](const Item& it) -> int {
    const Req R = req_of(g, it.r);
    if (it.i >= R.Tq) return 0;  // padding query tile of a shorter request (varlen): no work
    if (DENSE) return (int)req_row_count(R, g.T, it.i) * TR;
    return count[((long long)it.r * g.Hkv + it.h) * g.Tq + it.i] * TR;
  };
  auto row_list = [&](const Item& it) -> const int32_t* {
    return list + ((long long)it.r * g.Hkv + it.h) * g.causal_per_head + req_row_offset(req_of(g, it.r), g.T, it.i);
  };
  // tiles in DESCENDING j (diagonal / local band first: the running max settles on the first step)
  auto tile_at_c = [&](const int32_t* lst, int cnt, int n) -> int {
    const int pos = cnt - 1 - n;
    if (DENSE) return pos;
    return TR == 1 ? __ldg(lst + pos) : 2 * __ldg(lst + (pos >> 1)) + (pos & 1);
  };
  uint32_t ring_n = 0;
  auto next_item = [&](int& idx, int& cnt) -> bool {
    const int e = ring_n & 3;
    mbar_wait(it_full + e, (ring_n >> 2) & 1);
    idx = ring[2 * e];
    cnt = ring[2 * e + 1];
    __syncwarp();
    if (lane == 0) mbar_arrive(it_empty + e);
    ++ring_n;
    return idx >= 0;
  };
  // one ring step of K (kvsel 0) or V (kvsel 1) by a whole warp (see attention2.cu load_step)
  auto load_step = [&](int kvsel, uint32_t ks, const int32_t* lst, int cnt, int s, const Item& it) {
    const int ns_ = kvsel ? C::VS : C::KS;
    const int st = ks % ns_;
    uint64_t* full = (kvsel ? v_full : k_full) + st;
    mbar_wait((kvsel ? v_empty : k_empty) + st, ((ks / ns_) & 1) ^ 1);
    const bool two = 2 * s + 1 < cnt;
    int jl = 0;
    if (lane < (two ? 2 : 1)) jl = tile_at_c(lst, cnt, 2 * s + lane);
    const int ja = __shfl_sync(0xffffffffu, jl, 0), jb = __shfl_sync(0xffffffffu, jl, 1);
    if (lane == 0) mbar_arrive_expect_tx(full, (two ? 2 : 1) * BN * D * 2);
    __syncwarp();
    unsigned char* dst = smem + (kvsel ? C::OFF_V : C::OFF_K) + st * C::SLOT;
    const CUtensorMap* map = kvsel ? &tmV : &tmK;
    if (!PAGED) {
      const int ntile = two ? 2 : 1;
      if (lane < ntile * (D / 64)) {
        const int hf = lane / (D / 64), cc = lane % (D / 64);
        tma_load_4d(dst + cc * C::CHUNK + hf * C::HALF, map, full, cc * 64, (hf ? jb : ja) * BN, it.h / g.kvdiv,
                    it.r);
      }
    } else {
      const int ps = g.page_size, ppt = BN / ps;
      const int ntile = two ? 2 : 1;
      if (lane < ntile * ppt) {
        const int hf = lane / ppt, pc = lane % ppt;
        const int npl = (req_of(g, it.r).Nkv + ps - 1) / ps;
        const int lp = (hf ? jb : ja) * ppt + pc;
        const int phys = __ldg(page_table + (long long)it.r * g.max_pages + (lp < npl ? lp : 0));
        for (int cc = 0; cc < D / 64; ++cc)
          tma_load_4d(dst + cc * C::CHUNK + hf * C::HALF + pc * ps * 128, map, full, cc * 64, it.h / g.kvdiv, 0,
                      phys);
      }
    }
  };

  if (warp == 0) {
    // ================================ TMA producer (K) + item scheduling ================================
    uint32_t ks = 0;
    int idx = blockIdx.x;
    for (;;) {
      const bool live = idx < n_items;
      const Item it = decode_item<SLICE>(g, live ? idx : 0, NC);
      const int cnt = live ? row_count(it) : 0;
      {
        const int e = ring_n & 3;
        mbar_wait(it_empty + e, ((ring_n >> 2) & 1) ^ 1);
        if (lane == 0) {
          ring[2 * e] = live ? idx : -1;
          ring[2 * e + 1] = cnt;
          mbar_arrive(it_full + e);
        }
        __syncwarp();
        ++ring_n;
      }
      if (!live) break;
      int nidx = 0;  // the next item (greedy longest-first list scheduling through the counter)
      if (lane == 0) nidx = sched ? (int)gridDim.x + atomicAdd(sched, 1) : idx + (int)gridDim.x;
      nidx = __shfl_sync(0xffffffffu, nidx, 0);
      if (cnt > 0) {
        const int32_t* lst = DENSE ? nullptr : row_list(it);
        const int ns = (cnt + 1) / 2;
        for (int s = 0; s < ns; ++s, ++ks) load_step(0, ks, lst, cnt, s, it);
      }
      idx = nidx;
    }
  } else if (warp == 2) {
    // ================================ TMA producer (Q) ================================
    uint32_t nit = 0;
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      if (cnt == 0) continue;
      const uint32_t my_it = nit++;
      const int qsl = my_it % C::QS;
      mbar_wait(q_empty + qsl, ((my_it / C::QS) & 1) ^ 1);
      if (lane == 0) {
        int nb = 0;
        for (int s = 0; s < hpq; ++s)
          if (it.c * hpq + s < g.m) nb += D / 64;
        mbar_arrive_expect_tx(q_full + qsl, nb * 64 * g.T * 2);
      }
      __syncwarp();
      const int s = lane / (D / 64), cc = lane % (D / 64);  // lane = (head slot, d-chunk)
      const int pl = it.c * hpq + s;
      if (s < hpq && pl < g.m)
        tma_load_4d(smem + C::OFF_Q + qsl * C::QBYTES + cc * (BM * 128) + s * (g.T * 128), &tmQ, q_full + qsl,
                    cc * 64, it.i * g.T, it.h * g.m + pl, it.r);
    }
  } else if (warp == 3) {
    // ================================ TMA producer (V) ================================
    uint32_t ks = 0;
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      if (cnt == 0) continue;
      const int32_t* lst = DENSE ? nullptr : row_list(it);
      const int ns = (cnt + 1) / 2;
      for (int s = 0; s < ns; ++s, ++ks) load_step(1, ks, lst, cnt, s, it);
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // Per step s (global step gs, S buffer b = gs & 1): S(s) = Q K_s^T into buffer b — free, because
    // PV(s-2), which read P(s-2) there, was issued before it (tcgen05 MMAs of one thread execute in
    // order) — then, once P(s-1) is stored, O += P(s-1) V_{s-1}.  So S(s) runs while the softmax works
    // on S(s-1): the softmax never waits for its own PV.
    const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(smem + C::OFF_V), C::CHUNK, 1024);
    uint32_t ks0 = 0, nit = 0, gs0 = 0;
    auto issue_PV = [&](uint32_t b, uint32_t vslot, int ntile, bool acc_first) {
      const uint32_t idO = idesc_bf16(BM, D, 0, 1);
      const uint64_t b0 = dV + (uint64_t)((vslot * C::SLOT) >> 4);
      const uint32_t aP = tmem + C::COL_S + b * 128;
#pragma unroll 8
      for (int kk = 0; kk < ntile * 4; ++kk)  // P of key tile a at columns [0, 32), of tile b at [64, 96)
        umma_f16_ts_warp(tmem + C::COL_O, aP + kk * 8 + (kk >= 4 ? 32 : 0), b0 + (uint64_t)((kk * 2048) >> 4), idO,
                         (acc_first || kk > 0) ? 1u : 0u);
    };
    auto issue_S = [&](uint32_t b, int qsl, uint32_t kslot, int ntile) {
      const uint32_t idS = ntile == 2 ? idesc_bf16(BM, 2 * BN, 0, 0) : idesc_bf16(BM, BN, 0, 0);
      const uint64_t a0 = dQ + (uint64_t)((qsl * C::QBYTES) >> 4), b0 = dK + (uint64_t)((kslot * C::SLOT) >> 4);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t offa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
        const uint32_t offb = ((kk >> 2) * C::CHUNK + (kk & 3) * 32) >> 4;
        umma_f16_ss_warp(tmem + C::COL_S + b * 128, a0 + offa, b0 + offb, idS, kk > 0 ? 1u : 0u);
      }
      umma_commit_warp(s_full + b);
    };
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      (void)it;
      if (cnt == 0) continue;
      const uint32_t my_it = nit++;
      const int qsl = my_it % C::QS;
      const int ns = (cnt + 1) / 2;
      for (int s = 0; s < ns; ++s) {
        const uint32_t ksn = ks0 + s, kst = ksn % C::KS, gs = gs0 + s;
        mbar_wait(k_full + kst, (ksn / C::KS) & 1);
        if (s == 0) mbar_wait(q_full + qsl, (my_it / C::QS) & 1);
        tc_fence_after();
        issue_S(gs & 1, qsl, kst, 2 * s + 1 < cnt ? 2 : 1);
        umma_commit_warp(k_empty + kst);
        if (s == ns - 1 && !otma) umma_commit_warp(q_empty + qsl);  // every S MMA of the item issued
        if (s > 0) {  // O += P(s-1) V(s-1): every step but the last holds two tiles
          const uint32_t vsn = ksn - 1, vst = vsn % C::VS;
          mbar_wait(v_full + vst, (vsn / C::VS) & 1);
          mbar_wait(p_full + ((gs - 1) & 1), ((gs - 1) >> 1) & 1);
          if (s == 1) mbar_wait(o_free, (my_it & 1) ^ 1);
          tc_fence_after();
          issue_PV((gs - 1) & 1, vst, 2, s > 1);
          umma_commit_warp(pv_done);
          umma_commit_warp(v_empty + vst);
        }
      }
      // tail: O += P(ns-1) V(ns-1)
      const uint32_t vsn = ks0 + ns - 1, vst = vsn % C::VS, gl = gs0 + ns - 1;
      mbar_wait(v_full + vst, (vsn / C::VS) & 1);
      mbar_wait(p_full + (gl & 1), (gl >> 1) & 1);
      if (ns == 1) mbar_wait(o_free, (my_it & 1) ^ 1);
      tc_fence_after();
      issue_PV(gl & 1, vst, cnt - 2 * (ns - 1), ns > 1);
      umma_commit_warp(pv_done);
      umma_commit_warp(o_full);
      umma_commit_warp(v_empty + vst);
      ks0 += ns;
      gs0 += ns;
    }
  } else {
    // ================================ softmax / epilogue (two column halves) ================================
    const int hh = (warp - 4) >> 2;  // column half: kept tile hh of each step
    const int lg = warp & 3;         // TMEM lane group of this warp
    const int row = lg * 32 + lane;  // row of the Q tile = TMEM lane
    const uint32_t lane_addr = (uint32_t)(lg * 32) << 16;
    const uint32_t tO = tmem + lane_addr + C::COL_O + hh * 64;
    const float c2 = g.scale * 1.4426950408889634f;  // softmax scale in the exp2 domain
    uint32_t gs = 0, nit = 0;
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      const int slot = row / g.T;
      const int pl = it.c * hpq + slot;
      const int t = it.i * g.T + (row % g.T);
      const Req Rq = req_of(g, it.r);  // this request's logical dims (varlen)
      const bool valid = slot < hpq && pl < g.m && t < Rq.Nq;
      const int p = it.h * g.m + pl;
      __nv_bfloat16* orow = O + (long long)it.r * g.os0 + (long long)p * g.os1 + (long long)t * g.os2;
      if (cnt == 0) {  // cannot happen for masks from bfla_expand_rescue (sink + band); defined anyway
        if (valid && hh == 0) {
          for (int c = 0; c < D; ++c) orow[c] = __float2bfloat16(0.0f);
          if (lse) lse[((long long)it.r * g.Hq + p) * g.Nq + t] = -INFINITY;
        }
        continue;
      }
      const uint32_t my_it = nit++;
      const int32_t* lst = DENSE ? nullptr : row_list(it);
      const int ns = (cnt + 1) / 2;
      float m_run = -INFINITY, l_run = 0.0f;
      for (int s = 0; s < ns; ++s, ++gs) {
        const uint32_t b = gs & 1;
        const uint32_t tS = tmem + lane_addr + C::COL_S + b * 128;
        const bool two = 2 * s + 1 < cnt;
        const int ja = tile_at_c(lst, cnt, 2 * s), jb = two ? tile_at_c(lst, cnt, 2 * s + 1) : 0;
        mbar_wait(s_full + b, (gs >> 1) & 1);
        tc_fence_after();
        // token-exact causality inside each tile (Eq. 27): key j*64 + c visible iff <= N_c + t
        const int la = Rq.Nc + t - ja * BN, lb = two ? Rq.Nc + t - jb * BN : -1;
        const bool own = hh == 0 || two, oth = hh == 1 || two;
        const int lim_own = hh ? lb : la, lim_oth = hh ? la : lb;
        float mrow = -INFINITY;
        if (oth) {  // the other half's S columns: their max only (the row max is shared)
#pragma unroll
          for (int ch = 0; ch < 2; ++ch) {
            float u[32];
            tmem_ld32(tS + (1 - hh) * 64 + ch * 32, u);
            tmem_wait_ld();
            if (lim_oth < BN - 1) {
#pragma unroll
              for (int c = 0; c < 32; ++c)
                if (ch * 32 + c > lim_oth) u[c] = -INFINITY;
            }
            float a = max3f(u[0], u[1], u[2]), b2 = max3f(u[16], u[17], u[18]);
#pragma unroll
            for (int c = 3; c < 15; c += 2) {
              a = max3f(a, u[c], u[c + 1]);
              b2 = max3f(b2, u[16 + c], u[16 + c + 1]);
            }
            mrow = max3f(mrow, fmaxf(a, u[15]), fmaxf(b2, u[31]));
          }
        }
        float v[64];
        if (own) {
          tmem_ld32(tS + hh * 64, v);
          tmem_ld32(tS + hh * 64 + 32, v + 32);
          tmem_wait_ld();
          if (lim_own < BN - 1) {
#pragma unroll
            for (int c = 0; c < BN; ++c)
              if (c > lim_own) v[c] = -INFINITY;
          }
          mrow = fmaxf(mrow, row_max64(v));
        }
        bar_sync_n(1, 256);  // every S column of the buffer has been read: P may overwrite them
        const float mx = mrow * c2;
        float alpha = 1.0f;
        // lazy rescale (identical inputs in both halves -> the same m_run): raise the running max only
        // when it grows by more than kLazy (P <= 2^kLazy keeps bf16 P, fp32 l and O in range)
        if (mx > m_run + kLazy || (m_run == -INFINITY && mx > -INFINITY)) {
          alpha = ex2_approx(m_run - mx);  // 0 when m_run = -inf
          l_run *= alpha;
          m_run = mx;
        }
        if (s > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
          // O must hold PV(s-1) before it is scaled (S(s) was committed before PV(s-1) was issued)
          mbar_wait(pv_done, (gs - 1) & 1);
          tc_fence_after();
#pragma unroll 1
          for (int cc = 0; cc < 64; cc += 32) {
            float ov[32];
            tmem_ld32(tO + cc, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] *= alpha;
            tmem_st32(tO + cc, ov);
          }
        }
        const float msub = m_run == -INFINITY ? 0.0f : m_run;
        float2 ls[4];
        ls[0] = ls[1] = ls[2] = ls[3] = make_float2(0.f, 0.f);
        if (own) {
          // p = 2^(s c2 - m) in pairs (FFMA2); POLY selects the pairs on the FMA pipe (rel. err 8e-5, far
          // below bf16 rounding of P), the rest on MUFU.EX2; P of this half -> its own S columns [0, 32)
          const float2 c22 = make_float2(c2, c2), nm2 = make_float2(-msub, -msub);
#pragma unroll
          for (int ch = 0; ch < 4; ++ch) {
            uint32_t pk[8];
#pragma unroll
            for (int e2 = 0; e2 < 8; ++e2) {
              const int e = ch * 8 + e2;
              const float2 x = __ffma2_rn(make_float2(v[2 * e], v[2 * e + 1]), c22, nm2);
              float2 pr;
              if ((POLY >> (e % 8)) & 1) {
                pr = exp2_poly2(x);
              } else {
                pr.x = ex2_approx(x.x);
                pr.y = ex2_approx(x.y);
              }
              ls[e & 3] = __fadd2_rn(ls[e & 3], pr);
              pk[e2] = pack_bf16x2(pr.x, pr.y);
            }
            tmem_st8(tS + hh * 64 + ch * 8, pk);
          }
        }
        l_run += ((ls[0].x + ls[0].y) + (ls[1].x + ls[1].y)) + ((ls[2].x + ls[2].y) + (ls[3].x + ls[3].y));
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + b);
      }
      // epilogue: l = l_half0 + l_half1 (fixed order); O / l -> bf16; LSE = (m + log2 l) ln 2.  With otma, O
      // is staged (SW128) in this item's Q slot — free once the last S MMA is done — and TMA-stored.
      mbar_wait(o_full, my_it & 1);
      tc_fence_after();
      lx[hh * 128 + row] = l_run;
      bar_sync_n(1, 256);
      const float l_tot = lx[row] + lx[128 + row];
      const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
      const int qsl = my_it % C::QS;
      unsigned char* qs = smem + C::OFF_Q + qsl * C::QBYTES;
#pragma unroll 1
      for (int cc = 0; cc < 64; cc += 32) {
        float ov[32];
        tmem_ld32(tO + cc, ov);
        tmem_wait_ld();
        if (cc == 32) {  // own O columns read from TMEM: the next item's first PV may overwrite them
          tc_fence_before();
          mbar_arrive(o_free);
        }
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(ov[2 * e] * inv_l, ov[2 * e + 1] * inv_l);
        if (otma) {
          unsigned char* rb = qs + hh * (BM * 128) + row * 128;  // d-chunk hh, row `row`
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = (cc >> 3) + e;
            st_shared_v4(rb + ((k ^ (row & 7)) << 4), w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          }
        } else if (valid) {
          uint4* dst = reinterpret_cast<uint4*>(orow + hh * 64 + cc);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
        }
      }
      if (valid && lse && hh == 0)
        lse[((long long)it.r * g.Hq + p) * g.Nq + t] =
            l_tot > 0.0f ? (m_run + log2f(l_tot)) * 0.6931471805599453f : -INFINITY;
      if (otma) {
        fence_proxy_async_smem();
        bar_sync_n(2, 256);
        if (warp == 4 && lane == 0) {
          for (int s = 0; s < hpq; ++s) {
            const int pls = it.c * hpq + s;
            if (pls >= g.m) continue;
            for (int dc = 0; dc < D / 64; ++dc)
              tma_store_4d(&tmO, qs + dc * (BM * 128) + s * (g.T * 128), dc * 64, it.i * g.T, it.h * g.m + pls,
                           it.r);
          }
          bulk_commit();
          bulk_wait_read0();  // the smem has been read: a later item's Q may land there
          mbar_arrive(q_empty + qsl);
        }
      }
    }
    if (otma && warp == 4 && lane == 0) bulk_wait_all();  // O stores complete before exit
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <bool PAGED, bool DENSE>
int launch3_t(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count, const int32_t* pt,
              void* o, float* lse, int n_items, int hpq, int NC, int num_sms, cudaStream_t st, int* sched) {
  const int grid = n_items < num_sms ? n_items : num_sms;
  auto go = [&](auto kern) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg3::SMEM_TOTAL);
    if (e != cudaSuccess) return (int)e;
    kern<<<grid, Cfg3::THREADS, Cfg3::SMEM_TOTAL, st>>>(maps.q, maps.k, maps.v, maps.o, maps.o_ok, g, list, count, pt,
                                                         static_cast<__nv_bfloat16*>(o), lse, n_items, hpq, NC, sched);
    count_launch();
    return (int)cudaGetLastError();
  };
#ifndef BFLA_POLY_MASK3
#define BFLA_POLY_MASK3 0x22
#endif
  constexpr int PM = BFLA_POLY_MASK3;
  if constexpr (!DENSE)
    if (g.nrows) return go(k_attn3<PAGED, false, PM, true>);  // work slice (bfla_sparse_prefill_rows)
  return go(k_attn3<PAGED, DENSE, PM>);
}

}  // namespace

// head_dim 128, one 128-row Q tile per item (T / 64 heads of T rows), two kept tiles per step.
int launch_attention3(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                      const int32_t* page_table, int dense, void* o, float* lse, int num_sms, cudaStream_t st,
                      int* sched) {
  const int hpq = BM / g.T;
  const int NC = (g.m + hpq - 1) / hpq;
  const long long items = (g.nrows ? (long long)g.nrows : (long long)g.B * g.Hkv * g.Tq) * NC;
  if (items == 0) return 0;
  if (items > 0x7fffffff) return (int)cudaErrorInvalidValue;
  const int n = (int)items;
  if (g.paged) {
    if (dense) return launch3_t<true, true>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched);
    return launch3_t<true, false>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched);
  }
  if (dense) return launch3_t<false, true>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched);
  return launch3_t<false, false>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched);
}

}  // namespace bfla
