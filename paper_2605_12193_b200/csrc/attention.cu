// attention.cu — fused sparse causal prefill of BFLA (Eq. 27) and its dense twin (Eq. 1).
//
// One work item = (request r, KV head h, row chunk c, query tile i).  All m query heads of the
// head group H_h (Eq. 8) share the item's kept-KV-tile list (the mask is per KV head after the OR,
// R8), so their T-row query tiles are stacked into 128-row MMA tiles (GQA packing): with T = 64,
// one 128-row tile holds 2 heads; NQT (1 or 2) tiles per CTA share every K/V tile loaded.
//
// Warp roles (1 CTA per SM, persistent over a static LPT-ordered item sequence):
//   warp 0        TMA producer: Q tiles per item, then K_j / V_j for every kept tile j (ring of
//                 K/V stage slots, mbarrier full/empty pairs).  Contiguous [B,H,N,d] via a 4-D
//                 tensor map, or vLLM pages [P,page,H,d] gathered page by page into the same
//                 swizzled smem layout.
//   warp 1        MMA issuer (one thread): S_q = Q_q K_j^T into TMEM (M=128, N=64, K=d) and
//                 O_q += P_q V_j (M=128, N=d, K=64), tcgen05.mma kind::f16, fp32 accumulators.
//   warp 2        TMEM allocator (512 columns).
//   warps 4..     one 128-thread softmax warpgroup per Q tile; thread = one query row (= one
//                 TMEM lane): loads S, applies the token-exact causal frontier, online softmax in
//                 the exp2 domain with lazy rescaling (the running max is only raised when it
//                 grows by > 8, so O in TMEM is rescaled rarely), writes P (bf16) to swizzled
//                 smem for the PV MMA, and finally O / l -> bf16 -> global (+ LSE).
// Dropped tiles are never loaded nor computed: they contribute exactly nothing (Eq. 27's -inf).
#include <cuda_bf16.h>

#include <cstdlib>

#include "attn_common.cuh"
#include "common.cuh"
#include "kernels.h"

namespace bfla {

namespace {
using namespace attn;

constexpr int BM = 128;  // MMA M (rows of a Q tile)
constexpr int BN = 64;   // KV tile = T

template <int D, int NQT, int SPL>
struct Cfg {
  static constexpr int KST = D == 128 ? 3 : 2;     // K stages (S runs two tiles ahead)
  static constexpr int VST = (D == 128 && SPL == 1) ? 3 : 2;  // V stages
  static constexpr int QBYTES = BM * D * 2;       // one 128-row Q tile
  static constexpr int KVBYTES = BN * D * 2;      // one K (or V) tile
  static constexpr int PBYTES = BM * BN * 2;      // one P tile
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + NQT * QBYTES;
  static constexpr int OFF_V = OFF_K + KST * KVBYTES;
  static constexpr int OFF_P = OFF_V + VST * KVBYTES;
  static constexpr int OFF_BAR = OFF_P + 2 * NQT * PBYTES;  // P double buffer per Q tile
  static constexpr int NBAR = 2 + 2 * KST + 2 * VST + 10 * NQT + 2 * 4;  // + item ring full/empty
  static constexpr int OFF_RED = OFF_BAR + ((NBAR * 8 + 16 + 127) / 128) * 128;  // row-max exchange
  static constexpr int OFF_RING = OFF_RED + (SPL == 2 ? NQT * 2 * 2 * 128 * 4 : 0);  // [NQT][parity][half][row]
  static constexpr int SMEM_TOTAL = OFF_RING + 4 * 8;  // item ring: (index, kept-tile count) x 4
  static constexpr int THREADS = 128 + 128 * SPL * NQT;  // 4 control warps + SPL softmax warpgroups per Q tile
  // TMEM columns: S_q double buffer at 128 q + 64 b (d=128) / 64 b (d=256); O_q from column 256
  static constexpr int COL_S = 0;
  static constexpr int COL_O = 256;
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
};

template <int D, int NQT, bool PAGED, bool DENSE, int SPL, bool SLICE = false>
__global__ void __launch_bounds__(Cfg<D, NQT, SPL>::THREADS, 1)
    k_attn(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
           const __grid_constant__ CUtensorMap tmV, Geom g, const int32_t* __restrict__ list,
           const int32_t* __restrict__ count, const int32_t* __restrict__ page_table,
           __nv_bfloat16* __restrict__ O, float* __restrict__ lse, int n_items, int hpq, int NC,
           int* __restrict__ sched) {
  using C = Cfg<D, NQT, SPL>;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (smem_u32(smem) & 1023) __trap();  // SW128 operands need 1024-byte alignment (no static smem here)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;
  uint64_t* q_empty = bars + 1;
  uint64_t* k_full = bars + 2;
  uint64_t* k_empty = k_full + C::KST;
  uint64_t* v_full = k_empty + C::KST;
  uint64_t* v_empty = v_full + C::VST;
  uint64_t* s_full = v_empty + C::VST;  // [NQT][2]: S_q(n) landed in TMEM buffer n % 2
  uint64_t* p_full = s_full + 2 * NQT;     // [NQT][2]: P_q(n) written to smem buffer n % 2 (128 arrivals)
  uint64_t* p_free = p_full + 2 * NQT;     // [NQT][2]: PV_q(n) done (P buffer n % 2 free, O includes PV(n))
  uint64_t* o_full = p_free + 2 * NQT;     // [NQT]: last PV of the item done
  uint64_t* o_free = o_full + NQT;         // [NQT]: epilogue has read O (128 arrivals)
  uint64_t* it_full = o_free + NQT;        // [4]: item ring entry published (Q/K producer)
  uint64_t* it_empty = it_full + 4;        // [4]: entry read by the V producer, the MMA warp, softmax warps
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + C::NBAR);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_RING);  // [4][2]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int s = 0; s < C::KST; ++s) {
      mbar_init(k_full + s, 1);
      mbar_init(k_empty + s, 1);
    }
    for (int s = 0; s < C::VST; ++s) {
      mbar_init(v_full + s, 1);
      mbar_init(v_empty + s, 1);
    }
    for (int q = 0; q < NQT; ++q) {
      mbar_init(s_full + 2 * q, 1);
      mbar_init(s_full + 2 * q + 1, 1);
      mbar_init(p_full + 2 * q, 128 * SPL);
      mbar_init(p_full + 2 * q + 1, 128 * SPL);
      mbar_init(p_free + 2 * q, 1);
      mbar_init(p_free + 2 * q + 1, 1);
      mbar_init(o_full + q, 1);
      mbar_init(o_free + q, 128 * SPL);
    }
    for (int e = 0; e < 4; ++e) {
      mbar_init(it_full + e, 1);
      mbar_init(it_empty + e, 2 + 4 * NQT * SPL);
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
  const int heads_in_chunk = NQT * hpq;

  // 64-key tiles (BN); a T = 128 mask tile is two of them (see attention2.cu)
  const int TR = g.T / BN;
  auto row_count = [&](const Item& it) -> int {
    const Req R = req_of(g, it.r);
    if (it.i >= R.Tq) return 0;  // padding query tile of a shorter request (varlen): no work
    if (DENSE) return (int)req_row_count(R, g.T, it.i) * TR;
    const int n = count[((long long)it.r * g.Hkv + it.h) * g.Tq + it.i];
    if (!g.kv_range) return n * TR;
    // split-KV: only the row's kept tiles inside [kv_lo, kv_hi) (the list is ascending in j)
    const int32_t* l = list + ((long long)it.r * g.Hkv + it.h) * g.causal_per_head + req_row_offset(R, g.T, it.i);
    return (list_lower_bound(l, n, g.kv_hi) - list_lower_bound(l, n, g.kv_lo)) * TR;
  };
  auto tile64 = [&](const int32_t* lst, int n) -> int {  // n-th 64-key tile of the row, ascending
    if (DENSE) return n;
    return TR == 1 ? __ldg(lst + n) : 2 * __ldg(lst + (n >> 1)) + (n & 1);
  };
  // Item sequence (as attention2.cu): the Q/K producer takes the CTA's first item statically and the
  // next ones from a global counter (longest-first greedy list scheduling) or round-robin without one,
  // and publishes (index, kept-tile count) in a 4-entry smem ring that every other role reads in order.
  uint32_t ring_n = 0;
  auto next_item = [&](int& idx, int& cnt, bool whole_warp) -> bool {
    const int e = ring_n & 3;
    mbar_wait(it_full + e, (ring_n >> 2) & 1);
    idx = ring[2 * e];
    cnt = ring[2 * e + 1];
    if (whole_warp) {
      __syncwarp();
      if (lane == 0) mbar_arrive(it_empty + e);
    } else {
      mbar_arrive(it_empty + e);
    }
    ++ring_n;
    return idx >= 0;
  };
  auto row_list = [&](const Item& it) -> const int32_t* {
    const int32_t* l =
        list + ((long long)it.r * g.Hkv + it.h) * g.causal_per_head + req_row_offset(req_of(g, it.r), g.T, it.i);
    if (!g.kv_range) return l;
    return l + list_lower_bound(l, count[((long long)it.r * g.Hkv + it.h) * g.Tq + it.i], g.kv_lo);
  };

  // one K (kvsel = 0) or V (kvsel = 1) tile j of item `it` into ring slot kv % stages
  auto load_kv = [&](int kvsel, uint32_t kv, int j, const Item& it) {
    const int nst = kvsel ? C::VST : C::KST;
    const int st = kv % nst;
    const uint32_t ph = (kv / nst) & 1;
    uint64_t* full = (kvsel ? v_full : k_full) + st;
    mbar_wait((kvsel ? v_empty : k_empty) + st, ph ^ 1);
    mbar_arrive_expect_tx(full, C::KVBYTES);
    unsigned char* dst = smem + (kvsel ? C::OFF_V : C::OFF_K) + st * C::KVBYTES;
    const CUtensorMap* map = kvsel ? &tmV : &tmK;
    if (!PAGED) {
      for (int cc = 0; cc < D / 64; ++cc)
        tma_load_4d(dst + cc * (BN * 128), map, full, cc * 64, j * BN, it.h / g.kvdiv, it.r);
    } else {
      // vLLM pages: the 64-token tile is BN/ps page boxes of (64 cols x ps rows); a page past the
      // request's last logical page (ragged tail) is replaced by its first page (finite data; those
      // keys are masked by causality and get P = 0).
      const int ps = g.page_size;
      const int npl = (req_of(g, it.r).Nkv + ps - 1) / ps;
      const int32_t* table = page_table + (long long)it.r * g.max_pages;
      for (int pc = 0; pc < BN / ps; ++pc) {
        const int lp = j * BN / ps + pc;
        const int phys = __ldg(table + (lp < npl ? lp : 0));
        for (int cc = 0; cc < D / 64; ++cc)
          tma_load_4d(dst + cc * (BN * 128) + pc * ps * 128, map, full, cc * 64, it.h / g.kvdiv, 0, phys);
      }
    }
  };

  if (warp == 0) {
    // ================================ TMA producer (Q, K) ================================
    if (lane == 0) {
      uint32_t kv = 0, nit = 0;
      for (int idx = blockIdx.x;;) {
        const bool live = idx < n_items;
        const Item it = decode_item<SLICE>(g, live ? idx : 0, NC);
        const int cnt = live ? row_count(it) : 0;
        {  // publish (idx, cnt) — or the end marker
          const int e = ring_n & 3;
          mbar_wait(it_empty + e, ((ring_n >> 2) & 1) ^ 1);
          ring[2 * e] = live ? idx : -1;
          ring[2 * e + 1] = cnt;
          mbar_arrive(it_full + e);
          ++ring_n;
        }
        if (!live) break;
        const int nidx = sched ? (int)gridDim.x + atomicAdd(sched, 1) : idx + (int)gridDim.x;
        if (cnt == 0) {
          idx = nidx;
          continue;
        }
        const int32_t* lst = DENSE ? nullptr : row_list(it);
        const uint32_t my_it = nit++;
        // Q: for each tile q and head slot s, D/64 boxes of (64 cols x 64 rows)
        mbar_wait(q_empty, (my_it & 1) ^ 1);
        int nq_boxes = 0;
        for (int q = 0; q < NQT; ++q)
          for (int s = 0; s < hpq; ++s)
            if (it.c * heads_in_chunk + q * hpq + s < g.m) nq_boxes += D / 64;
        mbar_arrive_expect_tx(q_full, nq_boxes * 64 * g.T * 2);
        for (int q = 0; q < NQT; ++q)
          for (int s = 0; s < hpq; ++s) {
            const int pl = it.c * heads_in_chunk + q * hpq + s;
            if (pl >= g.m) continue;
            const int p = it.h * g.m + pl;
            for (int cc = 0; cc < D / 64; ++cc)
              tma_load_4d(smem + C::OFF_Q + q * C::QBYTES + cc * (BM * 128) + s * (g.T * 128), &tmQ, q_full,
                          cc * 64, it.i * g.T, p, it.r);
          }
        // warm L2 with the next item's Q (it is read from HBM exactly once)
        if (nidx < n_items) {
          const Item nx = decode_item<SLICE>(g, nidx, NC);
          for (int q = 0; q < NQT; ++q)
            for (int s = 0; s < hpq; ++s) {
              const int pl = nx.c * heads_in_chunk + q * hpq + s;
              if (pl >= g.m) continue;
              for (int cc = 0; cc < D / 64; ++cc)
                tma_prefetch_4d(&tmQ, cc * 64, nx.i * g.T, nx.h * g.m + pl, nx.r);
            }
        }
        for (int n = 0; n < cnt; ++n, ++kv) {
          const int j = tile64(lst, n);
          load_kv(0, kv, j, it);
        }
        idx = nidx;
      }
    }
  } else if (warp == 3) {
    // ================================ TMA producer (V) ================================
    // V has its own ring and thread so that K loads (needed two tiles ahead by the S MMAs) never
    // queue behind a V slot that is still being read.
    if (lane == 0) {
      uint32_t kv = 0;
      for (int idx, cnt; next_item(idx, cnt, false);) {
        const Item it = decode_item<SLICE>(g, idx, NC);
        if (cnt == 0) continue;
        const int32_t* lst = DENSE ? nullptr : row_list(it);
        for (int n = 0; n < cnt; ++n, ++kv) load_kv(1, kv, tile64(lst, n), it);
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // Per item: S_q(0), S_q(1) up front; then for each tile n: PV_q(n) as soon as P_q(n) is ready,
    // followed by S_q(n+2) into the TMEM buffer S_q(n) just vacated — so the tensor core always has
    // the next S ready while the softmax warps work on the current one.  The whole warp runs this
    // loop converged; one elected lane issues each tcgen05 instruction.
    constexpr uint32_t idS = idesc_bf16(BM, BN, 0, 0);
    constexpr uint32_t idO = idesc_bf16(BM, D, 0, 1);
    // descriptor bases; advancing a SW128 descriptor = adding (bytes >> 4) to its start-address field
    const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(smem + C::OFF_V), BN * 128, 1024);
    const uint64_t dP = sdesc_sw128(smem_u32(smem + C::OFF_P), 16, 1024);
    uint32_t kv0 = 0, nit = 0, tc0 = 0;  // kv0: tiles loaded before this item; tc0: tiles before
    auto issue_S = [&](int q, uint32_t tcn, uint32_t st) {
      const uint32_t dS = tmem + C::COL_S + q * 2 * BN + (tcn & 1) * BN;
      const uint64_t a0 = dQ + (uint64_t)((q * C::QBYTES) >> 4), b0 = dK + (uint64_t)((st * C::KVBYTES) >> 4);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t off = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
        const uint32_t offk = ((kk >> 2) * (BN * 128) + (kk & 3) * 32) >> 4;
        umma_f16_ss_warp(dS, a0 + off, b0 + offk, idS, kk > 0 ? 1u : 0u);
      }
      umma_commit_warp(s_full + 2 * q + (tcn & 1));
    };
    for (int idx, cnt; next_item(idx, cnt, true);) {
      if (cnt == 0) continue;
      const uint32_t my_it = nit++;
      mbar_wait(q_full, my_it & 1);
      tc_fence_after();
      const int pre = cnt < 2 ? cnt : 2;
      for (int n = 0; n < pre; ++n) {
        const uint32_t st = (kv0 + n) % C::KST;
        mbar_wait(k_full + st, ((kv0 + n) / C::KST) & 1);
        tc_fence_after();
#pragma unroll
        for (int q = 0; q < NQT; ++q) issue_S(q, tc0 + n, st);
        umma_commit_warp(k_empty + st);
        if (n == cnt - 1) umma_commit_warp(q_empty);
      }
      for (int n = 0; n < cnt; ++n) {
        const uint32_t kvn = kv0 + n, stv = kvn % C::VST;
        mbar_wait(v_full + stv, (kvn / C::VST) & 1);
        const bool more = n + 2 < cnt;
        const uint32_t stk = (kvn + 2) % C::KST;
        tc_fence_after();
        const uint32_t pb = (tc0 + n) & 1;
#pragma unroll
        for (int q = 0; q < NQT; ++q) {
          mbar_wait(p_full + 2 * q + pb, ((tc0 + n) >> 1) & 1);
          if (n == 0) mbar_wait(o_free + q, (my_it & 1) ^ 1);  // epilogue of the previous item read O
          tc_fence_after();
          const uint64_t a0 = dP + (uint64_t)(((2 * q + pb) * C::PBYTES) >> 4);
          const uint64_t b0 = dV + (uint64_t)((stv * C::KVBYTES) >> 4);
#pragma unroll
          for (int kk = 0; kk < BN / 16; ++kk)
            umma_f16_ss_warp(tmem + C::COL_O + q * D, a0 + (uint64_t)((kk * 32) >> 4),
                             b0 + (uint64_t)((kk * 2048) >> 4), idO, (n > 0 || kk > 0) ? 1u : 0u);
          umma_commit_warp(p_free + 2 * q + pb);
          if (n == cnt - 1) umma_commit_warp(o_full + q);
          if (more) {
            if (q == 0) {
              mbar_wait(k_full + stk, ((kvn + 2) / C::KST) & 1);
              tc_fence_after();
            }
            issue_S(q, tc0 + n + 2, stk);
          }
        }
        umma_commit_warp(v_empty + stv);
        if (more) {
          umma_commit_warp(k_empty + stk);
          if (n + 2 == cnt - 1) umma_commit_warp(q_empty);  // every S MMA of the item has been issued
        }
      }
      kv0 += cnt;
      tc0 += cnt;
    }
  } else if (warp >= 4) {
    // ================================ softmax / epilogue ================================
    // Two warpgroups per Q tile: thread (half, row) owns columns [32 half, 32 half + 32) of its row
    // of S and [D/2 half, D/2 half + D/2) of O.  The row max is exchanged through smem once per
    // tile (named barrier per Q tile); the running sum l stays split until the epilogue.
    constexpr int NCOL = BN / SPL;       // S columns per thread
    const int q = (warp - 4) / (4 * SPL);
    const int half = SPL == 2 ? ((warp - 4) >> 2) & 1 : 0;
    const int lg = warp & 3;              // TMEM lane group of this warp
    const int row = lg * 32 + lane;       // row of Q tile q = TMEM lane
    const uint32_t lane_addr = (uint32_t)(lg * 32) << 16;
    const uint32_t tS0 = tmem + lane_addr + C::COL_S + q * 2 * BN + half * NCOL;
    constexpr int DH = D / SPL;
    const uint32_t tO = tmem + lane_addr + C::COL_O + q * D + half * DH;
    const float c2 = g.scale * 1.4426950408889634f;  // softmax scale in the exp2 domain
    unsigned char* sPq = smem + C::OFF_P + 2 * q * C::PBYTES;  // + (tc & 1) * PBYTES
    float* red = reinterpret_cast<float*>(smem + C::OFF_RED) + q * 512;  // [tc & 1][half][row] (SPL = 2)
    const uint32_t bar_id = 1 + q;
    auto pair_sync = [&]() {
      if (SPL == 2) asm volatile("bar.sync %0, 256;" ::"r"(bar_id) : "memory");
    };
    uint32_t tc = 0, nit = 0;
    for (int idx, cnt; next_item(idx, cnt, true);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      const int slot = row / g.T;
      const int pl = it.c * heads_in_chunk + q * hpq + slot;
      const int t = it.i * g.T + (row % g.T);
      const Req Rq = req_of(g, it.r);  // this request's logical dims (varlen)
      const bool valid = slot < hpq && pl < g.m && t < Rq.Nq;
      const int p = it.h * g.m + pl;
      __nv_bfloat16* orow = O + (long long)it.r * g.os0 + (long long)p * g.os1 + (long long)t * g.os2 + half * DH;
      if (cnt == 0) {  // cannot happen for masks from bfla_expand_rescue (sink + band); defined anyway
        if (valid) {
          for (int c = 0; c < DH; ++c) orow[c] = __float2bfloat16(0.0f);
          if (lse && half == 0) lse[((long long)it.r * g.Hq + p) * g.Nq + t] = -INFINITY;
          for (int mi = 0; mi < g.n_mirror; ++mi) {
            for (int c = 0; c < DH; ++c) (static_cast<__nv_bfloat16*>(g.mo[mi]) + (orow - O))[c] = __float2bfloat16(0.0f);
            if (lse && half == 0 && g.ml[mi]) g.ml[mi][((long long)it.r * g.Hq + p) * g.Nq + t] = -INFINITY;
          }
          if (g.mco)
            for (int c = 0; c < DH; c += 8) multimem_st16(static_cast<__nv_bfloat16*>(g.mco) + (orow - O) + c, 0u, 0u, 0u, 0u);
          if (lse && half == 0 && g.mcl) multimem_st_f32(g.mcl + ((long long)it.r * g.Hq + p) * g.Nq + t, -INFINITY);
        }
        continue;
      }
      const uint32_t my_it = nit++;
      const int32_t* lst = DENSE ? nullptr : row_list(it);
      float m_run = -INFINITY, l_run = 0.0f;
      for (int n = 0; n < cnt; ++n, ++tc) {
        const int j = tile64(lst, n);
        mbar_wait(s_full + 2 * q + (tc & 1), (tc >> 1) & 1);
        tc_fence_after();
        float s[NCOL];
#pragma unroll
        for (int c0 = 0; c0 < NCOL; c0 += 32) tmem_ld32(tS0 + (tc & 1) * BN + c0, s + c0);
        tmem_wait_ld();
        // token-exact causality inside the tile (Eq. 27): key j*64 + NCOL half + c visible iff <= N_c + t
        const int lim = Rq.Nc + t - j * BN - half * NCOL;
        if (lim < NCOL - 1) {
#pragma unroll
          for (int c = 0; c < NCOL; ++c)
            if (c > lim) s[c] = -INFINITY;
        }
        constexpr int NCH = NCOL / 16;  // independent FMNMX3 chains of 16
        float mc[NCH];
#pragma unroll
        for (int k2 = 0; k2 < NCH; ++k2) {
          float a = max3f(s[16 * k2], s[16 * k2 + 1], s[16 * k2 + 2]);
#pragma unroll
          for (int c = 3; c < 15; c += 2) a = max3f(a, s[16 * k2 + c], s[16 * k2 + c + 1]);
          mc[k2] = fmaxf(a, s[16 * k2 + 15]);
        }
#pragma unroll
        for (int w2 = NCH / 2; w2 >= 1; w2 /= 2)
#pragma unroll
          for (int k2 = 0; k2 < w2; ++k2) mc[k2] = fmaxf(mc[k2], mc[k2 + w2]);
        float mrow = mc[0];
        if (SPL == 2) {
          float* rslot = red + (tc & 1) * 256;
          rslot[half * 128 + row] = mrow;
          pair_sync();
          mrow = fmaxf(rslot[row], rslot[128 + row]);
        }
        const float mx = mrow * c2;
        // lazy rescale: raise the running max only when it grows by more than 8 (2^8 headroom in
        // P and l); both halves see the same mx, so they take the same decision
        const bool need = mx > m_run + 8.0f || (m_run == -INFINITY && mx > -INFINITY);
        float alpha = 1.0f;
        if (need) {
          alpha = ex2_approx(m_run - mx);  // 0 when m_run = -inf
          l_run *= alpha;
          m_run = mx;
        }
        const float msub = m_run == -INFINITY ? 0.0f : m_run;
        // p = 2^(s c2 - m): pairs through FFMA2; 1 of every 4 pairs evaluates 2^x on the FMA pipe
        // (rel. err 8e-5 << bf16 rounding of P), the rest on MUFU.EX2.
        const float2 c22 = make_float2(c2, c2), nm2 = make_float2(-msub, -msub);
        float2 ls[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t pk[NCOL / 2];
#pragma unroll
        for (int c = 0; c < NCOL; c += 2) {
          const float2 x = __ffma2_rn(make_float2(s[c], s[c + 1]), c22, nm2);
          float2 pr;
          if ((c / 2) % 4 == 1) {
            pr = exp2_poly2(x);
          } else {
            pr.x = ex2_approx(x.x);
            pr.y = ex2_approx(x.y);
          }
          ls[(c / 2) & 3] = __fadd2_rn(ls[(c / 2) & 3], pr);
          pk[c / 2] = pack_bf16x2(pr.x, pr.y);
        }
        l_run += ((ls[0].x + ls[0].y) + (ls[1].x + ls[1].y)) + ((ls[2].x + ls[2].y) + (ls[3].x + ls[3].y));
        // P buffer tc % 2 was last read by PV_q(tc - 2); an O rescale additionally needs PV_q(tc - 1)
        // (O must contain it).  PV latency is hidden behind a whole softmax step in the common case.
        if (tc >= 2) mbar_wait(p_free + 2 * q + (tc & 1), ((tc - 2) >> 1) & 1);
        const bool resc = n > 0 && __any_sync(0xffffffffu, alpha != 1.0f);
        if (resc) mbar_wait(p_free + 2 * q + ((tc - 1) & 1), ((tc - 1) >> 1) & 1);
        tc_fence_after();
        if (resc) {
#pragma unroll 1
          for (int cc = 0; cc < DH; cc += 32) {
            float ov[32];
            tmem_ld32(tO + cc, ov);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) ov[e] *= alpha;
            tmem_st32(tO + cc, ov);
          }
          tmem_wait_st();
        }
        // P row -> smem, 128B-swizzled K-major (16-byte chunk cc of row r at cc ^ (r & 7))
        unsigned char* prow = sPq + (tc & 1) * C::PBYTES + row * 128;
#pragma unroll
        for (int cc = 0; cc < NCOL / 8; ++cc)
          *reinterpret_cast<uint4*>(prow + (((half * (NCOL / 8) + cc) ^ (row & 7)) << 4)) =
              make_uint4(pk[4 * cc], pk[4 * cc + 1], pk[4 * cc + 2], pk[4 * cc + 3]);
        fence_proxy_async_smem();
        tc_fence_before();
        mbar_arrive(p_full + 2 * q + (tc & 1));
      }
      // epilogue: combine the two partial sums; O / l -> bf16 -> global; LSE = (m + log2 l) ln 2
      float l_tot = l_run;
      if (SPL == 2) {
        float* lslot = red + (tc & 1) * 256;  // the slot parity tc hasn't been written for this item
        lslot[half * 128 + row] = l_run;
        pair_sync();
        l_tot = lslot[row] + lslot[128 + row];
      }
      mbar_wait(o_full + q, my_it & 1);
      tc_fence_after();
      const float inv_l = l_tot > 0.0f ? 1.0f / l_tot : 0.0f;
#pragma unroll 1
      for (int cc = 0; cc < DH; cc += 32) {
        float ov[32];
        tmem_ld32(tO + cc, ov);
        tmem_wait_ld();
        if (valid) {
          uint32_t w[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(ov[2 * e] * inv_l, ov[2 * e + 1] * inv_l);
          uint4* dst = reinterpret_cast<uint4*>(orow + cc);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          for (int mi = 0; mi < g.n_mirror; ++mi) {  // fused exchange (bfla_sparse_prefill_mirrored)
            uint4* md = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(g.mo[mi]) + (orow - O) + cc);
#pragma unroll
            for (int e = 0; e < 4; ++e) md[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          }
          if (g.mco) {  // NVLS multicast: one store per 16 bytes reaches every member GPU
            __nv_bfloat16* mc = static_cast<__nv_bfloat16*>(g.mco) + (orow - O) + cc;
#pragma unroll
            for (int e = 0; e < 4; ++e) multimem_st16(mc + 8 * e, w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          }
        }
      }
      if (valid && lse && half == 0) {
        const long long li = ((long long)it.r * g.Hq + p) * g.Nq + t;
        const float lv = l_tot > 0.0f ? (m_run + log2f(l_tot)) * 0.6931471805599453f : -INFINITY;
        lse[li] = lv;
        for (int mi = 0; mi < g.n_mirror; ++mi)
          if (g.ml[mi]) g.ml[mi][li] = lv;
        if (g.mcl) multimem_st_f32(g.mcl + li, lv);
      }
      tc_fence_before();
      mbar_arrive(o_free + q);
      pair_sync();  // partner has read lslot before the slot is reused by the next item's tile tc
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

}  // namespace

size_t attn_smem_bytes(int D, int nqt) {
  if (D == 128) return nqt == 2 ? Cfg<128, 2, 1>::SMEM_TOTAL : Cfg<128, 1, 1>::SMEM_TOTAL;
  return Cfg<256, 1, 1>::SMEM_TOTAL;
}

template <int D, int NQT, bool PAGED, bool DENSE, int SPL>
static int launch_t(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                    const int32_t* pt, void* o, float* lse, int n_items, int hpq, int NC, int num_sms,
                    cudaStream_t st, int* sched) {
  using C = Cfg<D, NQT, SPL>;
  auto kern = k_attn<D, NQT, PAGED, DENSE, SPL>;
  if constexpr (!DENSE && SPL == 1)
    if (g.nrows) kern = k_attn<D, NQT, PAGED, false, 1, true>;  // work slice (bfla_sparse_prefill_rows)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, C::SMEM_TOTAL);
  if (e != cudaSuccess) return (int)e;
  const int grid = n_items < num_sms ? n_items : num_sms;
  kern<<<grid, C::THREADS, C::SMEM_TOTAL, st>>>(maps.q, maps.k, maps.v, g, list, count, pt,
                                          static_cast<__nv_bfloat16*>(o), lse, n_items, hpq, NC, sched);
  count_launch();
  return (int)cudaGetLastError();
}

// Rows of one item: NQT 128-row tiles, each holding hpq = 128/T heads of T rows; NQT = 2 when the
// group has more than one tile of rows and TMEM allows (d = 128: 2 x (64 S + 128 O) columns).
int launch_attention(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                     const int32_t* page_table, int dense, void* o, float* lse, int num_sms, cudaStream_t st,
                     int* sched) {
  const int hpq = BM / g.T;
  const int nqt = (g.D == 128 && g.m > hpq) ? 2 : 1;
  const int NC = (g.m + nqt * hpq - 1) / (nqt * hpq);
  const long long items = (g.nrows ? (long long)g.nrows : (long long)g.B * g.Hkv * g.Tq) * NC;
  if (items == 0) return 0;
  const int n = (int)items;
  // softmax warpgroups per Q tile: 1 (default) or 2 (BFLA_SOFTMAX_SPLIT=2, A/B experiments)
  static const int spl = experiment_knob("BFLA_SOFTMAX_SPLIT", 1) == 2 ? 2 : 1;
#define BFLA_GO(D_, Q_, P_, X_)                                                                          \
  return spl == 2                                                                                        \
             ? launch_t<D_, Q_, P_, X_, 2>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched) \
             : launch_t<D_, Q_, P_, X_, 1>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched)
  const bool paged = g.paged != 0;
  if (g.D == 128 && nqt == 2) {
    if (paged) { if (dense) BFLA_GO(128, 2, true, true); else BFLA_GO(128, 2, true, false); }
    else { if (dense) BFLA_GO(128, 2, false, true); else BFLA_GO(128, 2, false, false); }
  } else if (g.D == 128) {
    if (paged) { if (dense) BFLA_GO(128, 1, true, true); else BFLA_GO(128, 1, true, false); }
    else { if (dense) BFLA_GO(128, 1, false, true); else BFLA_GO(128, 1, false, false); }
  } else {
    if (paged) { if (dense) BFLA_GO(256, 1, true, true); else BFLA_GO(256, 1, true, false); }
    else { if (dense) BFLA_GO(256, 1, false, true); else BFLA_GO(256, 1, false, false); }
  }
#undef BFLA_GO
}

}  // namespace bfla
