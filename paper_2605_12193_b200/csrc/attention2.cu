// attention2.cu — fused sparse causal prefill (Eq. 27) and dense twin (Eq. 1), head_dim 128,
// processing the kept-tile list TWO TILES PER STEP.
//
// Any two kept KV tiles (j_a, j_b) of a row fill rows 0-63 / 64-127 of one K (and V) ring slot, so
// S = Q [K_a; K_b]^T is a single full-rate M128 x N128 tcgen05 MMA chain (an N=64 MMA reading both
// operands from shared memory runs at 2/3 rate: operand bandwidth) and O += P [V_a; V_b] is one K=128
// chain.  The mask granularity stays T = 64 (R10): pairing is an execution detail — each half is
// masked with its own tile's token-exact causal frontier, and a lone last tile runs as an N=64 step.
//
// P is written by the softmax threads straight into TMEM over the S columns it came from (packed
// bf16 pairs, row = lane) and consumed by the PV MMA as its A operand ("TS" form), so shared memory
// holds only Q and the K/V rings.  The two Q tiles (GQA packing: 2 heads x 64 rows each) ping-pong:
// while one softmax warpgroup works, the tensor core runs the other tile's PV and next S.
//
// Roles: warp 0 TMA Q + K, warp 3 TMA V, warp 1 MMA issue (converged, elect.sync), warp 2 TMEM
// allocation, warps 4.. one softmax warpgroup per Q tile (thread = row = TMEM lane).  setmaxnreg
// moves registers from the first warpgroup (96) to the softmax warpgroups (200), which read the
// whole 128-column S row of a step with one TMEM round trip, take the row max first, apply the lazy
// rescale rule and only then compute the exponentials (MAXFIRST; BFLA_MAXFIRST=0 selects the older
// single-pass-with-redo variant).  Timeline instrumentation: -DBFLA_TRACE (tools/attn_trace.py).
#include <cuda_bf16.h>

#include <cstdlib>

#include "attn_common.cuh"
#include "common.cuh"
#include "kernels.h"

namespace bfla {

#ifdef BFLA_TRACE
// Timeline instrumentation (trace build only: libbfla_trace.so, tools/attn_trace.py).  CTAs below
// kTraceCtas record (code, clock64) events per warp role into g_trace[cta][role][kTraceN].
__device__ unsigned long long* g_trace = nullptr;
constexpr int kTraceCtas = 4, kTraceRoles = 6, kTraceN = 8192;
extern "C" int bfla_debug_set_trace(void* buf) {
  return (int)cudaMemcpyToSymbol(g_trace, &buf, sizeof(buf));
}
#define TRACE(role, code)                                                                              \
  do {                                                                                                 \
    if (g_trace && blockIdx.x < kTraceCtas && (threadIdx.x & 31) == 0 && tr_n[role] < kTraceN) {       \
      g_trace[((size_t)blockIdx.x * kTraceRoles + (role)) * kTraceN + tr_n[role]++] =                  \
          ((unsigned long long)(code) << 56) | ((unsigned long long)clock64() & 0xFFFFFFFFFFFFFFull);  \
    }                                                                                                  \
  } while (0)
#else
#define TRACE(role, code) \
  do {                    \
  } while (0)
#endif

namespace {
using namespace attn;

constexpr int D = 128;
constexpr int BM = 128;   // MMA M (rows of a Q tile)
constexpr int BN = 64;    // mask tile T
constexpr int RS = 128;   // K/V rows per ring slot (two tiles)
// lazy-rescale headroom (log2 units): p = 2^(x - m_run) <= 2^24; O <= 2^24 * N_kv * |V| << fp32 max
constexpr float kLazy = 24.0f;

template <int NQT, bool PAGED = false, int SPLIT = 1>
struct Cfg2 {
  // BFLA_QRING=1: Q ring of NQT + 1 tiles (the next item's first Q tile loads while this item still
  // holds its tiles) at the price of a 2-deep K ring.  Default off: a 3-deep K ring measured better
  // (K loads arrive ~2 us after their slot frees; sparse 32K 1.014 -> 1.005 ms, dense 7.81 -> 7.29 ms)
#ifndef BFLA_QRING
#define BFLA_QRING 0
#endif
  static constexpr bool QR = BFLA_QRING && !PAGED;
  static constexpr int QS = QR ? NQT + 1 : NQT, KS = QR ? 2 : 3, VS = NQT == 2 ? 2 : 3;
  static constexpr int QBYTES = BM * D * 2;       // 32 KB
  static constexpr int SLOT = RS * D * 2;         // 32 KB (two 64-row tiles)
  static constexpr int HALF = BN * 128;           // bytes of one 64-row half of a 64-column chunk
  static constexpr int CHUNK = RS * 128;          // bytes of one 64-column chunk of a slot
  static constexpr int OFF_Q = 0;
  static constexpr int OFF_K = OFF_Q + QS * QBYTES;
  static constexpr int OFF_V = OFF_K + KS * SLOT;
  static constexpr int OFF_BAR = OFF_V + VS * SLOT;
  static constexpr int NBAR = 2 * QS + 2 * KS + 2 * VS + 5 * NQT + 2 * 4;  // + item ring full/empty, p_half
  static constexpr int OFF_RING = OFF_BAR + NBAR * 8 + 16;  // int2 (item index, kept-tile count) x 4
  static constexpr int OFF_LX = OFF_RING + 4 * 8;  // SPLIT: row sums of the two column halves [NQT][2][128]
  static constexpr int SMEM_TOTAL = OFF_LX + (SPLIT == 2 ? NQT * 2 * 128 * 4 : 0);
  static constexpr int THREADS = 128 + 128 * SPLIT * NQT;
  static constexpr int COL_S = 0;    // S_q / P_q at columns [128 q, 128 q + 128)
  static constexpr int COL_O = 256;  // O_q at [256 + 128 q, ...)
  static_assert(SMEM_TOTAL <= 232448, "shared memory budget");
};

// SMX: softmax variant — 0 fused single pass with exact redo, 1 max-first whole row per thread
// (MAXFIRST, default).  (Splitting a Q tile's 128 columns over two warpgroups with a row-max
// exchange was measured 10% slower: the exponential phases of all softmax warps then coincide.)
// BFLA_SPLIT_P (default 1; 0 for A/B): the PV of a two-tile step is issued in halves — tile a's 4 MMAs
// as soon as its P is in TMEM (p_half), tile b's after p_full — so PV_a overlaps the softmax of tile b
// and the softmax -> MMA -> softmax chain of a Q tile shortens by PV_a.  Measured (same box, 5 runs):
// sparse 32K 0.964 -> 0.937 ms, 128K 9.31 -> 8.95 ms, dense 32K 6.89 -> 6.75-6.85 ms; O bit-identical.
// Not kept: a 3/4 split (p_half after 96 keys: 0.951 ms), the split with half of tile b's exponentials
// run before the wait on tile a's stores (0.940 / 8.84 ms: equal within noise), the row sum taken
// from the stored bf16 P after the arrive (1.013 ms: the deferred adds delay the next step), and both
// softmax warpgroups sharing each Q tile by column halves with a smem row-max exchange (correct on the
// parity suite, but 1.046 vs 0.935 ms / 10.38 vs 9.25 ms at 128K: the TMEM load, exchange and P-store
// latencies are then paid twice per step per warpgroup).
#ifndef BFLA_SPLIT_P
#define BFLA_SPLIT_P 1
#endif
template <int NQT, bool PAGED, bool DENSE, int SMX, int POLY, bool SLICE = false>
__global__ void __launch_bounds__(Cfg2<NQT, PAGED>::THREADS, 1)
    k_attn2(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmK,
            const __grid_constant__ CUtensorMap tmV, const __grid_constant__ CUtensorMap tmO,
            const __grid_constant__ MirrorMaps tmM, int otma, Geom g, const int32_t* __restrict__ list,
            const int32_t* __restrict__ count, const int32_t* __restrict__ page_table,
            __nv_bfloat16* __restrict__ O, float* __restrict__ lse, int n_items, int hpq, int NC, int opts,
            int* __restrict__ sched) {
  constexpr bool MAXFIRST = SMX >= 1;
  constexpr bool SPLITP = BFLA_SPLIT_P && SMX == 1;  // split PV issue (the SMX = 1 softmax arrives p_half)
  constexpr int SPL = 1;
  using C = Cfg2<NQT, PAGED>;
  extern __shared__ __align__(1024) unsigned char smem[];
  if (smem_u32(smem) & 1023) __trap();  // SW128 operands need 1024-byte alignment (no static smem here)
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
  uint64_t* q_full = bars + 0;          // [QS]: Q ring slot loaded
  uint64_t* q_empty = bars + C::QS;     // [QS]: Q ring slot free (last S done / staged O stored from it)
  uint64_t* k_full = bars + 2 * C::QS;
  uint64_t* k_empty = k_full + C::KS;
  uint64_t* v_full = k_empty + C::KS;
  uint64_t* v_empty = v_full + C::VS;
  uint64_t* s_full = v_empty + C::VS;  // [NQT]: S_q(s) in TMEM (also: PV_q(s-1) done)
  uint64_t* p_full = s_full + NQT;     // [NQT]: P_q(s) in TMEM (128 arrivals)
  uint64_t* o_full = p_full + NQT;     // [NQT]: last PV of the item done
  uint64_t* o_free = o_full + NQT;     // [NQT]: epilogue has read O (128 arrivals)
  uint64_t* it_full = o_free + NQT;    // [4]: item ring entry published (K producer)
  uint64_t* it_empty = it_full + 4;    // [4]: entry read by every other role (11 warps)
  uint64_t* p_half = it_empty + 4;     // [NQT]: P_q of the step's first kept tile in TMEM (BFLA_SPLIT_P)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * C::QS + 2 * C::KS + 2 * C::VS + 5 * NQT + 8);
  volatile int* ring = reinterpret_cast<volatile int*>(smem + C::OFF_RING);  // [4][2]

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
    for (int q = 0; q < NQT; ++q) {
      mbar_init(s_full + q, 1);
      mbar_init(p_full + q, 128 * SPL);
      mbar_init(o_full + q, 1);
      mbar_init(o_free + q, 128 * SPL);
      mbar_init(p_half + q, 128 * SPL);
    }
    for (int e = 0; e < 4; ++e) {
      mbar_init(it_full + e, 1);
      mbar_init(it_empty + e, 3 + 4 * NQT * SPL);  // warps 1, 2, 3 and the softmax warps
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
  // Q tile q of the CTA's my_it-th item lives in ring slot qslot; qpar = parity of that slot's fill
  auto qslot = [&](uint32_t my_it, int q) -> int { return (int)((NQT * my_it + q) % C::QS); };
  auto qpar = [&](uint32_t my_it, int q) -> uint32_t { return ((NQT * my_it + q) / C::QS) & 1; };
  // registers (NQT = 2, MAXFIRST): the producer / MMA warpgroup needs few, the softmax warpgroups
  // hold a whole S row (128 fp32) plus its packed P: 128 x 96 + 256 x 200 <= 384 x 168 (the launch
  // allocation).  Each setmaxnreg dominates its role's code.
#ifdef BFLA_TRACE
  int tr_n[kTraceRoles] = {0, 0, 0, 0, 0, 0};
#endif

  // The kernel works in 64-key tiles (BN); a mask tile of T = 128 is two of them,
  // so counts scale by TR = T / 64 and the n-th 64-key tile of a row is half (n & 1) of list entry n / 2
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
  auto row_list = [&](const Item& it) -> const int32_t* {
    const int32_t* l =
        list + ((long long)it.r * g.Hkv + it.h) * g.causal_per_head + req_row_offset(req_of(g, it.r), g.T, it.i);
    if (!g.kv_range) return l;
    return l + list_lower_bound(l, count[((long long)it.r * g.Hkv + it.h) * g.Tq + it.i], g.kv_lo);
  };
  // tiles are visited in DESCENDING j (diagonal / local band first): the largest scores usually sit
  // near the diagonal, so the running max settles on the first step and the lazy-max fast path holds
  auto tile_at_c = [&](const int32_t* lst, int cnt, int n) -> int {
    const int pos = cnt - 1 - n;  // ascending position among the row's 64-key tiles
    if (DENSE) return pos;
    return TR == 1 ? __ldg(lst + pos) : 2 * __ldg(lst + (pos >> 1)) + (pos & 1);
  };
  // Item sequence.  The K producer (furthest ahead) picks items — the CTA's first is blockIdx.x, the
  // next ones come from a global counter (greedy longest-first list scheduling: items are ordered by
  // descending row length, so a CTA that finishes early takes the next heaviest item) or, without a
  // counter, blockIdx.x + k gridDim.x — and publishes (index, kept-tile count) in a 4-entry smem ring;
  // every other role (one warp at a time) reads the ring in order.  Index -1 ends the sequence.
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

  // One ring step of K (kvsel = 0) or V (kvsel = 1), issued by a whole warp: lanes fetch the list
  // entries and page-table entries concurrently (no chain of dependent global loads on one thread)
  // and each lane issues its own TMA boxes.  Tile a fills rows 0-63 of the slot, tile b rows 64-127.
  auto load_step = [&](int kvsel, uint32_t ks, const int32_t* lst, int cnt, int s, const Item& it) {
    const int ns_ = kvsel ? C::VS : C::KS;
    const int st = ks % ns_;
    uint64_t* full = (kvsel ? v_full : k_full) + st;
    mbar_wait((kvsel ? v_empty : k_empty) + st, ((ks / ns_) & 1) ^ 1);
    const bool two = 2 * s + 1 < cnt;
    // lane 0 / 1: list entries of tiles a / b (descending j, see tile_at_c)
    int jl = 0;
    if (lane < (two ? 2 : 1)) jl = tile_at_c(lst, cnt, 2 * s + lane);
    const int ja = __shfl_sync(0xffffffffu, jl, 0), jb = __shfl_sync(0xffffffffu, jl, 1);
    if (lane == 0) mbar_arrive_expect_tx(full, (two ? 2 : 1) * BN * D * 2);
    __syncwarp();
    unsigned char* dst = smem + (kvsel ? C::OFF_V : C::OFF_K) + st * C::SLOT;
    const CUtensorMap* map = kvsel ? &tmV : &tmK;
    if (!PAGED) {
      // lane = (tile, d-chunk)
      const int ntile = two ? 2 : 1;
      if (lane < ntile * (D / 64)) {
        const int hf = lane / (D / 64), cc = lane % (D / 64);
        tma_load_4d(dst + cc * C::CHUNK + hf * C::HALF, map, full, cc * 64, (hf ? jb : ja) * BN, it.h / g.kvdiv,
                    it.r);
      }
    } else {
      // lane = (tile, page of the tile): BN / page_size page boxes of (64 columns x ps rows) per
      // d-chunk; a page past the request's last logical page (ragged tail) is replaced by its first
      // page (finite data; those keys are masked by causality and get P = 0)
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

  if (warp < 4) {
#ifndef BFLA_REG_PROD
#define BFLA_REG_PROD 96
#define BFLA_REG_SMX 200
#endif
    if (NQT == 2 && SMX == 1) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(BFLA_REG_PROD) : "memory");
  if (warp == 0) {
    // ================================ TMA producer (K) ================================
    {
      uint32_t ks = 0;
      int idx = blockIdx.x;
      for (;;) {
        const bool live = idx < n_items;
        const Item it = decode_item<SLICE>(g, live ? idx : 0, NC);
        const int cnt = live ? row_count(it) : 0;
        {  // publish (idx, cnt) — or the end marker
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
        int nidx = 0;  // the next item, fetched before this one's loads so the atomic's latency hides
        if (lane == 0) nidx = sched ? (int)gridDim.x + atomicAdd(sched, 1) : idx + (int)gridDim.x;
        nidx = __shfl_sync(0xffffffffu, nidx, 0);
        if (cnt > 0) {
          const int32_t* lst = DENSE ? nullptr : row_list(it);
          const int ns = (cnt + 1) / 2;
          for (int s = 0; s < ns; ++s, ++ks) {
            load_step(0, ks, lst, cnt, s, it);
            TRACE(1, 6);
          }
        }
        idx = nidx;
      }
    }
  } else if (warp == 2) {
    // ================================ TMA producer (Q) ================================
    // Q tile q of the next item is loaded as soon as its smem is free: after the last S_q MMA (STG
    // epilogue) or after O_q, staged through the same smem, has been read by the TMA store.
    uint32_t nit = 0;
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      if (cnt == 0) continue;
      const uint32_t my_it = nit++;
#pragma unroll
      for (int q = 0; q < NQT; ++q) {
        const int qsl = qslot(my_it, q);
        mbar_wait(q_empty + qsl, qpar(my_it, q) ^ 1);
        if (q == 0) TRACE(5, 14);
        if (lane == 0) {
          int nb = 0;
          for (int s = 0; s < hpq; ++s)
            if (it.c * heads_in_chunk + q * hpq + s < g.m) nb += D / 64;
          mbar_arrive_expect_tx(q_full + qsl, nb * 64 * g.T * 2);
        }
        __syncwarp();
        {  // lane = (head slot, d-chunk)
          const int s = lane / (D / 64), cc = lane % (D / 64);
          const int pl = it.c * heads_in_chunk + q * hpq + s;
          if (s < hpq && pl < g.m)
            tma_load_4d(smem + C::OFF_Q + qsl * C::QBYTES + cc * (BM * 128) + s * (g.T * 128), &tmQ, q_full + qsl,
                        cc * 64, it.i * g.T, it.h * g.m + pl, it.r);
        }
      }
      if (!sched && !(opts & 1) && lane == 0 && idx + (int)gridDim.x < n_items) {  // warm L2: next item's Q
        const Item nx = decode_item<SLICE>(g, idx + gridDim.x, NC);
        for (int q = 0; q < NQT; ++q)
          for (int s = 0; s < hpq; ++s) {
            const int pl = nx.c * heads_in_chunk + q * hpq + s;
            if (pl >= g.m) continue;
            for (int cc = 0; cc < D / 64; ++cc) tma_prefetch_4d(&tmQ, cc * 64, nx.i * g.T, nx.h * g.m + pl, nx.r);
          }
      }
    }
  } else if (warp == 3) {
    // ================================ TMA producer (V) ================================
    {
      uint32_t ks = 0;
      for (int idx, cnt; next_item(idx, cnt);) {
        const Item it = decode_item<SLICE>(g, idx, NC);
        if (cnt == 0) continue;
        const int32_t* lst = DENSE ? nullptr : row_list(it);
        const int ns = (cnt + 1) / 2;
        for (int s = 0; s < ns; ++s, ++ks) {
          load_step(1, ks, lst, cnt, s, it);
          TRACE(2, 7);
        }
      }
    }
  } else if (warp == 1) {
    // ================================ MMA issuer ================================
    // Step s: [PV_q(s-1) (A = P_q in TMEM), S_q(s)] per Q tile.  S_q(s) overwrites the TMEM columns
    // P_q(s-1) occupies, after the PV that reads them (tcgen05 MMAs of one thread execute in order).
    const uint64_t dQ = sdesc_sw128(smem_u32(smem + C::OFF_Q), 16, 1024);
    const uint64_t dK = sdesc_sw128(smem_u32(smem + C::OFF_K), 16, 1024);
    const uint64_t dV = sdesc_sw128(smem_u32(smem + C::OFF_V), C::CHUNK, 1024);
    uint32_t ks0 = 0, nit = 0, st0 = 0;
    auto issue_PV = [&](int q, uint32_t vslot, int ntile, bool acc_first, int kk0 = 0) {
      const uint32_t idO = idesc_bf16(BM, D, 0, 1);
      const uint64_t b0 = dV + (uint64_t)((vslot * C::SLOT) >> 4);
      const uint32_t aP = tmem + C::COL_S + q * 128;
#pragma unroll 8
      for (int kk = kk0; kk < ntile * 4; ++kk)
        umma_f16_ts_warp(tmem + C::COL_O + q * D, aP + kk * 8,
                         b0 + (uint64_t)((kk * 2048) >> 4), idO, (acc_first || kk > 0) ? 1u : 0u);
    };
    // BFLA_SPLIT_P: PV of a two-tile step in two halves — tile a's 4 MMAs as soon as its P is in TMEM
    // (p_half), tile b's after p_full — so PV_a overlaps the softmax of tile b
    uint32_t hph = 0;  // two-tile steps whose p_half has been consumed (same count for every q)
    auto issue_PV_split = [&](int q, uint32_t vslot, uint32_t pfull_par, bool acc_first, bool first_of_item,
                              uint32_t my_it, int ntile = 2) {
      mbar_wait(p_half + q, hph & 1);
      if (first_of_item) mbar_wait(o_free + q, (my_it & 1) ^ 1);
      tc_fence_after();
      issue_PV(q, vslot, 1, acc_first);  // tile a: keys 0..63, P columns 0..31
      mbar_wait(p_full + q, pfull_par);
      tc_fence_after();
      if (ntile == 2) issue_PV(q, vslot, 2, true, 4);  // tile b
    };
    auto issue_S = [&](int q, int qsl, uint32_t kslot, int ntile) {
      const uint32_t idS = ntile == 2 ? idesc_bf16(BM, 2 * BN, 0, 0) : idesc_bf16(BM, BN, 0, 0);
      const uint64_t a0 = dQ + (uint64_t)((qsl * C::QBYTES) >> 4), b0 = dK + (uint64_t)((kslot * C::SLOT) >> 4);
#pragma unroll
      for (int kk = 0; kk < D / 16; ++kk) {
        const uint32_t offa = ((kk >> 2) * (BM * 128) + (kk & 3) * 32) >> 4;
        const uint32_t offb = ((kk >> 2) * C::CHUNK + (kk & 3) * 32) >> 4;
        umma_f16_ss_warp(tmem + C::COL_S + q * 128, a0 + offa, b0 + offb, idS, kk > 0 ? 1u : 0u);
      }
      umma_commit_warp(s_full + q);
    };
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      (void)it;
      if (cnt == 0) continue;
      const uint32_t my_it = nit++;
      const int ns = (cnt + 1) / 2;
      TRACE(0, 24);
      for (int s = 0; s < ns; ++s) {
        const uint32_t ksn = ks0 + s, kst = ksn % C::KS;
        mbar_wait(k_full + kst, (ksn / C::KS) & 1);
        TRACE(0, 1);
        uint32_t vst = 0;
        if (s > 0) {
          vst = (ksn - 1) % C::VS;
          mbar_wait(v_full + vst, ((ksn - 1) / C::VS) & 1);
          TRACE(0, 2);
        }
        tc_fence_after();
        const int nt = 2 * s + 1 < cnt ? 2 : 1;
#pragma unroll
        for (int q = 0; q < NQT; ++q) {
          if (s > 0) {  // O_q += P_q(s-1) [V]
            if constexpr (SPLITP) {
              issue_PV_split(q, vst, (st0 + s - 1) & 1, s > 1, s == 1, my_it);
              if (q == NQT - 1) ++hph;
            } else {
            mbar_wait(p_full + q, (st0 + s - 1) & 1);
            TRACE(0, 3 + 16 * q);
            if (s == 1) mbar_wait(o_free + q, (my_it & 1) ^ 1);
            tc_fence_after();
            issue_PV(q, vst, 2, s > 1);  // every step but the last holds two tiles
            }
          }
          const int qsl = qslot(my_it, q);
          if (s == 0) {
            mbar_wait(q_full + qsl, qpar(my_it, q));
            if (q == 0) TRACE(0, 15);
            tc_fence_after();
          }
          issue_S(q, qsl, kst, nt);
          TRACE(0, 4 + 16 * q);
          if (s == ns - 1 && !otma) umma_commit_warp(q_empty + qsl);  // every S_q MMA of the item issued
        }
        umma_commit_warp(k_empty + kst);
        if (s > 0) umma_commit_warp(v_empty + vst);
      }
      // tail: O_q += P_q(ns-1) [V]
      const uint32_t ksl = ks0 + ns - 1, vst = ksl % C::VS;
      mbar_wait(v_full + vst, (ksl / C::VS) & 1);
      tc_fence_after();
      const int ntl = cnt - 2 * (ns - 1);
#pragma unroll
      for (int q = 0; q < NQT; ++q) {
        if (SPLITP && ntl == 2) {
          issue_PV_split(q, vst, (st0 + ns - 1) & 1, ns > 1, ns == 1, my_it, ntl);
          if (q == NQT - 1) ++hph;
        } else {
        mbar_wait(p_full + q, (st0 + ns - 1) & 1);
        TRACE(0, 5 + 16 * q);
        if (ns == 1) mbar_wait(o_free + q, (my_it & 1) ^ 1);
        tc_fence_after();
        issue_PV(q, vst, ntl, ns > 1);
        }
        umma_commit_warp(o_full + q);
      }
      umma_commit_warp(v_empty + vst);
      ks0 += ns;
      st0 += ns;
    }
  }
  } else {
    if (NQT == 2 && SMX == 1) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(BFLA_REG_SMX) : "memory");

    // ================================ softmax / epilogue ================================
    const int q = (warp - 4) >> 2;
    const int lg = warp & 3;         // TMEM lane group of this warp
    const int row = lg * 32 + lane;  // row of Q tile q = TMEM lane
    const uint32_t lane_addr = (uint32_t)(lg * 32) << 16;
    const uint32_t tS = tmem + lane_addr + C::COL_S + q * 128;
    const uint32_t tO = tmem + lane_addr + C::COL_O + q * D;
    const float c2 = g.scale * 1.4426950408889634f;  // softmax scale in the exp2 domain
    uint32_t st = 0, nit = 0;
    for (int idx, cnt; next_item(idx, cnt);) {
      const Item it = decode_item<SLICE>(g, idx, NC);
      const int slot = row / g.T;
      const int pl = it.c * heads_in_chunk + q * hpq + slot;
      const int t = it.i * g.T + (row % g.T);
      const Req Rq = req_of(g, it.r);  // this request's logical dims (varlen)
      const bool valid = slot < hpq && pl < g.m && t < Rq.Nq;
      const int p = it.h * g.m + pl;
      __nv_bfloat16* orow = O + (long long)it.r * g.os0 + (long long)p * g.os1 + (long long)t * g.os2;
      if (cnt == 0) {  // cannot happen for masks from bfla_expand_rescue (sink + band); defined anyway
        if (valid) {
          for (int c = 0; c < D; ++c) orow[c] = __float2bfloat16(0.0f);
          if (lse) lse[((long long)it.r * g.Hq + p) * g.Nq + t] = -INFINITY;
          for (int mi = 0; mi < g.n_mirror; ++mi) {
            for (int c = 0; c < D; ++c) (static_cast<__nv_bfloat16*>(g.mo[mi]) + (orow - O))[c] = __float2bfloat16(0.0f);
            if (lse && g.ml[mi]) g.ml[mi][((long long)it.r * g.Hq + p) * g.Nq + t] = -INFINITY;
          }
          if (g.mco)
            for (int c = 0; c < D; c += 8) multimem_st16(static_cast<__nv_bfloat16*>(g.mco) + (orow - O) + c, 0u, 0u, 0u, 0u);
          if (lse && g.mcl) multimem_st_f32(g.mcl + ((long long)it.r * g.Hq + p) * g.Nq + t, -INFINITY);
        }
        continue;
      }
      const uint32_t my_it = nit++;
      const int32_t* lst = DENSE ? nullptr : row_list(it);
      const int ns = (cnt + 1) / 2;
      float m_run = -INFINITY, l_run = 0.0f;
      for (int s = 0; s < ns; ++s, ++st) {
        const bool two = 2 * s + 1 < cnt;
        const int ja = tile_at_c(lst, cnt, 2 * s), jb = two ? tile_at_c(lst, cnt, 2 * s + 1) : 0;
        mbar_wait(s_full + q, st & 1);
        if (lg == 0) TRACE(3 + q, 8);
        tc_fence_after();
        // token-exact causality inside each tile (Eq. 27): key j*64 + c visible iff <= N_c + t
        const int la = Rq.Nc + t - ja * BN, lb = two ? Rq.Nc + t - jb * BN : -1;
        // p = 2^(s c2 - m) in pairs (FFMA2); 1 of every 4 pairs on the FMA pipe (rel. err 8e-5 << bf16
        // rounding of P), the rest on MUFU.EX2.  Results are packed bf16 pairs, stored after the step.
        uint32_t pk[64];
        float2 ls[4];
        auto exps64 = [&](const float* v, int hf, float msub) {
          const float2 c22 = make_float2(c2, c2), nm2 = make_float2(-msub, -msub);
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float2 x = __ffma2_rn(make_float2(v[2 * e], v[2 * e + 1]), c22, nm2);
            float2 pr;
#ifdef BFLA_WHATIF_NOEXP
            if (true) {  // timing what-if (A/B builds only): no exponential at all
              pr = x;
            } else
#endif
            if ((POLY >> (e % 8)) & 1) {  // POLY: bit mask over e mod 8 of the pairs on the FMA pipe
              pr = exp2_poly2(x);
            } else {
              pr.x = ex2_approx(x.x);
              pr.y = ex2_approx(x.y);
            }
            ls[e & 3] = __fadd2_rn(ls[e & 3], pr);
            pk[hf * 32 + e] = pack_bf16x2(pr.x, pr.y);
          }
        };
        auto load64 = [&](float* v, int hf) {
          tmem_ld32(tS + hf * 64, v);
          tmem_ld32(tS + hf * 64 + 32, v + 32);
          tmem_wait_ld();
          const int lim = hf ? lb : la;
          if (lim < BN - 1) {
#pragma unroll
            for (int c = 0; c < BN; ++c)
              if (c > lim) v[c] = -INFINITY;
          }
        };
        auto max64 = [&](const float* v) { return row_max64(v); };
        if (MAXFIRST) {
          // whole S row in registers with ONE TMEM round trip (setmaxnreg gives the softmax
          // warpgroups 224 registers); row max first, then the lazy rule, then exponentials.  P of
          // the first tile goes to TMEM while the second tile's exponentials run.
          float v[128];
#ifdef BFLA_WHATIF_NOLOAD  // timing what-if (A/B builds only): S never read from TMEM
#pragma unroll
          for (int c = 0; c < 128; ++c) v[c] = l_run * 1e-30f + (float)(c & 15);
#else
          tmem_ld32(tS, v);
          tmem_ld32(tS + 32, v + 32);
          if (two) {
            tmem_ld32(tS + 64, v + 64);
            tmem_ld32(tS + 96, v + 96);
          }
          tmem_wait_ld();
#endif
          if (lg == 0) TRACE(3 + q, 16);
          if (la < BN - 1) {
#pragma unroll
            for (int c = 0; c < BN; ++c)
              if (c > la) v[c] = -INFINITY;
          }
          if (two && lb < BN - 1) {
#pragma unroll
            for (int c = 0; c < BN; ++c)
              if (c > lb) v[BN + c] = -INFINITY;
          }
          float mrow = max64(v);
          if (two) mrow = fmaxf(mrow, max64(v + BN));
          const float mx = mrow * c2;
          float alpha = 1.0f;
          // lazy rescale: raise the running max only when it grows by more than kLazy (P <= 2^kLazy:
          // bf16 P, fp32 l and O stay far inside their range)
          if (mx > m_run + kLazy || (m_run == -INFINITY && mx > -INFINITY)) {
            alpha = ex2_approx(m_run - mx);  // 0 when m_run = -inf
            l_run *= alpha;
            m_run = mx;
          }
          const float msub = m_run == -INFINITY ? 0.0f : m_run;
          ls[0] = ls[1] = ls[2] = ls[3] = make_float2(0.f, 0.f);
          if (SPLITP && s > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
            // PV of tile a may start before this step's P is complete: rescale O first (O is
            // complete through PV(s-1): the s_full commit covers every earlier MMA)
#pragma unroll 1
            for (int cc = 0; cc < D; cc += 32) {
              float ov[32];
              tmem_ld32(tO + cc, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] *= alpha;
              tmem_st32(tO + cc, ov);
            }
          }
          exps64(v, 0, msub);
          tmem_st16(tS, pk);
          tmem_st16(tS + 16, pk + 16);
          if (lg == 0) TRACE(3 + q, 17);
          if (two) {
            if (SPLITP) {  // tile a's P (and any O rescale) visible to the MMA warp
              tmem_wait_st();
              tc_fence_before();
              mbar_arrive(p_half + q);
            }
            exps64(v + BN, 1, msub);
            tmem_st16(tS + 32, pk + 32);
            tmem_st16(tS + 48, pk + 48);
          }
          if (lg == 0) TRACE(3 + q, 9);
          if (!SPLITP && s > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
            // O is complete through PV(s-1): the s_full commit covers every earlier MMA
#pragma unroll 1
            for (int cc = 0; cc < D; cc += 32) {
              float ov[32];
              tmem_ld32(tO + cc, ov);
              tmem_wait_ld();
#pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] *= alpha;
              tmem_st32(tO + cc, ov);
            }
          }
          l_run += ((ls[0].x + ls[0].y) + (ls[1].x + ls[1].y)) + ((ls[2].x + ls[2].y) + (ls[3].x + ls[3].y));
        } else {
          // fast path (running max known): one TMEM pass against m_run, checking the max on the way;
          // valid unless some row's max grew by more than 8 (then the lazy rule moves m_run)
          bool done = false;
          float alpha = 1.0f;
          if (__all_sync(0xffffffffu, m_run != -INFINITY)) {
            ls[0] = ls[1] = ls[2] = ls[3] = make_float2(0.f, 0.f);
            float mrow;
            {
              float v[64];
              load64(v, 0);
              if (lg == 0) TRACE(3 + q, 16);
              mrow = max64(v);
              exps64(v, 0, m_run);
              if (lg == 0) TRACE(3 + q, 17);
            }
            if (two) {
              float v[64];
              load64(v, 1);
              if (lg == 0) TRACE(3 + q, 18);
              mrow = fmaxf(mrow, max64(v));
              exps64(v, 1, m_run);
            }
            done = !__any_sync(0xffffffffu, mrow * c2 > m_run + kLazy);
            if (lg == 0) TRACE(3 + q, 9);
          }
          if (!done) {
            // exact path: row max first (S is still intact in TMEM: no P has been stored yet)
            float mrow;
            {
              float v[64];
              load64(v, 0);
              mrow = max64(v);
            }
            if (two) {
              float v[64];
              load64(v, 1);
              mrow = fmaxf(mrow, max64(v));
            }
            const float mx = mrow * c2;
            // lazy rescale: raise the running max only when it grows by more than kLazy (P <= 2^kLazy:
            // bf16 P, fp32 l and O stay far inside their range); TMEM traffic below is warp-uniform
            if (mx > m_run + kLazy || (m_run == -INFINITY && mx > -INFINITY)) {
              alpha = ex2_approx(m_run - mx);  // 0 when m_run = -inf
              l_run *= alpha;
              m_run = mx;
            }
            const float msub = m_run == -INFINITY ? 0.0f : m_run;
            ls[0] = ls[1] = ls[2] = ls[3] = make_float2(0.f, 0.f);
            {
              float v[64];
              load64(v, 0);
              exps64(v, 0, msub);
            }
            if (two) {
              float v[64];
              load64(v, 1);
              exps64(v, 1, msub);
            }
          }
          if (s > 0 && __any_sync(0xffffffffu, alpha != 1.0f)) {
            // O is complete through PV(s-1): the s_full commit covers every earlier MMA
  #pragma unroll 1
            for (int cc = 0; cc < D; cc += 32) {
              float ov[32];
              tmem_ld32(tO + cc, ov);
              tmem_wait_ld();
  #pragma unroll
              for (int e = 0; e < 32; ++e) ov[e] *= alpha;
              tmem_st32(tO + cc, ov);
            }
          }
          l_run += ((ls[0].x + ls[0].y) + (ls[1].x + ls[1].y)) + ((ls[2].x + ls[2].y) + (ls[3].x + ls[3].y));
          // P -> TMEM over the S columns it came from (packed bf16 pairs)
          tmem_st16(tS, pk);
          tmem_st16(tS + 16, pk + 16);
          if (two) {
            tmem_st16(tS + 32, pk + 32);
            tmem_st16(tS + 48, pk + 48);
          }
        }
        tmem_wait_st();
        tc_fence_before();
        mbar_arrive(p_full + q);
        if (lg == 0) TRACE(3 + q, 10);
      }
      // epilogue: O / l -> bf16 -> global; LSE (natural log) = (m + log2 l) ln 2.  With otma, O is
      // staged (SW128) in this tile's Q smem — free once the last PV is done — and written by TMA
      // stores: per-thread row stores (32 rows per warp instruction) clog the LSU/MIO path the
      // producers and the MMA issuer share (measured 6% of the kernel).
      mbar_wait(o_full + q, my_it & 1);
      if (lg == 0) TRACE(3 + q, 12);
      tc_fence_after();
      const float inv_l = l_run > 0.0f ? 1.0f / l_run : 0.0f;
      const int qsl = qslot(my_it, q);
      unsigned char* qs = smem + C::OFF_Q + qsl * C::QBYTES;
#pragma unroll 1
      for (int cc = 0; cc < D; cc += 32) {
        float ov[32];
        tmem_ld32(tO + cc, ov);
        tmem_wait_ld();
        if (cc == D - 32) {  // O_q fully read from TMEM: the next item's PV may overwrite it
          tc_fence_before();
          mbar_arrive(o_free + q);
        }
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 16; ++e) w[e] = pack_bf16x2(ov[2 * e] * inv_l, ov[2 * e + 1] * inv_l);
        if (g.mco && valid) {  // NVLS: the switch replicates the row into every member GPU's O
          __nv_bfloat16* mc = static_cast<__nv_bfloat16*>(g.mco) + (orow - O) + cc;
#pragma unroll
          for (int e = 0; e < 4; ++e) multimem_st16(mc + 8 * e, w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
        }
        if (otma) {
          // row `row` of the 128-row tile, 16-byte pieces k = (cc % 64) / 8 .. + 3 of d-chunk cc / 64
          unsigned char* rb = qs + (cc / 64) * (BM * 128) + row * 128;
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int k = ((cc % 64) >> 3) + e;
            st_shared_v4(rb + ((k ^ (row & 7)) << 4), w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          }
        } else if (valid && !(opts & 2)) {
          uint4* dst = reinterpret_cast<uint4*>(orow + cc);
#pragma unroll
          for (int e = 0; e < 4; ++e) dst[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          for (int mi = 0; mi < g.n_mirror; ++mi) {
            uint4* md = reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(g.mo[mi]) + (orow - O) + cc);
#pragma unroll
            for (int e = 0; e < 4; ++e) md[e] = make_uint4(w[4 * e], w[4 * e + 1], w[4 * e + 2], w[4 * e + 3]);
          }
        }
      }
      if (valid && lse) {
        const long long li = ((long long)it.r * g.Hq + p) * g.Nq + t;
        const float lv = l_run > 0.0f ? (m_run + log2f(l_run)) * 0.6931471805599453f : -INFINITY;
        lse[li] = lv;
        for (int mi = 0; mi < g.n_mirror; ++mi)
          if (g.ml[mi]) g.ml[mi][li] = lv;
        if (g.mcl) multimem_st_f32(g.mcl + li, lv);
      }
      if (lg == 0) TRACE(3 + q, 25);
      if (otma) {
        fence_proxy_async_smem();
        asm volatile("bar.sync %0, 128;" ::"r"(1 + q) : "memory");
        if (lg == 0) TRACE(3 + q, 26);
        if (warp == 4 + 4 * q && lane == 0) {
          for (int s = 0; s < hpq; ++s) {
            const int pls = it.c * heads_in_chunk + q * hpq + s;
            if (pls >= g.m) continue;
            for (int dc = 0; dc < D / 64; ++dc) {
              tma_store_4d(&tmO, qs + dc * (BM * 128) + s * (g.T * 128), dc * 64, it.i * g.T, it.h * g.m + pls,
                           it.r);
              for (int mi = 0; mi < g.n_mirror; ++mi)  // fused exchange: the same tile into every mirror
                tma_store_4d(&tmM.m[mi], qs + dc * (BM * 128) + s * (g.T * 128), dc * 64, it.i * g.T,
                             it.h * g.m + pls, it.r);
            }
          }
          bulk_commit();
          bulk_wait_read0();     // the smem has been read: Q of the next item may land there
          mbar_arrive(q_empty + qsl);
          TRACE(3 + q, 27);
        }
      }
      if (lg == 0) TRACE(3 + q, 13);
    }
    if (otma && warp == 4 + 4 * q && lane == 0) bulk_wait_all();  // O stores complete before exit
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc<512>(tmem);
  }
}

template <int NQT, bool PAGED, bool DENSE>
int launch2_t(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count, const int32_t* pt,
              void* o, float* lse, int n_items, int hpq, int NC, int num_sms, cudaStream_t st, int* sched) {
  // softmax variant (see k_attn2; default 1) and experiment switches (bit 0: no Q prefetch): A/B builds only
  static const int smx = experiment_knob("BFLA_SMX", 1) == 0 ? 0 : 1;
  static const int opts = experiment_knob("BFLA_ATTN_OPTS", 0);
  const int grid = n_items < num_sms ? n_items : num_sms;
  auto go = [&](auto kern, int smem, int threads) -> int {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return (int)e;
    kern<<<grid, threads, smem, st>>>(maps.q, maps.k, maps.v, maps.o, maps.mo, maps.o_ok, g, list, count, pt,
                                      static_cast<__nv_bfloat16*>(o), lse, n_items, hpq, NC, opts, sched);
    count_launch();
    return (int)cudaGetLastError();
  };
  // exponential pairs with e mod 8 == 1 (1 in 8) on the FMA pipe.  Round 1 measured 1/4 best of 0, 1/8,
  // 1/4, 3/8, 1/2; after the split PV issue (round 2, same box, 2 runs each): 0 0.920, 1/8 0.919, 1/4
  // 0.925, 3/8 0.946 ms sparse 32K; 128K equal within 0.1 % (profiles/r2_s3a_poly_ab.jsonl)
#ifndef BFLA_POLY_MASK
#define BFLA_POLY_MASK 0x02
#endif
  constexpr int PM = BFLA_POLY_MASK;
  using C = Cfg2<NQT, PAGED>;
  if constexpr (!DENSE)
    if (g.nrows) return go(k_attn2<NQT, PAGED, false, 1, PM, true>, C::SMEM_TOTAL, C::THREADS);  // work slice
  if (smx == 0) return go(k_attn2<NQT, PAGED, DENSE, 0, PM>, C::SMEM_TOTAL, C::THREADS);
  return go(k_attn2<NQT, PAGED, DENSE, 1, PM>, C::SMEM_TOTAL, C::THREADS);
}

}  // namespace

// head_dim 128 only (two 32 KB K/V slots per ring stage do not fit next to Q at d = 256).
int launch_attention2(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                      const int32_t* page_table, int dense, void* o, float* lse, int num_sms, cudaStream_t st,
                      int* sched) {
  const int hpq = BM / g.T;
  const int nqt = g.m > hpq ? 2 : 1;
  const int NC = (g.m + nqt * hpq - 1) / (nqt * hpq);
  const long long items = (g.nrows ? (long long)g.nrows : (long long)g.B * g.Hkv * g.Tq) * NC;
  if (items == 0) return 0;
  const int n = (int)items;
#define BFLA_GO2(Q_, P_, X_) \
  return launch2_t<Q_, P_, X_>(g, maps, list, count, page_table, o, lse, n, hpq, NC, num_sms, st, sched)
  if (nqt == 2) {
    if (g.paged) { if (dense) BFLA_GO2(2, true, true); else BFLA_GO2(2, true, false); }
    else { if (dense) BFLA_GO2(2, false, true); else BFLA_GO2(2, false, false); }
  } else {
    if (g.paged) { if (dense) BFLA_GO2(1, true, true); else BFLA_GO2(1, true, false); }
    else { if (dense) BFLA_GO2(1, false, true); else BFLA_GO2(1, false, false); }
  }
#undef BFLA_GO2
}

}  // namespace bfla
