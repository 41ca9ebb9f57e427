// api.cu — the C ABI of include/bfla.h: validation, geometry, workspace carving, TMA descriptor
// encoding and kernel launches.  No allocation, no device synchronisation, no global mutable
// state beyond the thread-local error detail and a launch counter.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <mutex>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX3: named ranges for nsys / ncu --nvtx, no link dependency

#include "../../include/bfla.h"
#include "common.cuh"
#include "kernels.h"

namespace bfla {

// One NVTX range per entry point (host-side enqueue span; the kernels it launches nest under it in nsys)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static std::atomic<unsigned long long> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

static thread_local char g_err[512] = "";

static bfla_status fail(bfla_status st, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return st;
}

static bool pow2(int x) { return x > 0 && (x & (x - 1)) == 0; }
static long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// ---- driver entry point for TMA descriptors (no link-time dependency on libcuda) -------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

// Side stream + fork/join events for the concurrent key-norm kernel inside one bfla_block_mask call.
// One set per (host thread, device): a call records its fork and join and waits on them before it
// returns to the caller, all from its own thread, so concurrent calls from different threads never
// see each other's events (cudaStreamWaitEvent takes the record made by the same thread just before).
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
static SideStream* side_stream() {
  static thread_local SideStream per_dev[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  SideStream& ss = per_dev[dev];
  if (!ss.s) {
    if (cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking) != cudaSuccess) return nullptr;
    if (cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      return nullptr;  // run the norms on the caller's stream instead
    }
  }
  return &ss;
}

static int num_sms_current() {
  int dev = 0, n = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
  return n;
}

static bfla_status encode_4d(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_b[3],
                             const uint32_t box[4]) {
  EncodeTiledFn fn = get_encode();
  if (!fn) return fail(BFLA_ERR_CUDA, "cuTensorMapEncodeTiled unavailable (no CUDA driver?)");
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t s[3] = {strides_b[0], strides_b[1], strides_b[2]};
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, s, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(BFLA_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return BFLA_OK;
}

static bool encode_4d_quiet(CUtensorMap* map, const void* base, const uint64_t dims[4], const uint64_t strides_b[3],
                            const uint32_t box[4]) {
  EncodeTiledFn fn = get_encode();
  if (!fn) return false;
  cuuint64_t d[4] = {dims[0], dims[1], dims[2], dims[3]};
  cuuint64_t s[3] = {strides_b[0], strides_b[1], strides_b[2]};
  cuuint32_t bx[4] = {box[0], box[1], box[2], box[3]};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), d, s, bx, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// ---- validation -> geometry -----------------------------------------------------------------
static bfla_status make_geom(const bfla_problem* P, const bfla_config* cfg, Geom* g) {
  if (!P) return fail(BFLA_ERR_INVALID_ARGUMENT, "problem is NULL");
  if (!P->q || !P->k || !P->v || !P->o) return fail(BFLA_ERR_INVALID_ARGUMENT, "q/k/v/o pointer is NULL");
  if (P->batch < 1 || P->h_q < 1 || P->h_kv < 1) return fail(BFLA_ERR_INVALID_ARGUMENT, "batch/h_q/h_kv must be >= 1");
  if (P->h_q % P->h_kv) return fail(BFLA_ERR_INVALID_ARGUMENT, "h_q %% h_kv != 0 (GQA, Eq. 3)");
  if (P->n_q < 1 || P->n_kv < P->n_q)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "need 1 <= n_q <= n_kv (N_c = n_kv - n_q >= 0, Eq. 11)");
  if (P->head_dim != 128 && P->head_dim != 256)
    return fail(BFLA_ERR_UNSUPPORTED, "head_dim %d not built (128, 256)", P->head_dim);
  if (P->kv_layout != BFLA_KV_CONTIGUOUS && P->kv_layout != BFLA_KV_PAGED)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "kv_layout");
  memset(g, 0, sizeof(*g));
  g->B = P->batch;
  g->Hq = P->h_q;
  g->Hkv = P->h_kv;
  g->m = P->h_q / P->h_kv;
  g->kvdiv = 1;
  g->Hkv_real = P->h_kv;
  g->D = P->head_dim;
  g->Nq = P->n_q;
  g->Nkv = P->n_kv;
  g->Nc = P->n_kv - P->n_q;
  g->head_offset = P->head_offset;
  g->scale = P->softmax_scale > 0.f ? P->softmax_scale : (float)(1.0 / std::sqrt((double)P->head_dim));
  g->qs0 = P->q_stride[0];
  g->qs1 = P->q_stride[1];
  g->qs2 = P->q_stride[2];
  g->os0 = P->o_stride[0];
  g->os1 = P->o_stride[1];
  g->os2 = P->o_stride[2];
  g->paged = P->kv_layout == BFLA_KV_PAGED;
  // TMA / 16-byte vector rules
  auto a16 = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  if (!a16(P->q) || !a16(P->k) || !a16(P->v) || !a16(P->o))
    return fail(BFLA_ERR_MISALIGNED, "q/k/v/o base must be 16-byte aligned");
  for (int d = 0; d < 3; ++d)
    if ((P->q_stride[d] % 8) || (P->o_stride[d] % 8) || P->q_stride[d] <= 0 || P->o_stride[d] <= 0)
      return fail(BFLA_ERR_MISALIGNED, "q/o strides must be positive multiples of 8 elements (16 B)");
  if (g->paged) {
    if (!P->page_table) return fail(BFLA_ERR_INVALID_ARGUMENT, "paged layout needs page_table");
    if (P->page_size != 16 && P->page_size != 32 && P->page_size != 64)
      return fail(BFLA_ERR_UNSUPPORTED, "page_size %d not built (16, 32, 64)", P->page_size);
    if (P->num_pages < 1 || (long long)P->max_pages_per_seq * P->page_size < P->n_kv)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "max_pages_per_seq * page_size < n_kv");
    g->page_size = P->page_size;
    g->num_pages = P->num_pages;
    g->max_pages = P->max_pages_per_seq;
  } else {
    for (int d = 0; d < 3; ++d)
      if ((P->kv_stride[d] % 8) || P->kv_stride[d] <= 0)
        return fail(BFLA_ERR_MISALIGNED, "kv strides must be positive multiples of 8 elements (16 B)");
    g->kvs0 = P->kv_stride[0];
    g->kvs1 = P->kv_stride[1];
    g->kvs2 = P->kv_stride[2];
  }
  int b = 64, gg = 64, T = 64;
  if (cfg) {
    b = cfg->block_b;
    gg = cfg->group_g;
    T = cfg->tile_t;
    if (!pow2(b) || !pow2(gg) || !pow2(T)) return fail(BFLA_ERR_INVALID_ARGUMENT, "b, g, T must be powers of two");
    if (b % gg) return fail(BFLA_ERR_INVALID_ARGUMENT, "g must divide b (Eq. 6)");
    if (b % T) return fail(BFLA_ERR_INVALID_ARGUMENT, "T must divide b (Eq. 19)");
    if (cfg->pool != BFLA_POOL_FLATTEN && cfg->pool != BFLA_POOL_MEAN) return fail(BFLA_ERR_INVALID_ARGUMENT, "pool");
    if (cfg->select != BFLA_SELECT_MASS && cfg->select != BFLA_SELECT_RATIO)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "select");
    if (!(cfg->gamma > 0.f && cfg->gamma <= 1.f)) return fail(BFLA_ERR_INVALID_ARGUMENT, "gamma must be in (0, 1] (Eq. 17)");
    if (cfg->select == BFLA_SELECT_RATIO && !(cfg->keep_ratio > 0.f && cfg->keep_ratio <= 1.f))
      return fail(BFLA_ERR_INVALID_ARGUMENT, "keep_ratio must be in (0, 1]");
    if (!(cfg->rho >= 0.f && cfg->rho <= 1.f)) return fail(BFLA_ERR_INVALID_ARGUMENT, "rho must be in [0, 1] (Eq. 25)");
    if (cfg->eta < 0 || cfg->n_local < 0 || cfg->n_sink < 0)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "eta, n_local, n_sink must be >= 0");
    if (T != 64 && T != 128) return fail(BFLA_ERR_UNSUPPORTED, "tile_t %d not built (64, 128)", T);
    if (cfg->mask_groups != BFLA_MASK_PER_KV_HEAD && cfg->mask_groups != BFLA_MASK_PER_Q_HEAD)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "mask_groups");
    if (cfg->certify_slack != 0.f && !(cfg->certify_slack >= 1.f))
      return fail(BFLA_ERR_INVALID_ARGUMENT, "certify_slack must be 0 or >= 1 (it can only widen tau)");
    if (cfg->mask_groups == BFLA_MASK_PER_Q_HEAD) {
      // one mask group per query head (Eq. 18 literal): groups of size 1 over KV head p / m
      g->kvdiv = g->m;
      g->Hkv = g->Hq;
      g->m = 1;
      g->head_offset = P->head_offset * g->kvdiv;  // psi's global index is the query head's
    }
  }
  g->b = b;
  g->g = gg;
  g->G = b / gg;
  g->T = T;
  g->rb = b / T;
  g->Lq = (int)cdiv(g->Nq, b);
  g->Lkv = (int)cdiv(g->Nkv, b);
  g->Lw = (int)cdiv(g->Lkv, 32);
  g->Tq = (int)cdiv(g->Nq, T);
  g->Tkv = (int)cdiv(g->Nkv, T);
  g->Tw = (int)cdiv(g->Tkv, 32);
  g->lens = P->seqlens;
  // list capacity per (r, h): the closed-form causal count (uniform batch) or the full tile rectangle
  // (varlen: every request's causal set fits inside it)
  g->causal_per_head = g->lens ? (long long)g->Tq * g->Tkv : causal_row_offset(*g, g->Tq);
  // int32 indices inside the kernels: recompute units (head row, KV block) and the prefill items
  if (cfg && (long long)g->B * g->Hq * g->Lq * g->Lkv >= (1LL << 31))
    return fail(BFLA_ERR_UNSUPPORTED, "batch * h_q * L_q * L_kv = %lld >= 2^31 (int32 unit indices)",
                (long long)g->B * g->Hq * g->Lq * g->Lkv);
  if ((long long)g->B * g->Hq * g->Tq >= (1LL << 31)) return fail(BFLA_ERR_UNSUPPORTED, "too many query tiles");
  return BFLA_OK;
}

// ---- workspace layout -------------------------------------------------------------------------
struct WsLayout {
  size_t S, qbar, kbar, coarse, tbits, list, count, stats, qn, kn, flagged, units, nflag, sched, kgather, tcpart, total;
};
static size_t al(size_t x) { return (x + 255) & ~size_t(255); }
static WsLayout ws_layout(const Geom& g, bool dense = false) {
  WsLayout L;
  size_t o = 0;
  if (dense) {  // the dense comparator (config == NULL) uses only the item counter
    memset(&L, 0, sizeof(L));
    L.sched = 0;
    L.total = al(16);
    return L;
  }
  L.S = o;
  o += al((size_t)g.B * g.Hq * g.Lq * g.Lkv * 4);
  L.qbar = o;
  o += al((size_t)g.B * g.Hq * g.Lq * g.D * 4);
  L.kbar = o;
  o += al((size_t)g.B * g.Hkv * g.Lkv * g.D * 4);
  L.coarse = o;  // internal mask buffers (used when bfla_prefill gets mask == NULL)
  o += al((size_t)g.B * g.Hkv * g.Lq * g.Lw * 4);
  L.tbits = o;
  o += al((size_t)g.B * g.Hkv * g.Tq * g.Tw * 4);
  L.list = o;
  o += al((size_t)g.B * g.Hkv * g.causal_per_head * 4);
  L.count = o;
  o += al((size_t)g.B * g.Hkv * g.Tq * 4);
  L.stats = o;
  o += al(sizeof(bfla_stats));
  L.qn = o;  // fast Stage-1 scores: block norms, flagged rows, gathered paged K
  o += al((size_t)g.B * g.Hq * g.Lq * 4);
  L.kn = o;
  o += al((size_t)g.B * g.Hkv * g.Lkv * 4);
  L.flagged = o;
  o += al((size_t)g.B * g.Hq * g.Lq * 4);
  L.units = o;  // recompute units (flagged row, KV block) of every flagged row's band, int32
  o += al((size_t)g.B * g.Hq * g.Lq * g.Lkv * 4);
  L.nflag = o;  // flagged-row and recompute-unit counters, then the split-K tile counters (one memset)
  o += al(16 + tc_tick_bytes(g));
  L.sched = o;  // attention item counter (dynamic scheduling)
  o += al(16);
  L.kgather = o;
  if (g.paged) o += al((size_t)g.B * g.Hkv_real * g.Nkv * g.D * 2);
  L.tcpart = o;  // split-K partial accumulators of the tensor-core scores (small tile grids only)
  o += al(tc_part_bytes(g));
  L.total = o;
  return L;
}

static bfla_status cuda_check(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(BFLA_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return BFLA_OK;
}

// tau: |S_tc - S_canonical| <= tau * ||x|| * ||y|| for one g*C-long group dot product.
// Canonical side, worst case (no probabilistic model): every product x_k y_k of the canonical order
// (g token chains of C FMAs, then g - 1 adds, §4 item 2) passes through at most C + g - 1
// round-to-nearest operations, so |S_c - S_exact| <= gamma_{C+g-1} sum|x_k y_k| with
// gamma_n = n u / (1 - n u) <= (C + g) u here (the classical recursive-summation bound; the tests
// pin it on adversarial inputs).  Tensor-core side: n/16 K=16 MMA steps into an fp32 accumulator,
// bounded by 2 (n/16) u even if every step truncated; + 2 u per split-K partial added in fp32
// (the last split of a tile adds them in k_s1_tc_scores).  Cauchy-Schwarz: sum|x_k y_k| <= ||x|| ||y||.  `slack` >= 1 (bfla_config
// certify_slack) only widens tau: more rows are recomputed, the mask cannot change.
static float certify_tau(const Geom& g, float slack) {
  const double n = (double)g.g * g.D, u = std::ldexp(1.0, -24);
  const double canon = ((double)g.D + g.g) * u / (1.0 - ((double)g.D + g.g) * u);
  double tau = canon + u * (n / 8.0 + 2.0 * tc_splits(g));
  if (slack > 1.0f) tau *= slack;
  return (float)(tau * (1.0 + 1e-6));  // rounding the bound to fp32 must not shrink it
}

static bool tc_eligible(const Geom& g, const bfla_problem* P, const bfla_config* cfg, const bfla_mask* mask) {
  if (cfg->pool != BFLA_POOL_FLATTEN || cfg->scores_path != BFLA_SCORES_AUTO || mask->kept_mass) return false;
  // ragged tails / varlen requests: the tensor maps cover the buffer's full groups and the scores
  // kernel uses full groups only; k_s1_ragged_fixup rewrites the partial groups' block scores
  if (g.Nq < g.g || g.Nkv < g.g) return false;  // no full group at all: the canonical path
  if (g.G > 16) return false;  // the score epilogue max-pools G <= 16 groups per block (g = 1: canonical)
  if (g.qs2 != g.D) return false;                    // group rows = contiguous token runs
  if (!g.paged && g.kvs2 != g.D) return false;
  if ((g.qs1 % 8) || (g.qs0 % 8) || (!g.paged && ((g.kvs1 % 8) || (g.kvs0 % 8)))) return false;
  return true;
}

static bfla_status run_block_mask(const Geom& g, const bfla_config* cfg, bfla_mask* mask, unsigned char* ws,
                                  const bfla_problem* P, cudaStream_t st) {
  const WsLayout L = ws_layout(g);
  float* S = reinterpret_cast<float*>(ws + L.S);
  unsigned long long* stats = reinterpret_cast<unsigned long long*>(mask->stats);
  const int32_t* pt = g.paged ? P->page_table : nullptr;
  // c_alpha = log2(e) / sqrt(C) rounded once to fp32 (DESIGN.md §4 item 4; alpha = 1/sqrt(C), Eq. 15)
  const float c_alpha = (float)(1.4426950408889634 / std::sqrt((double)g.D));
  if (tc_eligible(g, P, cfg, mask)) {
    // fast path: tcgen05 scores -> certified selection -> canonical recompute of uncertified rows
    float* qn = reinterpret_cast<float*>(ws + L.qn);
    float* kn = reinterpret_cast<float*>(ws + L.kn);
    int32_t* flagged = reinterpret_cast<int32_t*>(ws + L.flagged);
    int32_t* nflag = reinterpret_cast<int32_t*>(ws + L.nflag);
    int32_t* ulist = reinterpret_cast<int32_t*>(ws + L.units);
    const void* kc = g.paged ? static_cast<const void*>(ws + L.kgather) : P->k;  // paged K: gathered copy
    Geom gk = g;  // geometry of the K operand as the score kernels see it (gathered = contiguous)
    if (g.paged) {
      gk.paged = 0;
      gk.kvs2 = g.D;
      gk.kvs1 = (long long)g.Nkv * g.D;
      gk.kvs0 = (long long)g.Hkv_real * g.Nkv * g.D;
    }
    // every tensor map is encoded before the first enqueue: a failure leaves the stream untouched
    CUtensorMap tmA, tmB;
    bfla_status s;
    {
      // floor(N / g) group rows: a partial last group is never read (rows past it are zero-filled)
      const uint64_t dims[4] = {(uint64_t)g.g * g.D, (uint64_t)(g.Nq / g.g), (uint64_t)g.Hq, (uint64_t)g.B};
      const uint64_t str[3] = {(uint64_t)g.g * g.D * 2, (uint64_t)g.qs1 * 2, (uint64_t)g.qs0 * 2};
      const uint32_t box[4] = {64, 128, 1, 1};
      if ((s = encode_4d(&tmA, P->q, dims, str, box)) != BFLA_OK) return s;
    }
    {
      const uint64_t dims[4] = {(uint64_t)g.g * g.D, (uint64_t)(g.Nkv / g.g), (uint64_t)g.Hkv_real, (uint64_t)g.B};
      const uint64_t str[3] = {(uint64_t)g.g * g.D * 2, (uint64_t)gk.kvs1 * 2, (uint64_t)gk.kvs0 * 2};
      const uint32_t box[4] = {64, (uint32_t)kTcBBox, 1, 1};  // 128-row boxes (64-row boxes measured 1.5x slower)
      if ((s = encode_4d(&tmB, kc, dims, str, box)) != BFLA_OK) return s;
    }
    CUtensorMap tmB64;  // 64-row boxes of the same K view: B halves of the CTA-pair kernel's half tiles
    {
      const uint64_t dims[4] = {(uint64_t)g.g * g.D, (uint64_t)(g.Nkv / g.g), (uint64_t)g.Hkv_real, (uint64_t)g.B};
      const uint64_t str[3] = {(uint64_t)g.g * g.D * 2, (uint64_t)gk.kvs1 * 2, (uint64_t)gk.kvs0 * 2};
      const uint32_t box[4] = {64, 64, 1, 1};
      if ((s = encode_4d(&tmB64, kc, dims, str, box)) != BFLA_OK) return s;
    }
    CUtensorMap rq, rk;  // token-row maps (64 x 64 SW128 boxes) for the TMA-staged recompute
    bool rmaps;
    {
      const uint64_t dq[4] = {(uint64_t)g.D, (uint64_t)g.Nq, (uint64_t)g.Hq, (uint64_t)g.B};
      const uint64_t sq[3] = {(uint64_t)g.qs2 * 2, (uint64_t)g.qs1 * 2, (uint64_t)g.qs0 * 2};
      const uint64_t dk[4] = {(uint64_t)g.D, (uint64_t)g.Nkv, (uint64_t)g.Hkv_real, (uint64_t)g.B};
      const uint64_t sk[3] = {(uint64_t)gk.kvs2 * 2, (uint64_t)gk.kvs1 * 2, (uint64_t)gk.kvs0 * 2};
      const uint32_t box[4] = {64, 64, 1, 1};
      rmaps = encode_4d_quiet(&rq, P->q, dq, sq, box) && encode_4d_quiet(&rk, kc, dk, sk, box);
    }
    if (stats) cudaMemsetAsync(stats, 0, sizeof(bfla_stats), st);
    if (g.paged) launch_paged_gather(g, P->k, P->page_table, ws + L.kgather, st);
    // query-group norms come from the scores kernel (epilogue warps, no extra HBM bytes); key-group
    // norms (HBM-bound, K only) run on this thread's side stream concurrently, joined before the
    // selection.  The fork is recorded before the scores kernel but the norms are launched after it, so
    // the score CTAs (one per SM, all of its shared memory) are dispatched first and the norm CTAs fill
    // the remaining thread slots — launched first, the norm CTAs took every slot and the two kernels
    // ran back to back
    static const bool q_norms_separate = experiment_knob("BFLA_QNORM_KERNEL", 0) == 1;  // A/B builds only
    SideStream* ss = side_stream();
    if (ss) cudaEventRecord(ss->fork, st);
    float* tcpart = tc_part_bytes(g) ? reinterpret_cast<float*>(ws + L.tcpart) : nullptr;  // split-K partials
    cudaMemsetAsync(nflag, 0, 16 + tc_tick_bytes(g), st);  // flagged rows, recompute units, split-K tickets
    const int tc_err = launch_tc_scores(gk, tmA, tmB, S, q_norms_separate ? nullptr : qn, st, tcpart,
                                        reinterpret_cast<int*>(reinterpret_cast<unsigned char*>(nflag) + 16), &tmB64);
    if (ss) {
      cudaStreamWaitEvent(ss->s, ss->fork, 0);
      launch_block_norms(gk, P->q, kc, qn, kn, ss->s, q_norms_separate);
      cudaEventRecord(ss->join, ss->s);
    } else {
      launch_block_norms(gk, P->q, kc, qn, kn, st, q_norms_separate);
    }
    const bool ragged = g.lens || (g.Nq % g.g) || (g.Nkv % g.g);
    if (!tc_err && ragged && launch_ragged_fixup(gk, P->q, kc, S, st)) {
      if (ss) cudaStreamWaitEvent(st, ss->join, 0);
      return fail(BFLA_ERR_CUDA, "ragged fixup launch failed");
    }
    if (ss) cudaStreamWaitEvent(st, ss->join, 0);  // joined even on failure: never leave a fork open
    if (tc_err) return fail(BFLA_ERR_CUDA, "tc scores launch failed (%d)", tc_err);
    const int sms = num_sms_current();
    launch_select(g, S, c_alpha, cfg->select, cfg->gamma, cfg->keep_ratio, mask->coarse_bits, nullptr, stats, st,
                  1, qn, kn, certify_tau(g, cfg->certify_slack), flagged, nflag, sms, ulist);
    if (launch_recompute_rows(gk, P->q, kc, nullptr, flagged, nflag, ulist, nflag + 1, S, sms, st, rmaps ? &rq : nullptr,
                              rmaps ? &rk : nullptr))
      return fail(BFLA_ERR_CUDA, "recompute launch failed");
    launch_select(g, S, c_alpha, cfg->select, cfg->gamma, cfg->keep_ratio, mask->coarse_bits, nullptr, stats, st,
                  2, nullptr, nullptr, 0.f, flagged, nflag, sms);
    return cuda_check("bfla_block_mask launch");
  }
  if (stats) cudaMemsetAsync(stats, 0, sizeof(bfla_stats), st);
  if (cfg->pool == BFLA_POOL_FLATTEN) {
    if (launch_flatten_scores(g, P->q, P->k, pt, S, st)) return fail(BFLA_ERR_UNSUPPORTED, "G not built");
  } else {
    launch_mean_scores(g, P->q, P->k, pt, reinterpret_cast<float*>(ws + L.qbar), reinterpret_cast<float*>(ws + L.kbar),
                       S, st);
  }
  launch_select(g, S, c_alpha, cfg->select, cfg->gamma, cfg->keep_ratio, mask->coarse_bits, mask->kept_mass, stats, st);
  return cuda_check("bfla_block_mask launch");
}

static bfla_status run_expand(const Geom& g, const bfla_config* cfg, bfla_mask* mask, cudaStream_t st) {
  launch_expand_rescue(g, mask->coarse_bits, cfg->n_sink, cfg->n_local, cfg->eta, (double)cfg->rho, cfg->seed,
                       mask->tile_bits, mask->tile_list, mask->tile_count, mask->tile_label,
                       reinterpret_cast<unsigned long long*>(mask->stats), st);
  return cuda_check("bfla_expand_rescue launch");
}

static bfla_status run_attention(const Geom& g, const bfla_problem* P, const int32_t* list, const int32_t* count,
                                 int dense, cudaStream_t st, int32_t* sched = nullptr) {
  AttnMaps maps;
  bfla_status s;
  {
    const uint64_t dims[4] = {(uint64_t)g.D, (uint64_t)g.Nq, (uint64_t)g.Hq, (uint64_t)g.B};
    const uint64_t str[3] = {(uint64_t)g.qs2 * 2, (uint64_t)g.qs1 * 2, (uint64_t)g.qs0 * 2};
    const uint32_t box[4] = {64, (uint32_t)g.T, 1, 1};
    if ((s = encode_4d(&maps.q, P->q, dims, str, box)) != BFLA_OK) return s;
    // O through TMA stores when its layout allows (16-byte aligned base and strides) and rows are not
    // varlen padding (those must stay untouched); otherwise the kernel stores rows directly
    const uint64_t ostr[3] = {(uint64_t)g.os2 * 2, (uint64_t)g.os1 * 2, (uint64_t)g.os0 * 2};
    const bool oal = ((uintptr_t)P->o % 16 == 0) && ostr[0] % 16 == 0 && ostr[1] % 16 == 0 && ostr[2] % 16 == 0;
    static const bool no_otma = experiment_knob("BFLA_OTMA", 1) == 0;  // A/B builds only
    maps.o_ok = 0;
    if (oal && !g.lens && !no_otma && encode_4d_quiet(&maps.o, P->o, dims, ostr, box)) maps.o_ok = 1;
    // mirrors (fused exchange): TMA store maps with O's layout; if any cannot be encoded, every row
    // (local and mirrored) goes through per-thread stores
    for (int k = 0; k < g.n_mirror && maps.o_ok; ++k)
      if (((uintptr_t)g.mo[k] % 16) || !encode_4d_quiet(&maps.mo.m[k], g.mo[k], dims, ostr, box)) maps.o_ok = 0;
  }
  if (!g.paged) {
    const uint64_t dims[4] = {(uint64_t)g.D, (uint64_t)g.Nkv, (uint64_t)g.Hkv_real, (uint64_t)g.B};
    const uint64_t str[3] = {(uint64_t)g.kvs2 * 2, (uint64_t)g.kvs1 * 2, (uint64_t)g.kvs0 * 2};
    const uint32_t box[4] = {64, 64, 1, 1};
    if ((s = encode_4d(&maps.k, P->k, dims, str, box)) != BFLA_OK) return s;
    if ((s = encode_4d(&maps.v, P->v, dims, str, box)) != BFLA_OK) return s;
  } else {
    const uint64_t dims[4] = {(uint64_t)g.D, (uint64_t)g.Hkv_real, (uint64_t)g.page_size, (uint64_t)g.num_pages};
    const uint64_t str[3] = {(uint64_t)g.D * 2, (uint64_t)g.Hkv_real * g.D * 2,
                             (uint64_t)g.page_size * g.Hkv_real * g.D * 2};
    const uint32_t box[4] = {64, 1, (uint32_t)g.page_size, 1};
    if ((s = encode_4d(&maps.k, P->k, dims, str, box)) != BFLA_OK) return s;
    if ((s = encode_4d(&maps.v, P->v, dims, str, box)) != BFLA_OK) return s;
  }
  // d = 128: the paired-tile kernel (attention2.cu); d = 256 (or BFLA_ATTN=1): one tile per step
  static const bool v1 = experiment_knob("BFLA_ATTN", 0) == 1;  // A/B builds only
  const int32_t* pt = g.paged ? P->page_table : nullptr;
  static const bool no_dyn = experiment_knob("BFLA_DYN_SCHED", 1) == 0;  // A/B builds: static round-robin
  if (no_dyn) sched = nullptr;
  if (sched) cudaMemsetAsync(sched, 0, sizeof(int32_t), st);
  int e = (g.D == 128 && !v1)
              ? launch_attention2(g, maps, list, count, pt, dense, P->o, P->lse, num_sms_current(), st, sched)
              : launch_attention(g, maps, list, count, pt, dense, P->o, P->lse, num_sms_current(), st, sched);
  if (e) return fail(BFLA_ERR_CUDA, "attention launch: %s", cudaGetErrorString((cudaError_t)e));
  return cuda_check("attention launch");
}

static bfla_status check_mask(const Geom& g, const bfla_mask* mask, bool need_coarse, bool need_tiles) {
  if (!mask) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask is NULL");
  if (need_coarse && !mask->coarse_bits) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask->coarse_bits is NULL");
  if (need_tiles) {
    if (!mask->tile_bits || !mask->tile_list || !mask->tile_count)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "mask tile buffers are NULL");
    if (mask->tile_list_capacity < (long long)g.B * g.Hkv * g.causal_per_head)
      return fail(BFLA_ERR_CAPACITY, "tile_list_capacity %lld < %lld", (long long)mask->tile_list_capacity,
                  (long long)g.B * g.Hkv * g.causal_per_head);
  }
  return BFLA_OK;
}

}  // namespace bfla

using namespace bfla;

extern "C" {

size_t bfla_workspace_size(const bfla_problem* problem, const bfla_config* config) {
  Geom g;
  if (make_geom(problem, config, &g) != BFLA_OK) return 0;
  return ws_layout(g, config == nullptr).total;
}

int64_t bfla_tile_list_capacity(const bfla_problem* problem, const bfla_config* config) {
  Geom g;
  const bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return -(int64_t)s;
  return (int64_t)g.B * g.Hkv * g.causal_per_head;
}

bfla_status bfla_block_mask(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask, void* ws,
                            size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_block_mask");
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if ((s = check_mask(g, mask, true, false)) != BFLA_OK) return s;
  if (!ws || ws_bytes < ws_layout(g).total) return fail(BFLA_ERR_WORKSPACE, "workspace too small");
  return run_block_mask(g, config, mask, static_cast<unsigned char*>(ws), problem, static_cast<cudaStream_t>(stream));
}

bfla_status bfla_expand_rescue(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask, void* ws,
                               size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_expand_rescue");
  (void)ws;
  (void)ws_bytes;
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if ((s = check_mask(g, mask, true, true)) != BFLA_OK) return s;
  return run_expand(g, config, mask, static_cast<cudaStream_t>(stream));
}

bfla_status bfla_sparse_prefill(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_sparse_prefill");
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if (!mask || !mask->tile_list || !mask->tile_count) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask lists are NULL");
  // the workspace is optional here: with it, items are scheduled dynamically (a counter in ws)
  const WsLayout L = ws_layout(g);
  int32_t* sched = (ws && ws_bytes >= L.total) ? reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + L.sched)
                                                : nullptr;
  return run_attention(g, problem, mask->tile_list, mask->tile_count, 0, static_cast<cudaStream_t>(stream), sched);
}

bfla_status bfla_sparse_prefill_rows(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                     int64_t row_begin, int64_t row_end, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_sparse_prefill_rows");
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if (!mask || !mask->tile_list || !mask->tile_count) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask lists are NULL");
  const int64_t rows = (int64_t)g.B * g.Hkv * g.Tq;
  if (row_begin < 0 || row_end < row_begin || row_end > rows)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                (long long)row_end, (long long)rows);
  if (row_end == row_begin) return BFLA_OK;  // an empty slice enqueues nothing
  g.row0 = (int)row_begin;
  g.nrows = (int)(row_end - row_begin);
  const WsLayout L = ws_layout(g);
  int32_t* sched = (ws && ws_bytes >= L.total) ? reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + L.sched)
                                                : nullptr;
  return run_attention(g, problem, mask->tile_list, mask->tile_count, 0, static_cast<cudaStream_t>(stream), sched);
}

bfla_status bfla_sparse_prefill_mirrored(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                         int64_t row_begin, int64_t row_end, const bfla_mirrors* mirrors, void* ws,
                                         size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_sparse_prefill_mirrored");
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if (!mask || !mask->tile_list || !mask->tile_count) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask lists are NULL");
  if (mirrors) {
    if (mirrors->n < 0 || mirrors->n > BFLA_MAX_MIRRORS)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "mirrors->n = %d outside [0, %d]", mirrors->n, BFLA_MAX_MIRRORS);
    for (int k = 0; k < mirrors->n; ++k) {
      if (!mirrors->o[k]) return fail(BFLA_ERR_INVALID_ARGUMENT, "mirrors->o[%d] is NULL", k);
      if (((uintptr_t)mirrors->o[k] % 16) || (mirrors->lse[k] && ((uintptr_t)mirrors->lse[k] % 4)))
        return fail(BFLA_ERR_MISALIGNED, "mirror %d misaligned", k);
      g.mo[k] = mirrors->o[k];
      g.ml[k] = problem->lse ? mirrors->lse[k] : nullptr;
    }
    g.n_mirror = mirrors->n;
    if (mirrors->multicast_o) {
      if (((uintptr_t)mirrors->multicast_o % 16) || (mirrors->multicast_lse && ((uintptr_t)mirrors->multicast_lse % 4)))
        return fail(BFLA_ERR_MISALIGNED, "multicast address misaligned");
      g.mco = mirrors->multicast_o;
      g.mcl = problem->lse ? mirrors->multicast_lse : nullptr;
    }
  }
  const int64_t rows = (int64_t)g.B * g.Hkv * g.Tq;
  if (!(row_begin == 0 && row_end == 0)) {
    if (row_begin < 0 || row_end < row_begin || row_end > rows)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                  (long long)row_end, (long long)rows);
    if (row_end == row_begin) return BFLA_OK;
    if (row_begin != 0 || row_end != rows) {
      g.row0 = (int)row_begin;
      g.nrows = (int)(row_end - row_begin);
    }
  }
  const WsLayout L = ws_layout(g);
  int32_t* sched = (ws && ws_bytes >= L.total) ? reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + L.sched)
                                                : nullptr;
  return run_attention(g, problem, mask->tile_list, mask->tile_count, 0, static_cast<cudaStream_t>(stream), sched);
}

bfla_status bfla_sparse_prefill_kvrange(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                        int64_t kv_tile_begin, int64_t kv_tile_end, int64_t row_begin,
                                        int64_t row_end, void* ws, size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_sparse_prefill_kvrange");
  if (!config) return fail(BFLA_ERR_INVALID_ARGUMENT, "config is NULL");
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if (!mask || !mask->tile_list || !mask->tile_count) return fail(BFLA_ERR_INVALID_ARGUMENT, "mask lists are NULL");
  if (!problem->lse) return fail(BFLA_ERR_INVALID_ARGUMENT, "split-KV partials need problem->lse");
  if (kv_tile_begin < 0 || kv_tile_end < kv_tile_begin)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "kv tile range [%lld, %lld)", (long long)kv_tile_begin,
                (long long)kv_tile_end);
  g.kv_range = 1;
  g.kv_lo = (int)std::min<int64_t>(kv_tile_begin, (int64_t)g.Tkv);
  g.kv_hi = (int)std::min<int64_t>(kv_tile_end, (int64_t)g.Tkv);
  const int64_t rows = (int64_t)g.B * g.Hkv * g.Tq;
  if (!(row_begin == 0 && row_end == 0)) {
    if (row_begin < 0 || row_end < row_begin || row_end > rows)
      return fail(BFLA_ERR_INVALID_ARGUMENT, "row range [%lld, %lld) outside [0, %lld)", (long long)row_begin,
                  (long long)row_end, (long long)rows);
    if (row_end == row_begin) return BFLA_OK;
    if (row_begin != 0 || row_end != rows) {
      g.row0 = (int)row_begin;
      g.nrows = (int)(row_end - row_begin);
    }
  }
  const WsLayout L = ws_layout(g);
  int32_t* sched = (ws && ws_bytes >= L.total) ? reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + L.sched)
                                                : nullptr;
  return run_attention(g, problem, mask->tile_list, mask->tile_count, 0, static_cast<cudaStream_t>(stream), sched);
}

bfla_status bfla_merge_partials(const bfla_problem* problem, const bfla_partials* parts, void* stream) {
  NvtxRange nvtx_("bfla_merge_partials");
  Geom g;
  bfla_status s = make_geom(problem, nullptr, &g);
  if (s != BFLA_OK) return s;
  if (!parts || parts->n < 1 || parts->n > BFLA_MAX_PARTS)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "parts->n outside [1, %d]", BFLA_MAX_PARTS);
  MergeParts mp;
  mp.n = parts->n;
  for (int k = 0; k < parts->n; ++k) {
    if (!parts->o[k] || !parts->lse[k]) return fail(BFLA_ERR_INVALID_ARGUMENT, "part %d is NULL", k);
    if ((uintptr_t)parts->o[k] % 16) return fail(BFLA_ERR_MISALIGNED, "part %d O not 16-byte aligned", k);
    mp.o[k] = parts->o[k];
    mp.lse[k] = parts->lse[k];
  }
  if (launch_merge_partials(g, mp, problem->o, problem->lse, static_cast<cudaStream_t>(stream)))
    return cuda_check("bfla_merge_partials launch");
  return cuda_check("bfla_merge_partials launch");
}

bfla_status bfla_balance_rows(const int32_t* tile_count, int32_t batch, int32_t h_kv, int32_t tq, int32_t row_overhead,
                              int32_t parts, int64_t* bounds) {
  if (!tile_count || !bounds || batch < 1 || h_kv < 1 || tq < 1 || parts < 1 || row_overhead < 0)
    return fail(BFLA_ERR_INVALID_ARGUMENT, "balance_rows: bad argument");
  const int64_t n = (int64_t)batch * h_kv * tq;
  // cost of LPT row rho = (r * h_kv + h) * tq + (tq - 1 - i): its kept tiles + a per-row overhead
  auto cost = [&](int64_t rho) -> int64_t {
    const int64_t seg = rho / tq, i = tq - 1 - rho % tq;
    const int32_t c = tile_count[seg * tq + i];
    return (int64_t)(c > 0 ? c : 0) + row_overhead;
  };
  int64_t total = 0, lo = 0;
  for (int64_t rho = 0; rho < n; ++rho) {
    const int64_t c = cost(rho);
    total += c;
    lo = c > lo ? c : lo;
  }
  // smallest bottleneck M such that greedy contiguous packing needs <= parts pieces (exact optimum
  // of the linear partition problem: greedy packing is optimal for a fixed M)
  auto pieces = [&](int64_t M) -> int64_t {
    int64_t k = 1, acc = 0;
    for (int64_t rho = 0; rho < n; ++rho) {
      const int64_t c = cost(rho);
      if (acc + c > M) {
        ++k;
        acc = 0;
      }
      acc += c;
    }
    return k;
  };
  int64_t hi = total;
  if (lo < (total + parts - 1) / parts) lo = (total + parts - 1) / parts;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (pieces(mid) <= parts) hi = mid;
    else lo = mid + 1;
  }
  // cut greedily at the optimum M, but never leave fewer rows than parts still to fill: rows are
  // handed out so that every part gets at least one row when n >= parts
  int64_t acc = 0, p = 0;
  bounds[0] = 0;
  for (int64_t rho = 0; rho < n; ++rho) {
    const int64_t c = cost(rho);
    const bool must = (n - rho) <= (parts - 1 - p);  // remaining rows only just cover remaining parts
    if (p < parts - 1 && rho > bounds[p] && (acc + c > lo || must)) {
      bounds[++p] = rho;
      acc = 0;
    }
    acc += c;
  }
  while (p < parts) bounds[++p] = n;
  return BFLA_OK;
}

bfla_status bfla_prefill(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask, void* ws,
                         size_t ws_bytes, void* stream) {
  NvtxRange nvtx_("bfla_prefill");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  Geom g;
  bfla_status s = make_geom(problem, config, &g);
  if (s != BFLA_OK) return s;
  if (!config) {  // dense causal (Eq. 1); a workspace, if given, enables dynamic item scheduling
    const WsLayout Ld = ws_layout(g, true);
    int32_t* sched = (ws && ws_bytes >= Ld.total) ? reinterpret_cast<int32_t*>(static_cast<unsigned char*>(ws) + Ld.sched)
                                                   : nullptr;
    return run_attention(g, problem, nullptr, nullptr, 1, st, sched);
  }
  const WsLayout L = ws_layout(g);
  if (!ws || ws_bytes < L.total) return fail(BFLA_ERR_WORKSPACE, "workspace too small");
  unsigned char* w = static_cast<unsigned char*>(ws);
  bfla_mask local;
  if (!mask) {
    memset(&local, 0, sizeof(local));
    local.coarse_bits = reinterpret_cast<uint32_t*>(w + L.coarse);
    local.tile_bits = reinterpret_cast<uint32_t*>(w + L.tbits);
    local.tile_list = reinterpret_cast<int32_t*>(w + L.list);
    local.tile_list_capacity = (long long)g.B * g.Hkv * g.causal_per_head;
    local.tile_count = reinterpret_cast<int32_t*>(w + L.count);
    mask = &local;
  }
  if ((s = check_mask(g, mask, true, true)) != BFLA_OK) return s;
  if ((s = run_block_mask(g, config, mask, w, problem, st)) != BFLA_OK) return s;
  if ((s = run_expand(g, config, mask, st)) != BFLA_OK) return s;
  return run_attention(g, problem, mask->tile_list, mask->tile_count, 0, st,
                       reinterpret_cast<int32_t*>(w + L.sched));
}

const char* bfla_status_string(bfla_status status) {
  switch (status) {
    case BFLA_OK: return "BFLA_OK";
    case BFLA_ERR_INVALID_ARGUMENT: return "BFLA_ERR_INVALID_ARGUMENT";
    case BFLA_ERR_UNSUPPORTED: return "BFLA_ERR_UNSUPPORTED";
    case BFLA_ERR_MISALIGNED: return "BFLA_ERR_MISALIGNED";
    case BFLA_ERR_WORKSPACE: return "BFLA_ERR_WORKSPACE";
    case BFLA_ERR_CAPACITY: return "BFLA_ERR_CAPACITY";
    case BFLA_ERR_CUDA: return "BFLA_ERR_CUDA";
  }
  return "BFLA_UNKNOWN_STATUS";
}

const char* bfla_last_error(void) { return g_err; }

uint64_t bfla_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"
