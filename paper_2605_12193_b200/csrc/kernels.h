// kernels.h — internal launch functions (host side) of the BFLA sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.cuh"

namespace bfla {

void count_launch();

// Stage 1 scores (Eq. 9-10): FLATTEN (canonical SIMT fp32 chain) or MEAN.
int launch_flatten_scores(const Geom& g, const void* q, const void* k, const int32_t* page_table, float* S,
                          cudaStream_t st);
void launch_mean_scores(const Geom& g, const void* q, const void* k, const int32_t* page_table, float* qbar,
                        float* kbar, float* S, cudaStream_t st);
// Stage 1 selection (Eq. 13-18 + OR over H_h)
size_t select_smem_bytes(const Geom& g, int nwarps);
void launch_select(const Geom& g, const float* S, float c_alpha, int select, float gamma, float keep_ratio,
                   uint32_t* coarse, float* kept_mass, unsigned long long* stats, cudaStream_t st, int mode = 0,
                   const float* qn = nullptr, const float* kn = nullptr, float tau = 0.f,
                   int32_t* flagged = nullptr, int32_t* n_flagged = nullptr, int num_sms = 148,
                   int32_t* ulist = nullptr);
// Fast Stage-1 scores (tcgen05) + certification support (stage1_tc.cu)
constexpr int kTcTileN = 256;  // key groups per score tile (MMA N)
constexpr int kTcBBox = 128;   // key-group rows per TMA box of a score B stage
constexpr int kTcCluster = 2;
constexpr int kTcPair = 1;     // CTA-pair (cta_group::2) score kernel for clusters of two  // score CTAs per cluster (query heads sharing each K stage by multicast)
size_t tc_scores_smem();
// qn (optional): the scores kernel also writes the query-group norm bounds (Gram diagonal)
int launch_tc_scores(const Geom& g, const CUtensorMap& tmA, const CUtensorMap& tmB, float* S, float* qn,
                     cudaStream_t st, float* part = nullptr, int* tick = nullptr,
                     const CUtensorMap* tmB64 = nullptr);  // 64-row B boxes (CTA-pair kernel, half tiles)
int tc_splits(const Geom& g);
size_t tc_part_bytes(const Geom& g);
size_t tc_tick_bytes(const Geom& g);
// canonical rewrite of the block scores of partial groups (ragged n mod g != 0, varlen requests)
int launch_ragged_fixup(const Geom& g, const void* q, const void* k, float* S, cudaStream_t st);
// with_q = false: key-group norms only (the scores kernel wrote the query norms)
void launch_block_norms(const Geom& g, const void* q, const void* k, float* qn, float* kn, cudaStream_t st,
                        bool with_q = true);
// tmQ / tmK (optional): {D, N, H, B} maps with 64 x 64 SW128 boxes for the TMA-staged variant
int launch_recompute_rows(const Geom& g, const void* q, const void* k, const int32_t* pt, const int32_t* flagged,
                          const int32_t* n_flagged, const int32_t* ulist, const int32_t* n_units, float* S,
                          int num_sms, cudaStream_t st,
                          const CUtensorMap* tmQ = nullptr, const CUtensorMap* tmK = nullptr);
void launch_paged_gather(const Geom& g, const void* kcache, const int32_t* pt, void* kout, cudaStream_t st);
// Stage 2 (Eq. 19-26)
void launch_expand_rescue(const Geom& g, const uint32_t* coarse, int n_sink, int n_local, int eta, double rho,
                          uint64_t seed, uint32_t* tile_bits, int32_t* list, int32_t* count, uint8_t* label,
                          unsigned long long* stats, cudaStream_t st);

// split-KV merge (merge.cu): O / LSE of up to 8 KV-range partials, each with the problem's O layout
struct MergeParts {
  int n;
  const void* o[8];
  const float* lse[8];
};
int launch_merge_partials(const Geom& g, const MergeParts& mp, void* o, float* lse, cudaStream_t st);

// Sparse / dense prefill (Eq. 27 / Eq. 1) — tcgen05 + TMEM + TMA.
struct MirrorMaps {
  CUtensorMap m[7];  // O mirrors as TMA store targets (attention2 epilogue, Geom::n_mirror of them)
};
struct AttnMaps {
  CUtensorMap q, k, v;
  CUtensorMap o;  // O as a TMA store target (attention2 epilogue), valid when o_ok (and every mirror map)
  int o_ok = 0;
  MirrorMaps mo;
};
size_t attn_smem_bytes(int D, int nqt);
int launch_attention(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                     const int32_t* page_table, int dense, void* o, float* lse, int num_sms, cudaStream_t st,
                     int* sched = nullptr);
// head_dim 128: two kept tiles per step, P in TMEM (attention2.cu)
// sched: optional device int (zeroed by the caller) for dynamic item scheduling; NULL = static
int launch_attention2(const Geom& g, const AttnMaps& maps, const int32_t* list, const int32_t* count,
                      const int32_t* page_table, int dense, void* o, float* lse, int num_sms, cudaStream_t st,
                      int* sched = nullptr);
}  // namespace bfla
