/*
 * bfla.h — C ABI of the B200 (sm_100a) BFLA hot path.  ABI version 1.
 *
 * Block-Filtered Long-Context Attention (arXiv 2605.12193).  Citations "P:n" are lines of the
 * paper's text; "Eq. k" its equations; R1..R22 the readings listed in DESIGN.md §3.
 *
 * Conventions (all entry points):
 *  - Tensor pointers are DEVICE pointers (cudaMalloc / PyTorch CUDA tensors) unless stated.
 *    The caller owns every buffer; the library never allocates, frees, or keeps a pointer past
 *    the work it enqueues.  Parameter structs are read before the call returns.
 *  - All work is enqueued on `stream` (a cudaStream_t passed as void*; NULL = legacy stream).
 *    No entry point synchronises the device.
 *  - Validation is synchronous and happens before any launch: on a non-OK status nothing has
 *    been enqueued and outputs are untouched.  Faults inside kernels surface at the caller's
 *    next synchronisation as a CUDA error.
 *  - Identical inputs give identical output bits (masks, lists, O, LSE): no atomics decide any
 *    value (atomics only accumulate integer statistics).
 *  - Calls are reentrant and may come from several host threads at once: the only state kept
 *    between calls is per host thread (the detail string of bfla_last_error(), and the side stream
 *    + events bfla_block_mask forks its key-norm kernel onto, created on a thread's first call per
 *    device and joined back into `stream` before the call returns) plus a process-wide atomic
 *    launch counter.
 *  - Element strides are in ELEMENTS (bf16 = 2 bytes); the head_dim axis must be contiguous.
 */
#ifndef BFLA_H_
#define BFLA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BFLA_ABI_VERSION 1

typedef enum {
    BFLA_OK = 0,
    BFLA_ERR_INVALID_ARGUMENT = 1, /* a paper invariant is violated: Hq % Hkv != 0 (Eq. 3), Nq > Nkv or
                                      Nq < 1 (Eq. 11, N_c >= 0), b/g/T not powers of two, g does not divide b
                                      (Eq. 6), T does not divide b (Eq. 19), gamma not in (0,1] (Eq. 17),
                                      keep_ratio not in (0,1], rho not in [0,1] (Eq. 25), eta < 0, n_local < 0,
                                      n_sink < 0, NULL required pointer                                       */
    BFLA_ERR_UNSUPPORTED = 2,      /* valid but not built: head_dim not in {128, 256}, T not in {64, 128},
                                      FLATTEN with non-contiguous tokens, page_size not in {16, 32, 64}     */
    BFLA_ERR_MISALIGNED = 3,       /* TMA rules: base address % 16 B, strides % 16 B                         */
    BFLA_ERR_WORKSPACE = 4,        /* ws_bytes < bfla_workspace_size(...) or ws == NULL                       */
    BFLA_ERR_CAPACITY = 5,         /* mask->tile_list_capacity < bfla_tile_list_capacity(...)                */
    BFLA_ERR_CUDA = 6              /* a CUDA runtime/driver call failed; detail in bfla_last_error()          */
} bfla_status;

enum { BFLA_KV_CONTIGUOUS = 0, BFLA_KV_PAGED = 1 };
/* Stage-1 pooling (R1): FLATTEN = flattening-g pooling + max over group pairs (Eq. 6-10, the
   paper's operator, default); MEAN = per-block mean of Q and of K, one dot product per block pair
   (the north_star's wording; an HBM-bound variant). */
enum { BFLA_POOL_FLATTEN = 0, BFLA_POOL_MEAN = 1 };
/* Stage-1 selection: MASS = smallest prefix with mass >= gamma (Eq. 16-18); RATIO = the top
   ceil(keep_ratio * n_causal) blocks per row (north_star's "keep ratio", R9). */
enum { BFLA_SELECT_MASS = 0, BFLA_SELECT_RATIO = 1 };
/* How FLATTEN block scores are computed.  Both give the canonical mask bit for bit:
   AUTO = tcgen05 scores + per-row certification + canonical recompute of the rows it cannot certify
   (used when Q/K token rows are contiguous, n_q and n_kv are multiples of g, and kept_mass is not
   requested; otherwise CANONICAL); CANONICAL = every score on the fp32 FMA pipes in canonical order. */
enum { BFLA_SCORES_AUTO = 0, BFLA_SCORES_CANONICAL = 1 };
/* Mask groups: PER_KV_HEAD (default) ORs the m query heads' Stage-1 masks into one mask per KV head
   (R8; enables GQA packing in the prefill kernel); PER_Q_HEAD keeps Eq. 18 literal — one mask per
   query head p, Stage 2 (Eq. 19-26) per query head, psi (Eq. 25) indexed by the global query head —
   and the mask buffers then have h_q rows where the comments below say h_kv. */
enum { BFLA_MASK_PER_KV_HEAD = 0, BFLA_MASK_PER_Q_HEAD = 1 };

/* One attention layer call: Q/K/V in the paper's head-first layout (Eq. 2), GQA m = h_q / h_kv
   (Eq. 3), head group H_h = {h m, ..., h m + m - 1} (Eq. 8); the batch index is the paper's
   request index r (Eq. 20, 27).  N_c = n_kv - n_q (Eq. 11): chunked prefill is a request whose
   query chunk is the LAST n_q tokens of its n_kv-token KV sequence (uniform over the batch). */
typedef struct {
    int32_t batch, h_q, h_kv, head_dim;
    int32_t n_q, n_kv;
    float softmax_scale;   /* <= 0 -> 1/sqrt(head_dim) (Eq. 1, Eq. 27)                                 */
    int32_t head_offset;   /* global index of local KV head 0 (a multi-GPU shard passes rank*h_kv);
                              used only by psi (Eq. 25) so sharded masks equal unsharded ones       */
    const void* q;         /* bf16 [batch][h_q][n_q][head_dim] with element strides q_stride        */
    int64_t q_stride[3];   /* (batch, head, token); head_dim contiguous                                */
    void* o;               /* bf16 output, same shape as q, strides o_stride                           */
    int64_t o_stride[3];
    float* lse;            /* optional fp32 [batch][h_q][n_q] natural-log LSE of the scaled scores
                              over the attended keys; NULL = not written                               */
    int32_t kv_layout;     /* BFLA_KV_CONTIGUOUS | BFLA_KV_PAGED                                       */
    const void* k;         /* contiguous: bf16 [batch][h_kv][n_kv][head_dim] with strides kv_stride;
                              paged (vLLM): bf16 [num_pages][page_size][h_kv][head_dim], dense      */
    const void* v;
    int64_t kv_stride[3];  /* contiguous only: (batch, head, token)                                    */
    int32_t page_size, num_pages, max_pages_per_seq;
    const int32_t* page_table; /* paged only: device int32 [batch][max_pages_per_seq], logical page
                                  n of request r lives at physical page page_table[r][n]           */
    const int32_t* seqlens;    /* optional device int32 [batch][2] = (n_q_r, n_kv_r): variable-length
                                  batch (requests of different lengths / chunk offsets).  Must satisfy
                                  1 <= n_q_r <= n_kv_r, n_q_r <= n_q, n_kv_r <= n_kv (not checked: device
                                  memory).  n_q / n_kv are then the padded extents of every buffer;
                                  request r's queries are rows 0..n_q_r-1 of its Q/O slice, its keys
                                  rows 0..n_kv_r-1 (or its first n_kv_r paged tokens); other O/LSE rows
                                  are not written.  Stage-1 scores use the canonical path.  NULL =
                                  every request has (n_q, n_kv).                                    */
} bfla_problem;

/* Method knobs.  Defaults of the paper's strong operating point:
   b=256, g=64, gamma=0.99, n_local=8, rho=0, eta=16; T=64 and n_sink=1 are our readings (R10, R12). */
typedef struct {
    int32_t block_b;    /* b: coarse block size (Eq. 4), power of two                                   */
    int32_t group_g;    /* g: flattening group (Eq. 6), power of two dividing b; any G = b/g (tensor-core
                           scores for G <= 16, e.g. b=1024 g=64; canonical SIMT above, e.g. g=1) */
    int32_t tile_t;     /* T: attention tile (Eq. 19), divides b; 64 and 128 built                      */
    int32_t pool;       /* BFLA_POOL_*                                                                  */
    int32_t select;     /* BFLA_SELECT_*                                                                */
    float gamma;        /* mass threshold (Eq. 17), (0, 1]; 1 keeps every causal block (R7)           */
    float keep_ratio;   /* (0, 1], used when select == RATIO                                           */
    int32_t n_sink;     /* sink tile columns (Eq. 22, R12)                                              */
    int32_t n_local;    /* band width in tiles (Eq. 21, R11): tiles [d_i - n_local, d_i]              */
    int32_t eta;        /* stride-rescue period (Eq. 24); 0 = off                                      */
    float rho;          /* random-rescue probability (Eq. 25), [0, 1]                                  */
    uint64_t seed;      /* s of Eq. 24-25                                                               */
    int32_t scores_path; /* BFLA_SCORES_* (FLATTEN only; MEAN is always canonical)                      */
    int32_t mask_groups; /* BFLA_MASK_* (0 = per KV head, the default)                                  */
    float certify_slack; /* AUTO scores: factor >= 1 applied to the certification bound tau;
                            a wider bound only sends more rows to the canonical recompute — the mask
                            is the same bit for bit — so tests use it to exercise the recompute.
                            0 = 1 (default); values in (0, 1) or negative are INVALID_ARGUMENT, so no
                            setting can weaken the certification.                                     */
} bfla_config;

/* Statistics, accumulated with integer atomics (values are order independent). */
typedef struct {
    uint64_t causal_tiles;    /* sum over (r, h) of causal tiles (R20, kappa denominator)             */
    uint64_t kept_tiles;      /* sum of kept tiles (kappa numerator)                                   */
    uint64_t label[6];        /* kept tiles by provenance: [1] mass [2] sink [3] band [4] stride [5] random */
    uint64_t rows;            /* Stage-1 rows (r, p, i)                                                */
    uint64_t rows_exact_tie;  /* rows whose cut falls between two equal probabilities (R6, reported)  */
    uint64_t blocks_kept;     /* sum over rows of r* (blocks kept per query head before the OR)       */
    uint64_t rows_flagged;    /* AUTO scores: head rows (r,p,i) the certification could not prove     */
    uint64_t rows_recomputed; /* AUTO scores: head rows recomputed in the canonical order              */
    uint64_t reserved[3];
} bfla_stats;

/* Caller-owned device buffers written by Stage 1 / Stage 2.  Shapes use
   Lq = ceil(n_q/b), Lkv = ceil(n_kv/b), Tq = ceil(n_q/T), Tkv = ceil(n_kv/T). */
typedef struct {
    uint32_t* coarse_bits;  /* [batch][h_kv][Lq][ceil(Lkv/32)]: Eq. 18 after the OR over H_h (R8);
                               bit j%32 of word j/32                                              */
    uint32_t* tile_bits;    /* [batch][h_kv][Tq][ceil(Tkv/32)]: final M^tile (Eq. 26)             */
    int32_t* tile_list;     /* kept KV tile indices, ascending j; row (r,h,i) starts at
                               ((r*h_kv + h) * C + c_i) where C = causal tiles per (r,h) and
                               c_i = causal tiles of rows < i (closed form, no scan)            */
    int64_t tile_list_capacity; /* entries available in tile_list                              */
    int32_t* tile_count;    /* [batch][h_kv][Tq]: kept tiles per row                                  */
    uint8_t* tile_label;    /* optional [batch][h_kv][Tq][Tkv]: 0 drop/non-causal, 1 mass, 2 sink,
                               3 band, 4 stride, 5 random (precedence in that order, R13)          */
    float* kept_mass;       /* optional [batch][h_q][Lq]: sum of kept A (Eq. 17 check)               */
    bfla_stats* stats;      /* optional device bfla_stats (zeroed by bfla_block_mask)                */
} bfla_mask;

/* Bytes of device scratch the entry points need for (problem, config); 0 if the pair is invalid.
   config == NULL (the dense comparator of bfla_prefill) needs only the 256-byte scheduling counter. */
size_t bfla_workspace_size(const bfla_problem* problem, const bfla_config* config);
/* Entries tile_list must hold: batch * h_kv * (causal tiles per (r,h)); with seqlens, batch * h_kv *
   ceil(n_q/T) * ceil(n_kv/T).  On invalid (problem, config) it returns the NEGATED bfla_status
   (e.g. -BFLA_ERR_UNSUPPORTED) with the detail in bfla_last_error(). */
int64_t bfla_tile_list_capacity(const bfla_problem* problem, const bfla_config* config);

/* Stage 1 (Eq. 4-18 + GQA OR): pooling, block scores (Eq. 9-10), causal mask (Eq. 11-14),
   block softmax with alpha = 1/sqrt(head_dim) (Eq. 15), keep-mass / keep-ratio selection
   (Eq. 16-18), OR over each head group.  Writes mask->coarse_bits (+ kept_mass, stats).
   The decision follows the canonical fp32 arithmetic of DESIGN.md §4, so coarse_bits are bit-exact
   against the CPU oracle (see BFLA_SCORES_* for how the scores are obtained). */
bfla_status bfla_block_mask(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask,
                            void* ws, size_t ws_bytes, void* stream);

/* Stage 2 (Eq. 19-26): expansion to the T-tile grid with tile causality, local band
   (Eq. 21, R11), sink (Eq. 22, R12), stride rescue (Eq. 24) and random rescue (Eq. 25) of the
   dropped set (Eq. 23), final union (Eq. 26, R16).  Reads mask->coarse_bits; writes tile_bits,
   tile_list, tile_count (+ tile_label, stats).  Integer only: bit-exact by construction. */
bfla_status bfla_expand_rescue(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask,
                               void* ws, size_t ws_bytes, void* stream);

/* Fused sparse causal prefill (Eq. 27): for every (r, h, query tile i) and all m query
   heads of H_h, exact online-softmax attention over the kept KV tiles of mask->tile_list (ascending
   j), token-exact causal masking inside frontier tiles, dropped tiles contribute nothing.  Writes
   problem->o (+ lse).  tcgen05/TMEM/TMA kernel, bf16 in, fp32 accumulation, P rounded to bf16. */
bfla_status bfla_sparse_prefill(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                void* ws, size_t ws_bytes, void* stream);
/* (ws is optional for bfla_sparse_prefill and for the dense bfla_prefill: when it is given — at least
   bfla_workspace_size bytes — the kernel schedules its work items dynamically through a counter kept
   in ws; with ws == NULL it uses a static round-robin order.  Results are identical either way.) */

/* Work slice of the sparse prefill (balanced sharding): the same computation as
   bfla_sparse_prefill restricted to the prefill rows rho in [row_begin, row_end) of the LPT row order
   rho = (r * h_kv + h) * Tq + (Tq - 1 - i) — (request, head group) major, query tile i DESCENDING
   (h ranges over mask groups: h_q of them in PER_Q_HEAD mode); inside the slice the rows run in
   descending i with its (r, h) segments interleaved (longest first).  A row writes the O (+ LSE) rows
   i*T .. i*T+T-1 of every query head of its group; rows outside the slice are not touched.  Results
   are bit-identical to the unsliced call on the rows written (every row is computed by one CTA,
   independently of the schedule).  Errors: BFLA_ERR_INVALID_ARGUMENT unless
   0 <= row_begin <= row_end <= batch * h_kv * Tq; an empty slice enqueues nothing. */
bfla_status bfla_sparse_prefill_rows(const bfla_problem* problem, const bfla_config* config, const bfla_mask* mask,
                                     int64_t row_begin, int64_t row_end, void* ws, size_t ws_bytes, void* stream);

/* Fused output exchange: the prefill epilogue stores every O row (+ LSE row) it
   produces into up to BFLA_MAX_MIRRORS further buffers as well as problem->o / problem->lse — e.g. the
   same head chunk of every peer GPU's full-layer O, mapped into this device's address space (NVLink
   P2P / symmetric memory).  The exchange then overlaps the computation tile by tile instead of
   following it as a separate all-gather; the caller orders the peers' reads after the kernel (a
   device-side barrier across the ranks).  mirrors->o[k] uses problem->o's element offsets and strides
   (same shape), mirrors->lse[k] problem->lse's (NULL: LSE not mirrored; ignored if problem->lse is
   NULL).  Pointers: device-accessible, 16-byte aligned (else BFLA_ERR_MISALIGNED); never dereferenced
   on the host.  row_begin = row_end = 0 means every row, otherwise the slice semantics of
   bfla_sparse_prefill_rows.  n = 0 is exactly bfla_sparse_prefill(_rows).  Errors as those calls, plus
   BFLA_ERR_INVALID_ARGUMENT for n outside [0, BFLA_MAX_MIRRORS] or a NULL o[k].
   multicast_o / multicast_lse (optional, NULL = unused): NVLS multicast addresses (e.g. the
   multicast_ptr of a torch symmetric-memory buffer) with problem->o's / problem->lse's layout; every
   O / LSE row is also written through `multimem.st` to them, so the NVSwitch replicates it into every
   member GPU's buffer (one store per row instead of one per peer).  16-byte aligned. */
#define BFLA_MAX_MIRRORS 7
typedef struct {
    int32_t n;
    void* o[BFLA_MAX_MIRRORS];
    float* lse[BFLA_MAX_MIRRORS];
    void* multicast_o;
    float* multicast_lse;
} bfla_mirrors;
bfla_status bfla_sparse_prefill_mirrored(const bfla_problem* problem, const bfla_config* config,
                                         const bfla_mask* mask, int64_t row_begin, int64_t row_end,
                                         const bfla_mirrors* mirrors, void* ws, size_t ws_bytes, void* stream);

/* Split-KV (a row too long for one GPU or one SM): the sparse prefill restricted to the kept
   tiles j (mask tile index, T units) in [kv_tile_begin, kv_tile_end) — Eq. 27 over that subset of each
   row's kept tiles; a row with none writes O = 0 and LSE = -inf — over the LPT rows [row_begin, row_end)
   (0, 0 = every row; bfla_sparse_prefill_rows semantics), so a scheduler can hand out (row slice, KV
   range) pieces.  problem->lse is required (the merge needs it).  Errors as bfla_sparse_prefill_rows,
   plus BFLA_ERR_INVALID_ARGUMENT unless 0 <= kv_tile_begin <= kv_tile_end, or if problem->lse is NULL. */
bfla_status bfla_sparse_prefill_kvrange(const bfla_problem* problem, const bfla_config* config,
                                        const bfla_mask* mask, int64_t kv_tile_begin, int64_t kv_tile_end,
                                        int64_t row_begin, int64_t row_end, void* ws, size_t ws_bytes,
                                        void* stream);
/* Merge of KV-range partials: for every row, with M = max_k LSE_k and w_k = exp(LSE_k - M),
   O = sum_k w_k O_k / sum_k w_k and LSE = M + log(sum_k w_k) — the online softmax of Eq. 27 over the
   union of the ranges (exact up to the bf16 rounding of each O_k).  parts->o[k] / parts->lse[k]: device
   buffers with problem->o / problem->lse's layout (ranges that do not overlap, e.g. from
   bfla_sparse_prefill_kvrange).  Writes problem->o and, if not NULL, problem->lse; q/k/v are not read
   (but must be valid pointers).  Errors: BFLA_ERR_INVALID_ARGUMENT for n outside [1, BFLA_MAX_PARTS]
   or a NULL part; BFLA_ERR_MISALIGNED for parts not 16-byte aligned. */
#define BFLA_MAX_PARTS 8
typedef struct {
    int32_t n;
    const void* o[BFLA_MAX_PARTS];
    const float* lse[BFLA_MAX_PARTS];
} bfla_partials;
bfla_status bfla_merge_partials(const bfla_problem* problem, const bfla_partials* parts, void* stream);

/* Host-only (no GPU, no CUDA call): cost-balanced contiguous partition of the LPT row order into
   `parts` slices for bfla_sparse_prefill_rows (§8 f2: per-head kappa differs, so equal head counts per
   GPU are not equal work; P:443 runs 8 GPUs without naming a scheme).  tile_count is a HOST copy of
   mask->tile_count ([batch][h_kv][tq], kept tiles per row, Eq. 26); the cost of a row is
   tile_count + row_overhead (the per-row fixed cost in tile units).  Writes bounds[0..parts]
   (bounds[0] = 0, bounds[parts] = batch * h_kv * tq, non-decreasing): slice k = [bounds[k],
   bounds[k+1]).  The bottleneck max_k cost(slice k) is the minimum over all contiguous partitions
   (bisection on the bottleneck with greedy packing); when there are at least `parts` rows every slice
   is non-empty.  Errors: BFLA_ERR_INVALID_ARGUMENT on NULL pointers or non-positive sizes. */
bfla_status bfla_balance_rows(const int32_t* tile_count, int32_t batch, int32_t h_kv, int32_t tq, int32_t row_overhead,
                              int32_t parts, int64_t* bounds);

/* The whole path: Stage 1 -> Stage 2 -> sparse prefill.  config == NULL runs DENSE causal attention
   (Eq. 1, the comparator) with the same kernel.  mask == NULL keeps the mask buffers inside ws. */
bfla_status bfla_prefill(const bfla_problem* problem, const bfla_config* config, bfla_mask* mask, void* ws,
                         size_t ws_bytes, void* stream);

/* Human-readable status name and the calling thread's detail for its last non-OK status. */
const char* bfla_status_string(bfla_status status);
const char* bfla_last_error(void);
/* Launch counter: number of kernels this process has enqueued through the library (for bench). */
uint64_t bfla_kernel_launches(void);

#ifdef __cplusplus
}
#endif
#endif /* BFLA_H_ */
