/*
 * bfla_oracle.c — plain, slow, obviously-correct CPU oracle for the BFLA hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  The product path
 * (paper_2605_12193_b200/, libbfla.so) never links, imports or calls it, and the two share
 * no code, headers, tables or constants.
 *
 * Citations: "P:n" = PAPER.md line n (arXiv 2605.12193, BFLA); "Eq. k" = the paper's
 * equation k.  Readings R1..R21 are listed in DESIGN.md §3 (the canonical numerics of the
 * mask, which the paper does not fix, are DESIGN.md §4 / "canonical numerics").
 *
 * Every function here follows the paper's definition in the paper's order.  Floating point:
 *   - attention (Eq. 1, Eq. 27) is computed in fp64;
 *   - the Stage-1 mask arithmetic (Eq. 9-18) is computed in the canonical fp32 order of
 *     DESIGN.md §4 so that masks can be compared bit for bit.
 * Compile with -O2 -ffp-contract=off -mfma (fmaf must be the single-rounding hardware FMA).
 *
 * Parity pins: see tests/test_oracle_*.py (each function's pin is named in its comment).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_POOL_FLATTEN 0
#define ORC_POOL_MEAN 1
#define ORC_SELECT_MASS 0
#define ORC_SELECT_RATIO 1

/* Tile labels (provenance), precedence mass > sink > band > stride > random (R13). */
#define LBL_DROP 0
#define LBL_MASS 1
#define LBL_SINK 2
#define LBL_BAND 3
#define LBL_STRIDE 4
#define LBL_RANDOM 5

static int ceil_div(int a, int b) { return (a + b - 1) / b; }
static int imin(int a, int b) { return a < b ? a : b; }
static int imax(int a, int b) { return a > b ? a : b; }

/* ------------------------------------------------------------------------------------------
 * Eq. 11-13: causal block mask.  e_i = min(N_c + (i+1)b - 1, N_kv - 1), p_j = j b,
 * keep iff p_j <= e_i.  Used with b = block size (Stage 1) and b = T (tile level, R13).
 * Pin: closed forms, tests/test_oracle_stage1.py::test_causal_block_mask_*.
 * ---------------------------------------------------------------------------------------- */
int orc_causal(int i, int j, int blk, int n_q, int n_kv) {
    long n_c = (long)n_kv - (long)n_q;
    long e_i = n_c + (long)(i + 1) * blk - 1;
    if (e_i > n_kv - 1) e_i = n_kv - 1;
    long p_j = (long)j * blk;
    return p_j <= e_i;
}

/* ------------------------------------------------------------------------------------------
 * Eq. 4-7: blocking + flattening-g pooling.  Phi(X)[h,l,u, t*C + c] =
 * X[h, l*b + u*g + t, c] for in-range tokens, 0 for padding (R2, R3).  Writes
 * out[H][L][G][g*C] and valid[H? no: per block][G] = 1 iff group u of block l holds >= 1 real
 * token (padding-only groups are excluded from Eq. 10's max, R3).
 * Pin: SPEC hand layout N=5,b=4,g=2, round-trip.
 * ---------------------------------------------------------------------------------------- */
void orc_flatten(const float* x, int H, int N, int C, int b, int g, float* out, uint8_t* valid) {
    int L = ceil_div(N, b), G = b / g;
    for (int h = 0; h < H; ++h)
        for (int l = 0; l < L; ++l)
            for (int u = 0; u < G; ++u) {
                float* dst = out + (((size_t)h * L + l) * G + u) * (size_t)g * C;
                for (int t = 0; t < g; ++t) {
                    int tok = l * b + u * g + t;
                    for (int c = 0; c < C; ++c)
                        dst[(size_t)t * C + c] = tok < N ? x[((size_t)h * N + tok) * C + c] : 0.0f;
                }
                if (h == 0) valid[(size_t)l * G + u] = (uint8_t)(l * b + u * g < N);
            }
}

/* Canonical fp32 dot product of two C-vectors (DESIGN.md §4 item 2): acc = 0; acc = fma(x_c, y_c,
 * acc) for c ascending.  Single-rounding FMA, no reassociation.  (MEAN scores, and one token pair of
 * a FLATTEN group dot below.) */
static float dot_canon(const float* x, const float* y, int n) {
    float acc = 0.0f;
    for (int k = 0; k < n; ++k) acc = fmaf(x[k], y[k], acc);
    return acc;
}

/* Canonical fp32 FLATTEN group dot (DESIGN.md §4 item 2, reading R2): the flattened g*C vectors are
 * g consecutive tokens of C channels (index t*C + c, Eq. 7), so Phi(Q).Phi(K) = sum_t q_t . k_t.
 * Each token pair is a canonical C-long FMA chain (c ascending); the g token dots are then added in
 * ascending t with fp32 adds: acc = 0; acc = acc + dot_canon(x_t, y_t).  Padding tokens are exact
 * zeros and add exact zeros. */
static float dot_canon_flat(const float* x, const float* y, int g, int C) {
    float acc = 0.0f;
    for (int t = 0; t < g; ++t) acc = acc + dot_canon(x + (size_t)t * C, y + (size_t)t * C, C);
    return acc;
}

/* ------------------------------------------------------------------------------------------
 * Eq. 9-10, 14: block scores.
 *   FLATTEN: S[p,i,j] = max over valid (u,v) of Phi(Q)[p,i,u] . Phi(K)[h,j,v]   (h = p / m, Eq. 8)
 *   MEAN (north_star variant, R1): qbar = (sum_t q_t) / n_tokens (fp32, t ascending), same for k;
 *         S[p,i,j] = qbar . kbar (canonical dot over c ascending).
 *   Non-causal (Eq. 13) entries are -inf (Eq. 14).
 * q: [Hq][Nq][C], k: [Hkv][Nkv][C] (fp32 widening of the bf16 inputs), S: [Hq][Lq][Lkv].
 * Pin: g=1 -> block max of Q K^T; g=b -> trace of the diagonal block of Q K^T; naive 6-loop
 * (S:180-182); MEAN on integer inputs vs numpy; tests/test_oracle_stage1.py.
 * ---------------------------------------------------------------------------------------- */
void orc_block_scores(const float* q, const float* k, int Hq, int Hkv, int Nq, int Nkv, int C,
                      int b, int g, int pool, float* S) {
    int Lq = ceil_div(Nq, b), Lkv = ceil_div(Nkv, b), m = Hq / Hkv;
    if (pool == ORC_POOL_FLATTEN) {
        int G = b / g;
        size_t gc = (size_t)g * C;
        float* pq = (float*)malloc(sizeof(float) * (size_t)Hq * Lq * G * gc);
        float* pk = (float*)malloc(sizeof(float) * (size_t)Hkv * Lkv * G * gc);
        uint8_t* vq = (uint8_t*)malloc((size_t)Lq * G);
        uint8_t* vk = (uint8_t*)malloc((size_t)Lkv * G);
        orc_flatten(q, Hq, Nq, C, b, g, pq, vq);
        orc_flatten(k, Hkv, Nkv, C, b, g, pk, vk);
#pragma omp parallel for collapse(2) schedule(dynamic)
        for (int p = 0; p < Hq; ++p)
            for (int i = 0; i < Lq; ++i) {
                int h = p / m;
                for (int j = 0; j < Lkv; ++j) {
                    float best = -INFINITY;
                    if (orc_causal(i, j, b, Nq, Nkv)) {
                        for (int u = 0; u < G; ++u) {
                            if (!vq[(size_t)i * G + u]) continue;
                            const float* x = pq + (((size_t)p * Lq + i) * G + u) * gc;
                            for (int v = 0; v < G; ++v) {
                                if (!vk[(size_t)j * G + v]) continue;
                                const float* y = pk + (((size_t)h * Lkv + j) * G + v) * gc;
                                float s = dot_canon_flat(x, y, g, C);
                                if (s > best) best = s;
                            }
                        }
                    }
                    S[((size_t)p * Lq + i) * Lkv + j] = best;
                }
            }
        free(pq); free(pk); free(vq); free(vk);
    } else {
        float* mq = (float*)malloc(sizeof(float) * (size_t)Hq * Lq * C);
        float* mk = (float*)malloc(sizeof(float) * (size_t)Hkv * Lkv * C);
        for (int pass = 0; pass < 2; ++pass) {
            const float* x = pass ? k : q;
            int H = pass ? Hkv : Hq, N = pass ? Nkv : Nq, L = pass ? Lkv : Lq;
            float* mo = pass ? mk : mq;
            for (int h = 0; h < H; ++h)
                for (int l = 0; l < L; ++l) {
                    int t0 = l * b, t1 = imin(N, (l + 1) * b);
                    for (int c = 0; c < C; ++c) {
                        float acc = 0.0f;
                        for (int t = t0; t < t1; ++t) acc = acc + x[((size_t)h * N + t) * C + c];
                        mo[((size_t)h * L + l) * C + c] = acc / (float)(t1 - t0);
                    }
                }
        }
        for (int p = 0; p < Hq; ++p)
            for (int i = 0; i < Lq; ++i)
                for (int j = 0; j < Lkv; ++j)
                    S[((size_t)p * Lq + i) * Lkv + j] =
                        orc_causal(i, j, b, Nq, Nkv)
                            ? dot_canon(mq + ((size_t)p * Lq + i) * C, mk + ((size_t)(p / m) * Lkv + j) * C, C)
                            : -INFINITY;
        free(mq); free(mk);
    }
}

/* ------------------------------------------------------------------------------------------
 * Canonical exp2 for t <= 0 (DESIGN.md §4 item 5): n = floor(t), f = t - n in [0,1),
 * p = degree-6 Horner polynomial in fp32 FMA, result = p * 2^n.  Returns 0 for t < -126.
 * Pin: |exp2_canon(t) - 2^t| <= 2 ulp over a dense sweep (tests/test_oracle_stage1.py).
 * ---------------------------------------------------------------------------------------- */
float orc_exp2_canon(float t) {
    if (t < -126.0f) return 0.0f;
    float fl = floorf(t);
    int n = (int)fl;
    float f = t - fl;
    float p = 0x1.cacdfep-13f;
    p = fmaf(p, f, 0x1.44bd4cp-10f);
    p = fmaf(p, f, 0x1.3d5822p-7f);
    p = fmaf(p, f, 0x1.c67ee4p-5f);
    p = fmaf(p, f, 0x1.ebfdf8p-3f);
    p = fmaf(p, f, 0x1.62e428p-1f);
    p = fmaf(p, f, 0x1p+0f);
    return ldexpf(p, n);
}

/* ------------------------------------------------------------------------------------------
 * Eq. 15: block softmax over the causal j of one row, alpha = 1/sqrt(C) (R5),
 * canonical fp32 (DESIGN.md §4 items 4-6):
 *   M = max_j S_j; c = (float)(log2(e)/sqrt(C)); t_j = (S_j - M) * c (two roundings);
 *   e_j = exp2_canon(t_j); Z = sum_j e_j (j ascending); A_j = e_j / Z.  Non-causal A_j = 0.
 * Pin: [0,0] -> [.5,.5], single block -> 1, [1,2] with C=4 vs double; rows sum to 1.
 * ---------------------------------------------------------------------------------------- */
void orc_block_softmax_row(const float* S, int n, int C, float* A) {
    float M = -INFINITY;
    for (int j = 0; j < n; ++j)
        if (S[j] > M) M = S[j];
    float c = (float)(1.4426950408889634 / sqrt((double)C));
    float Z = 0.0f;
    for (int j = 0; j < n; ++j) {
        if (S[j] == -INFINITY) { A[j] = 0.0f; continue; }
        float d = S[j] - M;
        float t = d * c;
        A[j] = orc_exp2_canon(t);
        Z = Z + A[j];
    }
    for (int j = 0; j < n; ++j) A[j] = A[j] / Z;
}

/* ------------------------------------------------------------------------------------------
 * Eq. 16-18: keep-mass selection on one row of probabilities A (n entries,
 * causal[j] marks causal blocks).  Order = (A desc, j asc) (R6); P_r = sequential fp32 prefix;
 * r* = min{r : P_r >= (float)gamma} (R7); if none, or gamma >= 1, all causal blocks are kept.
 * select == RATIO (north_star extension, R9): keep the first ceil(ratio * n_causal) blocks of the
 * order (S desc, j asc) when the scores S are given (the block softmax is monotone in S, so this is
 * the top-k by probability without fp32 underflow ties), else (A desc, j asc).
 * Outputs keep[j] in {0,1}; returns r*.  *kept_mass = P_{r*} (A summed in the selection order);
 * *p_prev = P_{r*-1} (0 if r*=1); *tie = 1 iff the cut falls between two equal sort keys (reported,
 * R6); order_out = the causal blocks in sort order.
 * Pin: S:207-209 examples, mass >= gamma, minimality, monotonicity in gamma.
 * ---------------------------------------------------------------------------------------- */
int orc_keep_select_keyed(const float* A, const float* S, const uint8_t* causal, int n, int select,
                          float gamma, float keep_ratio, uint8_t* keep, float* kept_mass, float* p_prev,
                          int* tie, int* order_out) {
    const float* key = (select == ORC_SELECT_RATIO && S) ? S : A;
    int* ord = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
    int nc = 0;
    for (int j = 0; j < n; ++j)
        if (causal[j]) ord[nc++] = j;
    /* insertion sort: (key desc, j asc) — stable on the ascending-j input */
    for (int a = 1; a < nc; ++a) {
        int x = ord[a], bpos = a - 1;
        while (bpos >= 0 && key[ord[bpos]] < key[x]) { ord[bpos + 1] = ord[bpos]; --bpos; }
        ord[bpos + 1] = x;
    }
    int r = nc;
    if (select == ORC_SELECT_RATIO) {
        double want = ceil((double)keep_ratio * (double)nc);
        r = (int)want;
        if (r < 1) r = 1;
        if (r > nc) r = nc;
    } else if (gamma < 1.0f) {
        float P = 0.0f;
        for (int t = 0; t < nc; ++t) {
            P = P + A[ord[t]];
            if (P >= gamma) { r = t + 1; break; }
        }
    }
    float P = 0.0f, Pp = 0.0f;
    for (int t = 0; t < r; ++t) { Pp = P; P = P + A[ord[t]]; }
    memset(keep, 0, (size_t)n);
    for (int t = 0; t < r; ++t) keep[ord[t]] = 1;
    if (kept_mass) *kept_mass = P;
    if (p_prev) *p_prev = Pp;
    if (tie) *tie = (r < nc) && (key[ord[r - 1]] == key[ord[r]]);
    if (order_out) memcpy(order_out, ord, sizeof(int) * (size_t)nc);
    free(ord);
    return r;
}

int orc_keep_select(const float* A, const uint8_t* causal, int n, int select, float gamma,
                    float keep_ratio, uint8_t* keep, float* kept_mass, float* p_prev, int* tie,
                    int* order_out) {
    return orc_keep_select_keyed(A, NULL, causal, n, select, gamma, keep_ratio, keep, kept_mass, p_prev, tie,
                                 order_out);
}

/* ------------------------------------------------------------------------------------------
 * Stage 1 end to end (Eq. 13-18, then the GQA union R8 feeding Eq. 20):
 *   S [Hq][Lq][Lkv] (from orc_block_scores) -> per query-head mass mask [Hq][Lq][Lkv] and
 *   coarse[h][i][j] = OR_{p in H_h} mass[p][i][j]  (Eq. 8 head groups).
 * Optional outputs (NULL = skip): A [Hq][Lq][Lkv], kept_mass / p_prev [Hq][Lq], rstar, tie,
 * gap [Hq][Lq] = S_{pi_r*} - S_{pi_{r*+1}} in score units (0 if none dropped).
 * Pin: invariants (mass >= gamma, minimality, OR), tests/test_oracle_stage1.py.
 * ---------------------------------------------------------------------------------------- */
void orc_select(const float* S, int Hq, int Hkv, int Nq, int Nkv, int C, int b, int select,
                float gamma, float keep_ratio, uint8_t* mass, uint8_t* coarse, float* A_out,
                float* kept_mass, float* p_prev, int* rstar, int* tie, float* gap) {
    int Lq = ceil_div(Nq, b), Lkv = ceil_div(Nkv, b), m = Hq / Hkv;
    memset(coarse, 0, (size_t)Hkv * Lq * Lkv);
#pragma omp parallel for collapse(2) schedule(dynamic)
    for (int p = 0; p < Hq; ++p)
        for (int i = 0; i < Lq; ++i) {
            const float* s = S + ((size_t)p * Lq + i) * Lkv;
            float* A = (float*)malloc(sizeof(float) * (size_t)Lkv);
            uint8_t* causal = (uint8_t*)malloc((size_t)Lkv);
            int* ord = (int*)malloc(sizeof(int) * (size_t)Lkv);
            for (int j = 0; j < Lkv; ++j) causal[j] = (uint8_t)orc_causal(i, j, b, Nq, Nkv);
            orc_block_softmax_row(s, Lkv, C, A);
            uint8_t* keep = mass + ((size_t)p * Lq + i) * Lkv;
            float km, pp;
            int tt;
            int r = orc_keep_select_keyed(A, s, causal, Lkv, select, gamma, keep_ratio, keep, &km, &pp, &tt, ord);
            int nc = 0;
            for (int j = 0; j < Lkv; ++j) nc += causal[j];
            size_t row = (size_t)p * Lq + i;
            if (A_out) memcpy(A_out + row * Lkv, A, sizeof(float) * (size_t)Lkv);
            if (kept_mass) kept_mass[row] = km;
            if (p_prev) p_prev[row] = pp;
            if (rstar) rstar[row] = r;
            if (tie) tie[row] = tt;
            if (gap) gap[row] = r < nc ? s[ord[r - 1]] - s[ord[r]] : 0.0f;
            free(A); free(causal); free(ord);
        }
    for (int p = 0; p < Hq; ++p)
        for (int i = 0; i < Lq; ++i)
            for (int j = 0; j < Lkv; ++j)
                if (mass[((size_t)p * Lq + i) * Lkv + j]) coarse[((size_t)(p / m) * Lq + i) * Lkv + j] = 1;
}

/* ------------------------------------------------------------------------------------------
 * Hashes chi and psi of Eq. 24-25 — "lightweight deterministic mixing function",
 * pinned by us (R15): mix64 = the SplitMix64 finalizer (Steele, Lea, Flood 2014).
 * Pin: SplitMix64 published first output for seed 0 = 0xE220A8397B1DCDAF; residue uniformity
 * (S:280); psi mean; tests/test_oracle_stage2.py.
 * ---------------------------------------------------------------------------------------- */
uint64_t orc_mix64(uint64_t x) {
    x ^= x >> 30;
    x *= 0xbf58476d1ce4e5b9ULL;
    x ^= x >> 27;
    x *= 0x94d049bb133111ebULL;
    x ^= x >> 31;
    return x;
}
uint64_t orc_chi(int i, int j, uint64_t s) {
    uint64_t key = ((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)j;
    return orc_mix64(key ^ s);
}
double orc_psi(int h, int i, int j, uint64_t s) {
    uint64_t key = ((uint64_t)(uint32_t)i << 32) | (uint64_t)(uint32_t)j;
    uint64_t z = orc_mix64(orc_mix64(key ^ s ^ 0xD1B54A32D192ED03ULL) ^ ((uint64_t)h * 0x9E3779B97F4A7C15ULL));
    return (double)(z >> 11) * 0x1p-53;
}

/* ------------------------------------------------------------------------------------------
 * Stage 2 (Eq. 19-26) for one request.  coarse: [Hkv][Lq][Lkv] (Eq. 18 after OR);
 * label out: [Hkv][Tq][Tkv] with LBL_* codes, 0 = dropped or non-causal.
 *  1. expansion Eq. 19-20: tile (i,j) inherits coarse block (i/rho_b, j/rho_b), then non-causal
 *     tiles (Eq. 11-13 at b = T) are cleared (R13 / S:258);
 *  2. band Eq. 21 (R11): j in [max(0, d_i - n_local), d_i], d_i = min(floor((N_c+(i+1)T-1)/T), Tkv-1);
 *  3. sink Eq. 22 (R12): j < n_sink;
 *  4. dropped set Eq. 23 (R13): causal and not kept after 1-3;
 *  5. stride rescue Eq. 24 (R14): eta > 0 and chi(i,j;s) mod eta == 0;
 *     random rescue Eq. 25 (R14): psi(h_global,i,j;s) < rho, h_global = head_offset + h;
 *  6. final mask Eq. 26 = union (R16).
 * Pin: S:261-263, density (2L-1)/(L(L+1)/2), binomial rate.
 * ---------------------------------------------------------------------------------------- */
void orc_expand_rescue(const uint8_t* coarse, int Hkv, int Nq, int Nkv, int b, int T, int n_sink,
                       int n_local, int eta, double rho, uint64_t seed, int head_offset,
                       uint8_t* label) {
    int Lq = ceil_div(Nq, b), Lkv = ceil_div(Nkv, b);
    int Tq = ceil_div(Nq, T), Tkv = ceil_div(Nkv, T), rb = b / T;
    long n_c = (long)Nkv - Nq;
    for (int h = 0; h < Hkv; ++h)
        for (int i = 0; i < Tq; ++i) {
            long fr = n_c + (long)(i + 1) * T - 1;
            int d_i = (int)(fr / T);
            if (d_i > Tkv - 1) d_i = Tkv - 1;
            for (int j = 0; j < Tkv; ++j) {
                uint8_t* L = label + ((size_t)h * Tq + i) * Tkv + j;
                *L = LBL_DROP;
                if (!orc_causal(i, j, T, Nq, Nkv)) continue;
                int I = i / rb, J = j / rb;
                (void)Lq;
                if (coarse[((size_t)h * Lq + I) * Lkv + J]) { *L = LBL_MASS; continue; }
                if (j < n_sink) { *L = LBL_SINK; continue; }
                if (j >= imax(0, d_i - n_local) && j <= d_i) { *L = LBL_BAND; continue; }
                if (eta > 0 && orc_chi(i, j, seed) % (uint64_t)eta == 0) { *L = LBL_STRIDE; continue; }
                if (rho > 0.0 && orc_psi(head_offset + h, i, j, seed) < rho) { *L = LBL_RANDOM; continue; }
            }
        }
}

/* ------------------------------------------------------------------------------------------
 * Eq. 27 with the additive mask materialised row by row, in fp64 (R17, R19):
 * for query head p (KV head h = p/m) and chunk token t (absolute position N_c + t), the
 * attended key set is {s : s <= N_c + t} intersect {s : label[h][t/T][s/T] != 0}; the output
 * is softmax(scale * q.k) over that set times V, max-shifted.  If label == NULL every causal
 * key is attended (dense causal SDPA, Eq. 1 — the keep-all comparator).
 * rows: nrows pairs (row_p[r], row_t[r]); out: [nrows][C] fp64; lse: [nrows] natural-log
 * log-sum-exp of the scaled scores (may be NULL).
 * Pin: brute-force numpy dense causal attention (keep-all), N=1 -> V row, constant scores ->
 * mean of causal V, skipping exactness, convex hull.
 * ---------------------------------------------------------------------------------------- */
void orc_masked_attention(const float* q, const float* k, const float* v, int Hq, int Hkv, int Nq,
                          int Nkv, int C, double scale, const uint8_t* label, int T, int nrows,
                          const int* row_p, const int* row_t, double* out, double* lse) {
    int m = Hq / Hkv, Tq = ceil_div(Nq, T), Tkv = ceil_div(Nkv, T);
    long n_c = (long)Nkv - Nq;
#pragma omp parallel for schedule(dynamic, 4)
    for (int r = 0; r < nrows; ++r) {
        int p = row_p[r], t = row_t[r], h = p / m;
        const float* qr = q + ((size_t)p * Nq + t) * C;
        long last = n_c + t;
        double* sc = (double*)malloc(sizeof(double) * (size_t)(last + 1));
        double mx = -INFINITY;
        for (long s = 0; s <= last; ++s) {
            int keep = label ? label[((size_t)h * Tq + t / T) * Tkv + s / T] != 0 : 1;
            if (!keep) { sc[s] = -INFINITY; continue; }
            const float* kr = k + ((size_t)h * Nkv + s) * C;
            double d = 0.0;
            for (int c = 0; c < C; ++c) d += (double)qr[c] * (double)kr[c];
            sc[s] = d * scale;
            if (sc[s] > mx) mx = sc[s];
        }
        double* o = out + (size_t)r * C;
        for (int c = 0; c < C; ++c) o[c] = 0.0;
        double Z = 0.0;
        for (long s = 0; s <= last; ++s) {
            if (sc[s] == -INFINITY) continue;
            double w = exp(sc[s] - mx);
            Z += w;
            const float* vr = v + ((size_t)h * Nkv + s) * C;
            for (int c = 0; c < C; ++c) o[c] += w * (double)vr[c];
        }
        for (int c = 0; c < C; ++c) o[c] /= Z;
        if (lse) lse[r] = mx + log(Z);
        free(sc);
    }
}

/* Number of causal tiles of one (request, KV head) (Eq. 11-13 at block size T): the kappa
 * denominator (R20).  Pin: T_q(T_q+1)/2 for square full tiles. */
long orc_causal_tiles(int Nq, int Nkv, int T) {
    long n = 0;
    int Tq = ceil_div(Nq, T), Tkv = ceil_div(Nkv, T);
    for (int i = 0; i < Tq; ++i)
        for (int j = 0; j < Tkv; ++j) n += orc_causal(i, j, T, Nq, Nkv);
    return n;
}
