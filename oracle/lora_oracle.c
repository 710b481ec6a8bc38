/*
 * ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, obviously correct fp64 CPU implementation of the batched
 * multi-adapter LoRA delta.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or helper with the CUDA path (paper_2401_11240_b200/).
 *
 * What it computes (the plain definition, no blocking, fusion or reordering):
 *   PAPER.md §2.1 Eq. (1):  y' = xW + xAB,  A in R^{H1 x r}, B in R^{r x H2}.
 *   PAPER.md §2.2, P:299-300 and §4.1: the LoRA output xAB is computed
 *   on the fly per request and "added to the base output".
 *   BASELINE.json north_star adds the per-adapter scale s_a:  y_t += s_a (x_t A_a) B_a.
 *
 * Layout reading (reading R3): A is given rank-major, A_st[j][k] =
 * A[k][j] ([r][H_in]), B as [r][H_out].  For every token t of segment i with
 * adapter a = adapter_ids[i] >= 0:
 *     v[j]      = sum_{k=0..H_in-1} x[t][k] * A_st[j][k]        (ascending k)
 *     v[j]      = v[j] * s_a
 *     y[t][n]   = y_in[t][n] + sum_{j=0..r-1} v[j] * B[j][n]     (ascending j)
 * Tokens of segments with adapter id < 0 are left untouched (reading R7).
 *
 * The per-token routine is shared by the serial and the OpenMP driver, so both
 * perform the identical sequence of fp64 operations (pin P14: bitwise equal).
 *
 * Build: gcc -O2 -fPIC -shared -fopenmp -ffp-contract=off (no -ffast-math).
 */
#include <stdint.h>
#include <stddef.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_OK 0
#define ORACLE_ERR_UNKNOWN_ADAPTER 1
#define ORACLE_ERR_ARG 2
#define ORACLE_MAX_RANK 4096

/* find the table row of adapter id `id`; -1 when absent (plain linear scan) */
static int find_adapter(int n_adapters, const int32_t *ad_id, int32_t id) {
    for (int i = 0; i < n_adapters; ++i)
        if (ad_id[i] == id) return i;
    return -1;
}

/* one token: the three displayed lines of the header comment */
static void delta_token(int H_in, int H_out, int r, double s,
                        const double *A, const double *B,
                        const double *x_t, const double *y_in_t, double *y_out_t,
                        double *v /* [r] scratch, also returned */) {
    for (int j = 0; j < r; ++j) {
        double acc = 0.0;
        for (int k = 0; k < H_in; ++k)
            acc += x_t[k] * A[(size_t)j * H_in + k];
        v[j] = acc * s;
    }
    for (int n = 0; n < H_out; ++n) {
        double acc = 0.0;
        for (int j = 0; j < r; ++j)
            acc += v[j] * B[(size_t)j * H_out + n];
        y_out_t[n] = y_in_t[n] + acc;
    }
}

/*
 * oracle_lora_delta
 *   seg_indptr [S+1]  CSR: segment i owns tokens [seg_indptr[i], seg_indptr[i+1])
 *   adapter_ids[S]    adapter of each segment, < 0 = none
 *   ad_id/ad_rank/ad_scale/ad_A/ad_B  the adapter table (n_adapters rows)
 *   x    [T][H_in]  fp64,  y_in [T][H_out] fp64,  y_out [T][H_out] fp64 (written for
 *                   every computed token; rows of id<0 tokens are copied from y_in)
 *   token_mask [T]  optional (NULL = all): only tokens with mask != 0 are computed
 *   v_out [T][v_stride] optional: the scaled rank-r intermediate s*(x_t A)
 *   n_threads       1 = serial; > 1 = OpenMP over tokens (same per-token code)
 * returns ORACLE_OK or an error code (unknown adapter id, bad CSR).
 */
int oracle_lora_delta(int H_in, int H_out, int S,
                      const int32_t *seg_indptr, const int32_t *adapter_ids,
                      int n_adapters, const int32_t *ad_id, const int32_t *ad_rank,
                      const double *ad_scale, const double *const *ad_A, const double *const *ad_B,
                      const double *x, const double *y_in, double *y_out,
                      const uint8_t *token_mask, double *v_out, int v_stride, int n_threads) {
    if (S < 0 || H_in <= 0 || H_out <= 0) return ORACLE_ERR_ARG;
    if (seg_indptr[0] != 0) return ORACLE_ERR_ARG;
    for (int i = 0; i < S; ++i) {
        if (seg_indptr[i + 1] < seg_indptr[i]) return ORACLE_ERR_ARG;
        if (adapter_ids[i] >= 0) {
            int a = find_adapter(n_adapters, ad_id, adapter_ids[i]);
            if (a < 0) return ORACLE_ERR_UNKNOWN_ADAPTER;
            if (ad_rank[a] < 1 || ad_rank[a] > ORACLE_MAX_RANK) return ORACLE_ERR_ARG;
            if (v_out && ad_rank[a] > v_stride) return ORACLE_ERR_ARG;
        }
    }
    const int T = seg_indptr[S];

    /* token -> segment map (plain loop) so the OpenMP driver can split tokens */
    int32_t tok_seg_stack[1];
    int32_t *tok_seg = tok_seg_stack;
    if (T > 0) tok_seg = (int32_t *)malloc(sizeof(int32_t) * (size_t)T);
    for (int i = 0; i < S; ++i)
        for (int t = seg_indptr[i]; t < seg_indptr[i + 1]; ++t) tok_seg[t] = i;

    int err = ORACLE_OK;
#pragma omp parallel for schedule(dynamic, 1) num_threads(n_threads) if (n_threads > 1)
    for (int t = 0; t < T; ++t) {
        if (token_mask && !token_mask[t]) continue;
        const int i = tok_seg[t];
        const double *y_in_t = y_in + (size_t)t * H_out;
        double *y_out_t = y_out + (size_t)t * H_out;
        if (adapter_ids[i] < 0) {
            for (int n = 0; n < H_out; ++n) y_out_t[n] = y_in_t[n];
            continue;
        }
        const int a = find_adapter(n_adapters, ad_id, adapter_ids[i]);
        double v_local[ORACLE_MAX_RANK];
        delta_token(H_in, H_out, ad_rank[a], ad_scale[a], ad_A[a], ad_B[a],
                    x + (size_t)t * H_in, y_in_t, y_out_t, v_local);
        if (v_out)
            for (int j = 0; j < ad_rank[a]; ++j) v_out[(size_t)t * v_stride + j] = v_local[j];
    }
    if (T > 0) free(tok_seg);
    return err;
}

/* number of OpenMP threads the runtime would use (for cpu_baseline reporting) */
int oracle_max_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}
