/*
 * lora_delta.h -- C ABI of the B200-native batched multi-adapter LoRA delta.
 *
 * The operation (§2.1 Eq. 1; §2.2; §4.1):
 * for every token t of a continuous batch whose segment maps to adapter a(t) of
 * rank r_a,
 *
 *        y_t  +=  s_a · (x_t · A_a) · B_a                       (no padding to max rank)
 *
 * where A_a ∈ R^{H_in×r_a}, B_a ∈ R^{r_a×H_out} (Eq. 1's A and B) and s_a is a
 * per-adapter scale (BASELINE.json north_star; s_a = 1 reproduces Eq. 1).
 * The delta is "added to the base output", in place.  Adapters live in
 * host memory and are loaded on demand into a paged HBM pool (the cold start,
 * P:353-392); lora_apply is invoked per layer without any host synchronisation
 * (P:612-657).
 *
 * Conventions shared by every call
 *  - Every call returns an lora_status; none aborts.  On failure the thread-local
 *    message from lora_last_error() names the offending operand, and a failed
 *    call has no side effects.
 *  - Asynchronous CUDA errors surface as LORA_ERR_CUDA on a later call.
 *  - Calls on one pool must be serialised by the caller (exclusive
 *    access for registration); distinct pools are independent.  lora_apply calls
 *    on one pool must be issued in a single stream order (the pool's scratch is
 *    reused stream-ordered).
 *  - Element types: LORA_F32 (fp32 storage, fp32 arithmetic) and LORA_BF16 (bf16
 *    storage, fp32 accumulation, one round-to-nearest-even rounding of y + delta).
 *  - A is passed rank-major, A_host[j][k] = A[k][j] (j < rank, k < hidden_in): row
 *    j is the j-th column of Eq. 1's A (PEFT's lora_A.weight layout).  B is passed
 *    row-major as Eq. 1's B, B_host[j][n].  (reading R3.)
 */
#ifndef LORA_DELTA_H
#define LORA_DELTA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LORA_ABI_VERSION 2
#define LORA_MAX_RANK 256          /* 1 <= rank <= min(LORA_MAX_RANK, hidden_in, hidden_out) */

typedef struct lora_pool lora_pool;   /* opaque; bound to the CUDA device current at create */
typedef struct lora_tp_comm lora_tp_comm;   /* opaque; one tensor-parallel group's NCCL communicator */
#define LORA_TP_UNIQUE_ID_BYTES 128          /* size of the group's rendezvous id (ncclUniqueId) */

typedef enum { LORA_F32 = 0, LORA_BF16 = 1 } lora_dtype;

typedef enum {
    LORA_OK = 0,
    LORA_ERR_ARG = 1,               /* null pointer, negative size, malformed CSR, x/y overlap */
    LORA_ERR_SHAPE = 2,             /* hidden sizes / rank out of range */
    LORA_ERR_ALIGN = 3,             /* hidden not a multiple of 8 (bf16) / 4 (f32); x,y not 16-B aligned */
    LORA_ERR_UNKNOWN_ADAPTER = 4,   /* id not loaded */
    LORA_ERR_EXISTS = 5,            /* id already loaded */
    LORA_ERR_POOL_FULL = 6,         /* page budget or adapter slots exhausted */
    LORA_ERR_NOT_PINNED = 7,        /* A_host/B_host not page-locked host memory */
    LORA_ERR_CUDA = 8,              /* a CUDA runtime error (sticky errors reported on the next call) */
    LORA_ERR_NCCL = 9,              /* tensor-parallel communicator error */
    LORA_ERR_UNSUPPORTED = 10       /* operation not available for this pool (e.g. apply on a host-only pool) */
} lora_status;

/* pool creation flags */
#define LORA_POOL_HOST_ONLY 1u     /* host mirror only: no device memory, no CUDA calls.  Loads
                                      allocate pages and record (rank, scale) without copying;
                                      lora_plan/debug calls work; lora_apply returns UNSUPPORTED.
                                      Used by the CPU tests of allocator and metadata. */

/* segment kinds exported in the metadata (M5) */
#define LORA_KIND_NONE    (-1)     /* id < 0 or empty segment: no work */
#define LORA_KIND_DECODE    0      /* 1 <= len < L_tc: SIMT decode kernel */
#define LORA_KIND_PREFILL   1      /* len >= L_tc: tensor-core (tcgen05) prefill kernel */

/* options for lora_set_option */
#define LORA_OPT_TC_THRESHOLD 1    /* L_tc (default 64); segments with len >= L_tc take the tcgen05 path.
                                      A value larger than any segment forces the SIMT path everywhere. */
#define LORA_OPT_RESERVE_TOKENS 2  /* pre-size scratch for this many tokens (avoids a cudaMalloc in apply) */
/* options 3 and 4 (round-1 decode hand-off / cluster-span experiments) are retired in ABI 2; DESIGN.md
   §6 keeps their measurements and that of the round-2 persistent streaming kernel */

#define LORA_OPT_PAD_MAX_RANK 5    /* comparison mode: 1 pads every adapter's
                                      decode work to the batch's max rank with the pool's all-zero
                                      page, i.e. the padded BGMV of Punica that the paper contrasts
                                      with MBGMV (§3.1).  Same result (zero rows
                                      add 0); more bytes and time.  Not for production. */

#define LORA_OPT_LOAD_KERNEL 6     /* 1: lora_load_adapter copies the rank rows with a zero-copy gather
                                      kernel on the side stream (SMs read the UVA-mapped pinned host
                                      rows over PCIe): c4 cold-start loads 26 -> ~41 GB/s effective,
                                      one 1 MB adapter in 18 us (56 GB/s).  0 (default): cudaMemcpyAsync
                                      per run of pages (also the fallback when the host rows have no
                                      device mapping).  Same bytes (tested bitwise), same ready-event
                                      semantics.  Not the default: after many kernel loads, some
                                      processes run every later decode apply ~5 % slower (a
                                      process-wide state: pools loaded by memcpy in the same process
                                      slow down too; profiles/r2_load_kernel_bimodal.txt). */

/*
 * lora_pool_create -- make an empty paged adapter pool for one projection shape.
 *   hidden_in, hidden_out  H_in, H_out of the adapted projection (Eq. 1's H1, H2).
 *   max_adapters           resident-adapter slot count (id -> pages table).
 *   dtype                  element type of x, y, A and B.
 *   max_total_rank         page budget: one page holds one rank component
 *                          (a_j ∈ R^{H_in}, b_j ∈ R^{H_out}); 0 means 64 * max_adapters.
 *                          Device bytes = max_total_rank * (H_in + H_out) * sizeof(dtype).
 *   out                    receives the pool handle.
 * Errors: SHAPE (hidden <= 0, max_adapters <= 0), ALIGN, CUDA (allocation).
 */
lora_status lora_pool_create(int hidden_in, int hidden_out, int max_adapters, lora_dtype dtype,
                             int max_total_rank, lora_pool** out);

/* lora_pool_create_ex -- as lora_pool_create with flags (LORA_POOL_HOST_ONLY). */
lora_status lora_pool_create_ex(int hidden_in, int hidden_out, int max_adapters, lora_dtype dtype,
                                int max_total_rank, unsigned flags, lora_pool** out);

/* lora_pool_destroy -- synchronises the pool's side streams and every stream the pool was
 * applied on, then frees pages, scratch, events and staging.  NULL is a no-op. */
lora_status lora_pool_destroy(lora_pool* p);

/*
 * lora_load_adapter -- the cold-start path (§2.3 C1).
 *   id      adapter id >= 0.
 *   rank    r, 1 <= r <= min(LORA_MAX_RANK, hidden_in, hidden_out).
 *   A_host  pinned host buffer [rank][hidden_in]  (rank-major A, see header).
 *   B_host  pinned host buffer [rank][hidden_out].
 *   scale   s_a (fp32).
 * Allocates the rank lowest-indexed free pages (ascending; reading R9), then
 * enqueues the host->HBM copies on one of the pool's side streams (8, round-robin, so
 * consecutive loads overlap) and records a ready event; it returns without waiting.  The buffers must stay valid and unmodified until
 * lora_adapter_ready reports 1; the library never frees them.  Physical reuse of pages
 * freed by lora_unload_adapter is ordered after the applies that read them (events).
 * Errors: ARG (id < 0, null buffer), SHAPE (rank), EXISTS, POOL_FULL, NOT_PINNED, CUDA.
 * Host-only pools ignore A_host/B_host (may be NULL).
 */
lora_status lora_load_adapter(lora_pool* p, int32_t id, int rank,
                              const void* A_host, const void* B_host, float scale);

/* lora_unload_adapter -- frees the adapter's slot and pages at call time (logical); the
 * pages are physically rewritten only after the applies already enqueued and the adapter's
 * own load have finished (every side stream waits on both). */
lora_status lora_unload_adapter(lora_pool* p, int32_t id);

/* lora_adapter_ready -- *ready = 1 once the adapter's load has completed (cudaEventQuery). */
lora_status lora_adapter_ready(lora_pool* p, int32_t id, int* ready);

/*
 * lora_apply -- y += s·(x·A)·B per token, for one batch (the GPU LoRA of PAPER.md §4.1).
 *   x            device [T][hidden_in],  pool dtype, rows contiguous, 16-B aligned.
 *   y            device [T][hidden_out], pool dtype, updated in place; must not overlap x.
 *   seg_indptr   HOST [num_segments+1], CSR: segment i owns tokens [seg_indptr[i], seg_indptr[i+1]);
 *                seg_indptr[0] = 0, non-decreasing; T = seg_indptr[num_segments].
 *   adapter_ids  HOST [num_segments]; id < 0 = no adapter (rows bitwise untouched);
 *                duplicates allowed.
 *   stream       cudaStream_t the work is enqueued on (NULL = legacy default stream).
 * Builds the canonical metadata on the host, makes `stream` wait for any adapter whose
 * load is still in flight, and launches the decode (SIMT) and prefill (tcgen05) kernels on
 * `stream`.  Never synchronises the host.  seg_indptr/adapter_ids are consumed before
 * return.  T = 0 or num_segments = 0 is a no-op.  Graph capture of `stream` is supported: inside
 * a capture nothing is allocated, synchronised or queried, and loads still in flight become
 * external event waits.  A batch that needs more scratch than the pool holds is refused there
 * (UNSUPPORTED, the capture stays valid): run that batch shape once outside the capture, or pre-size
 * with LORA_OPT_RESERVE_TOKENS.  Outgrown scratch is kept until lora_pool_destroy, so graphs captured
 * earlier stay valid when a later apply grows it.  The pool's scratch is shared by its applies: one
 * pool serves one stream (or graph) at a time.
 * Errors: ARG, ALIGN, UNKNOWN_ADAPTER, UNSUPPORTED (host-only pool; scratch growth during capture), CUDA.
 */
lora_status lora_apply(lora_pool* p, const void* x, void* y,
                       const int32_t* seg_indptr, const int32_t* adapter_ids,
                       int num_segments, void* stream);

/*
 * lora_apply_multi -- lora_apply on up to 4 pools that share one batch layout (e.g. the W_Q, W_K,
 * W_V projections of a layer, which the paper adapts together), fused into ONE launch
 * pair of the decode kernels (prefill tiles still launch per pool).  Same semantics as calling
 * lora_apply(pools[i], xs[i], ys[i], seg_indptr, adapter_ids, num_segments, stream) for each i;
 * the work of all pools shares the kernels' prologue/epilogue latency instead of paying it per
 * pool.  The pools must be distinct, on one device and of one dtype; the first pool's scratch is
 * used.  All plans are validated before anything is launched.
 * Errors: as lora_apply (the message names the offending pool index).
 */
lora_status lora_apply_multi(lora_pool* const* pools, const void* const* xs, void* const* ys, int n_pools,
                             const int32_t* seg_indptr, const int32_t* adapter_ids, int num_segments, void* stream);

/*
 * Tensor parallelism (BASELINE.json north_star: "A tensor-parallel variant splits B's output
 * dimension (and A's input dimension, with an NCCL all-reduce of the tiny rank-r intermediate over
 * NVLink) for 70B-sized projections").  The paper's own scheme replicates
 * A and splits only B, with no communication (§4.2 "Support model parallelism");
 * splitting A's input dimension too makes every GPU's adapter bytes scale as 1/tp at the cost of one
 * all-reduce of v = s-less x·A, [T x r] fp32 (c5 decode: 64 tokens x ranks 16..128 = 15,360 B).
 * A TP rank's pool holds the shards A[:, its H_in slice] and B[:, its H_out slice]: the pool's
 * hidden_in / hidden_out are the shard widths.  Column-parallel layers (q/k/v/gate/up: x replicated)
 * pass the rank's x columns as a strided view (x_ld = full width) and their own y shard;
 * row-parallel layers (o/down: x already sharded) pass their x shard and a strided view of the
 * partial, pre-all-reduce y (y_ld = full width), which the base layer's own all-reduce completes.
 *
 * lora_tp_unique_id -- ncclGetUniqueId into id_out[LORA_TP_UNIQUE_ID_BYTES]: rank 0 of the group calls
 *   it and hands the bytes to the other ranks (the Python binding broadcasts them through the
 *   torch.distributed process group).  Errors: ARG, NCCL (libnccl.so.2 is resolved at run time).
 * lora_tp_comm_create -- ncclCommInitRank for (tp_rank, tp_size) on the CUDA device current at the
 *   call; collective over the group.  The caller owns the handle and destroys it after the pools
 *   bound to it.  Errors: ARG, NCCL.
 * lora_tp_comm_destroy -- ncclCommDestroy.  NULL is a no-op.
 * lora_tp_init -- binds pool p to the group's communicator (NULL unbinds).  Errors: ARG (other device),
 *   UNSUPPORTED (host-only pool).
 * lora_apply_tp -- y[:, this rank's out slice] += s·(Σ_ranks x_k·A_k)·B_shard for one batch, all on
 *   `stream` without host synchronisation: the shrink kernel (partials over this rank's
 *   H_in slice, per 1,024-wide k-slice; the last CTA of each group-chunk to finish sums the slices in
 *   fixed order into the compact v [Σ_gc ntok x round_up(r, 4)] fp32), ncclAllReduce(SUM) of that
 *   compact v in place over the group, the expand kernel.  Every token takes the decode kernels.  Capturable in a CUDA
 *   graph (NCCL calls are).
 *     x   device, T rows of hidden_in elements, row stride x_ld elements (0 = hidden_in), 16-B aligned.
 *     y   device, T rows of hidden_out elements, row stride y_ld elements (0 = hidden_out), 16-B aligned.
 *   Errors: as lora_apply; ARG without lora_tp_init or with x_ld/y_ld below the widths; NCCL.
 * lora_load_adapter_shard -- lora_load_adapter of this rank's shard straight from the FULL pinned
 *   adapter: rows j of A_host [rank][a_ld] columns [a_col0, a_col0 + hidden_in) and of B_host
 *   [rank][b_ld] columns [b_col0, b_col0 + hidden_out), one cudaMemcpy2DAsync per run of pages on the
 *   pool's side stream (no host-side slice or re-pin).  Errors: as lora_load_adapter; SHAPE (columns
 *   outside the full rows), ALIGN (pitch or first column not 16-B aligned).
 *
 * The split calls for callers that run their own collective:
 * lora_apply_shrink -- shrink + k-reduce of this rank's partial v into v_out (device fp32, v_capacity
 *   floats, 4-B aligned): the compact layout above, size lora_metadata_view.v_floats of the same
 *   batch (lora_plan).  Identical batches on every rank give identical layouts, so an elementwise
 *   SUM all-reduce of v_out yields the full-H_in v.  Every token takes the decode kernels.
 * lora_apply_expand -- y[:, this rank's H_out slice] += s · v · B_shard for the batch of the
 *   immediately preceding lora_apply_shrink on this pool, reading the (all-reduced) compact v_in.
 * Errors: as lora_apply; ARG if v_capacity is too small or expand has no pending shrink; ALIGN if
 *   v_out / v_in is not 4-byte aligned.
 */
lora_status lora_tp_unique_id(void* id_out);
lora_status lora_tp_comm_create(const void* id, int tp_rank, int tp_size, lora_tp_comm** out);
lora_status lora_tp_comm_destroy(lora_tp_comm* comm);
lora_status lora_tp_init(lora_pool* p, lora_tp_comm* comm);
lora_status lora_apply_tp(lora_pool* p, const void* x, int64_t x_ld, void* y, int64_t y_ld, const int32_t* seg_indptr,
                          const int32_t* adapter_ids, int num_segments, void* stream);
lora_status lora_load_adapter_shard(lora_pool* p, int32_t id, int rank, const void* A_host, int64_t a_ld, int64_t a_col0,
                                    const void* B_host, int64_t b_ld, int64_t b_col0, float scale);
lora_status lora_apply_shrink(lora_pool* p, const void* x, const int32_t* seg_indptr, const int32_t* adapter_ids,
                              int num_segments, float* v_out, int64_t v_capacity, void* stream);
lora_status lora_apply_expand(lora_pool* p, void* y, const float* v_in, void* stream);

/* lora_apply_fused_base -- the delta fused into the base projection GEMM (
 * PAPER.md §4.1 P:548-550 "incorporate the operators of GPU LoRA computation into the base LLM
 * inference process"; Eq. 1 P:276-280 with the adapter scale):
 *     y_t = x_t · W + s_a · (x_t · A_a) · B_a      (id < 0: y_t = x_t · W)
 * in one tcgen05 kernel: every K stage's x tile feeds both x·W and x·A; V = s·(x·A) is rounded once
 * to bf16 and its expand accumulates into the base accumulator in TMEM; y is written once (never
 * read).  fp32 accumulation, one bf16 rounding of y.
 *   x    device [T][hidden_in] bf16, 16-B aligned.
 *   W    device [hidden_in][hidden_out] bf16 row-major (the base projection), 16-B aligned; not owned.
 *   y    device [T][hidden_out] bf16, 16-B aligned, OVERWRITTEN (not accumulated); must not overlap
 *        x or W.
 *   seg_indptr / adapter_ids / num_segments / stream: as lora_apply.  Every segment's tokens are
 *   covered by 128-token tiles of that segment (short segments waste tile rows: this path is for
 *   prefill batches).
 * Errors: ARG, ALIGN, UNKNOWN_ADAPTER, CUDA; UNSUPPORTED for an fp32 pool, hidden_in % 64 != 0,
 * hidden_out % 128 != 0, an adapter of rank > 128, or a batch whose tile records and page lists
 * exceed the 7,680-word parameter blob of one launch. */
lora_status lora_apply_fused_base(lora_pool* p, const void* x, const void* W, void* y, const int32_t* seg_indptr,
                                  const int32_t* adapter_ids, int num_segments, void* stream);

/* lora_plan -- build (and keep for lora_debug_metadata) the canonical metadata of a batch
 * without launching anything.  Pure host code; works on host-only pools. */
lora_status lora_plan(lora_pool* p, const int32_t* seg_indptr, const int32_t* adapter_ids,
                      int num_segments);

/* lora_set_option -- see LORA_OPT_*. */
lora_status lora_set_option(lora_pool* p, int option, int64_t value);

typedef struct {
    int32_t hidden_in, hidden_out, max_adapters, max_total_rank, dtype, elem_bytes;
    int32_t resident_adapters, free_pages, tc_threshold, device;
    int64_t pool_bytes;           /* device bytes of the page arrays */
    int64_t resident_bytes;       /* Σ over resident adapters of r·(H_in+H_out)·elem_bytes (pin P11) */
    int64_t kernel_launches;      /* CUDA kernels this pool has launched (all applies so far) */
} lora_pool_info_t;

lora_status lora_pool_info(lora_pool* p, lora_pool_info_t* out);

/* Canonical metadata of the last lora_plan / lora_apply (M1-M6).
 * Views point into pool-owned host memory, valid until the next plan/apply on the pool. */
typedef struct {
    int32_t T, S, G, L_tc;
    const int32_t* tok_seg;          /* [T]  M1 */
    const int32_t* group_id;         /* [G]  M2: distinct ids >= 0 owning >= 1 token, ascending */
    const int32_t* group_rank;       /* [G] */
    const float*   group_scale;      /* [G] */
    const int32_t* group_ntok;       /* [G] */
    const int32_t* group_page_off;   /* [G]  offset into pages */
    const int32_t* group_tok_off;    /* [G]  offset into group_tokens */
    const int32_t* group_tokens;     /* [T_adapted] M3: token indices per group, ascending */
    const int32_t* pages;            /* [sum_rank_groups] M4: each group's pages in rank order */
    const int32_t* seg_kind;         /* [S]  M5: LORA_KIND_* */
    int64_t n_seg;                   /* M6: segments with id >= 0 and >= 1 token (the paper's |S|) */
    int64_t max_rank;                /*     max rank over those segments */
    int64_t nseg_x_maxrank;          /*     |S|·max r  (Perf_BGMV feature) */
    int64_t sum_rank_seg;            /*     Σ_{i∈S} r  (Perf_MBGMV feature) */
    int64_t sum_rank_groups;         /*     Σ over distinct adapters of r (adapter bytes / (H_in+H_out)/b) */
    int64_t sum_rank_tokens;         /*     Σ_t r_{a(t)} (flops / 2(H_in+H_out)) */
    int32_t n_decode_units, n_prefill_tiles;   /* kernel work of the last apply (informational) */
    int32_t n_shrink_units, n_expand_units;    /* split of n_decode_units (shrink units come first) */
    int64_t v_floats;                          /* size of the compact k-reduced v (lora_apply_shrink) */
    int32_t reserved0, reserved1;
    int32_t n_prefill_ctas, prefill_cluster;   /* tcgen05 prefill grid of the last apply: CTAs
                                                  (tiles x CTAs per tile) and split-K cluster size
                                                  (1 = no split-K) */
} lora_metadata_view;

lora_status lora_debug_metadata(lora_pool* p, lora_metadata_view* out);

/* lora_debug_adapter_pages -- copies the adapter's page indices (rank order) into
 * pages[0..cap) and its rank into *rank. */
lora_status lora_debug_adapter_pages(lora_pool* p, int32_t id, int32_t* pages, int cap, int* rank);

/* lora_debug_read_pages -- synchronous D2H read-back of an adapter's pages into host
 * buffers laid out like lora_load_adapter's (pin P12).  Synchronises the side streams. */
lora_status lora_debug_read_pages(lora_pool* p, int32_t id, void* A_out, void* B_out);

/* lora_debug_set_trace -- profiling aid: when dev_buf (device memory, uint64 words) is non-NULL,
 * each decode-kernel launch records per work unit u the words [8u..8u+5] = (smid, t_wait,
 * t_issue, t_data, t_flag, t_done) in %globaltimer ns, and per CTA b the words
 * [8·n_units + 4b ..] = (t_start, t_end, smid).  The buffer must hold 8·n_units + 4·grid words.
 * NULL disables tracing (the default). */
lora_status lora_debug_set_trace(lora_pool* p, void* dev_buf);

/* thread-local message of the last failed call on this thread ("" if none). */
const char* lora_last_error(void);

int lora_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* LORA_DELTA_H */
