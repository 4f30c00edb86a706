/*
 * codec_b200.h -- C ABI of the B200-native prefix-shared decode-attention
 * path (CoDec, arXiv 2505.17694).
 *
 * Plain C types only: pointers, sizes, PODs. No torch / C++ types cross
 * this boundary. Every product entry point is reentrant: handles
 * (codec_index, codec_plan, codec_table, codec_kernel_timer) carry all
 * state, the last-error string is thread-local, and every device entry
 * point is asynchronous on the caller's stream (passed as `void*`, a
 * cudaStream_t). The only process-global buffers belong to the debug
 * flags CODEC_FLAG_TRACE / CODEC_FLAG_CTALOG (timelines for tools/).
 * Ownership: the caller owns every buffer; host-side handles are created
 * and freed here.
 *
 * Each entry point names the reference interface it replaces
 * (/root/reference/pkg/src/prefixdec/<file>:<line>).  Status codes map
 * 1:1 onto the reference's exception classes (errors.py:9-102); the
 * Python host layer raises the same class with codec_last_error() as the
 * message.
 */
#ifndef CODEC_B200_H
#define CODEC_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define CODEC_API __attribute__((visibility("default")))
#else
#define CODEC_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status */
typedef enum {
  CODEC_OK = 0,
  CODEC_ERR_CYCLE_DETECTED = 1,          /* errors.CycleDetected          */
  CODEC_ERR_DANGLING_PARENT = 2,         /* errors.DanglingParent         */
  CODEC_ERR_PATH_NOT_PREFIX_CHAIN = 3,   /* errors.PathNotPrefixChain     */
  CODEC_ERR_DIMENSION_MISMATCH = 4,      /* errors.DimensionMismatch      */
  CODEC_ERR_UNKNOWN_REQUEST = 5,         /* errors.UnknownRequest         */
  CODEC_ERR_UNKNOWN_NODE = 6,            /* errors.UnknownNode            */
  CODEC_ERR_SHAPE_MISMATCH = 7,          /* errors.ShapeMismatch          */
  CODEC_ERR_EMPTY_VISIBLE_SET = 8,       /* errors.EmptyVisibleSet        */
  CODEC_ERR_NO_VISIBLE_TOKENS = 9,       /* errors.NoVisibleTokens        */
  CODEC_ERR_PLAN_FOREST_MISMATCH = 10,   /* errors.PlanForestMismatch     */
  CODEC_ERR_INCOMPLETE_PARTIALS = 11,    /* errors.IncompletePartials     */
  CODEC_ERR_SEARCH_SPACE_OVERFLOW = 12,  /* errors.SearchSpaceOverflow    */
  CODEC_ERR_PROFILE_LOAD = 13,           /* errors.ProfileLoadError       */
  CODEC_ERR_INCOMPLETE_GRID = 14,        /* errors.IncompleteGrid         */
  CODEC_ERR_NON_POSITIVE_COST = 15,      /* errors.NonPositiveCost        */
  CODEC_ERR_DUPLICATE_KNOT = 16,         /* errors.DuplicateKnot          */
  CODEC_ERR_VALUE = 20,                  /* builtin ValueError            */
  CODEC_ERR_UNSUPPORTED = 30,            /* shape/dtype the kernels do not cover */
  CODEC_ERR_CUDA = 31                    /* CUDA runtime/launch failure   */
} codec_status;

/* Message of the last non-OK status returned on this thread. */
CODEC_API const char* codec_last_error(void);
/* ABI version (bumped on any incompatible change). */
CODEC_API int32_t codec_abi_version(void);

/* element types of q / k / v / partials */
typedef enum { CODEC_F32 = 0, CODEC_F64 = 1, CODEC_BF16 = 2 } codec_dtype;

/* ======================================================================
 * K0 -- forest indexing.  Replaces the index half of
 *   build_forest()            forest.py:160-251
 *   _preorder_offsets()       forest.py:148-157
 * Inputs are the structural parts of the node specs and request paths;
 * tensors stay with the caller. Raises the build_forest error classes
 * with the reference's messages.
 * ==================================================================== */
typedef struct codec_index codec_index;

CODEC_API int32_t codec_index_build(int32_t n_nodes,            /* incl. virtual root 0 */
                          const int32_t* parent,      /* [n_nodes]; parent[0] ignored */
                          const int64_t* length,      /* [n_nodes]; length[0] ignored (0) */
                          int32_t bs,
                          const int64_t* path_ptr,    /* [bs+1] CSR of request paths */
                          const int32_t* path_idx,
                          int64_t n_vis,              /* visible_len entries */
                          const int32_t* vis_node,    /* [n_vis] */
                          const int32_t* vis_req,     /* [n_vis] */
                          const int64_t* vis_count,   /* [n_vis] */
                          codec_index** out);
CODEC_API void codec_index_free(codec_index* ix);

typedef struct {
  int32_t n_nodes, bs;
  int64_t total_tokens;     /* sum of node lengths (pool tokens) */
  int64_t qset_nnz;         /* sum |I_n| */
  int64_t path_nnz;
} codec_index_info;
CODEC_API int32_t codec_index_info_get(const codec_index* ix, codec_index_info* info);
/* Copy out: node_off[n_nodes] (preorder kappa, forest.py:148-157),
 * qset_ptr[n_nodes+1], qset_idx[qset_nnz] (ascending I_n, forest.py:236-237),
 * qset_vis[qset_nnz] (visible count of that request in that node,
 * forest.py:128-132), children_ptr[n_nodes+1], children_idx[n_nodes-1]. Any
 * pointer may be NULL. */
CODEC_API int32_t codec_index_read(const codec_index* ix, int64_t* node_off, int64_t* qset_ptr,
                         int32_t* qset_idx, int64_t* qset_vis, int64_t* children_ptr,
                         int32_t* children_idx);

/* ======================================================================
 * Structural report of a forest snapshot.  Replaces validate()
 * forest.py:266-363: every invariant checked, violations reported (not
 * raised) in the reference's order with its messages. The caller flattens
 * the (possibly corrupted) forest: per node position i its id, parent,
 * length and K/V state (kv_state 0: not checked, 1: K and V shapes differ,
 * 2: keys.shape[1:] given as kv_tail[kv_tail_ptr[i], kv_tail_ptr[i+1]));
 * children / paths / query sets as CSR; visible_len as (node, request,
 * count) triples in node order; token_offset as stored.
 * ==================================================================== */
typedef enum {
  CODEC_VIOLATION_BAD_NODE_INDEX = 0,
  CODEC_VIOLATION_NON_EMPTY_ROOT = 1,
  CODEC_VIOLATION_EMPTY_NON_ROOT = 2,
  CODEC_VIOLATION_DIMENSION_MISMATCH = 3,
  CODEC_VIOLATION_CYCLE_DETECTED = 4,
  CODEC_VIOLATION_DANGLING_PARENT = 5,
  CODEC_VIOLATION_ADJACENCY_MISMATCH = 6,
  CODEC_VIOLATION_PATH_NOT_PREFIX_CHAIN = 7,
  CODEC_VIOLATION_QUERY_SET_UNSORTED = 8,
  CODEC_VIOLATION_QUERY_SET_PATH_MISMATCH = 9,
  CODEC_VIOLATION_VISIBLE_LEN_OUT_OF_RANGE = 10,
  CODEC_VIOLATION_FLATTEN_MISMATCH = 11
} codec_violation_code;
typedef struct codec_report codec_report;
CODEC_API int32_t codec_forest_validate(int32_t n_nodes, const int64_t* node_id, const int64_t* parent,
                                        const int64_t* length, const int32_t* kv_state, const int64_t* kv_tail_ptr,
                                        const int64_t* kv_tail, int64_t h_kv, int64_t d, const int64_t* children_ptr,
                                        const int64_t* children_idx, int32_t bs, const int64_t* path_ptr,
                                        const int64_t* path_idx, const int64_t* qset_ptr, const int64_t* qset_idx,
                                        int64_t n_vis, const int64_t* vis_node, const int64_t* vis_req,
                                        const int64_t* vis_count, const int64_t* token_offset,
                                        int64_t n_token_offset, codec_report** out);
CODEC_API int32_t codec_report_count(const codec_report* rep, int64_t* n);
/* record i: code, node / request (INT64_MIN = None), message (NUL-terminated, truncated to msg_cap) */
CODEC_API int32_t codec_report_get(const codec_report* rep, int64_t i, int32_t* code, int64_t* node,
                                   int64_t* request, char* msg, int64_t msg_cap);
CODEC_API void codec_report_free(codec_report* rep);

/* ======================================================================
 * K1 -- cost model, task division and schedule (host, float64, operation
 * order identical to the reference => bit-exact plans).
 * ==================================================================== */
typedef struct {
  int32_t n_nq, n_n;
  const int64_t* nq_knots;   /* [n_nq] strictly ascending */
  const int64_t* n_knots;    /* [n_n]  strictly ascending */
  const double* cost_ms;     /* [n_n][n_nq] row-major      */
} codec_cost_table;

/* load_profile() grid assembly (cost_model.py:102-150): profile rows in
 * file order -> sorted unique knots and the n-major grid; raises
 * DuplicateKnot / NonPositiveCost on the first offending row, then
 * IncompleteGrid on the first missing cell. grid NULL: sizing call (knot
 * counts only). */
CODEC_API int32_t codec_cost_grid(int64_t n_rows, const int64_t* row_nq, const int64_t* row_n,
                                  const double* row_cost, int32_t* n_nq, int32_t* n_n, int64_t* nq_knots,
                                  int64_t* n_knots, double* grid);
/* CostTable invariants (cost_model.py:39-53): grid shape (given as
 * grid_ndim / grid_shape) = (len(n), len(n_q)), strictly ascending positive
 * knots, positive costs. */
CODEC_API int32_t codec_cost_table_check(int32_t n_nq, const int64_t* nq_knots, int32_t n_n, const int64_t* n_knots,
                                         int32_t grid_ndim, const int64_t* grid_shape, const double* cost_ms);
/* estimate()            cost_model.py:68-84 */
CODEC_API double codec_estimate(const codec_cost_table* t, int64_t n_q, int64_t n);
/* slice_ranges()/canonical_division()   scheduler.py:81-92.
 * Writes up to `cap` (start, stop) pairs; *count gets the slice count. */
CODEC_API int32_t codec_slice_ranges(int64_t n, int64_t b, int64_t* start_stop, int64_t cap, int64_t* count);
/* lower_bound()         scheduler.py:106-131 */
CODEC_API int32_t codec_lower_bound(const codec_cost_table* t, int32_t n_tasks, const int64_t* task_nq,
                          const int64_t* task_n, int32_t m, double tol, double* cost_l);
/* division_caps()       scheduler.py:134-139 */
CODEC_API int32_t codec_division_caps(const codec_cost_table* t, int32_t n_tasks, const int64_t* task_nq,
                            const int64_t* task_n, double cost_l, int64_t* caps);
/* greedy_assign()       scheduler.py:142-155 */
CODEC_API int32_t codec_greedy_assign(int64_t n, const double* costs, int32_t m, int32_t* block_of,
                            double* loads);

typedef struct codec_plan codec_plan;
/* divide_and_schedule() scheduler.py:187-222. on_overflow: 0 = fallback,
 * 1 = raise SearchSpaceOverflow. */
CODEC_API int32_t codec_divide_and_schedule(const codec_cost_table* t, int32_t n_tasks,
                                  const int64_t* task_node, const int64_t* task_nq,
                                  const int64_t* task_n, int32_t m, int64_t search_limit,
                                  int32_t on_overflow, codec_plan** out);
/* plan_uniform_bk()     scheduler.py:225-233. cost_l: NaN means None. */
CODEC_API int32_t codec_plan_uniform(const codec_cost_table* t, int32_t n_tasks, const int64_t* task_node,
                           const int64_t* task_nq, const int64_t* task_n, int32_t m, int64_t bk,
                           double cost_l, codec_plan** out);
CODEC_API void codec_plan_free(codec_plan* p);

typedef struct {
  int32_t n_tasks, n_subtasks, blocks, truncated;
  double makespan_ms, cost_l_ms;   /* cost_l NaN == None */
} codec_plan_info;
CODEC_API int32_t codec_plan_info_get(const codec_plan* p, codec_plan_info* info);
/* DivisionPlan fields (scheduler.py:26-78); any pointer may be NULL. */
CODEC_API int32_t codec_plan_read(const codec_plan* p, int64_t* b_k, int32_t* sub_task, int64_t* sub_node,
                        int64_t* sub_start, int64_t* sub_stop, double* sub_cost,
                        int32_t* block_of, double* loads);

/* ======================================================================
 * Device task table -- the plan expanded for the GPU.  Replaces the job
 * construction of _split_phase() (executor.py:145-206: row filter :156,
 * per-row visible :187-190) and the per-request unit lists of
 * _reduce_one() (executor.py:209-231), validated like _plan_slices()
 * (executor.py:120-142).
 *
 * Each plan task owns a contiguous chunk of its node's query set (a
 * node-level plan, tasks_from_forest(), is the one-chunk case). Each
 * subtask x row tile becomes one "group". GEMV / generic groups run one CTA
 * per (group, local kv head); tensor-core groups are LPT-packed (the
 * reference's greedy rule, scheduler.py:142-155) onto sm_count/h_local
 * persistent CTAs per head, which walk their group lists in order.
 * ==================================================================== */
typedef struct {
  int32_t bs, h_q, h_kv, d;
  int32_t head_begin, head_end;   /* local kv-head shard [begin, end) */
  int32_t kv_dtype;               /* codec_dtype of q, k, v */
  int32_t flags;                  /* CODEC_FLAG_* */
  int64_t pool_tokens;            /* T: token stride of one head in the pool */
  int32_t sm_count;               /* SMs of the device (0 = 148); sizes the persistent TC grid */
  int32_t tc_sm_budget;           /* SMs the TC kernel may occupy (0 = all); the rest stay free
                                     for the GEMV kernel running concurrently on an aux stream */
  /* Paged KV (ABI v3). page_size 0: k / v are the contiguous node pool
   * (nodes at their preorder offsets). page_size P > 0 (a power of two
   * >= 128; bf16, d = 128, tensor-core + mma.sync suffix kernels only):
   * every node's tokens are split into pages of P tokens, node n owning
   * logical pages [base[n], base[n+1]) (codec_page_layout); k / v are
   * [h_local][pool_tokens][d] physical pools and page_table[logical page]
   * is the physical page (token rows [page * P, page * P + P) of every
   * head). Plan slices must start at multiples of 128 tokens (shared,
   * tensor-core nodes) / 32 tokens (suffix nodes) within their node. */
  int32_t page_size;
  int32_t reserved0;
  const int32_t* page_table;      /* device int32[n_logical_pages]; NULL when page_size == 0 */
} codec_dims;

/* Logical page layout of a paged pool: node n (node-id order) owns pages
 * [node_page_base[n], node_page_base[n + 1]), ceil(len_n / page_size) of
 * them; *n_pages = node_page_base[n_nodes]. node_page_base has n_nodes + 1
 * entries. */
CODEC_API int32_t codec_page_layout(const codec_index* ix, int32_t page_size, int64_t* node_page_base,
                                    int64_t* n_pages);

#define CODEC_FLAG_NO_TC      1   /* never use the tcgen05 shared-node kernel */
#define CODEC_FLAG_FORCE_TC   2   /* tcgen05 kernel for every eligible group */
#define CODEC_FLAG_NO_GEMV    4   /* generic kernel instead of the GEMV kernel */
/* launch-time phase selection (profiling: time one kernel of the step alone) */
#define CODEC_FLAG_SKIP_GENERIC 8
#define CODEC_FLAG_SKIP_TC      16
#define CODEC_FLAG_SKIP_GEMV    32
#define CODEC_FLAG_SKIP_MERGE   64
#define CODEC_FLAG_TRACE        128  /* record a clock64 timeline of TC CTA pair (0,0) (debug) */
#define CODEC_FLAG_DBG_NO_TMEM  256  /* TC softmax skips its TMEM S loads / P stores: timing only, wrong output (debug) */
#define CODEC_FLAG_DBG_NO_EXP   512  /* TC softmax skips the exponentials: timing only, wrong output (debug) */
#define CODEC_FLAG_CTALOG       1024 /* record {smid, start ns, end ns, cta} per TC / GEMV CTA (debug) */
#define CODEC_FLAG_GEMV_SIMT    2048 /* suffix groups on the CUDA-core GEMV kernel instead of the mma.sync one */
#define CODEC_FLAG_FUSED_MERGE  4096 /* the mma.sync suffix kernel folds each request's TC partials into its output
                                        instead of the merge kernel (opt-in: slower on cfg2 so far) */
#define CODEC_FLAG_DBG_NO_TC_UNITS 8192 /* TC kernel skips its shared-node units: timing only, wrong output (debug) */
#define CODEC_FLAG_DBG_NO_LOADS 32768 /* TC producers skip the K/V TMA loads: timing only, wrong output (debug) */
#define CODEC_FLAG_DBG_ISSUER_ONLY 131072 /* TC kernel runs only its MMA issuer, no waits: timing only (debug) */
#define CODEC_FLAG_MERGE_NO_PDL 262144 /* launch the merge plainly after the suffix kernel (measurement) */
#define CODEC_FLAG_NO_MULTI 524288 /* lightly shared slices on the tensor-core (or per-request) kernels instead of
                                       the multi-request mma.sync kernel */
#define CODEC_FLAG_COUNTED_MERGE 1048576 /* partial producers count per merge entry and the merge starts each entry
                                            as soon as it is complete (opt-in: measured no faster on cfg2/cfg3) */
#define CODEC_FLAG_DBG_NO_PWAIT 65536 /* with DBG_NO_TMEM: softmax skips the P-buffer (PV(t-2)) wait: timing only (debug) */
#define CODEC_FLAG_NO_TCT 4194304 /* lightly shared slices above the multi-request range on the M = 256 pair kernel
                                      instead of the transposed tensor-core kernel */
#define CODEC_FLAG_TCT_WIDE 8388608 /* the transposed tensor-core kernel also takes nodes of 65..128 query-head rows
                                       (its wide variant) instead of the pair kernel */
#define CODEC_FLAG_MERGE_ALL 2097152 /* every (request, kv head) output goes through the merge kernel, single-partial
                                        ones too (no direct writes by the split kernels): what the fused peer-store
                                        output gather (codec_decode_attention_gather) needs */

typedef struct codec_table codec_table;
CODEC_API int32_t codec_table_build(const codec_index* ix, const codec_dims* dims, int32_t n_tasks,
                          const int64_t* task_node, const int64_t* task_nq, int32_t n_sub,
                          const int32_t* sub_task, const int64_t* sub_start,
                          const int64_t* sub_stop, const int32_t* sub_block,
                          codec_table** out);
CODEC_API void codec_table_free(codec_table* t);

typedef struct {
  int32_t n_tc_groups, n_gemv_groups, n_gen_groups;   /* per kernel */
  int32_t n_rows, n_slots, n_merge;                    /* rows, partial slots, merged requests */
  int32_t gemv_rows;                                   /* q-row capacity of a GEMV group */
  int32_t off_tc, off_gemv, off_gen, off_rows;         /* int32 offsets into the blob */
  int32_t off_merge_req, off_merge_ptr, off_merge_slot;
  int32_t h_local;                                     /* head_end - head_begin */
  int32_t n_tc_blocks, off_tc_block_ptr;               /* persistent TC CTA pairs, their (group, head) unit CSR */
  int32_t max_merge;                                   /* most partials of one merged (request, head) */
  int32_t n_merge_fused;                               /* further merge entries (after the n_merge) that the
                                                          suffix kernel folds into its own output */
  int32_t n_multi_groups, off_multi;                   /* lightly shared slices (2..32/g requests) on the
                                                          multi-request mma.sync kernel */
  int32_t off_entry_of;                                /* [bs][h_local] merge entry of (request, kv head), -1 none */
  int32_t n_tct_groups;                                /* slices of 2+ requests of nodes with <= 64 query-head rows (128 with TCT_WIDE)
                                                          on the transposed tensor-core kernel: records right
                                                          after the multi-request ones (off_multi + 8 n_multi_groups) */
  int32_t tct_ctas;                                    /* its grid (CTAs loop over the (group, kv head) items):
                                                          one per item unless CODEC_TCT_CTAS caps it */
  int32_t n_tct_wide;                                  /* the last n_tct_wide of those groups have 65..128 rows
                                                          (the wide variant; the others <= 64) */
  int32_t merge_np;                                    /* the merge kernel's all-loads-in-flight width (4, 8, 16):
                                                          holds 95 % of the entries */
  int32_t reserved3;
  int64_t blob_len;                                    /* int32 elements */
  int64_t workspace_bytes;                             /* partial (o, m, l) storage */
} codec_table_info;
CODEC_API int32_t codec_table_info_get(const codec_table* t, codec_table_info* info);
/* Copy the int32 blob to host memory (caller uploads it to the device). */
CODEC_API int32_t codec_table_copy(const codec_table* t, int32_t* blob);

/* ======================================================================
 * The decode-attention step.  Replaces execute()  executor.py:296-308
 * (split phase + barrier + per-request LSE reduction + finalize), with
 * _kernels.pac_kernel (_kernels.pyx:16-54) as the per-tile math.
 *
 *   q      [bs][h_q_local][d]            (q dtype = kv_dtype)
 *   k, v   [h_local][pool_tokens][d]     head-major node pool, nodes at
 *                                        their preorder offsets (kappa)
 *   out    [bs][h_q_local][d]            float32 for BF16/F32, float64 for F64
 *   workspace, workspace_bytes
 *          >= info.workspace_bytes (checked), 256-byte aligned: partial
 *          (o, m, l) storage, then a tail whose first int32 is the step's
 *          TC completion counter (reset and used inside each call; a
 *          workspace must not be shared by calls in flight)
 * All device pointers; asynchronous on `stream`. Every check runs before
 * the first enqueue: a non-OK status leaves stream, output and workspace
 * untouched.
 * ==================================================================== */
/* Per-kernel device times of the calls made with this timer (profiling):
 * CUDA events around each kernel on the launching stream. One ring of up
 * to 4096 calls per handle; a handle must not be shared across threads. */
typedef struct codec_kernel_timer codec_kernel_timer;
CODEC_API int32_t codec_timer_create(codec_kernel_timer** out);
CODEC_API void codec_timer_free(codec_kernel_timer* timer);
/* ms[3 i + k] = call i's TC kernel, suffix + generic kernels, merge kernel.
 * Synchronizes on the recorded events, then clears the ring. */
CODEC_API int32_t codec_timer_read(codec_kernel_timer* timer, float* ms, int32_t max_calls, int32_t* n_calls);

/* The step with the GEMV / generic kernels forked onto `aux_stream`
 * (event fork/join on `stream`) so they run concurrently with the
 * tensor-core kernel; aux_stream NULL: one stream. timer NULL: no events
 * (a timer also serialises the kernels: the events sit between them). */
CODEC_API int32_t codec_decode_attention_ex(const codec_dims* dims, const codec_table_info* info,
                                            const int32_t* table_dev, const void* q, const void* k,
                                            const void* v, void* out, void* workspace, int64_t workspace_bytes,
                                            void* stream, void* aux_stream, codec_kernel_timer* timer);
CODEC_API int32_t codec_decode_attention(const codec_dims* dims, const codec_table_info* info,
                                         const int32_t* table_dev, const void* q, const void* k, const void* v,
                                         void* out, void* workspace, int64_t workspace_bytes, void* stream);

/* ======================================================================
 * Fused multi-GPU output gather. Replaces the NCCL
 * all-gather of the per-rank outputs (parallel.all_gather_heads /
 * gather_requests): the merge kernel of rank `self` stores every output
 * row it produces straight into all n_peers ranks' global output buffers
 * (peer stores over NVLink / NVSwitch), at row row_map[r] (r when NULL),
 * q heads [head0, head0 + h_q_local) of hq_global; its last CTA then bumps
 * counter `self` in every rank's flag array (system-scope atomics, after a
 * system fence). codec_peer_wait makes a stream wait until all n_peers
 * counters of the local flag array reached the next step's value -- the
 * gathered output is then complete on this rank. The table must be built
 * with CODEC_FLAG_MERGE_ALL (bf16 KV, d = 128). Buffers come from
 * codec_ipc_alloc on each rank, peers' handles are opened with
 * codec_ipc_open (the handles travel over any side channel: gloo / NCCL
 * all_gather_object). `done` (device int32, zero before the first call)
 * counts the merge CTAs of a call and is reset by the last one.
 * ==================================================================== */
typedef struct {
  int32_t n_peers, self;       /* ranks in the gather, this rank */
  int32_t hq_global, head0;    /* q heads per row of the global buffer, this rank's first one */
  void* const* peer_out;       /* device [n_peers]: float32 [rows][hq_global][128] of every rank */
  int32_t* const* peer_flags;  /* device [n_peers]: int32 [n_peers] arrival counters of every rank */
  const int32_t* row_map;      /* device [bs]: global row of local request r, NULL = r */
  int32_t* done;               /* device int32: merge CTAs finished in the current call */
} codec_peer_gather;
CODEC_API int32_t codec_decode_attention_gather(const codec_dims* dims, const codec_table_info* info,
                                                const int32_t* table_dev, const void* q, const void* k,
                                                const void* v, void* workspace, int64_t workspace_bytes,
                                                void* stream, void* aux_stream, const codec_peer_gather* pg);
/* Wait (on `stream`) until every flags[p], p < n_peers, is >= *expected + 1,
 * then store *expected + 1 (device int32 step counter of this rank). */
CODEC_API int32_t codec_peer_wait(const int32_t* flags, int32_t n_peers, int32_t* expected, void* stream);
/* Symmetric buffers: a cudaMalloc allocation (zeroed) plus its 64-byte
 * CUDA IPC handle; open / close a peer's handle in this process. */
CODEC_API int32_t codec_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle64);
/* Make `device` the calling thread's current device inside the library.
 * The library links its own (static) CUDA runtime, so the host's
 * cudaSetDevice / torch.cuda.set_device does not necessarily reach it;
 * one process per GPU calls this once per thread before its first call
 * (the Python layer does it in DecodeStep / PeerGather). */
CODEC_API int32_t codec_bind_device(int32_t device);
CODEC_API int32_t codec_ipc_free(void* dev_ptr);
CODEC_API int32_t codec_ipc_open(const void* handle64, void** dev_ptr);
CODEC_API int32_t codec_ipc_close(void* dev_ptr);

/* Debug builds only (compiled with -DCODEC_HANG_CHECK): a device pointer to
 * host-mapped int32[8 + 8 * 1000]; a TC-kernel mbarrier wait that spins for
 * ~2^20 polls appends (block.x, block.y, thread, barrier SMEM address,
 * phase) there. Returns CODEC_ERR_VALUE in normal builds. */
CODEC_API int32_t codec_debug_hang_buffer(void* dev_ptr);

/* Copy the TC timeline recorded under CODEC_FLAG_TRACE: n <= 1792 clock64
 * values, trace[(event * 2 + q_tile) * 64 + tile], events: 0 MMA saw P,
 * 1 MMA issued PV+next S, 2 softmax saw S, 3 softmax released P, 4 softmax
 * finished the row-max exchange. Debug only. */
CODEC_API int32_t codec_debug_trace(long long* host, int64_t n);
/* Copy the CTA log recorded under CODEC_FLAG_CTALOG: 4 int64 per record,
   TC CTAs at records [0, 4096), GEMV CTAs (blockIdx.y * gridDim.x +
   blockIdx.x) from record 4096 (debug). */
CODEC_API int32_t codec_debug_ctalog(long long* host, int64_t n);
/* ======================================================================
 * Device primitives with the reference's argument meaning.
 * ==================================================================== */
/* pac_kernel()  _kernels.pyx:16-54 / attention.py:88-117.
 * q [n_q][h_q][d], k/v [n][h_kv][d] (token-major, the reference layout),
 * visible int64 [n_q] (device, each in 1..n; NULL = all n), scale (the
 * reference passes 1/sqrt(d)); out [n_q][h_q][d], max_score / exp_sum
 * [n_q][h_q]: float32 for F32/BF16 inputs, float64 for F64. */
CODEC_API int32_t codec_pac(int32_t dtype, const void* q, const void* k, const void* v,
                  const int64_t* visible, int64_t n_q, int64_t h_q, int64_t n, int64_t h_kv,
                  int64_t d, double scale, void* out, void* max_score, void* exp_sum,
                  void* stream);
/* por()  attention.py:131-153, elementwise part (the whole-side-empty
 * identity is resolved by the host wrapper). a/b/result (out, m, s) with
 * out [count][d], m/s [count]; dtype F32 or F64. */
CODEC_API int32_t codec_por(int32_t dtype, int64_t count, int64_t d, const void* a_out, const void* a_m,
                  const void* a_s, const void* b_out, const void* b_m, const void* b_s,
                  void* r_out, void* r_m, void* r_s, void* stream);

/* merge_schedule()  executor.py:86-111 (mode 0: balanced rounds over
 * sum(slices_per_node) partials) / sequential_schedule()  :114-117 (mode 1:
 * path_len = total, P-1 rounds of (0, i)). Writes the (left, right) label
 * pairs (2 per pair, up to cap pairs) and round_ptr[n_rounds + 1] when both
 * are non-NULL; *n_pairs / *n_rounds always. */
CODEC_API int32_t codec_merge_schedule(int32_t mode, int64_t path_len, const int64_t* slices_per_node,
                                       int64_t n_counts, int64_t* pairs, int64_t* round_ptr, int64_t cap,
                                       int64_t* n_pairs, int64_t* n_rounds);
/* reduce_tree()'s fold + finalize math  executor.py:209-293 on the device:
 * request i merges partial slots slot[ptr[i] .. ptr[i+1]) (device int32
 * CSR) of part_out [n_slots][h_q][d], part_m / part_s [n_slots][h_q] (the
 * PartialResult fields, F32 or F64) into out [n_req][h_q][d]; out_s
 * [n_req][h_q] receives the merged exp-sum (0 = no visible token). */
CODEC_API int32_t codec_merge_partials(int32_t dtype, int32_t n_req, int32_t h_q, int32_t d, const int32_t* ptr,
                                       const int32_t* slot, const void* part_out, const void* part_m,
                                       const void* part_s, void* out, void* out_s, void* stream);

/* Pack token-major node tensors [len][h_kv][d] into the head-major pool
 * [h_local][pool_tokens][d] at token offset `tok0` (heads
 * [head_begin, head_begin + h_local)). Device pointers, same dtype. */
CODEC_API int32_t codec_pool_pack(int32_t dtype, const void* src, int64_t len, int64_t h_kv, int64_t d,
                        int32_t head_begin, int32_t h_local, void* pool, int64_t pool_tokens,
                        int64_t tok0, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* CODEC_B200_H */
