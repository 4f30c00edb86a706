// codec_decode_attention(): one decode-attention step over a device task
// table -- the B200 replacement of execute() (executor.py:296-308).
//
// Launch order on the caller's stream: tensor-core groups (shared nodes),
// GEMV groups (unshared suffixes), generic groups, then the LSE merge of
// requests with more than one partial (the reference's barrier +
// reduce_tree, executor.py:177-179, :267-293). Requests with a single
// partial were written straight to `out` by their split kernel.
#include <cuda_runtime.h>
#include <string.h>

#include "common.h"
#include "device_table.h"

namespace codec {
int32_t launch_tc(const int32_t* table, const codec_table_info& in, const void* q, const void* k, const void* v,
                  int64_t pool_tokens, int g, int h_local, int bs, void* out, void* part_o, void* part_ml,
                  cudaStream_t st, int flags, long long* ctalog, const int32_t* page_table, int page_shift,
                  int32_t* tc_done, const int32_t* entry_of, int32_t* cnt);
int32_t read_trace(long long* host, int64_t n);
int32_t set_hang_buffer(void* dev_ptr);
int32_t launch_gemv(int dtype, int d, int rows, const int32_t* table, int n_groups, int off_groups, int off_rows,
                    const void* q, const void* k, const void* v, int64_t pool_tokens, int g, int h_local,
                    void* out, void* part_o, void* part_ml, cudaStream_t st, long long* ctalog);
int32_t launch_mma_gemv(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q,
                        const void* k, const void* v, int64_t pool_tokens, int g, int h_local, void* out,
                        void* part_o, void* part_ml, int off_merge_ptr, int off_merge_slot, cudaStream_t st,
                        long long* ctalog, bool after_tc, const int32_t* page_table, int page_shift,
                        const int32_t* entry_of, int32_t* cnt);
int32_t launch_mma_multi(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q,
                         const void* k, const void* v, int64_t pool_tokens, int g, int h_local, void* out,
                         void* part_o, void* part_ml, cudaStream_t st, bool pdl, const int32_t* page_table,
                         int page_shift, int32_t* done, const int32_t* entry_of, int32_t* cnt);
int32_t launch_tct(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q, const void* k,
                   const void* v, int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                   cudaStream_t st, bool pdl, const int32_t* page_table, int page_shift, int32_t* done,
                   const int32_t* entry_of, int32_t* cnt, int max_ctas, int n_wide);
int32_t launch_generic_groups(int dtype, const int32_t* table, int n_groups, int off_groups, int off_rows,
                              const void* q, const void* k, const void* v, int64_t pool_tokens, int d, int g,
                              int hq_local, void* out, void* part_o, void* part_ml, cudaStream_t st);
int32_t launch_merge(int dtype, const int32_t* table, const codec_table_info& in, int d, int hq_local,
                     const void* part_o, const void* part_ml, void* out, cudaStream_t st, const int32_t* tc_done,
                     int tc_ctas, bool pdl, const int32_t* cnt, const codec_peer_gather* gather);
int32_t cuda_status(cudaError_t e, const char* what);
}  // namespace codec

using namespace codec;

namespace {
// Per-thread, per-device fork/join events for the aux-stream variant.
struct ForkJoin {
  int device = -1;
  cudaEvent_t fork = nullptr, join = nullptr;
};
int32_t fork_join_events(ForkJoin*& out) {
  thread_local ForkJoin slots[16];
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return codec::cuda_status(e, "cudaGetDevice");
  ForkJoin& fj = slots[dev & 15];
  if (fj.device != dev) {
    if (cudaEventCreateWithFlags(&fj.fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&fj.join, cudaEventDisableTiming) != cudaSuccess)
      return codec::fail(CODEC_ERR_CUDA, "event creation failed");
    fj.device = dev;
  }
  out = &fj;
  return CODEC_OK;
}
}  // namespace

namespace {
long long* g_ctalog = nullptr;  // debug CTA log (CODEC_FLAG_CTALOG), one per process
}

// Per-kernel timing (codec_kernel_timer, ABI v4): CUDA events around each
// kernel of a call on the caller's stream, so a benchmark can time every
// kernel inside its own timed region. One ring per handle -- nothing
// process-global on this path; a handle must not be shared by threads.
constexpr int kEvCalls = 4096;
struct codec_kernel_timer {
  cudaEvent_t ev[kEvCalls][4] = {};
  int n = 0;
};

namespace {
int32_t kev_record(codec_kernel_timer* tm, int slot, cudaStream_t st) {
  if (tm->n >= kEvCalls) return CODEC_OK;  // ring full: drop
  cudaEvent_t& e = tm->ev[tm->n][slot];
  if (!e && cudaEventCreate(&e) != cudaSuccess) return fail(CODEC_ERR_CUDA, "event create");
  if (cudaEventRecord(e, st) != cudaSuccess) return fail(CODEC_ERR_CUDA, "event record");
  return CODEC_OK;
}
}  // namespace

extern "C" int32_t codec_timer_create(codec_kernel_timer** out) {
  if (!out) return fail(CODEC_ERR_VALUE, "NULL argument");
  *out = new codec_kernel_timer();
  return CODEC_OK;
}

extern "C" void codec_timer_free(codec_kernel_timer* tm) {
  if (!tm) return;
  for (auto& call : tm->ev)
    for (auto& e : call)
      if (e) cudaEventDestroy(e);
  delete tm;
}

extern "C" int32_t codec_timer_read(codec_kernel_timer* tm, float* ms, int32_t max_calls, int32_t* n_calls) {
  if (!tm || !ms || !n_calls) return fail(CODEC_ERR_VALUE, "NULL argument");
  const int n = tm->n < max_calls ? tm->n : max_calls;
  for (int i = 0; i < n; ++i)
    for (int k = 0; k < 3; ++k) {
      float t = 0.f;
      if (cudaEventSynchronize(tm->ev[i][k + 1]) != cudaSuccess ||
          cudaEventElapsedTime(&t, tm->ev[i][k], tm->ev[i][k + 1]) != cudaSuccess)
        return fail(CODEC_ERR_CUDA, "event read");
      ms[3 * i + k] = t;
    }
  *n_calls = n;
  tm->n = 0;
  return CODEC_OK;
}

extern "C" int32_t codec_debug_ctalog(long long* host, int64_t n) {
  if (!g_ctalog) return fail(CODEC_ERR_VALUE, "no CTA log recorded");
  if (n > 4 * (int64_t)kCtaLogLen) n = 4 * (int64_t)kCtaLogLen;
  return codec::cuda_status(cudaMemcpy(host, g_ctalog, n * sizeof(long long), cudaMemcpyDeviceToHost), "ctalog copy");
}

static int32_t decode_impl(const codec_dims* dims, const codec_table_info* info, const int32_t* table_dev,
                           const void* q, const void* k, const void* v, void* out, void* workspace,
                           int64_t workspace_bytes, void* stream, void* aux_stream, codec_kernel_timer* timer,
                           const codec_peer_gather* gather) {
  // ---- every argument / eligibility check before the first enqueue: an
  // error leaves the stream, the output and the workspace untouched
  if (!dims || !info || !table_dev) return fail(CODEC_ERR_VALUE, "NULL argument");
  if (!q || !k || !v || !out || !workspace) return fail(CODEC_ERR_VALUE, "NULL device buffer");
  if (workspace_bytes < info->workspace_bytes)
    return fail(CODEC_ERR_VALUE, "workspace of %lld bytes, the table needs %lld", (long long)workspace_bytes,
                (long long)info->workspace_bytes);
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(CODEC_ERR_VALUE, "workspace must be 256-byte aligned");
  if ((reinterpret_cast<uintptr_t>(k) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) ||
      (reinterpret_cast<uintptr_t>(q) & 15))
    return fail(CODEC_ERR_VALUE, "q, k and v must be 16-byte aligned");
  if (dims->h_kv < 1 || dims->h_q % dims->h_kv != 0 || info->h_local != dims->head_end - dims->head_begin)
    return fail(CODEC_ERR_DIMENSION_MISMATCH, "dims do not match the table (h_q %d, h_kv %d, shard [%d, %d), "
                "table heads %d)", dims->h_q, dims->h_kv, dims->head_begin, dims->head_end, info->h_local);
  cudaStream_t st = (cudaStream_t)stream;
  const int g = dims->h_q / dims->h_kv;
  int page_shift = 0;
  if (dims->page_size) {
    if (dims->page_size < 128 || (dims->page_size & (dims->page_size - 1)) || !dims->page_table)
      return fail(CODEC_ERR_VALUE, "page_size %d must be a power of two >= 128 with a page table", dims->page_size);
    while ((1 << page_shift) < dims->page_size) ++page_shift;
  }
  const int h_local = info->h_local, hq_local = h_local * g, d = dims->d;
  const int64_t elem = dims->kv_dtype == CODEC_F64 ? 8 : 4;
  int64_t o_bytes = (int64_t)info->n_slots * hq_local * d * elem;
  o_bytes = (o_bytes + 255) / 256 * 256;
  void* part_o = workspace;
  void* part_ml = static_cast<uint8_t*>(workspace) + o_bytes;
  const bool do_tc = info->n_tc_groups && !(dims->flags & CODEC_FLAG_SKIP_TC);
  const bool do_gemv = info->n_gemv_groups && !(dims->flags & CODEC_FLAG_SKIP_GEMV);
  const bool do_gen = info->n_gen_groups && !(dims->flags & CODEC_FLAG_SKIP_GENERIC);
  const bool do_multi = info->n_multi_groups && !(dims->flags & CODEC_FLAG_SKIP_GEMV);
  const bool do_tct = info->n_tct_groups && !(dims->flags & CODEC_FLAG_SKIP_GEMV);
  if ((do_tc || do_multi || do_tct) && (dims->kv_dtype != CODEC_BF16 || d != 128 || g > 128))
    return fail(CODEC_ERR_UNSUPPORTED, "tensor-core / multi-request groups need bf16, d = 128");
  if (do_multi && g > 8) return fail(CODEC_ERR_UNSUPPORTED, "multi-request groups need <= 8 query heads per kv head");
  // The mma.sync suffix kernel is launched right after the TC kernel on the
  // same stream with programmatic dependent launch: its CTAs start on the
  // SMs the TC grid leaves once every TC CTA is resident (the TC grid gets
  // its SMs first; nothing co-resides with a TC CTA, which holds the SM's
  // whole register file and ~227 KB of SMEM). The merge, launched after the
  // suffix kernel, may then start before the TC grid finished, so it waits
  // for the TC CTAs' completion counter in the workspace (zeroed before the
  // TC launch, bumped by every TC CTA after its last write). The CUDA-core
  // GEMV / generic kernels fork onto the aux stream and join before the
  // merge.
  const bool mma_gemv = do_gemv && dims->kv_dtype == CODEC_BF16 && d == 128 && g <= 8 &&
                        !(dims->flags & CODEC_FLAG_GEMV_SIMT);
  if (do_gemv && !mma_gemv && page_shift)
    return fail(CODEC_ERR_UNSUPPORTED, "paged KV: suffix groups need the mma.sync kernel (bf16, d = 128, g <= 8)");
  if (do_gemv && !mma_gemv && info->gemv_rows != 4 && info->gemv_rows != 8)
    return fail(CODEC_ERR_UNSUPPORTED, "GEMV kernel: %d query-head rows per group", info->gemv_rows);
  if (do_gen && page_shift) return fail(CODEC_ERR_UNSUPPORTED, "paged KV: no generic-kernel groups");
  if (d > 512) return fail(CODEC_ERR_UNSUPPORTED, "head dim %d > 512", d);
  const bool fork = aux_stream != nullptr && do_tc && ((do_gemv && !mma_gemv) || do_gen);
  cudaStream_t side = fork ? (cudaStream_t)aux_stream : st;
  long long* ctalog = nullptr;
  if (dims->flags & CODEC_FLAG_CTALOG) {  // debug builds of a timeline: one process-global buffer
    if (!g_ctalog && cudaMalloc(&g_ctalog, 4 * sizeof(long long) * kCtaLogLen) != cudaSuccess)
      return fail(CODEC_ERR_CUDA, "ctalog alloc");
    ctalog = g_ctalog;
  }
  ForkJoin* fj = nullptr;
  if (fork) CODEC_TRY(fork_join_events(fj));
  const bool kev = timer != nullptr && !fork;

  // ---- enqueue
  if (ctalog && cudaMemsetAsync(g_ctalog, 0, 4 * sizeof(long long) * kCtaLogLen, st) != cudaSuccess)
    return fail(CODEC_ERR_CUDA, "ctalog clear");
  if (fork) {
    if (cudaEventRecord(fj->fork, st) != cudaSuccess || cudaStreamWaitEvent(side, fj->fork, 0) != cudaSuccess)
      return fail(CODEC_ERR_CUDA, "fork failed");
  }
  // completion counter of the TC and multi-request CTAs (the merge may
  // start before those grids end): the first word of the workspace tail
  int64_t ml_bytes = (int64_t)info->n_slots * hq_local * 2 * elem;
  ml_bytes = (ml_bytes + 255) / 256 * 256;
  int32_t* tc_done = reinterpret_cast<int32_t*>(static_cast<uint8_t*>(workspace) + o_bytes + ml_bytes);
  const int done_target = (do_tc ? 2 * info->n_tc_blocks : 0) + (do_multi ? info->n_multi_groups * h_local : 0) +
                          (do_tct ? info->n_tct_groups * h_local : 0);
  // early (programmatic) launches of the kernels after the TC kernel; not
  // with the fused merge, which reads the TC partials from the suffix kernel
  const bool early = info->n_merge_fused == 0 && !kev;
  const bool pdl = mma_gemv && (do_tc || do_multi || do_tct) && early;
  // Counted merge (opt-in): every partial producer (TC epilogue rows, mma.sync
  // suffix / multi CTAs) bumps its merge entry's counter after its stores,
  // and each merge CTA starts as soon as its entry is complete -- the merge
  // overlaps the other kernels' tail. Only when all producers are those
  // kernels (no CUDA-core GEMV / generic groups, no fused merge, the
  // merge128 kernel) and nothing is skipped.
  const int n_entries = info->n_merge + info->n_merge_fused;
  const bool counted = (dims->flags & CODEC_FLAG_COUNTED_MERGE) && info->n_merge > 0 && dims->kv_dtype == CODEC_BF16 &&
                       d == 128 &&
                       !do_gen && (!do_gemv || mma_gemv) && info->n_merge_fused == 0 &&
                       !(dims->flags & (CODEC_FLAG_SKIP_TC | CODEC_FLAG_SKIP_GEMV | CODEC_FLAG_SKIP_GENERIC));
  int32_t* cnt = counted ? tc_done + 64 : nullptr;  // the tail's 256-byte block, then the counters
  const int32_t* entry_of = table_dev + info->off_entry_of;
  const size_t tail_bytes = 256 + (counted ? (size_t)n_entries * 4 : 0);
  if ((done_target || counted) && cudaMemsetAsync(tc_done, 0, tail_bytes, st) != cudaSuccess)
    return fail(CODEC_ERR_CUDA, "tc counter reset");
  if (kev) CODEC_TRY(kev_record(timer, 0, st));
  if (do_tc)
    CODEC_TRY(launch_tc(table_dev, *info, q, k, v, dims->pool_tokens, g, h_local, dims->bs, out, part_o, part_ml, st,
                        dims->flags, ctalog, dims->page_table, page_shift, tc_done, entry_of, cnt));
  if (kev) CODEC_TRY(kev_record(timer, 1, st));
  // the transposed tensor-core kernel first: its CTAs are the longest of the
  // SMs the TC grid leaves (one per SM), the mma.sync grids fill in after
  if (do_tct)
    CODEC_TRY(launch_tct(table_dev, info->n_tct_groups, info->off_multi + kGroupInts * info->n_multi_groups,
                         info->off_rows, q, k, v, dims->pool_tokens, g, h_local, out, part_o, part_ml, st,
                         do_tc && early, dims->page_table, page_shift, tc_done, entry_of, cnt, info->tct_ctas,
                         info->n_tct_wide));
  if (do_multi)
    CODEC_TRY(launch_mma_multi(table_dev, info->n_multi_groups, info->off_multi, info->off_rows, q, k, v,
                               dims->pool_tokens, g, h_local, out, part_o, part_ml, st, (do_tc || do_tct) && early,
                               dims->page_table, page_shift, tc_done, entry_of, cnt));
  if (mma_gemv)
    CODEC_TRY(launch_mma_gemv(table_dev, info->n_gemv_groups, info->off_gemv, info->off_rows, q, k, v,
                              dims->pool_tokens, g, h_local, out, part_o, part_ml, info->off_merge_ptr,
                              info->off_merge_slot, st, ctalog, pdl, dims->page_table, page_shift, entry_of, cnt));
  else if (do_gemv)
    CODEC_TRY(launch_gemv(dims->kv_dtype, d, info->gemv_rows, table_dev, info->n_gemv_groups, info->off_gemv,
                          info->off_rows, q, k, v, dims->pool_tokens, g, h_local, out, part_o, part_ml, side,
                          ctalog));
  if (kev) CODEC_TRY(kev_record(timer, 2, st));
  if (do_gen)
    CODEC_TRY(launch_generic_groups(dims->kv_dtype, table_dev, info->n_gen_groups, info->off_gen, info->off_rows, q,
                                    k, v, dims->pool_tokens, d, g, hq_local, out, part_o, part_ml, side));
  if (fork) {
    if (cudaEventRecord(fj->join, side) != cudaSuccess || cudaStreamWaitEvent(st, fj->join, 0) != cudaSuccess)
      return fail(CODEC_ERR_CUDA, "join failed");
  }
  if (!(dims->flags & CODEC_FLAG_SKIP_MERGE))
    CODEC_TRY(launch_merge(dims->kv_dtype, table_dev, *info, d, hq_local, part_o, part_ml, out, st,
                           done_target ? tc_done : nullptr, done_target,
                           (mma_gemv || do_multi || do_tct || counted) && !fork && !kev &&
                               !(dims->flags & CODEC_FLAG_SKIP_GEMV) && !(dims->flags & CODEC_FLAG_MERGE_NO_PDL),
                           cnt, gather));
  if (kev) {
    CODEC_TRY(kev_record(timer, 3, st));
    ++timer->n;
  }
  return CODEC_OK;
}

extern "C" int32_t codec_decode_attention_ex(const codec_dims* dims, const codec_table_info* info,
                                             const int32_t* table_dev, const void* q, const void* k, const void* v,
                                             void* out, void* workspace, int64_t workspace_bytes, void* stream,
                                             void* aux_stream, codec_kernel_timer* timer) {
  return decode_impl(dims, info, table_dev, q, k, v, out, workspace, workspace_bytes, stream, aux_stream, timer,
                     nullptr);
}

// ---------------------------------------------------------------- fused gather
extern "C" int32_t codec_decode_attention_gather(const codec_dims* dims, const codec_table_info* info,
                                                 const int32_t* table_dev, const void* q, const void* k,
                                                 const void* v, void* workspace, int64_t workspace_bytes,
                                                 void* stream, void* aux_stream, const codec_peer_gather* pg) {
  if (!dims || !info || !pg) return fail(CODEC_ERR_VALUE, "NULL argument");
  if (!(dims->flags & CODEC_FLAG_MERGE_ALL))
    return fail(CODEC_ERR_VALUE, "the fused gather needs a table built with CODEC_FLAG_MERGE_ALL");
  if (dims->flags & (CODEC_FLAG_SKIP_MERGE | CODEC_FLAG_FUSED_MERGE | CODEC_FLAG_COUNTED_MERGE))
    return fail(CODEC_ERR_VALUE, "the fused gather needs the plain merge kernel");
  if (dims->kv_dtype != CODEC_BF16 || dims->d != 128)
    return fail(CODEC_ERR_UNSUPPORTED, "the fused gather needs bf16 KV and d = 128");
  if (pg->n_peers < 1 || pg->self < 0 || pg->self >= pg->n_peers || !pg->peer_out || !pg->peer_flags || !pg->done)
    return fail(CODEC_ERR_VALUE, "bad peer gather (%d peers, self %d)", pg->n_peers, pg->self);
  const int g = dims->h_kv > 0 ? dims->h_q / dims->h_kv : 0;
  const int hq_local = info->h_local * g;
  if (pg->head0 < 0 || pg->head0 + hq_local > pg->hq_global)
    return fail(CODEC_ERR_DIMENSION_MISMATCH, "q heads [%d, %d) outside the %d of the gathered rows", pg->head0,
                pg->head0 + hq_local, pg->hq_global);
  if (info->n_merge == 0) return fail(CODEC_ERR_VALUE, "the fused gather needs merge entries");
  // the split kernels write no output rows (MERGE_ALL): any non-NULL
  // pointer satisfies their signature
  return decode_impl(dims, info, table_dev, q, k, v, workspace, workspace, workspace_bytes, stream, aux_stream, nullptr,
                     pg);
}

namespace {
__global__ void peer_wait_kernel(const int32_t* flags, int n_peers, int32_t* expected) {
  const int32_t want = *expected + 1;
  for (int p = 0; p < n_peers; ++p) {
    int v;
    for (long long it = 0;; ++it) {
      asm volatile("ld.acquire.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(flags + p) : "memory");
      if (v >= want) break;
      if (it > (1ll << 26)) __trap();  // a peer that never arrives: trap rather than hang the GPU
      __nanosleep(200);
    }
  }
  *expected = want;
  __threadfence();
}
}  // namespace

extern "C" int32_t codec_peer_wait(const int32_t* flags, int32_t n_peers, int32_t* expected, void* stream) {
  if (!flags || !expected || n_peers < 1) return fail(CODEC_ERR_VALUE, "bad peer wait arguments");
  peer_wait_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(flags, n_peers, expected);
  return cuda_status(cudaGetLastError(), "peer wait launch");
}

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "codec_ipc_* pass 64-byte handles");
extern "C" int32_t codec_ipc_alloc(int64_t bytes, void** dev_ptr, void* handle64) {
  if (bytes <= 0 || !dev_ptr || !handle64) return fail(CODEC_ERR_VALUE, "bad ipc alloc arguments");
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, (size_t)bytes);
  if (e != cudaSuccess) return cuda_status(e, "ipc alloc");
  e = cudaMemset(p, 0, (size_t)bytes);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t*>(handle64), p);
  if (e != cudaSuccess) {
    cudaFree(p);
    return cuda_status(e, "ipc handle");
  }
  *dev_ptr = p;
  return CODEC_OK;
}
extern "C" int32_t codec_bind_device(int32_t device) {
  int cur = -1;
  if (device < 0) return fail(CODEC_ERR_VALUE, "bad device");
  if (cudaGetDevice(&cur) == cudaSuccess && cur == device) return CODEC_OK;
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) cudaGetLastError();  // not sticky: later launch checks must not see it
  return cuda_status(e, "cudaSetDevice");
}
extern "C" int32_t codec_ipc_free(void* dev_ptr) { return cuda_status(cudaFree(dev_ptr), "ipc free"); }
extern "C" int32_t codec_ipc_open(const void* handle64, void** dev_ptr) {
  if (!handle64 || !dev_ptr) return fail(CODEC_ERR_VALUE, "bad ipc open arguments");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle64, sizeof(h));
  return cuda_status(cudaIpcOpenMemHandle(dev_ptr, h, cudaIpcMemLazyEnablePeerAccess), "ipc open");
}
extern "C" int32_t codec_ipc_close(void* dev_ptr) { return cuda_status(cudaIpcCloseMemHandle(dev_ptr), "ipc close"); }

extern "C" int32_t codec_decode_attention(const codec_dims* dims, const codec_table_info* info,
                                          const int32_t* table_dev, const void* q, const void* k, const void* v,
                                          void* out, void* workspace, int64_t workspace_bytes, void* stream) {
  return codec_decode_attention_ex(dims, info, table_dev, q, k, v, out, workspace, workspace_bytes, stream, nullptr,
                                   nullptr);
}

extern "C" int32_t codec_debug_trace(long long* host, int64_t n) { return read_trace(host, n); }

// debug builds (CODEC_NVCC_EXTRA=-DCODEC_HANG_CHECK): where TC waits spin too long
extern "C" CODEC_API int32_t codec_debug_hang_buffer(void* dev_ptr) { return set_hang_buffer(dev_ptr); }
