// codec_decode_attention(): one decode-attention step over a device task
// table -- the B200 replacement of execute() (executor.py:296-308).
//
// Launch order on the caller's stream: tensor-core groups (shared nodes),
// GEMV groups (unshared suffixes), generic groups, then the LSE merge of
// requests with more than one partial (the reference's barrier +
// reduce_tree, executor.py:177-179, :267-293). Requests with a single
// partial were written straight to `out` by their split kernel.
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"

namespace codec {
int32_t launch_tc(const int32_t* table, const codec_table_info& in, const void* q, const void* k, const void* v,
                  int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                  cudaStream_t st);
int32_t launch_gemv(int dtype, int d, int rows, const int32_t* table, int n_groups, int off_groups, int off_rows,
                    const void* q, const void* k, const void* v, int64_t pool_tokens, int g, int h_local,
                    void* out, void* part_o, void* part_ml, cudaStream_t st);
int32_t launch_generic_groups(int dtype, const int32_t* table, int n_groups, int off_groups, int off_rows,
                              const void* q, const void* k, const void* v, int64_t pool_tokens, int d, int g,
                              int hq_local, void* out, void* part_o, void* part_ml, cudaStream_t st);
int32_t launch_merge(int dtype, const int32_t* table, const codec_table_info& in, int d, int hq_local,
                     const void* part_o, const void* part_ml, void* out, cudaStream_t st);
}  // namespace codec

using namespace codec;

extern "C" int32_t codec_decode_attention(const codec_dims* dims, const codec_table_info* info,
                                          const int32_t* table_dev, const void* q, const void* k, const void* v,
                                          void* out, void* workspace, void* stream) {
  if (!dims || !info || !table_dev) return fail(CODEC_ERR_VALUE, "NULL argument");
  if ((reinterpret_cast<uintptr_t>(workspace) & 255) != 0)
    return fail(CODEC_ERR_VALUE, "workspace must be 256-byte aligned");
  if ((reinterpret_cast<uintptr_t>(k) & 15) || (reinterpret_cast<uintptr_t>(v) & 15) ||
      (reinterpret_cast<uintptr_t>(q) & 15))
    return fail(CODEC_ERR_VALUE, "q, k and v must be 16-byte aligned");
  cudaStream_t st = (cudaStream_t)stream;
  const int g = dims->h_q / dims->h_kv;
  const int h_local = info->h_local, hq_local = h_local * g, d = dims->d;
  const int64_t elem = dims->kv_dtype == CODEC_F64 ? 8 : 4;
  int64_t o_bytes = (int64_t)info->n_slots * hq_local * d * elem;
  o_bytes = (o_bytes + 255) / 256 * 256;
  void* part_o = workspace;
  void* part_ml = static_cast<uint8_t*>(workspace) + o_bytes;
  if (info->n_tc_groups && !(dims->flags & CODEC_FLAG_SKIP_TC))
    CODEC_TRY(launch_tc(table_dev, *info, q, k, v, dims->pool_tokens, g, h_local, out, part_o, part_ml, st));
  if (info->n_gemv_groups && !(dims->flags & CODEC_FLAG_SKIP_GEMV))
    CODEC_TRY(launch_gemv(dims->kv_dtype, d, info->gemv_rows, table_dev, info->n_gemv_groups, info->off_gemv,
                          info->off_rows, q, k, v, dims->pool_tokens, g, h_local, out, part_o, part_ml, st));
  if (info->n_gen_groups && !(dims->flags & CODEC_FLAG_SKIP_GENERIC))
    CODEC_TRY(launch_generic_groups(dims->kv_dtype, table_dev, info->n_gen_groups, info->off_gen, info->off_rows, q,
                                    k, v, dims->pool_tokens, d, g, hq_local, out, part_o, part_ml, st));
  if (!(dims->flags & CODEC_FLAG_SKIP_MERGE))
    CODEC_TRY(launch_merge(dims->kv_dtype, table_dev, *info, d, hq_local, part_o, part_ml, out, st));
  return CODEC_OK;
}
