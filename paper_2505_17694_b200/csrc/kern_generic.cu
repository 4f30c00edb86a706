// Generic split-attention kernel (any dtype in {f32, f64, bf16}, any
// head dim <= 512), the LSE merge primitive and the KV pool packer.
//
// This is the CUDA restatement of the reference's per-(query, head)
// split-attention math, _kernels.pyx:25-54 / _kernels_py.py:35-52:
// scores q.k * scale over the visible prefix, online softmax across
// token chunks, output normalised by the exp-sum, (m, s) kept so the
// partial is mergeable. It serves
//   * codec_pac(): the drop-in for _kernels.pac_kernel (token-major K/V,
//     the reference layout), and
//   * decode groups the specialised kernels do not cover (f64, odd d).
// One CTA per (unit, query head); a unit is a query row (pac) or a
// (subtask, request) group (decode).
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"

namespace codec {

constexpr int kGenThreads = 128;
constexpr int kGenChunk = 1024;  // scores staged per pass (tokens)
constexpr int kGenMaxD = 512;

template <typename A> __device__ A block_reduce(A v, A* red, bool is_max) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  A r = red[0];
  for (int i = 1; i < kGenThreads / 32; ++i) r = is_max ? max(r, red[i]) : r + red[i];
  return r;
}

// One query row against `vis` tokens: k/v row t at k + t * tok_stride.
// Writes out[0..d) = normalised output, *m_out = max score, *s_out = exp-sum.
template <typename T, typename O>
__device__ void pac_row(const T* __restrict__ q, const T* __restrict__ k, const T* __restrict__ v,
                        int64_t tok_stride, int vis, int d, typename AccOf<T>::type scale, O* __restrict__ out,
                        O* m_out, O* s_out) {
  using A = typename AccOf<T>::type;
  __shared__ A qs[kGenMaxD];
  __shared__ A sc[kGenChunk];
  __shared__ A red[kGenThreads / 32];
  const int tid = threadIdx.x;
  for (int e = tid; e < d; e += kGenThreads) qs[e] = (A)to_f(q[e]);
  constexpr int kDpt = kGenMaxD / kGenThreads;
  A acc[kDpt];
#pragma unroll
  for (int i = 0; i < kDpt; ++i) acc[i] = 0;
  A m = neg_inf<A>(), l = 0;
  __syncthreads();
  for (int c0 = 0; c0 < vis; c0 += kGenChunk) {
    const int cn = min(kGenChunk, vis - c0);
    A cmax = neg_inf<A>();
    for (int i = tid; i < cn; i += kGenThreads) {
      const T* kr = k + (int64_t)(c0 + i) * tok_stride;
      A dot = 0;
      for (int e = 0; e < d; ++e) dot += qs[e] * (A)to_f(kr[e]);
      dot *= scale;
      sc[i] = dot;
      cmax = max(cmax, dot);
    }
    cmax = block_reduce<A>(cmax, red, true);
    const A m_new = max(m, cmax);
    const A r = exp_acc(m - m_new);  // 0 on the first chunk (m = -inf)
    A part = 0;
    for (int i = tid; i < cn; i += kGenThreads) {
      A p = exp_acc(sc[i] - m_new);
      sc[i] = p;
      part += p;
    }
    part = block_reduce<A>(part, red, false);  // also orders the sc[] writes
    l = l * r + part;
#pragma unroll
    for (int j = 0; j < kDpt; ++j) {
      const int e = tid + j * kGenThreads;
      if (e < d) {
        A a = acc[j] * r;
        const T* vc = v + (int64_t)c0 * tok_stride + e;
        for (int i = 0; i < cn; ++i) a += sc[i] * (A)to_f(vc[(int64_t)i * tok_stride]);
        acc[j] = a;
      }
    }
    m = m_new;
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < kDpt; ++j) {
    const int e = tid + j * kGenThreads;
    if (e < d) out[e] = (O)(acc[j] / l);
  }
  if (tid == 0) {
    if (m_out) *m_out = (O)m;
    if (s_out) *s_out = (O)l;
  }
}

// --- codec_pac: q [n_q][h_q][d], k/v [n][h_kv][d], grid (n_q, h_q)
template <typename T, typename O>
__global__ void __launch_bounds__(kGenThreads) pac_api_kernel(const T* q, const T* k, const T* v,
                                                              const int64_t* visible, int n, int h_q, int h_kv,
                                                              int d, double scale, O* out, O* mo, O* so) {
  const int i = blockIdx.x, h = blockIdx.y;
  const int g = h_q / h_kv, kh = h / g;
  const int vis = visible ? (int)visible[i] : n;
  const int64_t row = (int64_t)i * h_q + h;
  pac_row<T, O>(q + row * d, k + (int64_t)kh * d, v + (int64_t)kh * d, (int64_t)h_kv * d, vis, d,
                (typename AccOf<T>::type)scale, out + row * d, mo + row, so + row);
}

// --- decode groups (1 request each), grid (n_groups, hq_local)
template <typename T, typename O>
__global__ void __launch_bounds__(kGenThreads) gen_decode_kernel(const int32_t* __restrict__ table, int off_groups,
                                                                 int off_rows, const T* q, const T* kpool,
                                                                 const T* vpool, int64_t pool_tokens, int d,
                                                                 int g, int hq_local, double scale, O* out,
                                                                 O* part_o, O* part_ml) {
  const int32_t* grp = table + off_groups + blockIdx.x * kGroupInts;
  const int qh = blockIdx.y, kh = qh / g;
  const int32_t* row = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  const int req = row[0], vis = row[1], slot = row[2];
  const int64_t kv0 = ((int64_t)kh * pool_tokens + grp[kGrpKvTok]) * d;
  const T* qp = q + ((int64_t)req * hq_local + qh) * d;
  if (slot < 0) {
    pac_row<T, O>(qp, kpool + kv0, vpool + kv0, d, vis, d, (typename AccOf<T>::type)scale,
                  out + ((int64_t)req * hq_local + qh) * d, (O*)nullptr, (O*)nullptr);
  } else {
    const int64_t e = (int64_t)slot * hq_local + qh;
    pac_row<T, O>(qp, kpool + kv0, vpool + kv0, d, vis, d, (typename AccOf<T>::type)scale, part_o + e * d,
                  part_ml + 2 * e, part_ml + 2 * e + 1);
  }
}

// --- POR elementwise (attention.py:131-153): entries with s == 0 are empty
template <typename A>
__global__ void por_kernel(int64_t count, int d, const A* ao, const A* am, const A* as, const A* bo, const A* bm,
                           const A* bs, A* ro, A* rm, A* rs) {
  const int64_t i = blockIdx.x;
  if (i >= count) return;
  const A sa = as[i], sb = bs[i];
  const A m = max(am[i], bm[i]);
  const A wa = sa > 0 ? sa * exp_acc(am[i] - m) : (A)0;
  const A wb = sb > 0 ? sb * exp_acc(bm[i] - m) : (A)0;
  const A s = wa + wb;
  const A den = s > 0 ? s : (A)1;
  for (int e = threadIdx.x; e < d; e += blockDim.x)
    ro[i * d + e] = s > 0 ? (ao[i * d + e] * wa + bo[i * d + e] * wb) / den : (A)0;
  if (threadIdx.x == 0) {
    rm[i] = s > 0 ? m : neg_inf<A>();
    rs[i] = s;
  }
}

// --- pool pack: src [len][h_kv][d] -> pool [h_local][T][d] at tok0
template <typename W>
__global__ void pool_pack_kernel(const W* src, int64_t len, int h_kv, int64_t dw, int head_begin, int h_local,
                                 W* pool, int64_t pool_tokens, int64_t tok0) {
  const int64_t total = len * h_local * dw;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t e = i % dw;
    const int64_t t = (i / dw) % len;
    const int64_t h = i / (dw * len);
    pool[(h * pool_tokens + tok0 + t) * dw + e] = src[(t * h_kv + head_begin + h) * dw + e];
  }
}

int32_t cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return CODEC_OK;
  return fail(CODEC_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

int32_t launch_generic_groups(int dtype, const int32_t* table, int n_groups, int off_groups, int off_rows,
                              const void* q, const void* k, const void* v, int64_t pool_tokens, int d, int g,
                              int hq_local, void* out, void* part_o, void* part_ml, cudaStream_t st) {
  if (n_groups == 0) return CODEC_OK;
  if (d > kGenMaxD) return fail(CODEC_ERR_UNSUPPORTED, "head dim %d > %d", d, kGenMaxD);
  dim3 grid(n_groups, hq_local);
  const double scale = 1.0 / sqrt((double)d);
  if (dtype == CODEC_F64)
    gen_decode_kernel<double, double><<<grid, kGenThreads, 0, st>>>(
        table, off_groups, off_rows, (const double*)q, (const double*)k, (const double*)v, pool_tokens, d, g,
        hq_local, scale, (double*)out, (double*)part_o, (double*)part_ml);
  else if (dtype == CODEC_F32)
    gen_decode_kernel<float, float><<<grid, kGenThreads, 0, st>>>(
        table, off_groups, off_rows, (const float*)q, (const float*)k, (const float*)v, pool_tokens, d, g,
        hq_local, scale, (float*)out, (float*)part_o, (float*)part_ml);
  else
    gen_decode_kernel<__nv_bfloat16, float><<<grid, kGenThreads, 0, st>>>(
        table, off_groups, off_rows, (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v,
        pool_tokens, d, g, hq_local, scale, (float*)out, (float*)part_o, (float*)part_ml);
  return cuda_status(cudaGetLastError(), "generic decode launch");
}

}  // namespace codec

using namespace codec;

extern "C" int32_t codec_pac(int32_t dtype, const void* q, const void* k, const void* v, const int64_t* visible,
                             int64_t n_q, int64_t h_q, int64_t n, int64_t h_kv, int64_t d, double scale, void* out,
                             void* max_score, void* exp_sum, void* stream) {
  if (n_q < 1 || n < 1 || d < 1 || h_kv < 1 || h_q % h_kv != 0)
    return fail(CODEC_ERR_DIMENSION_MISMATCH, "bad pac shape n_q=%lld h_q=%lld n=%lld h_kv=%lld d=%lld",
                (long long)n_q, (long long)h_q, (long long)n, (long long)h_kv, (long long)d);
  if (d > kGenMaxD) return fail(CODEC_ERR_UNSUPPORTED, "head dim %lld > %d", (long long)d, kGenMaxD);
  if (n_q > 0x7fffffff || h_q > 65535) return fail(CODEC_ERR_UNSUPPORTED, "pac grid too large");
  cudaStream_t st = (cudaStream_t)stream;
  dim3 grid((unsigned)n_q, (unsigned)h_q);
  if (dtype == CODEC_F64)
    pac_api_kernel<double, double><<<grid, kGenThreads, 0, st>>>((const double*)q, (const double*)k,
                                                                  (const double*)v, visible, (int)n, (int)h_q,
                                                                  (int)h_kv, (int)d, scale, (double*)out,
                                                                  (double*)max_score, (double*)exp_sum);
  else if (dtype == CODEC_F32)
    pac_api_kernel<float, float><<<grid, kGenThreads, 0, st>>>((const float*)q, (const float*)k, (const float*)v,
                                                                visible, (int)n, (int)h_q, (int)h_kv, (int)d,
                                                                scale, (float*)out, (float*)max_score,
                                                                (float*)exp_sum);
  else if (dtype == CODEC_BF16)
    pac_api_kernel<__nv_bfloat16, float><<<grid, kGenThreads, 0, st>>>(
        (const __nv_bfloat16*)q, (const __nv_bfloat16*)k, (const __nv_bfloat16*)v, visible, (int)n, (int)h_q,
        (int)h_kv, (int)d, scale, (float*)out, (float*)max_score, (float*)exp_sum);
  else
    return fail(CODEC_ERR_UNSUPPORTED, "dtype %d", dtype);
  return cuda_status(cudaGetLastError(), "pac launch");
}

extern "C" int32_t codec_por(int32_t dtype, int64_t count, int64_t d, const void* a_out, const void* a_m,
                             const void* a_s, const void* b_out, const void* b_m, const void* b_s, void* r_out,
                             void* r_m, void* r_s, void* stream) {
  if (count < 1) return CODEC_OK;
  cudaStream_t st = (cudaStream_t)stream;
  if (dtype == CODEC_F64)
    por_kernel<double><<<(unsigned)count, 128, 0, st>>>(count, (int)d, (const double*)a_out, (const double*)a_m,
                                                        (const double*)a_s, (const double*)b_out,
                                                        (const double*)b_m, (const double*)b_s, (double*)r_out,
                                                        (double*)r_m, (double*)r_s);
  else if (dtype == CODEC_F32)
    por_kernel<float><<<(unsigned)count, 128, 0, st>>>(count, (int)d, (const float*)a_out, (const float*)a_m,
                                                       (const float*)a_s, (const float*)b_out, (const float*)b_m,
                                                       (const float*)b_s, (float*)r_out, (float*)r_m,
                                                       (float*)r_s);
  else
    return fail(CODEC_ERR_UNSUPPORTED, "por dtype %d", dtype);
  return cuda_status(cudaGetLastError(), "por launch");
}

extern "C" int32_t codec_pool_pack(int32_t dtype, const void* src, int64_t len, int64_t h_kv, int64_t d,
                                   int32_t head_begin, int32_t h_local, void* pool, int64_t pool_tokens,
                                   int64_t tok0, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const int64_t total = len * h_local * d;
  if (total == 0) return CODEC_OK;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  if (dtype == CODEC_F64)
    pool_pack_kernel<uint64_t><<<blocks, 256, 0, st>>>((const uint64_t*)src, len, (int)h_kv, d, head_begin, h_local,
                                                       (uint64_t*)pool, pool_tokens, tok0);
  else if (dtype == CODEC_F32)
    pool_pack_kernel<uint32_t><<<blocks, 256, 0, st>>>((const uint32_t*)src, len, (int)h_kv, d, head_begin, h_local,
                                                       (uint32_t*)pool, pool_tokens, tok0);
  else
    pool_pack_kernel<uint16_t><<<blocks, 256, 0, st>>>((const uint16_t*)src, len, (int)h_kv, d, head_begin, h_local,
                                                       (uint16_t*)pool, pool_tokens, tok0);
  return cuda_status(cudaGetLastError(), "pool pack launch");
}
