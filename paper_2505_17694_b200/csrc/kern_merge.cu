// K4: per-request log-sum-exp merge of split partials.
//
// Replaces reduce_tree()/_reduce_one() + por() + finalize()
// (executor.py:209-293, attention.py:131-161). For each request with two
// or more partials (its path-then-slice list from the task table) and
// each local query head:
//     M = max_p m_p,  L = sum_p s_p e^(m_p - M),
//     out = sum_p out_p s_p e^(m_p - M) / L
// which equals the reference's balanced pairwise por() fold up to
// rounding (the merge is associative/commutative in exact arithmetic,
// test_attention.py:160-180) but takes one pass over the partials.
// A merge entry is (request, local kv head): stream-K cuts the shared nodes
// per head, so the partial lists differ between heads. One warp per
// (entry, query head of that kv head); lanes cover the head dim.
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"

namespace codec {

// The TC grid may still be finishing when the merge starts (the suffix
// kernel before it was a programmatic dependent launch): wait until every
// TC CTA bumped the completion counter.
__device__ __forceinline__ void wait_tc_done(const int32_t* tc_done, int tc_ctas) {
  // launched as a programmatic dependent of the suffix kernel: wait for its
  // completion (and memory) first; a no-op for a plain launch
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (!tc_done) return;
  if (threadIdx.x == 0) {
    // bounded: the TC grid is resident and finishing (it was launched
    // before this kernel); a count that never arrives is a bug, and a trap
    // beats a hung GPU (~4 s of polling)
    int v;
    for (int it = 0;; ++it) {
      asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(tc_done) : "memory");
      if (v >= tc_ctas) break;
      if (it > (1 << 24)) __trap();
      __nanosleep(256);
    }
  }
  __syncthreads();
}

template <typename A, int DPL>
__global__ void __launch_bounds__(128) merge_kernel(const int32_t* __restrict__ table, int off_req, int off_ptr,
                                                    int off_slot, int n_merge, int g, int h_local, int d,
                                                    const A* __restrict__ part_o, const A* __restrict__ part_ml,
                                                    A* __restrict__ out, const int32_t* tc_done, int tc_ctas) {
  wait_tc_done(tc_done, tc_ctas);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const int k = blockIdx.y * 4 + warp;
  if (i >= n_merge || k >= g) return;
  const int hq_local = g * h_local;
  const int code = table[off_req + i], req = code / h_local, qh = (code % h_local) * g + k;
  const int p0 = table[off_ptr + i], p1 = table[off_ptr + i + 1];
  const int32_t* slots = table + off_slot;
  A M = neg_inf<A>();
  for (int p = p0; p < p1; ++p) {
    const int64_t e = (int64_t)slots[p] * hq_local + qh;
    if (part_ml[2 * e + 1] > 0) M = max(M, part_ml[2 * e]);
  }
  A acc[DPL];
#pragma unroll
  for (int j = 0; j < DPL; ++j) acc[j] = 0;
  A L = 0;
  for (int p = p0; p < p1; ++p) {
    const int64_t e = (int64_t)slots[p] * hq_local + qh;
    const A s = part_ml[2 * e + 1];
    if (!(s > 0)) continue;
    const A w = s * exp_acc(part_ml[2 * e] - M);
    L += w;
    const A* po = part_o + e * d;
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
      const int x = lane + 32 * j;
      if (x < d) acc[j] += w * po[x];
    }
  }
  A* dst = out + ((int64_t)req * hq_local + qh) * d;
#pragma unroll
  for (int j = 0; j < DPL; ++j) {
    const int x = lane + 32 * j;
    if (x < d) dst[x] = acc[j] / L;
  }
}

// d = 128, fp32 partials, any number of partials per entry: the (m, l)
// pairs 32 at a time across the lanes, then the output vectors four
// partials at a time with all four loads in flight (float4 per lane), so
// the merge costs a few memory latencies instead of one per partial.
// Fused output gather (codec_decode_attention_gather): every output row
// goes to all n_peers ranks' global buffers, then the grid's last CTA bumps
// this rank's arrival counter in every rank's flag array.
struct PeerDev {
  int n_peers, self, hq_global, head0;
  float* const* peer_out;
  int32_t* const* peer_flags;
  const int32_t* row_map;
  int32_t* done;
};

__device__ __forceinline__ void merge128_row(const int32_t* __restrict__ table, int off_req, int off_ptr,
                                             int off_slot, int i, int k, int g, int h_local, int lane,
                                             const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                             float* __restrict__ out, const PeerDev& pg);

// kFastNp: partials per entry merged with all their loads in flight at once,
// instantiated for 4 / 8 / 16 and chosen by the table (codec_table_info.
// merge_np: the smallest that holds 95 % of the entries; cfg2 <= 4, cfg3
// 10-13) -- the registers grow with it (16: 117 per thread, half the
// resident CTAs of 4, and a 5 us slower cfg2 merge); larger entries take
// merge128_row
template <int kFastNp>
__global__ void __launch_bounds__(128) merge128_kernel(const int32_t* __restrict__ table, int off_req, int off_ptr,
                                                       int off_slot, int n_merge, int g, int h_local,
                                                       const float* __restrict__ part_o,
                                                       const float* __restrict__ part_ml, float* __restrict__ out,
                                                       const int32_t* tc_done, int tc_ctas, const int32_t* cnt,
                                                       const PeerDev pg) {
  if (cnt) {
    // counted mode: no wait for whole grids -- this entry merges as soon
    // as its partial producers (TC epilogue rows, suffix / multi CTAs, all
    // resident already: this grid launched after the last of them started)
    // counted g rows per partial in, so the merge overlaps the tail of the
    // other kernels instead of following it
    if (threadIdx.x == 0 && blockIdx.x < n_merge) {
      const int need = g * (table[off_ptr + blockIdx.x + 1] - table[off_ptr + blockIdx.x]);
      int v;
      for (int it = 0;; ++it) {
        asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(cnt + blockIdx.x) : "memory");
        if (v >= need) break;
        if (it > (1 << 24)) __trap();  // a count that never arrives is a bug: trap, do not hang
        __nanosleep(128);
      }
    }
    __syncthreads();
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.x;
  const int k = blockIdx.y * 4 + warp;
  const bool active = i < n_merge && k < g;
  // The entry's task-table data (static) before waiting for the producers:
  // after the wait only the partials' loads remain, (m, l) and o of up to
  // kFastNp partials all in flight at once -- one memory latency instead of
  // three on the step's tail.
  const int hq_local = g * h_local;
  int req = 0, qh = 0, np = 0;
  int64_t ep[kFastNp] = {};
  if (active) {
    const int code = __ldg(table + off_req + i);
    req = code / h_local;
    qh = (code % h_local) * g + k;
    const int p0 = __ldg(table + off_ptr + i);
    np = __ldg(table + off_ptr + i + 1) - p0;
#pragma unroll
    for (int p = 0; p < kFastNp; ++p)
      if (p < np) ep[p] = (int64_t)__ldg(table + off_slot + p0 + p) * hq_local + qh;
  }
  if (!cnt) wait_tc_done(tc_done, tc_ctas);
  if (active && np <= kFastNp) {
    float2 ml[kFastNp];
    float4 o[kFastNp];
#pragma unroll
    for (int p = 0; p < kFastNp; ++p) {
      ml[p] = make_float2(0.f, 0.f);
      o[p] = make_float4(0.f, 0.f, 0.f, 0.f);
      if (p < np) {
        ml[p] = __ldg(reinterpret_cast<const float2*>(part_ml) + ep[p]);
        o[p] = __ldg(reinterpret_cast<const float4*>(part_o + ep[p] * 128) + lane);
      }
    }
    float M = neg_inf<float>();
#pragma unroll
    for (int p = 0; p < kFastNp; ++p)
      if (ml[p].y > 0) M = fmaxf(M, ml[p].x);
    float L = 0.f;
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int p = 0; p < kFastNp; ++p) {
      if (!(ml[p].y > 0)) continue;  // an empty partial (its o may be 0/0)
      const float w = ml[p].y * __expf(ml[p].x - M);
      L += w;
      acc.x += w * o[p].x;
      acc.y += w * o[p].y;
      acc.z += w * o[p].z;
      acc.w += w * o[p].w;
    }
    const float inv = 1.f / L;
    const float4 res = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
    if (pg.n_peers > 0) {
      const int64_t row = pg.row_map ? pg.row_map[req] : req;
      const int64_t off = (row * pg.hq_global + pg.head0 + qh) * 128;
      for (int p = 0; p < pg.n_peers; ++p) reinterpret_cast<float4*>(pg.peer_out[p] + off)[lane] = res;
    } else {
      reinterpret_cast<float4*>(out + ((int64_t)req * hq_local + qh) * 128)[lane] = res;
    }
  } else if (active) {
    merge128_row(table, off_req, off_ptr, off_slot, i, k, g, h_local, lane, part_o, part_ml, out, pg);
  }
  if (pg.n_peers > 0) {
    // every CTA's peer stores system-visible before it is counted; the
    // last CTA publishes this rank's rows to every rank
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int total = gridDim.x * gridDim.y;
      if (atomicAdd(pg.done, 1) == total - 1) {
        *pg.done = 0;  // every other CTA already counted: reset for the next call
        __threadfence_system();
        for (int p = 0; p < pg.n_peers; ++p) {
          int32_t* f = pg.peer_flags[p] + pg.self;
          asm volatile("red.release.sys.global.add.s32 [%0], 1;" ::"l"(f) : "memory");
        }
      }
    }
  }
}

__device__ __forceinline__ void merge128_row(const int32_t* __restrict__ table, int off_req, int off_ptr,
                                             int off_slot, int i, int k, int g, int h_local, int lane,
                                             const float* __restrict__ part_o, const float* __restrict__ part_ml,
                                             float* __restrict__ out, const PeerDev& pg) {
  const int hq_local = g * h_local;
  const int code = table[off_req + i], req = code / h_local, qh = (code % h_local) * g + k;
  const int p0 = table[off_ptr + i], np = table[off_ptr + i + 1] - p0;
  const int32_t* slots = table + off_slot + p0;
  // pass 1: the max over all partials, 32 (m, l) pairs per round in flight
  float M = neg_inf<float>();
  for (int b = 0; b < np; b += 32) {
    if (b + lane < np) {
      const float2 ml = __ldg(reinterpret_cast<const float2*>(part_ml) + (int64_t)slots[b + lane] * hq_local + qh);
      if (ml.y > 0) M = fmaxf(M, ml.x);
    }
  }
  M = warp_max(M);
  // pass 2: weights (lane p of round b holds partial b + p), then the
  // output vectors four partials at a time with all four loads in flight
  float L = 0.f;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int b = 0; b < np; b += 32) {
    float wl = 0.f;
    int64_t ep = 0;
    if (b + lane < np) {
      ep = (int64_t)slots[b + lane] * hq_local + qh;
      const float2 ml = __ldg(reinterpret_cast<const float2*>(part_ml) + ep);
      wl = ml.y > 0 ? ml.y * __expf(ml.x - M) : 0.f;
    }
    L += warp_sum(wl);
    const int nb = min(32, np - b);
    for (int c = 0; c < nb; c += 4) {
      float4 o[4];
      float w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int p = c + u;
        w[u] = __shfl_sync(0xffffffffu, wl, p & 31);
        const int64_t e = __shfl_sync(0xffffffffu, ep, p & 31);
        o[u] = (p < nb && w[u] > 0) ? __ldg(reinterpret_cast<const float4*>(part_o + e * 128) + lane)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float ww = (c + u < nb) ? w[u] : 0.f;
        acc.x += ww * o[u].x;
        acc.y += ww * o[u].y;
        acc.z += ww * o[u].z;
        acc.w += ww * o[u].w;
      }
    }
  }
  const float inv = 1.f / L;
  const float4 res = make_float4(acc.x * inv, acc.y * inv, acc.z * inv, acc.w * inv);
  if (pg.n_peers > 0) {
    const int64_t row = pg.row_map ? pg.row_map[req] : req;
    const int64_t off = (row * pg.hq_global + pg.head0 + qh) * 128;
    for (int p = 0; p < pg.n_peers; ++p) reinterpret_cast<float4*>(pg.peer_out[p] + off)[lane] = res;
  } else {
    reinterpret_cast<float4*>(out + ((int64_t)req * hq_local + qh) * 128)[lane] = res;
  }
}

int32_t cuda_status(cudaError_t e, const char* what);

// reduce_tree() on the device (codec_merge_partials): request i folds the
// partials slot[ptr[i] .. ptr[i+1]) given in the reference's PartialResult
// layout (out [slot][h_q][d] normalised, m / s [slot][h_q]); one warp per
// (request, head). Empty entries (s = 0) drop out; the exp-sum of the
// result goes to out_s so the host can raise NoVisibleTokens.
template <typename A>
__global__ void __launch_bounds__(128) merge_csr_kernel(const int32_t* __restrict__ ptr, const int32_t* __restrict__ slot,
                                                        int n_req, int h_q, int d, const A* __restrict__ po,
                                                        const A* __restrict__ pm, const A* __restrict__ ps,
                                                        A* __restrict__ out, A* __restrict__ out_s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t e = (int64_t)blockIdx.x * 4 + warp;
  if (e >= (int64_t)n_req * h_q) return;
  const int r = (int)(e / h_q), h = (int)(e % h_q);
  const int p0 = ptr[r], p1 = ptr[r + 1];
  A M = neg_inf<A>();
  for (int p = p0; p < p1; ++p) {
    const int64_t x = (int64_t)slot[p] * h_q + h;
    if (ps[x] > 0) M = max(M, pm[x]);
  }
  A L = 0;
  for (int p = p0; p < p1; ++p) {
    const int64_t x = (int64_t)slot[p] * h_q + h;
    if (ps[x] > 0) L += ps[x] * exp_acc(pm[x] - M);
  }
  A* dst = out + e * d;
  for (int c = lane; c < d; c += 32) {
    A acc = 0;
    for (int p = p0; p < p1; ++p) {
      const int64_t x = (int64_t)slot[p] * h_q + h;
      if (ps[x] > 0) acc += ps[x] * exp_acc(pm[x] - M) * po[x * d + c];
    }
    dst[c] = L > 0 ? acc / L : A(0);
  }
  if (lane == 0) out_s[e] = L;
}

int32_t launch_merge_csr(int dtype, int n_req, int h_q, int d, const int32_t* ptr, const int32_t* slot,
                         const void* po, const void* pm, const void* ps, void* out, void* out_s, cudaStream_t st) {
  const int64_t warps = (int64_t)n_req * h_q;
  if (warps == 0) return CODEC_OK;
  const dim3 grid((unsigned)((warps + 3) / 4));
  if (dtype == CODEC_F64)
    merge_csr_kernel<double><<<grid, 128, 0, st>>>(ptr, slot, n_req, h_q, d, (const double*)po, (const double*)pm,
                                                    (const double*)ps, (double*)out, (double*)out_s);
  else if (dtype == CODEC_F32)
    merge_csr_kernel<float><<<grid, 128, 0, st>>>(ptr, slot, n_req, h_q, d, (const float*)po, (const float*)pm,
                                                   (const float*)ps, (float*)out, (float*)out_s);
  else
    return fail(CODEC_ERR_UNSUPPORTED, "merge: partials must be float32 or float64");
  return cuda_status(cudaGetLastError(), "merge launch");
}

int32_t launch_merge(int dtype, const int32_t* table, const codec_table_info& in, int d, int hq_local,
                     const void* part_o, const void* part_ml, void* out, cudaStream_t st, const int32_t* tc_done,
                     int tc_ctas, bool pdl, const int32_t* cnt, const codec_peer_gather* gather) {
  PeerDev pg{0, 0, 0, 0, nullptr, nullptr, nullptr, nullptr};
  if (gather) {
    if (dtype == CODEC_F64 || d != 128) return fail(CODEC_ERR_UNSUPPORTED, "fused gather: bf16 / f32, d = 128 only");
    pg = PeerDev{gather->n_peers, gather->self, gather->hq_global, gather->head0,
                 reinterpret_cast<float* const*>(gather->peer_out), gather->peer_flags, gather->row_map, gather->done};
  }
  if (in.n_merge == 0) return CODEC_OK;
  const int h_local = in.h_local, g = hq_local / h_local;
  dim3 grid(in.n_merge, (g + 3) / 4);
#define CODEC_MERGE(A, DPL)                                                                                    \
  merge_kernel<A, DPL><<<grid, 128, 0, st>>>(table, in.off_merge_req, in.off_merge_ptr, in.off_merge_slot,     \
                                             in.n_merge, g, h_local, d, (const A*)part_o, (const A*)part_ml,    \
                                             (A*)out, tc_done, tc_ctas)
  if (d > 512) return fail(CODEC_ERR_UNSUPPORTED, "head dim %d > 512", d);
  if (dtype != CODEC_F64 && d == 128) {
    // after the suffix kernel on the same stream: programmatic dependent
    // launch, so the merge CTAs are resident when it retires (they wait in
    // griddepcontrol.wait, then for the TC counter)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(128);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    auto kern = in.merge_np <= 4 ? merge128_kernel<4> : in.merge_np <= 8 ? merge128_kernel<8> : merge128_kernel<16>;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, table, in.off_merge_req, in.off_merge_ptr, in.off_merge_slot,
                                       in.n_merge, g, h_local, (const float*)part_o, (const float*)part_ml,
                                       (float*)out, tc_done, tc_ctas, cnt, pg);
    if (e != cudaSuccess) return cuda_status(e, "merge launch");
    return cuda_status(cudaGetLastError(), "merge launch");
  }
  if (dtype == CODEC_F64) {
    if (d <= 128) CODEC_MERGE(double, 4); else CODEC_MERGE(double, 16);
  } else {
    if (d <= 128) CODEC_MERGE(float, 4); else CODEC_MERGE(float, 16);
  }
#undef CODEC_MERGE
  return cuda_status(cudaGetLastError(), "merge launch");
}

}  // namespace codec

extern "C" int32_t codec_merge_partials(int32_t dtype, int32_t n_req, int32_t h_q, int32_t d, const int32_t* ptr,
                                        const int32_t* slot, const void* part_out, const void* part_m,
                                        const void* part_s, void* out, void* out_s, void* stream) {
  if (n_req < 0 || h_q < 1 || d < 1) return codec::fail(CODEC_ERR_DIMENSION_MISMATCH, "bad merge dims (%d, %d, %d)",
                                                         n_req, h_q, d);
  if (!ptr || !slot || !part_out || !part_m || !part_s || !out || !out_s)
    return codec::fail(CODEC_ERR_VALUE, "NULL argument");
  return codec::launch_merge_csr(dtype, n_req, h_q, d, ptr, slot, part_out, part_m, part_s, out, out_s,
                                 (cudaStream_t)stream);
}
