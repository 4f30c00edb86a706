// K3' (fp32 KV, d in {64, 256}, g <= 16, or CODEC_FLAG_GEMV_SIMT): unshared /
// lightly shared nodes -- bulk-async streamed, warp-shuffle GEMV split
// attention on CUDA cores. bf16 d=128 suffixes run on kern_mma.cu instead.
//
// Same math as the reference's pac_kernel (_kernels.pyx:25-54): scores
// q.k/sqrt(d) over the visible prefix, online softmax, normalised output
// plus (m, s). One CTA = (GEMV group = one request's slice of a node,
// one kv head) with its g query heads as R rows (GQA packing, rows >= g
// are zero padding).
//
// Memory path: the slice of one head is contiguous in the head-major pool
// ([h][T][d], nodes at their preorder offsets), so a producer lane streams
// it with 1D bulk async copies (cp.async.bulk, TMA engine, UBLKCP in SASS)
// into a 4-stage shared-memory ring guarded by mbarriers; 4 consumer
// warps read 16-byte vectors from smem.
//
// Math path: lane layout per warp step = NTS token slots x TPT lanes per
// token, each lane owning EPT contiguous elements of the head dim. The R
// partial dot products of a token are reduce-scattered across its TPT
// lanes (log2 R halving stages, then an all-reduce), which needs ~R-1
// shuffles per token instead of R*log2(TPT). Scores are kept in the
// log2 domain (q pre-scaled by log2(e)/sqrt(d)) so softmax uses ex2.approx.
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "tc_ptx.cuh"

namespace codec {

constexpr int kGemvWarps = 4;                  // consumer warps
constexpr int kGemvThreads = 32 * (kGemvWarps + 1);
constexpr int kGemvStages = 4;
constexpr int kGemvStageBytes = 8192;          // K (and V) bytes per stage

template <typename T, int D, int R>
struct GemvCfg {
  static constexpr int VEC = 16 / (int)sizeof(T);
  static constexpr int TPT = (D / VEC) < 32 ? (D / VEC) : 32;
  static constexpr int EPT = D / TPT;
  static constexpr int NVEC = EPT / VEC;  // 16-byte vectors per lane
  static constexpr int NTS = 32 / TPT;
  static constexpr int CT = kGemvStageBytes / (D * (int)sizeof(T));
  static constexpr int STEPS = CT / (kGemvWarps * NTS);
  static constexpr int LTPT = TPT == 32 ? 5 : TPT == 16 ? 4 : TPT == 8 ? 3 : TPT == 4 ? 2 : TPT == 2 ? 1 : 0;
  static constexpr int LR = R == 8 ? 3 : R == 4 ? 2 : R == 2 ? 1 : 0;
  static_assert(R <= TPT, "reduce-scatter needs R <= lanes per token");
  static_assert(STEPS >= 1, "stage too small");
  static_assert(EPT % VEC == 0, "lane chunk must be whole vectors");
};

template <typename T> __device__ __forceinline__ void load_vec(const T* p, float* f);
template <> __device__ __forceinline__ void load_vec<__nv_bfloat16>(const __nv_bfloat16* p, float* f) {
  uint4 v = *reinterpret_cast<const uint4*>(p);
  bf16x8_to_f32(v, f);
}
template <> __device__ __forceinline__ void load_vec<float>(const float* p, float* f) {
  float4 v = *reinterpret_cast<const float4*>(p);
  f[0] = v.x;
  f[1] = v.y;
  f[2] = v.z;
  f[3] = v.w;
}

template <typename T, int D, int R>
__global__ void __launch_bounds__(kGemvThreads) gemv_pac_kernel(const int32_t* __restrict__ table, int off_groups,
                                                                 int off_rows, const T* __restrict__ q,
                                                                 const T* __restrict__ kpool,
                                                                 const T* __restrict__ vpool, int64_t pool_tokens,
                                                                 int g, int hq_local, float qscale,
                                                                 float* __restrict__ out,
                                                                 float* __restrict__ part_o,
                                                                 float* __restrict__ part_ml,
                                                                 long long* __restrict__ ctalog) {
  const long long t_start = ctalog ? global_ns() : 0;
  using C = GemvCfg<T, D, R>;
  extern __shared__ __align__(128) uint8_t smem[];
  T* sk = reinterpret_cast<T*>(smem);                                  // [S][CT][D]
  T* sv = reinterpret_cast<T*>(smem + kGemvStages * kGemvStageBytes);  // [S][CT][D]
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + 2 * kGemvStages * kGemvStageBytes);
  uint64_t* empty = full + kGemvStages;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* grp = table + off_groups + blockIdx.x * kGroupInts;
  const int kh = blockIdx.y;
  const int len = grp[kGrpLen];
  const int32_t* row = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  const int req = row[0], vis = row[1], slot = row[2];
  const int n_tok = vis;  // visible tokens of this request within the slice
  const int nch = (n_tok + C::CT - 1) / C::CT;
  (void)len;
  const int64_t base = ((int64_t)kh * pool_tokens + grp[kGrpKvTok]) * D;

  if (tid == 0) {
    for (int s = 0; s < kGemvStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kGemvWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kGemvWarps) {
    // ---------------- producer: one lane streams K and V chunks
    if (lane == 0) {
      for (int c = 0; c < nch; ++c) {
        const int s = c % kGemvStages;
        if (c >= kGemvStages) mbar_wait(&empty[s], ((c / kGemvStages) - 1) & 1);
        const int ntok = min(C::CT, n_tok - c * C::CT);
        const uint32_t bytes = (uint32_t)(ntok * D * sizeof(T));
        mbar_arrive_expect_tx(&full[s], 2 * bytes);
        const int64_t src = base + (int64_t)c * C::CT * D;
        bulk_g2s(sk + (size_t)s * C::CT * D, kpool + src, bytes, &full[s]);
        bulk_g2s(sv + (size_t)s * C::CT * D, vpool + src, bytes, &full[s]);
      }
    }
  } else {
    // ---------------- consumers
    const int ts = lane / C::TPT, sub = lane % C::TPT;
    const int rr = (sub >> (C::LTPT - C::LR)) & (R - 1);  // row this lane owns after reduce-scatter
    float qf[R][C::EPT];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (r < g) {
        const T* qp = q + ((int64_t)req * hq_local + kh * g + r) * D + sub * C::EPT;
#pragma unroll
        for (int v = 0; v < C::NVEC; ++v) load_vec<T>(qp + v * C::VEC, &qf[r][v * C::VEC]);
#pragma unroll
        for (int e = 0; e < C::EPT; ++e) qf[r][e] *= qscale;
      } else {
#pragma unroll
        for (int e = 0; e < C::EPT; ++e) qf[r][e] = 0.f;
      }
    }
    float acc[R][C::EPT];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int e = 0; e < C::EPT; ++e) acc[r][e] = 0.f;
    float m_run = neg_inf<float>(), l_run = 0.f;

    for (int c = 0; c < nch; ++c) {
      const int s = c % kGemvStages;
      mbar_wait(&full[s], (c / kGemvStages) & 1);
      const T* ck = sk + (size_t)s * C::CT * D;
      const T* cv = sv + (size_t)s * C::CT * D;
      const int tok0 = c * C::CT;
      float sc[C::STEPS];
#pragma unroll
      for (int u = 0; u < C::STEPS; ++u) {
        const int lt = (warp * C::STEPS + u) * C::NTS + ts;
        float kf[C::EPT];
#pragma unroll
        for (int v = 0; v < C::NVEC; ++v) load_vec<T>(ck + lt * D + sub * C::EPT + v * C::VEC, &kf[v * C::VEC]);
        float part[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          float2 a = make_float2(0.f, 0.f);
#pragma unroll
          for (int e = 0; e < C::EPT; e += 2)
            a = tc::ffma2(make_float2(qf[r][e], qf[r][e + 1]), make_float2(kf[e], kf[e + 1]), a);
          part[r] = a.x + a.y;
        }
        // reduce-scatter R partials over the TPT lanes of this token
#pragma unroll
        for (int k = 0; k < C::LR; ++k) {
          const int half = R >> (k + 1);
          const int bit = C::TPT >> (k + 1);
          const bool upper = (sub & bit) != 0;
#pragma unroll
          for (int i = 0; i < half; ++i) {
            const float send = upper ? part[i] : part[i + half];
            const float keep = upper ? part[i + half] : part[i];
            part[i] = keep + __shfl_xor_sync(0xffffffffu, send, bit);
          }
        }
#pragma unroll
        for (int k = C::LR; k < C::LTPT; ++k) part[0] += __shfl_xor_sync(0xffffffffu, part[0], C::TPT >> (k + 1));
        sc[u] = (tok0 + lt < n_tok) ? part[0] : neg_inf<float>();
      }
      // online softmax for this lane's row
      float mx = sc[0];
#pragma unroll
      for (int u = 1; u < C::STEPS; ++u) mx = fmaxf(mx, sc[u]);
#pragma unroll
      for (int b = C::TPT; b < 32; b <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, b));
      // lazy rescale: the exponent reference only moves when this chunk's
      // max beats it by more than 2^8 (p <= 256 otherwise: exact enough in fp32)
      const bool need = mx > m_run + 8.f;
      const int src0 = ts * C::TPT;
      if (__any_sync(0xffffffffu, need)) {
        const float alpha = need ? fast_exp2(m_run - mx) : 1.f;  // 0 on the first chunk
        l_run *= alpha;
        m_run = need ? mx : m_run;
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float a = __shfl_sync(0xffffffffu, alpha, src0 + (r << (C::LTPT - C::LR)));
#pragma unroll
          for (int e = 0; e < C::EPT; ++e) acc[r][e] *= a;
        }
      }
      const bool dead = m_run == neg_inf<float>();
      float p[C::STEPS];
      float psum = 0.f;
#pragma unroll
      for (int u = 0; u < C::STEPS; ++u) {
        p[u] = dead ? 0.f : fast_exp2(sc[u] - m_run);
        psum += p[u];
      }
      l_run += psum;
#pragma unroll
      for (int u = 0; u < C::STEPS; ++u) {
        const int lt = (warp * C::STEPS + u) * C::NTS + ts;
        float vf[C::EPT];
#pragma unroll
        for (int v = 0; v < C::NVEC; ++v) load_vec<T>(cv + lt * D + sub * C::EPT + v * C::VEC, &vf[v * C::VEC]);
        if (tok0 + lt >= n_tok) {
#pragma unroll
          for (int e = 0; e < C::EPT; ++e) vf[e] = 0.f;  // stale smem may hold non-finite bits
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float pr = __shfl_sync(0xffffffffu, p[u], src0 + (r << (C::LTPT - C::LR)));
#pragma unroll
          for (int e = 0; e < C::EPT; e += 2) {
            const float2 a = tc::ffma2(make_float2(pr, pr), make_float2(vf[e], vf[e + 1]),
                                       make_float2(acc[r][e], acc[r][e + 1]));
            acc[r][e] = a.x;
            acc[r][e + 1] = a.y;
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // fold the token slots of this warp
#pragma unroll
    for (int b = C::TPT; b < 32; b <<= 1) {
      l_run += __shfl_xor_sync(0xffffffffu, l_run, b);
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < C::EPT; ++e) acc[r][e] += __shfl_xor_sync(0xffffffffu, acc[r][e], b);
    }
    // stash per-warp (m, l, acc) in the K ring once every consumer warp is
    // done reading it (named barrier over the 4 consumer warps)
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kGemvWarps) : "memory");
    float* wm = reinterpret_cast<float*>(smem) + warp * (R * (D + 2));
    if (ts == 0) {
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int e = 0; e < C::EPT; ++e) wm[2 * R + r * D + sub * C::EPT + e] = acc[r][e];
      if ((sub & ((1 << (C::LTPT - C::LR)) - 1)) == 0) {
        wm[rr] = m_run;
        wm[R + rr] = l_run;
      }
    }
  }
  __syncthreads();  // all chunks consumed (ring free) before the stash above is read
  // NOTE: the stash is written after the consumers' last mbarrier wait, and
  // the producer issues no copy after the last chunk, so the ring is idle.
  if (tid < 32 * kGemvWarps) {
    const float* wbase = reinterpret_cast<const float*>(smem);
    for (int idx = tid; idx < R * D; idx += 32 * kGemvWarps) {
      const int r = idx / D, e = idx % D;
      if (r >= g) continue;
      float M = neg_inf<float>();
#pragma unroll
      for (int w = 0; w < kGemvWarps; ++w) M = fmaxf(M, wbase[w * (R * (D + 2)) + r]);
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < kGemvWarps; ++w) {
        const float* wm = wbase + w * (R * (D + 2));
        const float mw = wm[r];
        if (mw == neg_inf<float>()) continue;
        const float sc = fast_exp2(mw - M);
        L += wm[R + r] * sc;
        O += wm[2 * R + r * D + e] * sc;
      }
      const int qh = kh * g + r;
      if (slot < 0) {
        out[((int64_t)req * hq_local + qh) * D + e] = O / L;
      } else {
        const int64_t ei = (int64_t)slot * hq_local + qh;
        part_o[ei * D + e] = O / L;
        if (e == 0) {
          part_ml[2 * ei] = M * 0.69314718055994530942f;  // back to natural-log units
          part_ml[2 * ei + 1] = L;
        }
      }
    }
  }
  if (ctalog) {
    __syncthreads();
    cta_log(ctalog, kCtaLogGemv + blockIdx.y * gridDim.x + blockIdx.x, t_start);
  }
}

int32_t cuda_status(cudaError_t e, const char* what);

template <typename T, int D, int R>
int32_t launch_gemv_t(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q,
                      const void* k, const void* v, int64_t pool_tokens, int g, int h_local, void* out,
                      void* part_o, void* part_ml, cudaStream_t st, long long* ctalog) {
  const int smem = 2 * kGemvStages * kGemvStageBytes + 2 * kGemvStages * 8;
  static_assert(kGemvWarps * R * (D + 2) * 4 <= kGemvStages * kGemvStageBytes * 2, "stash must fit the ring");
  auto kern = gemv_pac_kernel<T, D, R>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return cuda_status(e, "gemv smem attribute");
  e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return cuda_status(e, "gemv carveout attribute");
  const float qscale = (float)(1.4426950408889634 / sqrt((double)D));
  dim3 grid(n_groups, h_local);
  kern<<<grid, kGemvThreads, smem, st>>>(table, off_groups, off_rows, (const T*)q, (const T*)k, (const T*)v,
                                        pool_tokens, g, h_local * g, qscale, (float*)out, (float*)part_o,
                                        (float*)part_ml, ctalog);
  return cuda_status(cudaGetLastError(), "gemv launch");
}

int32_t launch_gemv(int dtype, int d, int rows, const int32_t* table, int n_groups, int off_groups, int off_rows,
                    const void* q, const void* k, const void* v, int64_t pool_tokens, int g, int h_local,
                    void* out, void* part_o, void* part_ml, cudaStream_t st, long long* ctalog) {
  if (n_groups == 0) return CODEC_OK;
#define CODEC_GEMV(T, D, R)                                                                                 \
  if (d == D && rows == R)                                                                                  \
  return launch_gemv_t<T, D, R>(table, n_groups, off_groups, off_rows, q, k, v, pool_tokens, g, h_local, out, \
                                part_o, part_ml, st, ctalog)
  if (dtype == CODEC_BF16) {
    CODEC_GEMV(__nv_bfloat16, 64, 4);
    CODEC_GEMV(__nv_bfloat16, 64, 8);
    CODEC_GEMV(__nv_bfloat16, 128, 4);
    CODEC_GEMV(__nv_bfloat16, 128, 8);
    CODEC_GEMV(__nv_bfloat16, 256, 4);
    CODEC_GEMV(__nv_bfloat16, 256, 8);
  } else if (dtype == CODEC_F32) {
    CODEC_GEMV(float, 64, 4);
    CODEC_GEMV(float, 64, 8);
    CODEC_GEMV(float, 128, 4);
    CODEC_GEMV(float, 128, 8);
    CODEC_GEMV(float, 256, 4);
    CODEC_GEMV(float, 256, 8);
  }
#undef CODEC_GEMV
  return fail(CODEC_ERR_UNSUPPORTED, "gemv: dtype %d d %d rows %d", dtype, d, rows);
}

}  // namespace codec
