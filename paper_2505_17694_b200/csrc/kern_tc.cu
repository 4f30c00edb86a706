// K2: shared-node split attention on the 5th-generation tensor cores.
//
// One CTA = (TC group, kv head): a KV slice [kv_tok, kv_tok + len) of a
// shared node and up to 128 query-head rows (128/g requests of the node's
// query set, each with its g query heads -- the GQA group becomes the M
// dimension, so sharing turns the per-request GEMVs into one dense
// contraction). Per 128-token tile j:
//     S   = Q K_j^T              tcgen05.mma M128 N128 K128, S in TMEM
//     P   = exp2(S*c - m)        softmax warps, online max/sum per row
//     O  += P V_j                tcgen05.mma M128 N128 K128, O in TMEM
// Math is the reference's pac_kernel (_kernels.pyx:25-54) per row; the
// partial (O/l, m, l) feeds the same LSE merge as the other kernels.
//
// Warp roles (192 threads): warp 0 = TMA producer (K and V rings, 2
// stages each, SWIZZLE_128B boxes of 128 tokens x 64 dims), warp 1 = TMEM
// allocator + single-thread MMA issuer, warps 2-5 = softmax / epilogue
// (thread = one query row = one TMEM lane). S_{j+1} is issued as soon as
// the softmax has pulled S_j into registers, so the QK^T of the next tile
// overlaps the exponentials of this one. P goes through shared memory
// (K-major SW128) as the A operand of the PV MMA; V is consumed MN-major
// straight from its TMA layout.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "tc_ptx.cuh"

namespace codec {

constexpr int kTcThreads = 192;
constexpr int kTcRows = 128;        // M
constexpr int kTcTok = 128;         // tokens per tile (N of QK^T, K of PV)
constexpr int kTcD = 128;           // head dim
constexpr int kTcTile = 128 * 128 * 2;  // bytes of one bf16 128x128 tile
constexpr int kTcKStages = 2;
constexpr int kTcVStages = 2;
constexpr int kOffQ = 0;
constexpr int kOffP = kOffQ + kTcTile;
constexpr int kOffK = kOffP + kTcTile;
constexpr int kOffV = kOffK + kTcKStages * kTcTile;
constexpr int kOffBar = kOffV + kTcVStages * kTcTile;
constexpr int kTcSmem = kOffBar + 256 + 1024;  // + barriers + alignment slack
constexpr uint32_t kTmemCols = 256;  // S: cols [0,128), O: cols [128,256)

struct TcBars {
  uint64_t q_full;
  uint64_t k_full[kTcKStages], k_empty[kTcKStages];
  uint64_t v_full[kTcVStages], v_empty[kTcVStages];
  uint64_t s_full, s_free, p_full, pv_done;
  uint32_t tmem_slot;
};

// byte offset of 16-byte chunk `c` (0..15 along a 128-element row) of row
// `r` in a K-major SWIZZLE_128B tile made of two 64-element atoms
__device__ __forceinline__ uint32_t sw128_off(int r, int c) {
  const int atom = c >> 3, cc = c & 7;
  return atom * (128 * 128) + r * 128 + ((cc ^ (r & 7)) << 4);
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_pac_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const int32_t* __restrict__ table, int off_groups, int off_rows,
                  const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, int hq_local,
                  float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  uint8_t* smem = smem_raw + (((raw_u32 + 1023) & ~1023u) - raw_u32);
  const uint32_t sbase = smem_u32(smem);
  TcBars* bars = reinterpret_cast<TcBars*>(smem + kOffBar);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* grp = table + off_groups + blockIdx.x * kGroupInts;
  const int kh = blockIdx.y;
  const int kv_tok = grp[kGrpKvTok];
  const int n_req = grp[kGrpNRows];
  const int32_t* rows = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  // tiles needed = max visible over the group's rows
  int max_vis = 0;
  for (int i = 0; i < n_req; ++i) max_vis = max(max_vis, rows[i * kRowInts + 1]);
  const int n_tiles = (max_vis + kTcTok - 1) / kTcTok;
  const int row_base = kh * (int)pool_tokens + kv_tok;  // row of the 2D pool view

  if (tid == 0) {
    mbar_init(&bars->q_full, 128);
    for (int s = 0; s < kTcKStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < kTcVStages; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    mbar_init(&bars->s_full, 1);
    mbar_init(&bars->s_free, 128);
    mbar_init(&bars->p_full, 128);
    mbar_init(&bars->pv_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tc::tmem_alloc(&bars->tmem_slot, kTmemCols);
  if (warp == 0 && lane == 0) {
    tc::prefetch_tmap(&tmk);
    tc::prefetch_tmap(&tmv);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;
  const uint32_t tmem_s = tmem, tmem_o = tmem + 128;

  if (warp == 0) {
    // ------------------------------------------------ TMA producer
    if (lane == 0) {
      for (int j = 0; j < n_tiles; ++j) {
        const int y = row_base + j * kTcTok;
        const int ks = j % kTcKStages;
        if (j >= kTcKStages) mbar_wait(&bars->k_empty[ks], ((j / kTcKStages) - 1) & 1);
        mbar_arrive_expect_tx(&bars->k_full[ks], kTcTile);
        uint8_t* kd = smem + kOffK + ks * kTcTile;
        tc::tma_load_2d(kd, &tmk, 0, y, &bars->k_full[ks]);
        tc::tma_load_2d(kd + 128 * 128, &tmk, 64, y, &bars->k_full[ks]);
        const int vs = j % kTcVStages;
        if (j >= kTcVStages) mbar_wait(&bars->v_empty[vs], ((j / kTcVStages) - 1) & 1);
        mbar_arrive_expect_tx(&bars->v_full[vs], kTcTile);
        uint8_t* vd = smem + kOffV + vs * kTcTile;
        tc::tma_load_2d(vd, &tmv, 0, y, &bars->v_full[vs]);
        tc::tma_load_2d(vd + 128 * 128, &tmv, 64, y, &bars->v_full[vs]);
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, 128, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16(128, 128, false, true);
      const uint32_t q_addr = sbase + kOffQ, p_addr = sbase + kOffP;
      auto issue_s = [&](int j) {
        const int ks = j % kTcKStages;
        mbar_wait(&bars->k_full[ks], (j / kTcKStages) & 1);
        tc::fence_after();
        const uint32_t k_addr = sbase + kOffK + ks * kTcTile;
#pragma unroll
        for (int k = 0; k < kTcD / 16; ++k) {
          const uint32_t koff = (k >> 2) * (128 * 128) + (k & 3) * 32;
          tc::mma_f16_ss(tmem_s, tc::smem_desc(q_addr + koff, 16, 1024), tc::smem_desc(k_addr + koff, 16, 1024),
                         idesc_s, k > 0 ? 1u : 0u);
        }
        tc::commit(&bars->k_empty[ks]);
        tc::commit(&bars->s_full);
      };
      mbar_wait(&bars->q_full, 0);
      if (n_tiles > 0) issue_s(0);
      for (int j = 0; j < n_tiles; ++j) {
        if (j + 1 < n_tiles) {
          mbar_wait(&bars->s_free, j & 1);  // softmax holds S_j in registers
          issue_s(j + 1);
        }
        const int vs = j % kTcVStages;
        mbar_wait(&bars->v_full[vs], (j / kTcVStages) & 1);
        mbar_wait(&bars->p_full, j & 1);
        tc::fence_after();
        const uint32_t v_addr = sbase + kOffV + vs * kTcTile;
#pragma unroll
        for (int k = 0; k < kTcTok / 16; ++k) {
          // A = P (K-major over tokens), B = V (MN-major: N = head dim)
          const uint32_t aoff = (k >> 2) * (128 * 128) + (k & 3) * 32;
          const uint32_t boff = k * 16 * 128;
          tc::mma_f16_ss(tmem_o, tc::smem_desc(p_addr + aoff, 16, 1024),
                         tc::smem_desc(v_addr + boff, 128 * 128, 1024), idesc_o, (j > 0 || k > 0) ? 1u : 0u);
        }
        tc::commit(&bars->v_empty[vs]);
        tc::commit(&bars->pv_done);
      }
    }
  } else {
    // ------------------------------------------------ softmax / epilogue
    const int quad = warp & 3;             // TMEM lane quadrant this warp may access
    const int r = quad * 32 + lane;        // query row == TMEM lane
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const int ridx = r / g;                // request slot within the group
    const bool valid = ridx < n_req;
    const int req = valid ? rows[ridx * kRowInts + 0] : 0;
    const int vis = valid ? rows[ridx * kRowInts + 1] : 0;
    const int slot = valid ? rows[ridx * kRowInts + 2] : 0;
    const int qh = kh * g + (r % g);
    // stage Q row r (K-major SW128)
    {
      uint8_t* qs = smem + kOffQ;
      const uint4* src = reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + qh) * kTcD);
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint4 v = valid ? src[c] : make_uint4(0, 0, 0, 0);
        *reinterpret_cast<uint4*>(qs + sw128_off(r, c)) = v;
      }
      tc::fence_proxy_async_smem();
      mbar_arrive(&bars->q_full);
    }
    const float cscale = 1.4426950408889634f * rsqrtf((float)kTcD);
    float m_run = neg_inf<float>(), l_run = 0.f;
    uint8_t* ps = smem + kOffP;
    for (int j = 0; j < n_tiles; ++j) {
      mbar_wait(&bars->s_full, j & 1);
      tc::fence_after();
      uint32_t sreg[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(tmem_s + lane_addr + c * 32, sreg + c * 32);
      tc::wait_ld();
      tc::fence_before();
      mbar_arrive(&bars->s_free);
      const int lim = vis - j * kTcTok;  // tokens of this tile visible to the row
      float mt = neg_inf<float>();
#pragma unroll
      for (int c = 0; c < 128; ++c) {
        float s = __uint_as_float(sreg[c]) * cscale;
        s = (c < lim) ? s : neg_inf<float>();
        sreg[c] = __float_as_uint(s);
        mt = fmaxf(mt, s);
      }
      const float m_new = fmaxf(m_run, mt);
      if (j > 0) {
        mbar_wait(&bars->pv_done, (j - 1) & 1);  // P buffer free, O settled
        tc::fence_after();
        const bool need = valid && m_new > m_run;
        if (__any_sync(0xffffffffu, need)) {  // tcgen05.ld/st are warp-collective
          const float alpha = need ? fast_exp2(m_run - m_new) : 1.f;
          l_run *= alpha;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            uint32_t o[32];
            tc::tmem_ld32(tmem_o + lane_addr + c * 32, o);
            tc::wait_ld();
#pragma unroll
            for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
            tc::tmem_st32(tmem_o + lane_addr + c * 32, o);
          }
          tc::wait_st();
        }
      }
      m_run = valid ? m_new : m_run;
      // P row -> bf16 K-major SW128
      float psum = 0.f;
#pragma unroll
      for (int c = 0; c < 16; ++c) {
        uint32_t w[4];
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          float p0 = valid ? fast_exp2(__uint_as_float(sreg[c * 8 + 2 * h]) - m_new) : 0.f;
          float p1 = valid ? fast_exp2(__uint_as_float(sreg[c * 8 + 2 * h + 1]) - m_new) : 0.f;
          __nv_bfloat162 b2 = __floats2bfloat162_rn(p0, p1);
          // accumulate l from the rounded values the MMA actually sees
          float2 rb = __bfloat1622float2(b2);
          psum += rb.x + rb.y;
          w[h] = *reinterpret_cast<uint32_t*>(&b2);
        }
        *reinterpret_cast<uint4*>(ps + sw128_off(r, c)) = make_uint4(w[0], w[1], w[2], w[3]);
      }
      l_run += psum;
      tc::fence_proxy_async_smem();
      tc::fence_before();
      mbar_arrive(&bars->p_full);
    }
    // epilogue: O / l
    if (n_tiles > 0) {
      mbar_wait(&bars->pv_done, (n_tiles - 1) & 1);
      tc::fence_after();
    }
    float* dst;
    if (slot < 0) {
      dst = out + ((int64_t)req * hq_local + qh) * kTcD;
    } else {
      const int64_t ei = (int64_t)slot * hq_local + qh;
      dst = part_o + ei * kTcD;
      if (valid) {
        part_ml[2 * ei] = m_run * 0.69314718055994530942f;
        part_ml[2 * ei + 1] = l_run;
      }
    }
    const float inv = 1.f / l_run;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      uint32_t o[32];
      tc::tmem_ld32(tmem_o + lane_addr + c * 32, o);
      tc::wait_ld();
      if (valid) {
#pragma unroll
        for (int i = 0; i < 32; i += 4)
          *reinterpret_cast<float4*>(dst + c * 32 + i) =
              make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                          __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
      }
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == 1) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int32_t cuda_status(cudaError_t e, const char* what);

static int32_t encode_pool_map(CUtensorMap* map, const void* pool, int64_t rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
      return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kTcD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kTcD * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CODEC_OK;
}

int32_t launch_tc(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q, const void* k,
                  const void* v, int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                  cudaStream_t st) {
  if (n_groups == 0) return CODEC_OK;
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_map(&mk, k, (int64_t)h_local * pool_tokens));
  CODEC_TRY(encode_pool_map(&mv, v, (int64_t)h_local * pool_tokens));
  cudaError_t e = cudaFuncSetAttribute(tc_pac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
  if (e != cudaSuccess) return cuda_status(e, "tc smem attribute");
  dim3 grid(n_groups, h_local);
  tc_pac_kernel<<<grid, kTcThreads, kTcSmem, st>>>(mk, mv, table, off_groups, off_rows, (const __nv_bfloat16*)q,
                                                   pool_tokens, g, h_local * g, (float*)out, (float*)part_o,
                                                   (float*)part_ml);
  return cuda_status(cudaGetLastError(), "tc launch");
}

}  // namespace codec
