// K3: unshared / lightly shared nodes (the per-request suffixes) on the
// warp-level tensor cores (mma.sync m16n8k16 bf16 -> f32, HMMA in SASS).
//
// Same math as the reference's pac_kernel (_kernels.pyx:25-54) for the g
// query heads of one request and one kv head over the request's visible
// part of one node slice: scores q.k/sqrt(d), online softmax, normalised
// output plus (m, s). One CTA = (GEMV group = one request's slice, one kv
// head); rows = the g <= 8 query heads (GQA packing, padded to n = 8).
//
// Why tensor cores for a GEMV: the suffix path is HBM-bound, but it runs
// concurrently with the persistent tcgen05 kernel on the same SMs, whose
// softmax needs most of the issue slots. Turned on its side -- S^T = K Q^T
// (m = 16 tokens, n = 8 heads, k = 16 of d) and O^T += V^T P^T (m = 16 of d,
// n = 8 heads, k = 16 tokens) -- one request-head costs ~3.5 warp
// instructions per token instead of ~40 on the CUDA cores (FFMA2 dots,
// bf16 converts, shuffles). P^T reaches the B-fragment layout with two
// movmatrix.trans per 16 tokens; no TMEM is used, so the kernel co-resides
// with the tcgen05 kernel (which owns all 512 TMEM columns).
//
// Memory path: one producer lane streams the slice with 3D TMA boxes of
// 32 whole token rows (8 KB, SWIZZLE_128B; one op each for K and V: the
// TMA unit's per-op cost, not bytes, limits small boxes) of the head-major
// pool into a 2-stage ring (6 CTAs per SM: measured better than 4 stages x
// 3 CTAs or 64-token stages); the swizzle makes the ldmatrix reads
// conflict-free. Two consumer warps take 16 tokens of each stage; each
// fences its generic-proxy reads of a stage before releasing it to the next
// TMA write (without the fence a stage was sometimes overwritten under a
// consumer's ldmatrix: wrong O, right l, tools/k3_race2.py).
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "mma_sync.cuh"
#include "tc_ptx.cuh"

namespace codec {

#ifndef CODEC_MMA_SUB
#define CODEC_MMA_SUB 1
#endif
#ifndef CODEC_SUFFIX_EVICT_FIRST
#define CODEC_SUFFIX_EVICT_FIRST 1
#endif
#ifndef CODEC_MMA_STAGES
#define CODEC_MMA_STAGES 2  // 2 x 16 KB per CTA, 6 CTAs per SM: more CTAs beat deeper rings (~5 % on cfg2)
#endif
// L2 prefetch beyond the SMEM ring: chunks ahead of the TMA loads (0: off),
// issued CODEC_MMA_PF_GROUP chunks per bulk-prefetch op (the SM's TMA unit
// pays per op, not per byte): more bytes in flight per CTA without SMEM
#ifndef CODEC_MMA_PF
#define CODEC_MMA_PF 0  // measured: 4 ahead (2 per op) slowed the suffix stream 90 -> 129 us on cfg2
#endif
#ifndef CODEC_MMA_PF_GROUP
#define CODEC_MMA_PF_GROUP 2
#endif
constexpr int kMmaWarps = 2;                       // consumer warps
constexpr int kMmaThreads = 32 * (kMmaWarps + 1);  // + producer warp
constexpr int kMmaStages = CODEC_MMA_STAGES;
constexpr int kMmaSub = CODEC_MMA_SUB;             // 16-token steps per consumer warp per stage
constexpr int kMmaCT = 16 * kMmaWarps * kMmaSub;   // tokens per stage
constexpr int kMmaD = 128;
constexpr int kFzMax = 8;                          // partials besides its own a fused merge folds in
constexpr int kMmaBox = kMmaCT * 256;              // one box: kMmaCT whole token rows
static_assert(kMmaCT <= 256, "TMA box rows");
constexpr int kMmaStageBytes = 2 * kMmaBox;        // K box + V box
constexpr int kMmaSmem = kMmaStages * kMmaStageBytes + 1024 /* align */ + 2 * kMmaStages * 8;

// byte offset of 16-byte chunk c (0..15 along d) of token row r in a
// [rows][2][64] SW128 box (line = 2 r + half, chunk XOR line % 8)
__device__ __forceinline__ uint32_t mma_sw(int r, int c) {
  const int line = 2 * r + (c >> 3);
  return line * 128 + (((c & 7) ^ (line & 7)) << 4);
}

__global__ void __launch_bounds__(kMmaThreads, 6)
    mma_pac_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                   const int32_t* __restrict__ table, int off_groups, int off_rows,
                   const __nv_bfloat16* __restrict__ q, const uint8_t* __restrict__ kpool,
                   const uint8_t* __restrict__ vpool, int64_t pool_tokens, int g, int hq_local,
                   float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml,
                   int off_merge_ptr, int off_merge_slot, long long* __restrict__ ctalog,
                   const int32_t* __restrict__ page_table, int page_shift, const int32_t* __restrict__ entry_of,
                   int32_t* __restrict__ cnt) {
  const long long t_start = ctalog ? global_ns() : 0;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // the merge may be scheduled early (it waits)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMmaStages * kMmaStageBytes);
  uint64_t* empty = full + kMmaStages;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* grp = table + off_groups + blockIdx.x * kGroupInts;
  const int kh = blockIdx.y;
  const int32_t* row = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  const int req = row[0], n_tok = row[1], slot = row[2];
  const int fz = row[3];  // >= 0: merge entry of (req, kv head 0): fold the TC partials in here
  const int nch = (n_tok + kMmaCT - 1) / kMmaCT;
  const int kv_tok = grp[kGrpKvTok];

  if (tid == 0) {
    for (int s = 0; s < kMmaStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kMmaWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kMmaWarps) {
    // ---------------- producer: one lane streams K and V boxes
    if (lane == 0) {
      tc::prefetch_tmap(&tmk);
      tc::prefetch_tmap(&tmv);
#if CODEC_SUFFIX_EVICT_FIRST
      const uint64_t pol = tc::policy_evict_first();  // read once: leave L2 to the shared-node tiles
#endif
      // pool row of chunk c (logical token; paged pool: a 32-token box
      // never crosses a page)
      auto chunk_row = [&](int c) {
        int x = kv_tok + c * kMmaCT;
        if (page_shift) x = (__ldg(page_table + (x >> page_shift)) << page_shift) | (x & ((1 << page_shift) - 1));
        return (int64_t)kh * pool_tokens + x;
      };
      // L2 prefetch of chunks [c0, c0 + n) (paged: chunk by chunk)
      auto prefetch = [&](int c0, int n) {
        if (c0 >= nch) return;
        n = min(n, nch - c0);
        if (!page_shift) {
          const int64_t y = chunk_row(c0);
          const uint32_t bytes = (uint32_t)min(n * kMmaCT, n_tok - c0 * kMmaCT) * 256;  // within the slice
          tc::bulk_prefetch_l2(kpool + y * 256, bytes);
          tc::bulk_prefetch_l2(vpool + y * 256, bytes);
        } else {
          for (int i = 0; i < n; ++i) {
            const int64_t y = chunk_row(c0 + i);
            tc::bulk_prefetch_l2(kpool + y * 256, kMmaBox);
            tc::bulk_prefetch_l2(vpool + y * 256, kMmaBox);
          }
        }
      };
      if (CODEC_MMA_PF > 0) prefetch(kMmaStages, CODEC_MMA_PF);
      for (int c = 0; c < nch; ++c) {
        const int s = c % kMmaStages;
        if (c >= kMmaStages) mbar_wait(&empty[s], ((c / kMmaStages) - 1) & 1);
        uint8_t* st = smem + s * kMmaStageBytes;
        const int y = (int)chunk_row(c);
        mbar_arrive_expect_tx(&full[s], kMmaStageBytes);
#if CODEC_SUFFIX_EVICT_FIRST
        tc::tma_load_3d_hint(st, &tmk, 0, 0, y, &full[s], pol);
        tc::tma_load_3d_hint(st + kMmaBox, &tmv, 0, 0, y, &full[s], pol);
#else
        tc::tma_load_3d(st, &tmk, 0, 0, y, &full[s]);
        tc::tma_load_3d(st + kMmaBox, &tmv, 0, 0, y, &full[s]);
#endif
        // keep CODEC_MMA_PF chunks beyond the ring requested, in groups
        if (CODEC_MMA_PF > 0 && c % CODEC_MMA_PF_GROUP == 0)
          prefetch(c + kMmaStages + CODEC_MMA_PF, CODEC_MMA_PF_GROUP);
      }
    }
  } else {
    // ---------------- consumers: 16 tokens of every stage each
    const int gid = lane >> 2, tig = lane & 3;
    const float cscale = 1.4426950408889634f * rsqrtf((float)kMmaD);
    // B fragments of Q^T (k = d, n = query head gid of this kv head)
    uint32_t qf[8][2];
    {
      const bool hv = gid < g;
      const uint32_t* qp = reinterpret_cast<const uint32_t*>(q + ((int64_t)req * hq_local + kh * g + (hv ? gid : 0)) * kMmaD);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qf[ks][0] = hv ? __ldg(qp + ks * 8 + tig) : 0u;
        qf[ks][1] = hv ? __ldg(qp + ks * 8 + 4 + tig) : 0u;
      }
    }
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {neg_inf<float>(), neg_inf<float>()};  // heads 2 tig, 2 tig + 1 (log2 units)
    float l_run[2] = {0.f, 0.f};                            // this lane's tokens only
    const int mat = lane >> 3, rr = lane & 7;
    for (int c = 0; c < nch; ++c) {
      const int s = c % kMmaStages;
      mbar_wait(&full[s], (c / kMmaStages) & 1);
      const uint32_t kb = smem_u32(smem + s * kMmaStageBytes), vb = kb + kMmaBox;
#pragma unroll 1
      for (int u = 0; u < kMmaSub; ++u) {
      const int wrow = 16 * (warp * kMmaSub + u);  // this step's first token row in the stage
      const int tk_qk = wrow + rr + ((mat & 1) << 3), ck_qk = mat >> 1;  // ldmatrix rows for S^T
      const int tk_pv = wrow + rr + ((mat >> 1) << 3), ck_pv = mat & 1;  // ldmatrix.trans rows for V^T
      // S^T (16 tokens x 8 heads) = K Q^T
      float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        uint32_t a[4];
        ldsm_x4(kb + mma_sw(tk_qk, 2 * ks + ck_qk), a);
        hmma(sc, a, qf[ks][0], qf[ks][1]);
      }
      // sc[0]: (token gid, head 2tig), [1]: (gid, 2tig+1), [2]: (gid+8, 2tig), [3]: (gid+8, 2tig+1)
      const int t0 = c * kMmaCT + wrow + gid;
      const bool va = t0 < n_tok, vb8 = t0 + 8 < n_tok;
      sc[0] = va ? sc[0] * cscale : neg_inf<float>();
      sc[1] = va ? sc[1] * cscale : neg_inf<float>();
      sc[2] = vb8 ? sc[2] * cscale : neg_inf<float>();
      sc[3] = vb8 ? sc[3] * cscale : neg_inf<float>();
      float mx0 = fmaxf(sc[0], sc[2]), mx1 = fmaxf(sc[1], sc[3]);
#pragma unroll
      for (int o = 4; o < 32; o <<= 1) {
        mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
        mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
      }
      // lazy rescale: the exponent reference moves only when a head's max
      // beats it by more than 2^8 (p <= 256 otherwise: exact enough in fp32)
      const bool n0 = mx0 > m_run[0] + 8.f, n1 = mx1 > m_run[1] + 8.f;
      if (__any_sync(0xffffffffu, n0 || n1)) {
        const float a0 = n0 ? fast_exp2(m_run[0] - mx0) : 1.f;  // 0 on a head's first live tile
        const float a1 = n1 ? fast_exp2(m_run[1] - mx1) : 1.f;
        l_run[0] *= a0;
        l_run[1] *= a1;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          acc[i][0] *= a0;
          acc[i][2] *= a0;
          acc[i][1] *= a1;
          acc[i][3] *= a1;
        }
        if (n0) m_run[0] = mx0;
        if (n1) m_run[1] = mx1;
      }
      const bool d0 = m_run[0] == neg_inf<float>(), d1 = m_run[1] == neg_inf<float>();
      const float p0 = d0 ? 0.f : fast_exp2(sc[0] - m_run[0]);
      const float p1 = d1 ? 0.f : fast_exp2(sc[1] - m_run[1]);
      const float p2 = d0 ? 0.f : fast_exp2(sc[2] - m_run[0]);
      const float p3 = d1 ? 0.f : fast_exp2(sc[3] - m_run[1]);
      l_run[0] += p0 + p2;
      l_run[1] += p1 + p3;
      // P^T as the B fragment (k = token, n = head): transpose the two 8x8 halves
      const uint32_t b0 = movm_t(pack2_bf16(p0, p1)), b1 = movm_t(pack2_bf16(p2, p3));
      // O^T (128 d x 8 heads) += V^T P^T
#pragma unroll
      for (int dm = 0; dm < 8; ++dm) {
        uint32_t a[4];
        ldsm_x4_t(vb + mma_sw(tk_pv, 2 * dm + ck_pv), a);
        hmma(acc[dm], a, b0, b1);
      }
      }
      // this warp's ldmatrix reads of the stage (generic proxy) before the
      // producer's next TMA write into it (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    // row sums over the lanes holding other tokens of the same heads
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], o);
      l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], o);
    }
    // stash (m, l, O^T) per warp in the ring (every stage consumed by now:
    // wait for the other consumer warp before overwriting)
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kMmaWarps) : "memory");
    float* wm = reinterpret_cast<float*>(smem) + warp * (16 + 8 * kMmaD);  // m[8], l[8], O[8][128]
    if (gid == 0) {
      wm[2 * tig] = m_run[0];
      wm[2 * tig + 1] = m_run[1];
      wm[8 + 2 * tig] = l_run[0];
      wm[8 + 2 * tig + 1] = l_run[1];
    }
#pragma unroll
    for (int dm = 0; dm < 8; ++dm) {
      const int dd = 16 * dm + gid;
      wm[16 + (2 * tig) * kMmaD + dd] = acc[dm][0];
      wm[16 + (2 * tig + 1) * kMmaD + dd] = acc[dm][1];
      wm[16 + (2 * tig) * kMmaD + dd + 8] = acc[dm][2];
      wm[16 + (2 * tig + 1) * kMmaD + dd + 8] = acc[dm][3];
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kMmaWarps) : "memory");
    const float* wb = reinterpret_cast<const float*>(smem);
    // fused merge: the other partials' slots and (m, l) of (req, kv head)
    float2* fz_ml = reinterpret_cast<float2*>(smem + 16384);       // [8 q heads][kFzMax]
    int* fz_slot = reinterpret_cast<int*>(smem + 16384 + 8 * kFzMax * 8);
    int fz_np = 0;
    if (fz >= 0) {
      const int entry = fz + kh;
      const int p0 = table[off_merge_ptr + entry] + 1;  // the own slot comes first
      fz_np = min(table[off_merge_ptr + entry + 1] - p0, kFzMax);
      const int h = tid / kFzMax, p = tid % kFzMax;
      if (h < g && p < fz_np) {
        const int sl = table[off_merge_slot + p0 + p];
        if (h == 0) fz_slot[p] = sl;
        fz_ml[h * kFzMax + p] = __ldg(reinterpret_cast<const float2*>(part_ml) + (int64_t)sl * hq_local + kh * g + h);
      }
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kMmaWarps) : "memory");
    }
#pragma unroll 4
    for (int idx = tid; idx < g * kMmaD; idx += 32 * kMmaWarps) {
      const int h = idx / kMmaD, e = idx % kMmaD;
      float M = neg_inf<float>();
#pragma unroll
      for (int w = 0; w < kMmaWarps; ++w) M = fmaxf(M, wb[w * (16 + 8 * kMmaD) + h]);
      float L = 0.f, O = 0.f;
#pragma unroll
      for (int w = 0; w < kMmaWarps; ++w) {
        const float* x = wb + w * (16 + 8 * kMmaD);
        if (x[h] == neg_inf<float>()) continue;
        const float f = fast_exp2(x[h] - M);
        L += x[8 + h] * f;
        O += x[16 + h * kMmaD + e] * f;
      }
      const int qh = kh * g + h;
      if (fz >= 0) {
        // fused merge (kern_merge.cu math): this suffix partial + the TC
        // pieces' partials of (req, kv head) -- they completed before this
        // kernel started; their (m, l) were staged in SMEM above
        const int np = fz_np;
        float Mn = M * 0.69314718055994530942f;  // natural-log units, like the stored partials
#pragma unroll
        for (int p = 0; p < kFzMax; ++p)
          if (p < np && fz_ml[h * kFzMax + p].y > 0.f) Mn = fmaxf(Mn, fz_ml[h * kFzMax + p].x);
        const float fo = __expf(M * 0.69314718055994530942f - Mn);
        float Lt = L * fo, Ot = O * fo;
        float ov[kFzMax];
#pragma unroll
        for (int p = 0; p < kFzMax; ++p)
          ov[p] = p < np ? __ldg(part_o + ((int64_t)fz_slot[p] * hq_local + qh) * kMmaD + e) : 0.f;
#pragma unroll
        for (int p = 0; p < kFzMax; ++p) {
          const float2 ml = fz_ml[h * kFzMax + p];
          const float w = (p < np && ml.y > 0.f) ? ml.y * __expf(ml.x - Mn) : 0.f;
          Lt += w;
          Ot += w * ov[p];
        }
        out[((int64_t)req * hq_local + qh) * kMmaD + e] = Ot / Lt;
      } else if (slot < 0) {
        out[((int64_t)req * hq_local + qh) * kMmaD + e] = O / L;
      } else {
        const int64_t ei = (int64_t)slot * hq_local + qh;
        part_o[ei * kMmaD + e] = O / L;
        if (e == 0) {
          part_ml[2 * ei] = M * 0.69314718055994530942f;  // natural-log units
          part_ml[2 * ei + 1] = L;
        }
      }
    }
    // readiness count of the merge entry of (req, kv head): g rows landed
    if (cnt && slot >= 0 && fz < 0) {
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"n"(32 * kMmaWarps) : "memory");
      if (tid == 0) {
        const int e = __ldg(entry_of + (int64_t)req * (hq_local / g) + kh);
        if (e >= 0) atomicAdd(cnt + e, g);
      }
    }
  }
  if (ctalog) {
    __syncthreads();
    cta_log(ctalog, kCtaLogGemv + blockIdx.y * gridDim.x + blockIdx.x, t_start);
  }
}

// ---------------------------------------------------------------------------
// K3m: lightly shared nodes -- a slice shared by 2..32/g requests (<= 32
// query-head rows) -- on the same warp-level tensor cores, so the node's
// K/V streams from HBM ONCE for all of them (the single-request kernel
// above would stream it once per request; the tcgen05 kernel would pad the
// rows to 256). The rows are split across consumer warps by columns: warp
// w owns query-head rows [8w, 8w + 8) of the group (n = 8 of m16n8k16) and
// runs every token of every stage for them, so each warp's (m, l, O^T) is
// final at the end -- no cross-warp merge. Rows of different requests see
// different visible counts (masks): the per-column limit masks the scores.
constexpr int kMultiWarps = 4;                          // consumer warps (<= 32 rows)
constexpr int kMultiThreads = 32 * (kMultiWarps + 1);   // + producer warp
constexpr int kMultiStages = 4;                         // fewer CTAs per SM than K3: a deeper ring
constexpr int kMultiCT = 32;                            // tokens per stage (two 16-token steps per warp)
constexpr int kMultiBox = kMultiCT * 256;               // one box: kMultiCT whole token rows
constexpr int kMultiStageBytes = 2 * kMultiBox;         // K box + V box
constexpr int kMultiSmem = kMultiStages * kMultiStageBytes + 1024 + 2 * kMultiStages * 8;

__global__ void __launch_bounds__(kMultiThreads, 3)
    mma_multi_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                     const int32_t* __restrict__ table, int off_groups, int off_rows,
                     const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, int hq_local,
                     float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml,
                     const int32_t* __restrict__ page_table, int page_shift, int32_t* __restrict__ done,
                     const int32_t* __restrict__ entry_of, int32_t* __restrict__ cnt) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + kMultiStages * kMultiStageBytes);
  uint64_t* empty = full + kMultiStages;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int32_t* grp = table + off_groups + blockIdx.x * kGroupInts;
  const int kh = blockIdx.y;
  const int32_t* rows = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  const int n_req = grp[kGrpNRows];
  const int n_cols = n_req * g;
  const int nbw = (n_cols + 7) >> 3;  // busy consumer warps
  const int nch = (grp[kGrpMaxVis] + kMultiCT - 1) / kMultiCT;
  const int kv_tok = grp[kGrpKvTok];

  if (tid == 0) {
    for (int s = 0; s < kMultiStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], nbw);
    }
    fence_barrier_init();
  }
  __syncthreads();

  if (warp == kMultiWarps) {
    // ---------------- producer: one lane streams 32-token K and V boxes
    if (lane == 0) {
      tc::prefetch_tmap(&tmk);
      tc::prefetch_tmap(&tmv);
#if CODEC_SUFFIX_EVICT_FIRST
      const uint64_t pol = tc::policy_evict_first();  // read once: leave L2 to the shared-node tiles
#endif
      for (int c = 0; c < nch; ++c) {
        const int s = c % kMultiStages;
        if (c >= kMultiStages) mbar_wait(&empty[s], ((c / kMultiStages) - 1) & 1);
        uint8_t* st = smem + s * kMultiStageBytes;
        int x = kv_tok + c * kMultiCT;  // paged pool: a 32-token box never crosses a page
        if (page_shift) x = (__ldg(page_table + (x >> page_shift)) << page_shift) | (x & ((1 << page_shift) - 1));
        const int y = kh * (int)pool_tokens + x;
        mbar_arrive_expect_tx(&full[s], kMultiStageBytes);
#if CODEC_SUFFIX_EVICT_FIRST
        tc::tma_load_3d_hint(st, &tmk, 0, 0, y, &full[s], pol);
        tc::tma_load_3d_hint(st + kMultiBox, &tmv, 0, 0, y, &full[s], pol);
#else
        tc::tma_load_3d(st, &tmk, 0, 0, y, &full[s]);
        tc::tma_load_3d(st + kMultiBox, &tmv, 0, 0, y, &full[s]);
#endif
      }
    }
  } else if (warp < nbw) {
    // ---------------- consumer warp: query-head rows [8 warp, 8 warp + 8)
    const int gid = lane >> 2, tig = lane & 3;
    const float cscale = 1.4426950408889634f * rsqrtf((float)kMmaD);
    const int c0 = 8 * warp;
    uint32_t qf[8][2];  // B fragments of Q^T: k = d, n = row c0 + gid
    {
      const int col = c0 + gid, ridx = col / g;
      const bool hv = col < n_cols;
      const int req = hv ? rows[ridx * kRowInts] : 0;
      const uint32_t* qp =
          reinterpret_cast<const uint32_t*>(q + ((int64_t)req * hq_local + kh * g + col % g) * kMmaD);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        qf[ks][0] = hv ? __ldg(qp + ks * 8 + tig) : 0u;
        qf[ks][1] = hv ? __ldg(qp + ks * 8 + 4 + tig) : 0u;
      }
    }
    // visible tokens of this lane's two score columns (0: padding column)
    const int ca = c0 + 2 * tig, cb = ca + 1;
    const int lim_a = ca < n_cols ? rows[(ca / g) * kRowInts + 1] : 0;
    const int lim_b = cb < n_cols ? rows[(cb / g) * kRowInts + 1] : 0;
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    float m_run[2] = {neg_inf<float>(), neg_inf<float>()};
    float l_run[2] = {0.f, 0.f};
    const int mat = lane >> 3, rr = lane & 7;
    for (int c = 0; c < nch; ++c) {
      const int s = c % kMultiStages;
      mbar_wait(&full[s], (c / kMultiStages) & 1);
      const uint32_t kb = smem_u32(smem + s * kMultiStageBytes), vb = kb + kMultiBox;
#pragma unroll
      for (int u = 0; u < kMultiCT / 16; ++u) {
        const int wrow = 16 * u;
        const int tk_qk = wrow + rr + ((mat & 1) << 3), ck_qk = mat >> 1;
        const int tk_pv = wrow + rr + ((mat >> 1) << 3), ck_pv = mat & 1;
        float sc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int ks = 0; ks < 8; ++ks) {
          uint32_t a[4];
          ldsm_x4(kb + mma_sw(tk_qk, 2 * ks + ck_qk), a);
          hmma(sc, a, qf[ks][0], qf[ks][1]);
        }
        // sc[0]: (token gid, col a), [1]: (gid, col b), [2]: (gid+8, a), [3]: (gid+8, b)
        const int t0 = c * kMultiCT + wrow + gid;
        sc[0] = t0 < lim_a ? sc[0] * cscale : neg_inf<float>();
        sc[1] = t0 < lim_b ? sc[1] * cscale : neg_inf<float>();
        sc[2] = t0 + 8 < lim_a ? sc[2] * cscale : neg_inf<float>();
        sc[3] = t0 + 8 < lim_b ? sc[3] * cscale : neg_inf<float>();
        float mx0 = fmaxf(sc[0], sc[2]), mx1 = fmaxf(sc[1], sc[3]);
#pragma unroll
        for (int o = 4; o < 32; o <<= 1) {
          mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, o));
          mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, o));
        }
        // lazy rescale (threshold 2^8, as in K3)
        const bool n0 = mx0 > m_run[0] + 8.f, n1 = mx1 > m_run[1] + 8.f;
        if (__any_sync(0xffffffffu, n0 || n1)) {
          const float a0 = n0 ? fast_exp2(m_run[0] - mx0) : 1.f;
          const float a1 = n1 ? fast_exp2(m_run[1] - mx1) : 1.f;
          l_run[0] *= a0;
          l_run[1] *= a1;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            acc[i][0] *= a0;
            acc[i][2] *= a0;
            acc[i][1] *= a1;
            acc[i][3] *= a1;
          }
          if (n0) m_run[0] = mx0;
          if (n1) m_run[1] = mx1;
        }
        const bool d0 = m_run[0] == neg_inf<float>(), d1 = m_run[1] == neg_inf<float>();
        const float p0 = d0 ? 0.f : fast_exp2(sc[0] - m_run[0]);
        const float p1 = d1 ? 0.f : fast_exp2(sc[1] - m_run[1]);
        const float p2 = d0 ? 0.f : fast_exp2(sc[2] - m_run[0]);
        const float p3 = d1 ? 0.f : fast_exp2(sc[3] - m_run[1]);
        l_run[0] += p0 + p2;
        l_run[1] += p1 + p3;
        const uint32_t b0 = movm_t(pack2_bf16(p0, p1)), b1 = movm_t(pack2_bf16(p2, p3));
#pragma unroll
        for (int dm = 0; dm < 8; ++dm) {
          uint32_t a[4];
          ldsm_x4_t(vb + mma_sw(tk_pv, 2 * dm + ck_pv), a);
          hmma(acc[dm], a, b0, b1);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
#pragma unroll
    for (int o = 4; o < 32; o <<= 1) {
      l_run[0] += __shfl_xor_sync(0xffffffffu, l_run[0], o);
      l_run[1] += __shfl_xor_sync(0xffffffffu, l_run[1], o);
    }
    // every consumer is past the ring: stage (m, l, O^T) of this warp's 8
    // rows there, then write each row as one 512-byte warp store
    asm volatile("bar.sync 1, %0;" ::"r"(32 * nbw) : "memory");
    float* wm = reinterpret_cast<float*>(smem) + warp * (16 + 8 * kMmaD);
    if (gid == 0) {
      wm[2 * tig] = m_run[0];
      wm[2 * tig + 1] = m_run[1];
      wm[8 + 2 * tig] = l_run[0];
      wm[8 + 2 * tig + 1] = l_run[1];
    }
#pragma unroll
    for (int dm = 0; dm < 8; ++dm) {
      const int dd = 16 * dm + gid;
      wm[16 + (2 * tig) * kMmaD + dd] = acc[dm][0];
      wm[16 + (2 * tig + 1) * kMmaD + dd] = acc[dm][1];
      wm[16 + (2 * tig) * kMmaD + dd + 8] = acc[dm][2];
      wm[16 + (2 * tig + 1) * kMmaD + dd + 8] = acc[dm][3];
    }
    __syncwarp();
    for (int j = 0; j < 8; ++j) {
      const int col = c0 + j;
      if (col >= n_cols) break;
      const int32_t* row = rows + (col / g) * kRowInts;
      const int req = row[0], slot = row[2], qh = kh * g + col % g;
      const float M = wm[j], L = wm[8 + j], inv = 1.f / L;
      const float4 o4 = reinterpret_cast<const float4*>(wm + 16 + j * kMmaD)[lane];
      const float4 r4 = make_float4(o4.x * inv, o4.y * inv, o4.z * inv, o4.w * inv);
      if (slot < 0) {
        reinterpret_cast<float4*>(out + ((int64_t)req * hq_local + qh) * kMmaD)[lane] = r4;
      } else {
        const int64_t ei = (int64_t)slot * hq_local + qh;
        reinterpret_cast<float4*>(part_o + ei * kMmaD)[lane] = r4;
        if (lane == 0) {
          part_ml[2 * ei] = M * 0.69314718055994530942f;  // natural-log units
          part_ml[2 * ei + 1] = L;
        }
        if (cnt) {  // readiness count of the merge entry of (req, kv head): one row landed
          __threadfence();
          __syncwarp();
          if (lane == 0) {
            const int e = __ldg(entry_of + (int64_t)req * (hq_local / g) + kh);
            if (e >= 0) atomicAdd(cnt + e, 1);
          }
        }
      }
    }
  }
  // completion count for the merge (it may start before this grid ends)
  __threadfence();
  __syncthreads();
  if (tid == 0 && done) atomicAdd(done, 1);
}

int32_t cuda_status(cudaError_t e, const char* what);
int32_t encode_pool_rows_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows);

int32_t launch_mma_gemv(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q,
                        const void* k, const void* v, int64_t pool_tokens, int g, int h_local, void* out,
                        void* part_o, void* part_ml, int off_merge_ptr, int off_merge_slot, cudaStream_t st,
                        long long* ctalog, bool after_tc, const int32_t* page_table, int page_shift,
                        const int32_t* entry_of, int32_t* cnt) {
  if (n_groups == 0) return CODEC_OK;
  if (g > 8) return fail(CODEC_ERR_UNSUPPORTED, "mma suffix kernel needs <= 8 query heads per kv head");
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_rows_map(&mk, k, (int64_t)h_local * pool_tokens, kMmaCT));
  CODEC_TRY(encode_pool_rows_map(&mv, v, (int64_t)h_local * pool_tokens, kMmaCT));
  cudaError_t e = cudaFuncSetAttribute(mma_pac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMmaSmem);
  if (e != cudaSuccess) return cuda_status(e, "mma smem attribute");
  e = cudaFuncSetAttribute(mma_pac_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  if (e != cudaSuccess) return cuda_status(e, "mma carveout attribute");
  // Programmatic dependent launch after the TC kernel: the suffix CTAs do
  // not read its output, so they may start on any SM the TC grid leaves
  // idle or has finished with (a running TC CTA holds its SM's whole
  // register file and shared memory, so nothing ever co-resides with it).
  // Not with the fused merge, which reads the TC partials.
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_groups, h_local);
  cfg.blockDim = dim3(kMmaThreads);
  cfg.dynamicSmemBytes = kMmaSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = after_tc ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, mma_pac_kernel, mk, mv, table, off_groups, off_rows, (const __nv_bfloat16*)q,
                         (const uint8_t*)k, (const uint8_t*)v, pool_tokens, g, h_local * g, (float*)out, (float*)part_o, (float*)part_ml, off_merge_ptr,
                         off_merge_slot, ctalog, page_table, page_shift, entry_of, cnt);
  if (e != cudaSuccess) return cuda_status(e, "mma gemv launch");
  return cuda_status(cudaGetLastError(), "mma gemv launch");
}

}  // namespace codec

namespace codec {
int32_t launch_mma_multi(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q,
                         const void* k, const void* v, int64_t pool_tokens, int g, int h_local, void* out,
                         void* part_o, void* part_ml, cudaStream_t st, bool pdl, const int32_t* page_table,
                         int page_shift, int32_t* done, const int32_t* entry_of, int32_t* cnt) {
  if (n_groups == 0) return CODEC_OK;
  if (g > 8) return fail(CODEC_ERR_UNSUPPORTED, "multi-request suffix kernel needs <= 8 query heads per kv head");
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_rows_map(&mk, k, (int64_t)h_local * pool_tokens, kMultiCT));
  CODEC_TRY(encode_pool_rows_map(&mv, v, (int64_t)h_local * pool_tokens, kMultiCT));
  cudaError_t e = cudaFuncSetAttribute(mma_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMultiSmem);
  if (e != cudaSuccess) return cuda_status(e, "multi smem attribute");
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(n_groups, h_local);
  cfg.blockDim = dim3(kMultiThreads);
  cfg.dynamicSmemBytes = kMultiSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, mma_multi_kernel, mk, mv, table, off_groups, off_rows, (const __nv_bfloat16*)q,
                         pool_tokens, g, h_local * g, (float*)out, (float*)part_o, (float*)part_ml, page_table,
                         page_shift, done, entry_of, cnt);
  if (e != cudaSuccess) return cuda_status(e, "multi launch");
  return cuda_status(cudaGetLastError(), "multi launch");
}
}  // namespace codec
