// K2t: lightly shared slices (2+ requests of nodes with <= 128 query-head
// rows) on the tcgen05 tensor cores, transposed -- SURVEY.md §8(a) a22 (the
// reference's pac_kernel, _kernels.pyx:16-54, for the nodes the M=256
// shared-node kernel would mostly pad).
//
// The shared-node kernel (kern_tc.cu) puts query-head rows on the MMA's M
// dimension: every KV tile costs an M=256 pair MMA plus a 256-row softmax
// whatever the rows, so a node read by 10 requests (40 rows) pays for 256.
// Here the tokens are M and the rows are N, so the work follows the rows:
//
//   S^T[tok][row]  = K_tile (M=128 tokens, K-major) x Q^T (N rows, K-major)
//   O^T[d][row]   += V_tile^T (M=128 d, MN-major view of the same TMA tile)
//                    x P^T (K=128 tokens, N rows; K-major, from SMEM)
//
// Two widths (template NG): NG = 1 takes up to 64 rows (4 softmax warps, P^T
// double-buffered), NG = 2 up to 128 rows (8 softmax warps, two column
// groups of 64 that share each S^T / P^T tile; P^T single-buffered so SMEM
// holds 128 rows of Q). A CTA loops over (slice group, kv head) items of the
// table (one per CTA by default). Warp roles: softmax (thread = token lane of
// S^T, then d lane of O^T), one TMA producer warp, one MMA issuer warp.
// TMEM: S^T double-buffered and O^T (3 x 64 NG columns).
//
// Softmax without a per-tile cross-thread max: every column keeps a
// reference m (log2 units, SMEM) and a tile exponentiates against it; only
// when a score passes m + 8 anywhere in its column group (bar.red.or over
// the group's 128 threads) -- always on an item's first tile, rarely after --
// the group takes the slow path: column maxima through SMEM, rescale of the
// per-thread row sums and of its O^T columns in TMEM (after the previous PV
// landed). The two column groups never synchronise with each other (their
// columns are independent). Row sums are per-thread partials over the
// thread's tokens, reduced once in the epilogue.
#include <algorithm>

#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "tc_ptx.cuh"

namespace codec {
namespace {

constexpr int kTctBN = 128;                     // tokens per KV tile (MMA M of S^T)
constexpr int kTctD = 128;                      // head dim (MMA M of O^T)
constexpr int kTileBytes = kTctBN * kTctD * 2;  // 32 KB: two SW128 atom columns [64 d][128 rows]
constexpr int kAtomTile = kTileBytes / 2;       // 16 KB
// narrow variant's K / V ring depths: 2 / 3 measured 80.1 vs 80.7 us on cfg3
// (2 / 2), 3 / 2 81.4; cfg4 unchanged
#ifndef CODEC_TCT_KSTAGES
#define CODEC_TCT_KSTAGES 2
#define CODEC_TCT_VSTAGES 3
#endif
constexpr int kMaxStages = 3;
constexpr float kRefSlack = 8.f;  // a score may pass its column reference by 2^8

template <int NG>
struct TctCfg {
  static constexpr int kRows = 64 * NG;                    // columns (rows of Q) per item, at most
  static constexpr int kSoftmaxWarps = 4 * NG;
  // NG = 2: three whole warpgroups (two idle warps) so setmaxnreg can move
  // registers from the role warps (56) to the softmax warps (224): 384 x 168
  // at launch covers 256 x 224 + 128 x 56
  static constexpr int kThreads = NG == 1 ? 6 * 32 : 12 * 32;
  static constexpr int kProducerWarp = kSoftmaxWarps, kMmaWarp = kSoftmaxWarps + 1;
  static constexpr int kRegsSoftmax = 224, kRegsOther = 56;
  static_assert(NG == 1 || 256 * kRegsSoftmax + 128 * kRegsOther <= kThreads * 168, "setmaxnreg pool");
  static constexpr int kQtBytes = kRows * kTctD * 2;      // Q rows (B of S^T), two atom columns
  static constexpr int kAtomQ = kQtBytes / 2;
  static constexpr int kPBuf = NG == 1 ? 2 : 1;           // P^T buffers
  static constexpr int kPtBytes = kRows * kTctBN * 2;     // P^T (B of O^T), rows x tokens, K-major
  static constexpr int kAtomP = kPtBytes / 2;
  static constexpr int kOffQ = 0;
  static constexpr int kOffK = kOffQ + kQtBytes;
  // K / V ring depths (the narrow variant's can be raised for experiments)
  static constexpr int kKSt = NG == 1 ? CODEC_TCT_KSTAGES : 2, kVSt = NG == 1 ? CODEC_TCT_VSTAGES : 2;
  static_assert(kKSt <= kMaxStages && kVSt <= kMaxStages, "ring depth");
  static constexpr int kOffV = kOffK + kKSt * kTileBytes;
  static constexpr int kOffP = kOffV + kVSt * kTileBytes;
  static constexpr int kOffRed = kOffP + kPBuf * kPtBytes;       // [4 quadrants][kRows] f32 column reductions
  static constexpr int kOffRow = kOffRed + 4 * kRows * 4;         // per column: vis, slot, out row, request
  static constexpr int kOffMisc = kOffRow + 4 * kRows * 4;        // [kRows] f32 m, min visible, [kRows] f32 m steps
  static constexpr int kOffDm = kOffMisc + kRows * 4 + 16;
  static constexpr int kOffBar = kOffDm + kRows * 4;
  static constexpr int kSmem = kOffBar + 256 + 1024;              // + alignment slack
  static_assert(kSmem <= 232448, "exceeds the 227 KB opt-in shared memory");
  static constexpr uint32_t kColS = 0, kColO = 2 * kRows, kTmemCols = NG == 1 ? 256 : 512;
};

struct TctBars {
  uint64_t k_full[kMaxStages], k_empty[kMaxStages], v_full[kMaxStages], v_empty[kMaxStages];
  uint64_t s_full[2], s_free[2], p_full[2], p_empty[2];
  uint64_t q_full, o_free;  // per item: Q rows staged / the epilogue read O^T
  uint64_t pv_done[4];  // PV(t) completes pv_done[t % 4]: a parity wait never sees a phase two behind
  uint32_t tmem_slot;
};

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
// bar.red.or over the n threads of named barrier id
__device__ __forceinline__ bool named_or(int id, int n, bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred p, q;\n\t"
      "setp.ne.u32 p, %1, 0;\n\t"
      "bar.red.or.pred q, %2, %3, p;\n\t"
      "selp.u32 %0, 1, 0, q;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id), "r"(n)
      : "memory");
  return r != 0;
}
// (volatile: keeps loop-invariant SMEM tables out of registers)
__device__ __forceinline__ int4 lds_v4(const void* p) {
  int4 v;
  asm volatile("ld.shared.v4.s32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(smem_u32(p)));
  return v;
}
__device__ __forceinline__ void sts_u16(uint32_t addr, unsigned short v) {
  asm volatile("st.shared.u16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

template <int N>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, uint32_t* r) {
  static_assert(N % 16 == 0, "16-column granules");
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tc::tmem_ld32(taddr + c, r + c);
  if constexpr (N % 32 == 16) tc::tmem_ld16(taddr + (N - 16), r + (N - 16));
}

// One column group's whole item for N (padded) columns starting at column
// c0: tiles, then the epilogue (row sums, O^T out of TMEM, one coalesced
// 128-byte warp store per row and d quarter). bar_or / bar_grp: the group's
// named barriers (128 threads).
template <int NG, int N>
__device__ __forceinline__ void softmax_unit(uint8_t* smem, TctBars* bars, uint32_t tmem, int jb, int n_tiles,
                                             int c0, int n_cols, int bar_or, int bar_grp, int kh, int g, int hq_local,
                                             float* __restrict__ out, float* __restrict__ part_o,
                                             float* __restrict__ part_ml, const int32_t* __restrict__ entry_of,
                                             int32_t* __restrict__ cnt) {
  using C = TctCfg<NG>;
  const int lane = threadIdx.x & 31, quad = (threadIdx.x >> 5) & 3;
  const int t = quad * 32 + lane;  // token lane of S^T, d lane of O^T
  const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
  const float cs = 1.4426950408889634f * rsqrtf((float)kTctD);
  const int32_t* rinfo = reinterpret_cast<const int32_t*>(smem + C::kOffRow);  // [4][kRows]: vis, slot, out row, req
  float* red = reinterpret_cast<float*>(smem + C::kOffRed);
  float* mref = reinterpret_cast<float*>(smem + C::kOffMisc);  // column references (uniform: read as broadcasts)
  float* dm = reinterpret_cast<float*>(smem + C::kOffDm);      // m_old - m_new of the last slow path
  const int min_vis = reinterpret_cast<const int32_t*>(smem + C::kOffMisc)[C::kRows];
  const uint32_t pbase = smem_u32(smem + C::kOffP);
  // this thread's byte within a P^T row: atom column (t / 64), 16-byte chunk
  // ((t % 64) / 8) XOR (row % 8), element t % 8
  const int patom = (t >> 6) * C::kAtomP, pchunk = (t & 63) >> 3, pin = (t & 7) * 2;

  float l[N];  // this thread's partial row sums
#pragma unroll
  for (int n = 0; n < N; ++n) l[n] = 0.f;
  if (t < 64) mref[c0 + t] = 0.f;  // tile 0 always takes the slow path: its x are absolute
  named_sync(bar_grp, 128);
  for (int j = 0; j < n_tiles; ++j) {
    const int jg = jb + j, b = jg & 1;  // the CTA's tile sequence runs on across its items
    mbar_wait(&bars->s_full[b], (jg >> 1) & 1);
    tc::fence_after();
    uint32_t sr[N];
    tmem_ld_cols<N>(tmem + lane_base + C::kColS + b * C::kRows + c0, sr);
    tc::wait_ld();
    tc::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->s_free[b]);
    // x = score * log2(e) / sqrt(d) - m, -inf past a column's visible tokens
    float x[N];
    const int tok = j * kTctBN + t;
    const bool masked = j * kTctBN + kTctBN > min_vis;  // a tile some column does not see whole
    float over = neg_inf<float>();
#pragma unroll
    for (int n = 0; n < N; n += 4) {
      const int4 m4 = lds_v4(mref + c0 + n);
      const float mm[4] = {__int_as_float(m4.x), __int_as_float(m4.y), __int_as_float(m4.z), __int_as_float(m4.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u) x[n + u] = fmaf(__uint_as_float(sr[n + u]), cs, -mm[u]);
      if (masked) {
        const int4 v4 = lds_v4(rinfo + c0 + n);
        const int vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (tok >= vv[u]) x[n + u] = neg_inf<float>();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) over = fmaxf(over, x[n + u]);
    }
    if (named_or(bar_or, 128, j == 0 || over > kRefSlack)) {
      // slow path: raise the references to this tile's column maxima (tile
      // 0: set them to its maxima; a column with no visible token keeps 0)
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float v = warp_max(x[n]);
        if (lane == 0) red[quad * C::kRows + c0 + n] = v;
      }
      named_sync(bar_grp, 128);
      if (t < N) {
        const int c = c0 + t;
        const float tm = fmaxf(fmaxf(red[c], red[C::kRows + c]), fmaxf(red[2 * C::kRows + c], red[3 * C::kRows + c]));
        // x is relative to the old m: the new m is m + up
        const float up = j == 0 ? (tm > neg_inf<float>() ? tm : 0.f) : fmaxf(tm, 0.f);
        dm[c] = -up;
        mref[c] += up;
      }
      named_sync(bar_grp, 128);
#pragma unroll
      for (int n = 0; n < N; n += 4) {
        const int4 d4 = lds_v4(dm + c0 + n);
        const float dd[4] = {__int_as_float(d4.x), __int_as_float(d4.y), __int_as_float(d4.z), __int_as_float(d4.w)};
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[n + u] += dd[u];
          if (j > 0) l[n + u] *= fast_exp2(dd[u]);
        }
      }
      if (j > 0) {  // O^T (thread = d lane) rescaled once PV(j - 1) landed; PV(j) waits for P(j)
        mbar_wait(&bars->pv_done[(jg - 1) & 3], ((jg - 1) >> 2) & 1);
        tc::fence_after();
#pragma unroll
        for (int c = 0; c < N; c += 16) {
          uint32_t o[16];
          tc::tmem_ld16(tmem + lane_base + C::kColO + c0 + c, o);
          tc::wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * fast_exp2(dm[c0 + c + u]));
          tc::tmem_st16(tmem + lane_base + C::kColO + c0 + c, o);
        }
        tc::wait_st();
      }
    }
    // P^T(j) into SMEM once the PV that last read its buffer landed
    const int pb_i = jg % C::kPBuf;
    if (jg >= C::kPBuf) mbar_wait(&bars->p_empty[pb_i], ((jg - C::kPBuf) / C::kPBuf) & 1);
    const uint32_t pb = pbase + pb_i * C::kPtBytes + patom + pin;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float p = fast_exp2(x[n]);
      l[n] += p;
      const int row = c0 + n;
      sts_u16(pb + row * 128 + ((pchunk ^ (row & 7)) << 4), __bfloat16_as_ushort(__float2bfloat16_rn(p)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> MMA operand reads
    tc::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->p_full[pb_i]);
  }

  // ---- epilogue: row sums over the CTA's tokens, then O^T / l
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const float v = warp_sum(l[n]);
    if (lane == 0) red[quad * C::kRows + c0 + n] = v;
  }
  named_sync(bar_grp, 128);
  const int jl = jb + n_tiles - 1;
  mbar_wait(&bars->pv_done[jl & 3], (jl >> 2) & 1);
  tc::fence_after();
  uint32_t o[N];
  tmem_ld_cols<N>(tmem + lane_base + C::kColO + c0, o);
  tc::wait_ld();
  tc::fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&bars->o_free);  // the next item's first PV may overwrite O^T
#pragma unroll
  for (int n = 0; n < N; ++n) {
    if (n < n_cols) {
      const int c = c0 + n;
      const float L = red[c] + red[C::kRows + c] + red[2 * C::kRows + c] + red[3 * C::kRows + c];
      const int slot = rinfo[C::kRows + c], orow = rinfo[2 * C::kRows + c];
      float* dst = (slot < 0 ? out : part_o) + (int64_t)orow * kTctD;
      asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(dst + t), "f"(__uint_as_float(o[n]) / L)
                   : "memory");
    }
  }
  if (t < n_cols && rinfo[C::kRows + c0 + t] >= 0) {
    const int c = c0 + t, orow = rinfo[2 * C::kRows + c];
    part_ml[2 * (int64_t)orow] = mref[c] * 0.69314718055994530942f;  // natural-log units
    part_ml[2 * (int64_t)orow + 1] = red[c] + red[C::kRows + c] + red[2 * C::kRows + c] + red[3 * C::kRows + c];
  }
  if (cnt) {  // readiness counts of the merge entries: every store of the group's rows fenced first
    __threadfence();
    named_sync(bar_grp, 128);
    if (t < n_cols && rinfo[C::kRows + c0 + t] >= 0 && (c0 + t) % g == 0) {
      const int e = __ldg(entry_of + (int64_t)rinfo[3 * C::kRows + c0 + t] * (hq_local / g) + kh);
      if (e >= 0) atomicAdd(cnt + e, g);  // the g rows of (request, kv head)
    }
  }
}

template <int NG>
__global__ void __launch_bounds__(TctCfg<NG>::kThreads, 1)
    tct_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
               const int32_t* __restrict__ table, int off_groups, int off_rows, int n_groups, int h_local,
               const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, float* __restrict__ out,
               float* __restrict__ part_o, float* __restrict__ part_ml, const int32_t* __restrict__ page_table,
               int page_shift, int32_t* __restrict__ done, const int32_t* __restrict__ entry_of,
               int32_t* __restrict__ cnt) {
  using C = TctCfg<NG>;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  TctBars* bars = reinterpret_cast<TctBars*>(smem + C::kOffBar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hq_local = g * h_local, n_items = n_groups * h_local;
  // item it = (group it / h_local, kv head it % h_local); a CTA takes items
  // blockIdx.x, + gridDim.x, ...
  struct Item {
    const int32_t* rows;
    int kh, n_cols, npad, n_tiles, kv_tok;
  };
  auto item = [&](int it) {
    const int32_t* grp = table + off_groups + (it / h_local) * kGroupInts;
    Item x;
    x.kh = it % h_local;
    x.rows = table + off_rows + grp[kGrpRowBegin] * kRowInts;
    x.n_cols = grp[kGrpNRows] * g;
    x.npad = (x.n_cols + 15) & ~15;
    x.n_tiles = (grp[kGrpMaxVis] + kTctBN - 1) / kTctBN;
    x.kv_tok = grp[kGrpKvTok];
    return x;
  };

  if (tid == 0) {
    for (int s = 0; s < kMaxStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->s_free[b], C::kSoftmaxWarps);
      mbar_init(&bars->p_full[b], C::kSoftmaxWarps);
      mbar_init(&bars->p_empty[b], 1);
    }
    mbar_init(&bars->q_full, C::kSoftmaxWarps);
    mbar_init(&bars->o_free, C::kSoftmaxWarps);
    for (int i = 0; i < 4; ++i) mbar_init(&bars->pv_done[i], 1);
    fence_barrier_init();
  }
  if (warp == C::kMmaWarp) tc::tmem_alloc(&bars->tmem_slot, C::kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;
  if constexpr (NG == 2) {
    if (warp >= C::kSoftmaxWarps)
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(C::kRegsOther));
    else
      asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(C::kRegsSoftmax));
  }

  if (warp < C::kSoftmaxWarps) {
    const int grp = warp >> 2;  // column group: columns [64 grp, 64 grp + 64)
    const int nsm = 32 * C::kSoftmaxWarps;
    int32_t* rinfo = reinterpret_cast<int32_t*>(smem + C::kOffRow);
    int32_t* minv = reinterpret_cast<int32_t*>(smem + C::kOffMisc) + C::kRows;
    int tiles_done = 0;  // tiles of this CTA's earlier items (barrier phases run on across items)
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = item(it);
      if (x.n_cols > C::kRows || (NG == 2 && x.n_cols <= 64)) __trap();  // the host routes by width
      // ---- per column: visible tokens, slot, output row, request; Q rows
      // (the previous item's S MMAs are complete: its tiles were consumed)
      if (tid == 0) *minv = 0x7fffffff;
      named_sync(1, nsm);
      if (tid < C::kRows) {
        int vis = 0, slot = 0, orow = 0, req = 0;
        if (tid < x.n_cols) {
          const int32_t* row = x.rows + (tid / g) * kRowInts;
          req = row[0];
          vis = row[1];
          slot = row[2];
          const int qh = x.kh * g + tid % g;
          orow = slot < 0 ? req * hq_local + qh : slot * hq_local + qh;
          atomicMin(minv, vis);
        }
        rinfo[tid] = vis;
        rinfo[C::kRows + tid] = slot;
        rinfo[2 * C::kRows + tid] = orow;
        rinfo[3 * C::kRows + tid] = req;
      }
      // Q rows as the K-major SW128 B operand: 16-byte chunk c of row n at
      // atom column c / 8, row n, chunk (c % 8) XOR (n % 8); padding rows zero
#pragma unroll
      for (int i = 0; i < (C::kRows * 16) / (32 * C::kSoftmaxWarps); ++i) {
        const int e = i * nsm + tid, n = e >> 4, c = e & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (n < x.n_cols) {
          const int req = __ldg(x.rows + (n / g) * kRowInts);
          v = __ldg(reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + x.kh * g + n % g) * kTctD) + c);
        }
        *reinterpret_cast<uint4*>(smem + C::kOffQ + (c >> 3) * C::kAtomQ + n * 128 + (((c & 7) ^ (n & 7)) << 4)) = v;
      }
      tc::fence_proxy_async_smem();
      named_sync(1, nsm);  // row info and min_vis before the softmax reads them
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->q_full);
      const int c0 = 64 * grp;
      const int cols = min(64, x.n_cols - c0), npad = min(64, x.npad - c0);
      const int bo = 2 + grp, bg = 4 + grp;
#define CODEC_TCT_UNIT(NN)                                                                                       \
  softmax_unit<NG, NN>(smem, bars, tmem, tiles_done, x.n_tiles, c0, cols, bo, bg, x.kh, g, hq_local, out, part_o, \
                       part_ml, entry_of, cnt)
      switch (npad) {
        case 16: CODEC_TCT_UNIT(16); break;
        case 32: CODEC_TCT_UNIT(32); break;
        case 48: CODEC_TCT_UNIT(48); break;
        default: CODEC_TCT_UNIT(64); break;
      }
#undef CODEC_TCT_UNIT
      tiles_done += x.n_tiles;
      named_sync(1, nsm);  // every thread's epilogue reads of the row info done before the next item's
    }
  } else if (warp == C::kProducerWarp) {
    // ---- TMA producer: K and V tiles, both SW128 atom columns in one op
    if (lane == 0) {
      tc::prefetch_tmap(&tmk);
      tc::prefetch_tmap(&tmv);
      const uint64_t pol = tc::policy_evict_first();  // read by this CTA only
      int jg = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item x = item(it);
        for (int j = 0; j < x.n_tiles; ++j, ++jg) {
          const int ks = jg % C::kKSt, vs = jg % C::kVSt;
          int xt = x.kv_tok + j * kTctBN;  // paged pool: a 128-token tile never crosses a page
          if (page_shift)
            xt = (__ldg(page_table + (xt >> page_shift)) << page_shift) | (xt & ((1 << page_shift) - 1));
          const int y = x.kh * (int)pool_tokens + xt;
          if (jg >= C::kKSt) mbar_wait(&bars->k_empty[ks], ((jg - C::kKSt) / C::kKSt) & 1);
          mbar_arrive_expect_tx(&bars->k_full[ks], kTileBytes);
          tc::tma_load_3d_hint(smem + C::kOffK + ks * kTileBytes, &tmk, 0, y, 0, &bars->k_full[ks], pol);
          if (jg >= C::kVSt) mbar_wait(&bars->v_empty[vs], ((jg - C::kVSt) / C::kVSt) & 1);
          mbar_arrive_expect_tx(&bars->v_full[vs], kTileBytes);
          tc::tma_load_3d_hint(smem + C::kOffV + vs * kTileBytes, &tmv, 0, y, 0, &bars->v_full[vs], pol);
        }
      }
    }
  } else if (warp == C::kMmaWarp) {
    // ---- MMA issuer: S^T(j), then PV(j - 1) (the tensor pipe computes
    // S^T(j + 1) while the softmax works on tile j)
    const uint32_t sbase = smem_u32(smem);
    int jg = 0, u = 0;
    auto pv = [&](int tp, int j_item, uint32_t idesc_o) {
      const int vb = tp % C::kVSt, pb = tp % C::kPBuf;
      mbar_wait(&bars->p_full[pb], (tp / C::kPBuf) & 1);
      mbar_wait(&bars->v_full[vb], (tp / C::kVSt) & 1);
      tc::fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < kTctBN / 16; ++k) {
          // A = V^T: MN-major, 64-d blocks 16 KB apart (LBO), 8-token groups 1 KB apart (SBO)
          const uint64_t av = tc::smem_desc(sbase + C::kOffV + vb * kTileBytes + k * 2048, kAtomTile, 1024);
          const uint64_t bp =
              tc::smem_desc(sbase + C::kOffP + pb * C::kPtBytes + (k >> 2) * C::kAtomP + (k & 3) * 32, 16, 1024);
          tc::mma_f16_ss(tmem + C::kColO, av, bp, idesc_o, (j_item > 0 || k > 0) ? 1u : 0u);
        }
        tc::commit(&bars->v_empty[vb]);
        tc::commit(&bars->p_empty[pb]);
        tc::commit(&bars->pv_done[tp & 3]);
      }
      __syncwarp();
    };
    for (int it = blockIdx.x; it < n_items; it += gridDim.x, ++u) {
      const Item x = item(it);
      const uint32_t idesc_s = tc::idesc_bf16(128, x.npad, false, false);
      const uint32_t idesc_o = tc::idesc_bf16(128, x.npad, true, false);
      mbar_wait(&bars->q_full, u & 1);
      for (int j = 0; j < x.n_tiles; ++j, ++jg) {
        const int s = jg & 1, ks = jg % C::kKSt;  // S buffer, K stage
        mbar_wait(&bars->k_full[ks], (jg / C::kKSt) & 1);
        if (jg >= 2) mbar_wait(&bars->s_free[s], ((jg - 2) >> 1) & 1);
        tc::fence_after();
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kTctD / 16; ++k) {
            const uint64_t ak =
                tc::smem_desc(sbase + C::kOffK + ks * kTileBytes + (k >> 2) * kAtomTile + (k & 3) * 32, 16, 1024);
            const uint64_t bq = tc::smem_desc(sbase + C::kOffQ + (k >> 2) * C::kAtomQ + (k & 3) * 32, 16, 1024);
            tc::mma_f16_ss(tmem + C::kColS + s * C::kRows, ak, bq, idesc_s, k > 0 ? 1u : 0u);
          }
          tc::commit(&bars->k_empty[ks]);
          tc::commit(&bars->s_full[s]);
        }
        __syncwarp();
        if (j >= 1) {
          pv(jg - 1, j - 1, idesc_o);
        } else if (u > 0) {
          mbar_wait(&bars->o_free, (u - 1) & 1);  // the previous item's epilogue read O^T
          tc::fence_after();
        }
      }
      pv(jg - 1, x.n_tiles - 1, idesc_o);
    }
    // every commit's arrival landed before the CTA exits (a late one would
    // hit the SMEM of the next CTA on this SM): the last phase of each
    for (int s = 0; s < C::kKSt; ++s) {
      const int uses = (jg - s + C::kKSt - 1) / C::kKSt;
      if (uses > 0) mbar_wait(&bars->k_empty[s], (uses - 1) & 1);
    }
    for (int s = 0; s < C::kVSt; ++s) {
      const int uses = (jg - s + C::kVSt - 1) / C::kVSt;
      if (uses > 0) mbar_wait(&bars->v_empty[s], (uses - 1) & 1);
    }
    for (int s = 0; s < C::kPBuf; ++s) {
      const int uses = (jg - s + C::kPBuf - 1) / C::kPBuf;
      if (uses > 0) mbar_wait(&bars->p_empty[s], (uses - 1) & 1);
    }
    for (int i = 0; i < 4; ++i) {
      const int uses = (jg - i + 3) / 4;
      if (uses > 0) mbar_wait(&bars->pv_done[i], (uses - 1) & 1);
    }
  }
  // completion count for the merge (it may start before this grid ends):
  // one per item, as the table's CTA count expects
  __threadfence();
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  if (tid == 0 && done) {
    int mine = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) ++mine;
    if (mine) atomicAdd(done, mine);
  }
  if (warp == C::kMmaWarp) tc::tmem_dealloc(tmem, C::kTmemCols);
}

template <int NG>
int32_t launch_tct_w(const CUtensorMap& mk, const CUtensorMap& mv, const int32_t* table, int n_groups, int off_groups,
                     int off_rows, const void* q, int64_t pool_tokens, int g, int h_local, void* out, void* part_o,
                     void* part_ml, cudaStream_t st, bool pdl, const int32_t* page_table, int page_shift,
                     int32_t* done, const int32_t* entry_of, int32_t* cnt, int max_ctas);

}  // namespace

int32_t cuda_status(cudaError_t e, const char* what);
int32_t encode_pool_halves_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows);

namespace {
template <int NG>
int32_t launch_tct_w(const CUtensorMap& mk, const CUtensorMap& mv, const int32_t* table, int n_groups, int off_groups,
                     int off_rows, const void* q, int64_t pool_tokens, int g, int h_local, void* out, void* part_o,
                     void* part_ml, cudaStream_t st, bool pdl, const int32_t* page_table, int page_shift,
                     int32_t* done, const int32_t* entry_of, int32_t* cnt, int max_ctas) {
  using C = TctCfg<NG>;
  cudaError_t e = cudaFuncSetAttribute(tct_kernel<NG>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  if (e != cudaSuccess) return cuda_status(e, "tct smem attribute");
  const int n_items = n_groups * h_local;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(max_ctas > 0 ? std::min(n_items, max_ctas) : n_items);
  cfg.blockDim = dim3(C::kThreads);
  cfg.dynamicSmemBytes = C::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, tct_kernel<NG>, mk, mv, table, off_groups, off_rows, n_groups, h_local,
                         (const __nv_bfloat16*)q, pool_tokens, g, (float*)out, (float*)part_o, (float*)part_ml,
                         page_table, page_shift, done, entry_of, cnt);
  if (e != cudaSuccess) return cuda_status(e, "tct launch");
  return cuda_status(cudaGetLastError(), "tct launch");
}
}  // namespace

// groups: the kKindTct records (multi-request table format) -- the first
// n_groups - n_wide of at most 64 rows, then n_wide of 65..128 rows -- as
// (group, local kv head) items; pdl: programmatic dependent of the previous
// launch (the wide grid follows the narrow one)
int32_t launch_tct(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q, const void* k,
                   const void* v, int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                   cudaStream_t st, bool pdl, const int32_t* page_table, int page_shift, int32_t* done,
                   const int32_t* entry_of, int32_t* cnt, int max_ctas, int n_wide) {
  if (n_groups == 0) return CODEC_OK;
  if (g > 64) return fail(CODEC_ERR_UNSUPPORTED, "transposed tensor-core kernel: g = %d > 64", g);
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_halves_map(&mk, k, (int64_t)h_local * pool_tokens, kTctBN));
  CODEC_TRY(encode_pool_halves_map(&mv, v, (int64_t)h_local * pool_tokens, kTctBN));
  const int n_narrow = n_groups - n_wide;
  if (n_narrow > 0)
    CODEC_TRY(launch_tct_w<1>(mk, mv, table, n_narrow, off_groups, off_rows, q, pool_tokens, g, h_local, out, part_o,
                              part_ml, st, pdl, page_table, page_shift, done, entry_of, cnt, max_ctas));
  if (n_wide > 0)
    CODEC_TRY(launch_tct_w<2>(mk, mv, table, n_wide, off_groups + kGroupInts * n_narrow, off_rows, q, pool_tokens, g,
                              h_local, out, part_o, part_ml, st, pdl || n_narrow > 0, page_table, page_shift, done,
                              entry_of, cnt, max_ctas));
  return CODEC_OK;
}

}  // namespace codec
