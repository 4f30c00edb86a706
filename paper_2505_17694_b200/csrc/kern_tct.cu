// K2t: lightly shared slices (17..64 query-head rows per CTA) on the
// tcgen05 tensor cores, transposed -- SURVEY.md §8(a) a22 (the reference's
// pac_kernel, _kernels.pyx:16-54, for the nodes between the multi-request
// mma.sync kernel and the M=256 shared-node kernel).
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
// One CTA = one (slice group, kv head), grid (groups, h_local) like the
// multi-request kernel, whose table records it shares. Warps 0-3 are the
// softmax (thread = token lane of S^T, then d lane of O^T), warp 4 the TMA
// producer, warp 5 the MMA issuer. TMEM: S^T double-buffered (2 x 64
// columns) and O^T (64 columns).
//
// Softmax without a per-tile cross-thread max: every column keeps a CTA-wide
// reference m (log2 units) and a tile exponentiates against it; only when a
// score passes m + 8 anywhere in the CTA (bar.red.or over the 128 softmax
// threads) -- always on the first tile, rarely after -- the tile takes the
// slow path: column maxima through SMEM, rescale of the per-thread row sums
// and of O^T in TMEM (after the previous PV landed). Row sums are per-thread
// partials over the thread's tokens, reduced once in the epilogue.
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
constexpr int kTctThreads = 6 * 32;
constexpr int kTileBytes = kTctBN * kTctD * 2;  // 32 KB: two SW128 atom columns [64 d][128 rows]
constexpr int kAtomTile = kTileBytes / 2;       // 16 KB
constexpr int kQtBytes = kTctRows * kTctD * 2;  // 16 KB: Q rows (B of S^T), atom columns of 64 rows
constexpr int kAtomQ = kQtBytes / 2;            // 8 KB
constexpr int kPtBytes = kTctRows * kTctBN * 2; // 16 KB: P^T (B of O^T), rows x tokens, K-major
constexpr int kAtomP = kPtBytes / 2;            // 8 KB
constexpr int kStages = 2;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + kQtBytes;
constexpr int kOffV = kOffK + kStages * kTileBytes;
constexpr int kOffP = kOffV + kStages * kTileBytes;
constexpr int kOffRed = kOffP + 2 * kPtBytes;           // [4 warps][64] f32 column reductions
constexpr int kOffRow = kOffRed + 4 * kTctRows * 4;     // per column: vis, slot, out row, request
constexpr int kOffMisc = kOffRow + 4 * kTctRows * 4;    // [64] f32 m, min visible, [64] f32 m steps
constexpr int kOffBar = kOffMisc + 2 * kTctRows * 4 + 16;
constexpr int kTctSmem = kOffBar + 256 + 1024;          // + alignment slack
static_assert(kTctSmem <= 232448, "exceeds the 227 KB opt-in shared memory");
constexpr uint32_t kColS = 0, kColO = 2 * kTctRows, kTmemCols = 256;
constexpr float kRefSlack = 8.f;  // a score may pass its column reference by 2^8

struct TctBars {
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
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
template <int N>
__device__ __forceinline__ void tmem_st_cols(uint32_t taddr, const uint32_t* r) {
#pragma unroll
  for (int c = 0; c + 32 <= N; c += 32) tc::tmem_st32(taddr + c, r + c);
  if constexpr (N % 32 == 16) tc::tmem_st16(taddr + (N - 16), r + (N - 16));
}

// The softmax warps' whole unit for N (padded) columns: tiles, then the
// epilogue (row sums, O^T out of TMEM, one coalesced 128-byte warp store
// per row and d quarter).
template <int N>
__device__ __forceinline__ void softmax_unit(uint8_t* smem, TctBars* bars, uint32_t tmem, int jb, int n_tiles, int n_cols,
                                             int kh, int g, int hq_local, float* __restrict__ out,
                                             float* __restrict__ part_o, float* __restrict__ part_ml,
                                             const int32_t* __restrict__ entry_of, int32_t* __restrict__ cnt) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  const float cs = 1.4426950408889634f * rsqrtf((float)kTctD);
  const int32_t* rinfo = reinterpret_cast<const int32_t*>(smem + kOffRow);  // [4][64]: vis, slot, out row, req
  float* red = reinterpret_cast<float*>(smem + kOffRed);
  float* misc = reinterpret_cast<float*>(smem + kOffMisc);
  const int min_vis = reinterpret_cast<const int32_t*>(smem + kOffMisc)[kTctRows];
  const uint32_t pbase = smem_u32(smem + kOffP);
  // this thread's byte within a P^T row: atom column (t / 64), 16-byte chunk
  // ((t % 64) / 8) XOR (row % 8), element t % 8
  const int t = tid, patom = (t >> 6) * kAtomP, pchunk = (t & 63) >> 3, pin = (t & 7) * 2;

  // column references m (log2 units) live in SMEM (uniform over the
  // threads, read as broadcasts); l = this thread's partial row sums
  float* mref = misc;                       // [64]
  float* dm = misc + kTctRows + 4;          // [64] m_old - m_new of the last slow path
  float l[N];
#pragma unroll
  for (int n = 0; n < N; ++n) l[n] = 0.f;
  if (t < kTctRows) mref[t] = 0.f;  // tile 0 always takes the slow path: its x are absolute
  named_sync(2, 128);
  for (int j = 0; j < n_tiles; ++j) {
    const int jg = jb + j, b = jg & 1;  // the CTA's tile sequence runs on across its items
    mbar_wait(&bars->s_full[b], (jg >> 1) & 1);
    tc::fence_after();
    uint32_t sr[N];
    tmem_ld_cols<N>(tmem + lane_base + kColS + b * kTctRows, sr);
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
      const int4 m4 = lds_v4(mref + n);
      const float mm[4] = {__int_as_float(m4.x), __int_as_float(m4.y), __int_as_float(m4.z), __int_as_float(m4.w)};
#pragma unroll
      for (int u = 0; u < 4; ++u) x[n + u] = fmaf(__uint_as_float(sr[n + u]), cs, -mm[u]);
      if (masked) {
        const int4 v4 = lds_v4(rinfo + n);
        const int vv[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (tok >= vv[u]) x[n + u] = neg_inf<float>();
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) over = fmaxf(over, x[n + u]);
    }
    if (named_or(1, 128, j == 0 || over > kRefSlack)) {
      // slow path: raise the references to this tile's column maxima (tile
      // 0: set them to its maxima; a column with no visible token keeps 0)
#pragma unroll
      for (int n = 0; n < N; ++n) {
        const float v = warp_max(x[n]);
        if (lane == 0) red[warp * kTctRows + n] = v;
      }
      named_sync(2, 128);
      if (t < N) {
        const float tm = fmaxf(fmaxf(red[t], red[kTctRows + t]), fmaxf(red[2 * kTctRows + t], red[3 * kTctRows + t]));
        // x is relative to the old m: the new m is m + up
        const float up = j == 0 ? (tm > neg_inf<float>() ? tm : 0.f) : fmaxf(tm, 0.f);
        dm[t] = -up;
        mref[t] += up;
      }
      named_sync(2, 128);
#pragma unroll
      for (int n = 0; n < N; n += 4) {
        const int4 d4 = lds_v4(dm + n);
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
          tc::tmem_ld16(tmem + lane_base + kColO + c, o);
          tc::wait_ld();
#pragma unroll
          for (int u = 0; u < 16; ++u) o[u] = __float_as_uint(__uint_as_float(o[u]) * fast_exp2(dm[c + u]));
          tc::tmem_st16(tmem + lane_base + kColO + c, o);
        }
        tc::wait_st();
      }
    }
    // P^T(j) into SMEM buffer b once PV(j - 2) read it
    if (jg >= 2) mbar_wait(&bars->p_empty[b], ((jg - 2) >> 1) & 1);
    const uint32_t pb = pbase + b * kPtBytes + patom + pin;
#pragma unroll
    for (int n = 0; n < N; ++n) {
      const float p = fast_exp2(x[n]);
      l[n] += p;
      sts_u16(pb + n * 128 + ((pchunk ^ (n & 7)) << 4), __bfloat16_as_ushort(__float2bfloat16_rn(p)));
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic stores -> MMA operand reads
    tc::fence_before();
    __syncwarp();
    if (lane == 0) mbar_arrive(&bars->p_full[b]);
  }

  // ---- epilogue: row sums over the CTA's tokens, then O^T / l
#pragma unroll
  for (int n = 0; n < N; ++n) {
    const float v = warp_sum(l[n]);
    if (lane == 0) red[warp * kTctRows + n] = v;
  }
  named_sync(2, 128);
  const int jl = jb + n_tiles - 1;
  mbar_wait(&bars->pv_done[jl & 3], (jl >> 2) & 1);
  tc::fence_after();
  uint32_t o[N];
  tmem_ld_cols<N>(tmem + lane_base + kColO, o);
  tc::wait_ld();
  tc::fence_before();
  __syncwarp();
  if (lane == 0) mbar_arrive(&bars->o_free);  // the next item's first PV may overwrite O^T
#pragma unroll
  for (int n = 0; n < N; ++n) {
    if (n < n_cols) {
      const float L = red[n] + red[kTctRows + n] + red[2 * kTctRows + n] + red[3 * kTctRows + n];
      const int slot = rinfo[kTctRows + n], orow = rinfo[2 * kTctRows + n];
      float* dst = (slot < 0 ? out : part_o) + (int64_t)orow * kTctD;
      asm volatile("st.global.L1::no_allocate.f32 [%0], %1;" ::"l"(dst + t), "f"(__uint_as_float(o[n]) / L)
                   : "memory");
    }
  }
  if (t < n_cols && rinfo[kTctRows + t] >= 0) {
    const int orow = rinfo[2 * kTctRows + t];
    part_ml[2 * (int64_t)orow] = mref[t] * 0.69314718055994530942f;  // natural-log units
    part_ml[2 * (int64_t)orow + 1] = red[t] + red[kTctRows + t] + red[2 * kTctRows + t] + red[3 * kTctRows + t];
  }
  if (cnt) {  // readiness counts of the merge entries: every store of the CTA's rows fenced first
    __threadfence();
    named_sync(2, 128);
    if (t < n_cols && rinfo[kTctRows + t] >= 0 && t % g == 0) {
      const int e = __ldg(entry_of + (int64_t)rinfo[3 * kTctRows + t] * (hq_local / g) + kh);
      if (e >= 0) atomicAdd(cnt + e, g);  // the g rows of (request, kv head)
    }
  }
}

__global__ void __launch_bounds__(kTctThreads, 1)
    tct_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
               const int32_t* __restrict__ table, int off_groups, int off_rows, int n_groups, int h_local,
               const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, float* __restrict__ out,
               float* __restrict__ part_o, float* __restrict__ part_ml, const int32_t* __restrict__ page_table,
               int page_shift, int32_t* __restrict__ done, const int32_t* __restrict__ entry_of,
               int32_t* __restrict__ cnt) {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  TctBars* bars = reinterpret_cast<TctBars*>(smem + kOffBar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int hq_local = g * h_local, n_items = n_groups * h_local;
  // item it = (group it / h_local, kv head it % h_local); a CTA takes items
  // blockIdx.x, + gridDim.x, ... (the grid fits in one wave beside the TC
  // grid, so the suffix kernel launched after it starts at once)
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
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&bars->s_full[b], 1);
      mbar_init(&bars->s_free[b], 4);
      mbar_init(&bars->p_full[b], 4);
      mbar_init(&bars->p_empty[b], 1);
    }
    mbar_init(&bars->q_full, 4);
    mbar_init(&bars->o_free, 4);
    for (int i = 0; i < 4; ++i) mbar_init(&bars->pv_done[i], 1);
    fence_barrier_init();
  }
  if (warp == 5) tc::tmem_alloc(&bars->tmem_slot, kTmemCols);
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;

  int tiles_total = 0;  // this CTA's tiles over all its items (barrier phases run on across items)
  if (warp < 4) {
    int32_t* rinfo = reinterpret_cast<int32_t*>(smem + kOffRow);
    int32_t* minv = reinterpret_cast<int32_t*>(smem + kOffMisc) + kTctRows;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      const Item x = item(it);
      if (x.n_cols > kTctRows) __trap();  // the host routes at most kTctRows rows here
      // ---- per column: visible tokens, slot, output row, request; Q rows
      // (the previous item's S MMAs are complete: its tiles were consumed)
      if (tid == 0) *minv = 0x7fffffff;
      named_sync(2, 128);
      if (tid < kTctRows) {
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
        rinfo[kTctRows + tid] = slot;
        rinfo[2 * kTctRows + tid] = orow;
        rinfo[3 * kTctRows + tid] = req;
      }
      // Q rows as the K-major SW128 B operand: 16-byte chunk c of row n at
      // atom column c / 8, row n, chunk (c % 8) XOR (n % 8); padding rows zero
#pragma unroll
      for (int i = 0; i < (kTctRows * 16) / 128; ++i) {
        const int e = i * 128 + tid, n = e >> 4, c = e & 15;
        uint4 v = make_uint4(0, 0, 0, 0);
        if (n < x.n_cols) {
          const int req = __ldg(x.rows + (n / g) * kRowInts);
          v = __ldg(reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + x.kh * g + n % g) * kTctD) + c);
        }
        *reinterpret_cast<uint4*>(smem + kOffQ + (c >> 3) * kAtomQ + n * 128 + (((c & 7) ^ (n & 7)) << 4)) = v;
      }
      tc::fence_proxy_async_smem();
      named_sync(2, 128);  // row info and min_vis before the softmax reads them
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars->q_full);
      switch (x.npad) {
        case 16: softmax_unit<16>(smem, bars, tmem, tiles_total, x.n_tiles, x.n_cols, x.kh, g, hq_local, out, part_o, part_ml, entry_of, cnt); break;
        case 32: softmax_unit<32>(smem, bars, tmem, tiles_total, x.n_tiles, x.n_cols, x.kh, g, hq_local, out, part_o, part_ml, entry_of, cnt); break;
        case 48: softmax_unit<48>(smem, bars, tmem, tiles_total, x.n_tiles, x.n_cols, x.kh, g, hq_local, out, part_o, part_ml, entry_of, cnt); break;
        default: softmax_unit<64>(smem, bars, tmem, tiles_total, x.n_tiles, x.n_cols, x.kh, g, hq_local, out, part_o, part_ml, entry_of, cnt); break;
      }
      tiles_total += x.n_tiles;
      named_sync(2, 128);  // every thread's epilogue reads of the row info done before the next item's
    }
  } else if (warp == 4) {
    // ---- TMA producer: K and V tiles, both SW128 atom columns in one op
    if (lane == 0) {
      tc::prefetch_tmap(&tmk);
      tc::prefetch_tmap(&tmv);
      const uint64_t pol = tc::policy_evict_first();  // read by this CTA only
      int jg = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        const Item x = item(it);
        for (int j = 0; j < x.n_tiles; ++j, ++jg) {
          const int s = jg & 1;
          int xt = x.kv_tok + j * kTctBN;  // paged pool: a 128-token tile never crosses a page
          if (page_shift)
            xt = (__ldg(page_table + (xt >> page_shift)) << page_shift) | (xt & ((1 << page_shift) - 1));
          const int y = x.kh * (int)pool_tokens + xt;
          if (jg >= kStages) mbar_wait(&bars->k_empty[s], ((jg - kStages) >> 1) & 1);
          mbar_arrive_expect_tx(&bars->k_full[s], kTileBytes);
          tc::tma_load_3d_hint(smem + kOffK + s * kTileBytes, &tmk, 0, y, 0, &bars->k_full[s], pol);
          if (jg >= kStages) mbar_wait(&bars->v_empty[s], ((jg - kStages) >> 1) & 1);
          mbar_arrive_expect_tx(&bars->v_full[s], kTileBytes);
          tc::tma_load_3d_hint(smem + kOffV + s * kTileBytes, &tmv, 0, y, 0, &bars->v_full[s], pol);
        }
      }
    }
  } else {
    // ---- MMA issuer: S^T(j), then PV(j - 1) (the tensor pipe computes
    // S^T(j + 1) while the softmax works on tile j)
    const uint32_t sbase = smem_u32(smem);
    int jg = 0, u = 0;
    auto pv = [&](int tp, int j_item, uint32_t idesc_o) {
      const int vb = tp & 1;
      mbar_wait(&bars->p_full[vb], (tp >> 1) & 1);
      mbar_wait(&bars->v_full[vb], (tp >> 1) & 1);
      tc::fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < kTctBN / 16; ++k) {
          // A = V^T: MN-major, 64-d blocks 16 KB apart (LBO), 8-token groups 1 KB apart (SBO)
          const uint64_t av = tc::smem_desc(sbase + kOffV + vb * kTileBytes + k * 2048, kAtomTile, 1024);
          const uint64_t bp = tc::smem_desc(sbase + kOffP + vb * kPtBytes + (k >> 2) * kAtomP + (k & 3) * 32, 16, 1024);
          tc::mma_f16_ss(tmem + kColO, av, bp, idesc_o, (j_item > 0 || k > 0) ? 1u : 0u);
        }
        tc::commit(&bars->v_empty[vb]);
        tc::commit(&bars->p_empty[vb]);
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
        const int s = jg & 1;
        mbar_wait(&bars->k_full[s], (jg >> 1) & 1);
        if (jg >= 2) mbar_wait(&bars->s_free[s], ((jg - 2) >> 1) & 1);
        tc::fence_after();
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kTctD / 16; ++k) {
            const uint64_t ak = tc::smem_desc(sbase + kOffK + s * kTileBytes + (k >> 2) * kAtomTile + (k & 3) * 32, 16, 1024);
            const uint64_t bq = tc::smem_desc(sbase + kOffQ + (k >> 2) * kAtomQ + (k & 3) * 32, 16, 1024);
            tc::mma_f16_ss(tmem + kColS + s * kTctRows, ak, bq, idesc_s, k > 0 ? 1u : 0u);
          }
          tc::commit(&bars->k_empty[s]);
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
    tiles_total = jg;
    // every commit's arrival landed before the CTA exits (a late one would
    // hit the SMEM of the next CTA on this SM): the last phase of each
    for (int s = 0; s < kStages; ++s) {
      const int uses = (tiles_total - s + 1) / 2;
      if (uses > 0) {
        mbar_wait(&bars->k_empty[s], (uses - 1) & 1);
        mbar_wait(&bars->v_empty[s], (uses - 1) & 1);
        mbar_wait(&bars->p_empty[s], (uses - 1) & 1);
      }
    }
    for (int i = 0; i < 4; ++i) {
      const int uses = (tiles_total - i + 3) / 4;
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
  if (warp == 5) tc::tmem_dealloc(tmem, kTmemCols);
}

}  // namespace

int32_t cuda_status(cudaError_t e, const char* what);
int32_t encode_pool_halves_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows);

// groups: the kKindTct records (multi-request table format), one CTA per
// (group, local kv head); pdl: programmatic dependent of the previous launch
int32_t launch_tct(const int32_t* table, int n_groups, int off_groups, int off_rows, const void* q, const void* k,
                   const void* v, int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                   cudaStream_t st, bool pdl, const int32_t* page_table, int page_shift, int32_t* done,
                   const int32_t* entry_of, int32_t* cnt, int max_ctas) {
  if (n_groups == 0) return CODEC_OK;
  if (g > kTctRows) return fail(CODEC_ERR_UNSUPPORTED, "transposed tensor-core kernel: g = %d > %d", g, kTctRows);
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_halves_map(&mk, k, (int64_t)h_local * pool_tokens, kTctBN));
  CODEC_TRY(encode_pool_halves_map(&mv, v, (int64_t)h_local * pool_tokens, kTctBN));
  cudaError_t e = cudaFuncSetAttribute(tct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTctSmem);
  if (e != cudaSuccess) return cuda_status(e, "tct smem attribute");
  cudaLaunchConfig_t cfg = {};
  const int n_items = n_groups * h_local;
  cfg.gridDim = dim3(max_ctas > 0 ? std::min(n_items, max_ctas) : n_items);
  cfg.blockDim = dim3(kTctThreads);
  cfg.dynamicSmemBytes = kTctSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  e = cudaLaunchKernelEx(&cfg, tct_kernel, mk, mv, table, off_groups, off_rows, n_groups, h_local,
                         (const __nv_bfloat16*)q, pool_tokens, g, (float*)out, (float*)part_o, (float*)part_ml,
                         page_table, page_shift, done, entry_of, cnt);
  if (e != cudaSuccess) return cuda_status(e, "tct launch");
  return cuda_status(cudaGetLastError(), "tct launch");
}

}  // namespace codec
