// K2: shared-node split attention on the 5th-generation tensor cores.
//
// Persistent CTA = (schedule block b, kv head h). It walks the TC groups
// the balancer assigned to block b (LPT over the SM slots, host_table.cpp);
// a group is a KV slice [kv_tok, kv_tok + len) of a shared node and up to
// 256 query-head rows (256/g requests of the node's query set with their g
// query heads: GQA packing turns the per-request GEMVs into one dense
// contraction). The rows form two M=128 tiles, Q0 and Q1, that share every
// K/V tile. Per 128-token KV tile t and Q tile i:
//     S_i = Q_i K_t^T      tcgen05.mma SS, M128 N128 K128, fp32 in TMEM
//     P_i = 2^(S_i c - m)  softmax warpgroup i (thread = row = TMEM lane),
//                          written back over S_i as bf16 (tcgen05.st)
//     O_i += P_i V_t       tcgen05.mma TS (A = P from TMEM), M128 N128 K128
// Per row this is the reference's pac_kernel math (_kernels.pyx:25-54);
// the partial (O/l, m, l) feeds the LSE merge (kern_merge.cu).
//
// Why this shape: the SS QK^T MMA already consumes SMEM bandwidth at its
// peak (A and B from SMEM), so P never goes through SMEM (TS MMA) and the
// 128-token tile halves the Q re-reads per token. The issue order
//     PV_0(t) S_0(t+1) PV_1(t) S_1(t+1)
// ping-pongs the two softmax warpgroups: while WG0 exponentiates S_0(t+1)
// the tensor pipe runs PV_1(t) and S_1(t+1). In-order tcgen05 execution
// makes S_i(t+1) (which overwrites P_i(t)) safe after PV_i(t), and the
// commit behind S_i(t) guarantees PV_i(t-1) landed before softmax i reads
// or rescales O_i.
//
// Warp roles (576 threads): 16 softmax warps -- (Q tile, column half, TMEM
// lane quadrant); a row's two 64-column halves exchange their max through
// SMEM -- warp 16 TMA producer (K/V 2-stage rings of 128x64 SWIZZLE_128B
// boxes), warp 17 TMEM allocator + single-thread MMA issuer. Two warps per
// row keep two independent instruction streams per scheduler, which the
// latency-bound exponential loop needs. Softmax: packed f32x2 math,
// exponentials split between MUFU.EX2 (5/8) and a degree-3 polynomial on
// the FMA pipe (3/8), lazy O rescale (only when a row max grows by > 2^8),
// masking only on a row's last tile.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "tc_ptx.cuh"

namespace codec {

constexpr int kTcSoftmaxWarps = 16;         // 2 Q tiles x 4 lane quadrants x 2 column halves
constexpr int kTcProducerWarp = kTcSoftmaxWarps;
constexpr int kTcMmaWarp = kTcSoftmaxWarps + 1;
constexpr int kTcThreads = 32 * (kTcSoftmaxWarps + 2);
constexpr int kTcBN = 128;                      // tokens per KV tile
constexpr int kTcD = 128;                       // head dim
constexpr int kTcKStages = 3;                   // K ring depth (K is needed one MMA earlier than V)
constexpr int kTcVStages = 2;                   // V ring depth
constexpr int kTcPrefetch = 3;                  // tiles ahead the producer warms L2
constexpr int kTileBytes = 128 * 128 * 2;       // 32 KB: one 128x128 bf16 tile (Q, K or V)
constexpr int kAtomBytes = kTileBytes / 2;      // 64-element-wide SW128 atom column
constexpr int kOffQ = 0;                                 // Q0, Q1
constexpr int kOffK = kOffQ + 2 * kTileBytes;            // K ring
constexpr int kOffV = kOffK + kTcKStages * kTileBytes;   // V ring
constexpr int kOffXch = kOffV + kTcVStages * kTileBytes; // row-max / row-sum exchange [2][2][128] f32
constexpr int kOffBar = kOffXch + 2 * 2 * 128 * 4;
// No alignment slack: the dynamic SMEM window starts 1024-aligned (behind the
// driver's 1 KB reservation) and the kernel traps if it ever does not.
constexpr int kTcSmem = kOffBar + 256;
static_assert(kTcSmem <= 232448, "exceeds the 227 KB opt-in shared memory");
constexpr uint32_t kTmemCols = 512;  // S0/P0 [0,128) S1/P1 [128,256) O0 [256,384) O1 [384,512)
constexpr float kRescaleLog2 = 8.f;

struct TcBars {
  uint64_t q_full;
  uint64_t k_full[kTcKStages], k_empty[kTcKStages];
  uint64_t v_full[kTcVStages], v_empty[kTcVStages];
  uint64_t s_full[2], p_full[2], o_done[2], o_free[2];
  uint32_t tmem_slot;
};

// 16-byte chunk c (0..15 along a 128-element row) of row r in a K-major
// SWIZZLE_128B 128x128 tile made of two 64-element atom columns
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (c >> 3) * kAtomBytes + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}

// 2^x on the FMA/ALU pipes (Cody-Waite split, degree-3 minimax on
// [-1/2, 1/2], rel. error 7.5e-5 -- below the bf16 rounding P gets anyway)
__device__ __forceinline__ float poly_exp2(float x) {
  x = fmaxf(x, -126.f);
  const float t = x + 12582912.f;  // 1.5 * 2^23: round-to-nearest into the mantissa
  const float f = x - (t - 12582912.f);
  float p = fmaf(0.05517153f, f, 0.24261101f);
  p = fmaf(p, f, 0.69326099f);
  p = fmaf(p, f, 0.99992808f);
  return __int_as_float(__float_as_int(p) + (__float_as_int(t) << 23));
}

// Two lanes of the same polynomial with packed f32x2 arithmetic
// (FADD2/FFMA2): ~5 issue slots per exponential instead of ~8.
__device__ __forceinline__ float2 poly_exp2x2(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 magic = make_float2(12582912.f, 12582912.f);
  const float2 t = tc::fadd2(x, magic);
  const float2 xi = tc::fadd2(t, make_float2(-12582912.f, -12582912.f));
  const float2 f = tc::fadd2(x, make_float2(-xi.x, -xi.y));
  float2 p = tc::ffma2(make_float2(0.05517153f, 0.05517153f), f, make_float2(0.24261101f, 0.24261101f));
  p = tc::ffma2(p, f, make_float2(0.69326099f, 0.69326099f));
  p = tc::ffma2(p, f, make_float2(0.99992808f, 0.99992808f));
  return make_float2(__int_as_float(__float_as_int(p.x) + (__float_as_int(t.x) << 23)),
                     __int_as_float(__float_as_int(p.y) + (__float_as_int(t.y) << 23)));
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

struct GroupView {
  int kv_tok, n_req, n_tiles;
  const int32_t* rows;
};

__device__ __forceinline__ GroupView group_view(const int32_t* table, int off_groups, int off_rows, int gidx) {
  const int32_t* grp = table + off_groups + gidx * kGroupInts;
  GroupView v;
  v.kv_tok = grp[kGrpKvTok];
  v.n_req = grp[kGrpNRows];
  v.rows = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  int max_vis = 0;
  for (int i = 0; i < v.n_req; ++i) max_vis = max(max_vis, v.rows[i * kRowInts + 1]);
  v.n_tiles = (max_vis + kTcBN - 1) / kTcBN;
  return v;
}

__global__ void __launch_bounds__(kTcThreads, 1)
    tc_pac_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const int32_t* __restrict__ table, int off_groups, int off_rows, int off_block_ptr,
                  const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, int hq_local,
                  float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml,
                  long long* __restrict__ trace) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();  // SWIZZLE_128B atoms need 1024-byte alignment
  TcBars* bars = reinterpret_cast<TcBars*>(smem + kOffBar);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int blk = blockIdx.x, kh = blockIdx.y;
  // optional timeline of CTA (0, 0): trace[(event * 2 + q tile) * 64 + tile]
  const bool tracing = trace != nullptr && blk == 0 && kh == 0;
  auto stamp = [&](int ev, int i, int tt) {
    if (tracing && tt < 64) trace[(ev * 2 + i) * 64 + tt] = clock64();
  };
  const int g_begin = table[off_block_ptr + blk], g_end = table[off_block_ptr + blk + 1];

  if (tid == 0) {
    mbar_init(&bars->q_full, 32 * kTcSoftmaxWarps);
    for (int s = 0; s < kTcKStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < kTcVStages; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], 256);
      mbar_init(&bars->o_done[i], 1);
      mbar_init(&bars->o_free[i], 256);
    }
    fence_barrier_init();
  }
  if (warp == kTcMmaWarp) tc::tmem_alloc(&bars->tmem_slot, kTmemCols);
  if (warp == kTcProducerWarp && lane == 0) {
    tc::prefetch_tmap(&tmk);
    tc::prefetch_tmap(&tmv);
  }
  tc::fence_before();
  __syncthreads();
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;

  if (warp == kTcProducerWarp) {
    // ================================================ TMA producer (whole warp, one lane issues)
    int t = 0;  // global KV tile counter (ring position)
    for (int gi = g_begin; gi < g_end; ++gi) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      const int row0 = kh * (int)pool_tokens + gv.kv_tok;
      if (tc::elect_one()) {  // warm L2 with the group's first tiles
        for (int j = 0; j < kTcPrefetch && j < gv.n_tiles; ++j) {
          tc::tma_prefetch_2d(&tmk, 0, row0 + j * kTcBN);
          tc::tma_prefetch_2d(&tmk, 64, row0 + j * kTcBN);
          tc::tma_prefetch_2d(&tmv, 0, row0 + j * kTcBN);
          tc::tma_prefetch_2d(&tmv, 64, row0 + j * kTcBN);
        }
      }
      __syncwarp();
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        const int ks = t % kTcKStages, vs = t % kTcVStages;
        const int y = row0 + j * kTcBN;
        if (t >= kTcKStages) mbar_wait(&bars->k_empty[ks], ((t / kTcKStages) - 1) & 1);
        if (tc::elect_one()) {
          mbar_arrive_expect_tx(&bars->k_full[ks], kTileBytes);
          uint8_t* kd = smem + kOffK + ks * kTileBytes;
          tc::tma_load_2d(kd, &tmk, 0, y, &bars->k_full[ks]);
          tc::tma_load_2d(kd + kAtomBytes, &tmk, 64, y, &bars->k_full[ks]);
          if (j + kTcPrefetch < gv.n_tiles) {
            const int yp = y + kTcPrefetch * kTcBN;
            tc::tma_prefetch_2d(&tmk, 0, yp);
            tc::tma_prefetch_2d(&tmk, 64, yp);
            tc::tma_prefetch_2d(&tmv, 0, yp);
            tc::tma_prefetch_2d(&tmv, 64, yp);
          }
        }
        __syncwarp();
        if (t >= kTcVStages) mbar_wait(&bars->v_empty[vs], ((t / kTcVStages) - 1) & 1);
        if (tc::elect_one()) {
          mbar_arrive_expect_tx(&bars->v_full[vs], kTileBytes);
          uint8_t* vd = smem + kOffV + vs * kTileBytes;
          tc::tma_load_2d(vd, &tmv, 0, y, &bars->v_full[vs]);
          tc::tma_load_2d(vd + kAtomBytes, &tmv, 64, y, &bars->v_full[vs]);
        }
        __syncwarp();
      }
    }
  } else if (warp == kTcMmaWarp) {
    // ================================================ MMA issuer
    // The whole warp runs the (warp-uniform) schedule so the descriptors stay
    // in uniform registers; one elected lane issues each batch of MMAs.
    // Descriptors are a base plus a compile-time start-address offset
    // (the low 14 bits hold addr >> 4).
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, kTcBN, false, false);
    constexpr uint32_t idesc_o = tc::idesc_bf16(128, kTcD, false, true);
    const uint64_t dq = tc::smem_desc(sbase + kOffQ, 16, 1024);
    const uint64_t dk = tc::smem_desc(sbase + kOffK, 16, 1024);
    const uint64_t dv = tc::smem_desc(sbase + kOffV, kAtomBytes, 1024);
    int t = 0;  // global tile counter
    int gq = 0;
    auto issue_s = [&](int i, int tt) {
      const int s = tt % kTcKStages;
      const uint64_t aq = dq + (uint64_t)((i * kTileBytes) >> 4);
      const uint64_t bk = dk + (uint64_t)((s * kTileBytes) >> 4);
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < kTcD / 16; ++k) {
          const uint64_t off = (uint64_t)((((k >> 2) * kAtomBytes) + (k & 3) * 32) >> 4);
          tc::mma_f16_ss(tmem + i * 128, aq + off, bk + off, idesc_s, k > 0 ? 1u : 0u);
        }
        tc::commit(&bars->s_full[i]);
        if (i == 1) tc::commit(&bars->k_empty[s]);
      }
      __syncwarp();
    };
    for (int gi = g_begin; gi < g_end; ++gi, ++gq) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (gv.n_tiles == 0) {  // (cannot happen: every row sees >= 1 token) keep gq in step
        --gq;
        continue;
      }
      mbar_wait(&bars->q_full, gq & 1);
      {
        const int s = t % kTcKStages;
        mbar_wait(&bars->k_full[s], (t / kTcKStages) & 1);
        tc::fence_after();
        issue_s(0, t);
        issue_s(1, t);
      }
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        const int s = t % kTcVStages;
        const bool more = j + 1 < gv.n_tiles;
        mbar_wait(&bars->v_full[s], (t / kTcVStages) & 1);
        if (more) mbar_wait(&bars->k_full[(t + 1) % kTcKStages], ((t + 1) / kTcKStages) & 1);
        const uint64_t bv = dv + (uint64_t)((s * kTileBytes) >> 4);
        for (int i = 0; i < 2; ++i) {
          mbar_wait(&bars->p_full[i], t & 1);                        // P_i(t) in TMEM
          if (j == 0 && gq > 0) mbar_wait(&bars->o_free[i], (gq - 1) & 1);  // epilogue read O_i
          tc::fence_after();
          if (lane == 0) stamp(0, i, t);
          const uint32_t p_tmem = tmem + i * 128;
          const uint32_t o_tmem = tmem + 256 + i * 128;
          if (tc::elect_one()) {
#pragma unroll
            for (int k = 0; k < kTcBN / 16; ++k)
              // tokens [16k, 16k+16) of P: columns 64*(k/4) + 8*(k%4) (each
              // column-half of the softmax packs its P over its own S columns)
              tc::mma_f16_ts(o_tmem, p_tmem + (k >> 2) * 64 + (k & 3) * 8, bv + (uint64_t)((k * 16 * 128) >> 4),
                             idesc_o, (j > 0 || k > 0) ? 1u : 0u);
            if (i == 1) tc::commit(&bars->v_empty[s]);
            if (!more) tc::commit(&bars->o_done[i]);
          }
          __syncwarp();
          if (more) issue_s(i, t + 1);
          if (lane == 0) stamp(1, i, t);
        }
      }
    }
  } else {
    // ================================================ softmax warps
    // warp = (Q tile wg, column half hf, lane quadrant quad); thread = one
    // row of the Q tile (TMEM lane) over 64 of the tile's 128 columns. The
    // two halves of a row meet through SMEM for the row max (named barrier
    // per (wg, quad) pair) and, at the end of a group, for the row sum.
    const int wg = warp >> 3;                 // Q tile
    const int hf = (warp >> 2) & 1;           // column half
    const int quad = warp & 3;                // TMEM lane quadrant
    const int r = quad * 32 + lane;           // row in the Q tile == TMEM lane
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    const uint32_t s_tmem = tmem + wg * 128 + lane_addr;
    const uint32_t o_tmem = tmem + 256 + wg * 128 + lane_addr + hf * 64;
    const uint32_t bar_id = 1 + wg * 4 + quad;  // pairs the two half-warps of these rows
    // [wg][hf][128]; single-buffered: a pair barrier before every write keeps
    // the partner's previous read ahead of the overwrite
    float* xch = reinterpret_cast<float*>(smem + kOffXch);
    auto xch_at = [&](int h) -> float* { return xch + (wg * 2 + h) * 128 + r; };
    auto pair_sync = [&]() { asm volatile("bar.sync %0, 64;" ::"r"(bar_id) : "memory"); };
    const float cscale = 1.4426950408889634f * rsqrtf((float)kTcD);
    const float2 c2 = make_float2(cscale, cscale);
    int t = 0, gq = 0;
    for (int gi = g_begin; gi < g_end; ++gi, ++gq) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (gv.n_tiles == 0) {
        --gq;
        continue;
      }
      const int grow = wg * 128 + r;          // row of the 256-row group
      const int ridx = grow / g;
      const bool valid = ridx < gv.n_req;
      const int req = valid ? gv.rows[ridx * kRowInts + 0] : 0;
      const int vis = valid ? gv.rows[ridx * kRowInts + 1] : 0;
      const int slot = valid ? gv.rows[ridx * kRowInts + 2] : 0;
      const int qh = kh * g + (grow % g);
      {  // stage my half of the Q row (K-major SW128); the previous group's S MMAs are complete
        uint8_t* qs = smem + kOffQ + wg * kTileBytes;
        const uint4* src = reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + qh) * kTcD);
#pragma unroll
        for (int c = hf * 8; c < hf * 8 + 8; ++c) {
          const uint4 v = valid ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
          *reinterpret_cast<uint4*>(qs + sw128(r, c)) = v;
        }
        tc::fence_proxy_async_smem();
        mbar_arrive(&bars->q_full);
      }
      float m_used = 0.f;  // exponent reference (log2 units), same in both halves
      float2 l2 = make_float2(0.f, 0.f);
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        mbar_wait(&bars->s_full[wg], t & 1);   // also: PV_wg(t-1) has landed (commit order)
        tc::fence_after();
        if (tid == wg * 256) stamp(2, wg, t);
        const int lim = vis - j * kTcBN - hf * 64;  // visible columns of my half
        const bool full = __all_sync(0xffffffffu, !valid || lim >= 64);
        const uint32_t my_s = s_tmem + hf * 64;
        // pass 1: max over my 64 columns
        float mx = neg_inf<float>();
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t sr[32];
          tc::tmem_ld32(my_s + c * 32, sr);
          tc::wait_ld();
          if (!full) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= lim) sr[i] = 0xff800000u;  // -inf
          }
#pragma unroll
          for (int i = 0; i < 32; i += 2) mx = fmaxf(mx, fmaxf(__uint_as_float(sr[i]), __uint_as_float(sr[i + 1])));
        }
        // meet the other half of the row (each half only ever writes P into
        // its own S columns, so no ordering beyond this exchange is needed)
        pair_sync();
        *xch_at(hf) = mx;
        pair_sync();
        mx = fmaxf(mx, *xch_at(hf ^ 1));
        if (tid == wg * 256) stamp(4, wg, t);
        const float mt = valid ? mx * cscale : 0.f;
        if (j == 0) {
          m_used = mt;
        } else {
          const bool need = mt > m_used + kRescaleLog2;
          if (__any_sync(0xffffffffu, need)) {  // tcgen05.ld/st are warp-collective
            const float alpha = need ? fast_exp2(m_used - mt) : 1.f;
            l2.x *= alpha;
            l2.y *= alpha;
#pragma unroll
            for (int c = 0; c < 2; ++c) {
              uint32_t o[32];
              tc::tmem_ld32(o_tmem + c * 32, o);
              tc::wait_ld();
#pragma unroll
              for (int i = 0; i < 32; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tc::tmem_st32(o_tmem + c * 32, o);
            }
            if (need) m_used = mt;
          }
        }
        // pass 2: P = 2^(S c - m) as bf16 pairs; S columns 64hf + [32c, 32c+32)
        // -> P columns 64hf + [16c, 16c+16), i.e. over my own consumed S
        const float2 nm = make_float2(-m_used, -m_used);
#pragma unroll
        for (int c = 0; c < 2; ++c) {
          uint32_t sr[32];
          tc::tmem_ld32(my_s + c * 32, sr);
          tc::wait_ld();
          if (!full) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (c * 32 + i >= lim) sr[i] = 0xff800000u;
          }
          uint32_t pw[16];
#pragma unroll
          for (int w = 0; w < 16; w += 4) {
            // 8 scores: 5 exponentials on the MUFU, 3 on the FMA pipe (a packed pair + 1)
            float2 x[4], p[4];
#pragma unroll
            for (int k = 0; k < 4; ++k)
              x[k] = tc::ffma2(make_float2(__uint_as_float(sr[2 * (w + k)]), __uint_as_float(sr[2 * (w + k) + 1])),
                               c2, nm);
            const float2 py = poly_exp2x2(make_float2(x[2].y, x[3].y));
            p[0] = make_float2(fast_exp2(x[0].x), fast_exp2(x[0].y));
            p[1] = make_float2(fast_exp2(x[1].x), poly_exp2(x[1].y));
            p[2] = make_float2(fast_exp2(x[2].x), py.x);
            p[3] = make_float2(fast_exp2(x[3].x), py.y);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              l2 = tc::fadd2(l2, p[k]);
              pw[w + k] = pack_bf16(p[k].x, p[k].y);
            }
          }
          tc::tmem_st16(my_s + c * 16, pw);
        }
        tc::wait_st();
        tc::fence_before();
        if (tid == wg * 256) stamp(3, wg, t);
        mbar_arrive(&bars->p_full[wg]);
      }
      // ---- epilogue: O / l once the group's last PV landed
      float l_run = l2.x + l2.y;
      pair_sync();
      *xch_at(hf) = l_run;
      pair_sync();
      l_run += *xch_at(hf ^ 1);
      mbar_wait(&bars->o_done[wg], gq & 1);
      tc::fence_after();
      float* dst;
      if (slot < 0) {
        dst = out + ((int64_t)req * hq_local + qh) * kTcD + hf * 64;
      } else {
        const int64_t ei = (int64_t)slot * hq_local + qh;
        dst = part_o + ei * kTcD + hf * 64;
        if (valid && hf == 0) {
          part_ml[2 * ei] = m_used * 0.69314718055994530942f;  // natural-log units
          part_ml[2 * ei + 1] = l_run;
        }
      }
      const float inv = 1.f / l_run;
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t o[32];
        tc::tmem_ld32(o_tmem + c * 32, o);
        tc::wait_ld();
        if (valid) {
#pragma unroll
          for (int i = 0; i < 32; i += 4)
            *reinterpret_cast<float4*>(dst + c * 32 + i) =
                make_float4(__uint_as_float(o[i]) * inv, __uint_as_float(o[i + 1]) * inv,
                            __uint_as_float(o[i + 2]) * inv, __uint_as_float(o[i + 3]) * inv);
        }
      }
      tc::fence_before();
      mbar_arrive(&bars->o_free[wg]);
    }
  }
  tc::fence_before();
  __syncthreads();
  if (warp == kTcMmaWarp) tc::tmem_dealloc(tmem, kTmemCols);
}

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int32_t cuda_status(cudaError_t e, const char* what);

static int32_t encode_pool_map(CUtensorMap* map, const void* pool, int64_t rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !p)
      return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kTcD, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kTcD * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)kTcBN};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CODEC_OK;
}

static long long* g_trace = nullptr;  // debug timeline (CODEC_FLAG_TRACE), one per process

int32_t launch_tc(const int32_t* table, const codec_table_info& in, const void* q, const void* k, const void* v,
                  int64_t pool_tokens, int g, int h_local, void* out, void* part_o, void* part_ml,
                  cudaStream_t st, bool trace) {
  if (trace && !g_trace) {
    if (cudaMalloc(&g_trace, 5 * 2 * 64 * sizeof(long long)) != cudaSuccess) return fail(CODEC_ERR_CUDA, "trace alloc");
    cudaMemsetAsync(g_trace, 0, 5 * 2 * 64 * sizeof(long long), st);
  }
  if (in.n_tc_groups == 0 || in.n_tc_blocks == 0) return CODEC_OK;
  CUtensorMap mk, mv;
  CODEC_TRY(encode_pool_map(&mk, k, (int64_t)h_local * pool_tokens));
  CODEC_TRY(encode_pool_map(&mv, v, (int64_t)h_local * pool_tokens));
  cudaError_t e = cudaFuncSetAttribute(tc_pac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
  if (e != cudaSuccess) return cuda_status(e, "tc smem attribute");
  dim3 grid(in.n_tc_blocks, h_local);
  tc_pac_kernel<<<grid, kTcThreads, kTcSmem, st>>>(mk, mv, table, in.off_tc, in.off_rows, in.off_tc_block_ptr,
                                                   (const __nv_bfloat16*)q, pool_tokens, g, h_local * g,
                                                   (float*)out, (float*)part_o, (float*)part_ml,
                                                   trace ? g_trace : nullptr);
  return cuda_status(cudaGetLastError(), "tc launch");
}

int32_t read_trace(long long* host, int64_t n) {
  if (!g_trace) return fail(CODEC_ERR_VALUE, "no trace recorded");
  if (n > 5 * 2 * 64) n = 5 * 2 * 64;
  return cuda_status(cudaMemcpy(host, g_trace, n * sizeof(long long), cudaMemcpyDeviceToHost), "trace copy");
}

}  // namespace codec
