// K2 variant (CODEC_FLAG_TC3): the shared-node kernel with THREE softmax
// warpgroups. Same pieces, pair structure, TMA producers and epilogue
// contract as kern_tc.cu; what changes is the tile pipeline:
//
//   * tile t belongs to softmax group t % 3; S is triple-buffered in TMEM
//     (S_b at columns [128 b, 128 b + 128)) and P(t) is written over the
//     first half of S(t)'s own columns, so TMEM holds S0 S1 S2 + O;
//   * S(t + 3) reuses buffer t % 3 once PV(t) has read P(t) (the S issuer
//     waits for PV(t)); each group then has three tiles of time for its
//     chain softmax(t) -> PV(t) -> S(t + 3), and the third group keeps
//     the MUFU busy while the other two wait on S or on the handoff --
//     kern_tc.cu's two groups phase-lock and leave the MUFU idle ~30 %;
//   * the row max still passes group to group every tile (shared O, lazy
//     rescale past 2^8), now around a ring of three;
//   * 512 threads: ptxas gets 128 registers per thread, so the softmax is
//     two-pass (row max over TMEM chunks, then the exponentials chunk by
//     chunk, P stored per chunk) and the epilogue reads O 32 columns at a
//     time into warp-private staging.
//
// Warps: 0-11 softmax (group = warp / 4, TMEM lane quadrant = warp % 4),
// 12 K producer, 13 TMEM allocator + S issuer (leader), 14 V producer + PV
// issuer (leader), 15 Q loads of later units.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "tc_ptx.cuh"

namespace codec {
namespace tc3 {

constexpr int kGroups = 3;
constexpr int kSoftmaxWarps = 4 * kGroups;
constexpr int kKWarp = kSoftmaxWarps, kMmaWarp = kSoftmaxWarps + 1, kVWarp = kSoftmaxWarps + 2,
              kQWarp = kSoftmaxWarps + 3;
constexpr int kThreads = 32 * (kSoftmaxWarps + 4);
constexpr int kBN = 128, kD = 128;
constexpr int kPrefetch = 4;
constexpr int kQBytes = 128 * 128 * 2, kQAtom = kQBytes / 2;
constexpr int kHalfBytes = 64 * 128 * 2, kKAtom = kHalfBytes / 2;
constexpr int kKStages = 4, kVStages = 5;
constexpr int kOffQ = 0;
constexpr int kOffK = kOffQ + 2 * kQBytes;
constexpr int kOffV = kOffK + kKStages * kHalfBytes;
constexpr int kOffMpub = kOffV + kVStages * kHalfBytes;  // [3 groups][128 rows] f32
constexpr int kOffLx = kOffMpub + kGroups * 128 * 4;      // [3 groups][128 rows] float2 (l, m)
constexpr int kOffBar = kOffLx + kGroups * 128 * 8;
constexpr int kSmem = kOffBar + 512;
static_assert(kSmem <= 232448, "exceeds the 227 KB opt-in shared memory");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColO = 384;
constexpr float kRescaleLog2 = 8.f;
constexpr int kGroupWarpArrivals = 2 * 4;
constexpr int kBarQ = 15;  // group 0's first-Q sync; the epilogue's counted-merge sync
// named barriers 1..12: row-max hand-off group g -> g + 1 (per lane quadrant); 13, 14: (l, m) hand-off

struct Bars {
  uint64_t k_full[kKStages], k_empty[kKStages];
  uint64_t v_full[kVStages], v_empty[kVStages];
  uint64_t q_full[2], q_empty[2], s_full[kGroups], p_full[kGroups];
  uint64_t epi_done[2];
  uint64_t q_tma[2];
  uint64_t pv_done[4];  // PV(t) completes pv_done[t % 4]
  uint64_t o_free;
  uint32_t tmem_slot;
};

__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (c >> 3) * kQAtom + r * 128 + (((c & 7) ^ (r & 7)) << 4);
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}

struct GroupView {
  int kv_tok, n_req, n_tiles, kh, qreq0;
  const int32_t* rows;
};
__device__ __forceinline__ GroupView group_view(const int32_t* table, int off_groups, int off_rows, int gidx) {
  const int32_t* grp = table + off_groups + gidx * kGroupInts;
  GroupView v;
  v.kv_tok = grp[kGrpKvTok];
  v.n_req = grp[kGrpNRows];
  v.kh = grp[kGrpHead];
  v.qreq0 = grp[kGrpQReq0];
  v.rows = table + off_rows + grp[kGrpRowBegin] * kRowInts;
  v.n_tiles = (grp[kGrpMaxVis] + kBN - 1) / kBN;
  return v;
}
struct TileCursor {
  const int32_t* table;
  int off_groups, off_rows, gi, g_end, n, j;
  GroupView gv;
  __device__ void open() {
    while (gi < g_end) {
      gv = group_view(table, off_groups, off_rows, gi);
      if (gv.n_tiles > 0) return;
      ++gi;
    }
  }
  __device__ bool done() const { return gi >= g_end; }
  __device__ void next() {
    if (++j < gv.n_tiles) return;
    j = 0;
    ++n;
    ++gi;
    open();
  }
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    tc3_pac_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                   const __grid_constant__ CUtensorMap tmq, const int32_t* __restrict__ table, int off_groups,
                   int off_rows, int off_block_ptr, const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g,
                   int hq_local, float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml,
                   const int32_t* __restrict__ page_table, int page_shift, int32_t* __restrict__ tc_done,
                   const int32_t* __restrict__ entry_of, int32_t* __restrict__ cnt) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();
  Bars* bars = reinterpret_cast<Bars*>(smem + kOffBar);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  auto prow = [&](int kh, int x) -> int {
    if (page_shift) x = (__ldg(page_table + (x >> page_shift)) << page_shift) | (x & ((1 << page_shift) - 1));
    return kh * (int)pool_tokens + x;
  };
  const bool leader = rank == 0;
  const int blk = blockIdx.x >> 1;
  auto ld_range = [&](int& gb, int& ge) {
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(gb) : "l"(table + off_block_ptr + blk));
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(ge) : "l"(table + off_block_ptr + blk + 1));
  };

  if (tid == 0) {
    for (int s = 0; s < kKStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < kVStages; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 2);
      mbar_init(&bars->q_empty[i], 1);
      mbar_init(&bars->epi_done[i], 4);
      mbar_init(&bars->q_tma[i], 1);
    }
    for (int i = 0; i < kGroups; ++i) {
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->p_full[i], kGroupWarpArrivals);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bars->pv_done[i], 1);
    mbar_init(&bars->o_free, kGroupWarpArrivals);
    fence_barrier_init();
  }
  if (warp == kMmaWarp) tc::tmem_alloc_pair(&bars->tmem_slot, kTmemCols);
  if (warp == kKWarp && lane == 0) {
    tc::prefetch_tmap(&tmk);
    tc::prefetch_tmap(&tmv);
  }
  tc::fence_before();
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;

  if (warp == kKWarp) {
    // ================================================ K producer (both CTAs)
    int g_begin, g_end;
    ld_range(g_begin, g_end);
    TileCursor pfc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
    pfc.open();
    int t_pf = 0;
    auto prefetch_to = [&](int limit) {
      for (; !pfc.done() && t_pf < limit; ++t_pf, pfc.next()) {
        const int xp = pfc.gv.kv_tok + pfc.j * kBN;
        const int ypk = prow(pfc.gv.kh, xp + 64 * rank), ypv = prow(pfc.gv.kh, xp);
        if (tc::elect_one()) {
          tc::tma_prefetch_3d(&tmk, 0, ypk, 0);
          tc::tma_prefetch_2d(&tmv, 64 * rank, ypv);
        }
        __syncwarp();
      }
    };
    prefetch_to(kPrefetch);
    int t = 0;
    for (int gi = g_begin; gi < g_end; ++gi) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        const int ks = t % kKStages;
        if (t >= kKStages) mbar_wait_relaxed(&bars->k_empty[ks], ((t / kKStages) - 1) & 1);
        if (tc::elect_one()) {
          if (leader) mbar_arrive_expect_tx(&bars->k_full[ks], 2 * kHalfBytes);
          const int yk = prow(gv.kh, gv.kv_tok + j * kBN + 64 * rank);
          tc::tma_load_3d_pair(smem + kOffK + ks * kHalfBytes, &tmk, 0, yk, 0, &bars->k_full[ks]);
        }
        __syncwarp();
        prefetch_to(t + 1 + kPrefetch);
      }
    }
  } else if (warp == kVWarp) {
    // ================================================ V producer (both CTAs) + PV issuer (leader)
    int g_begin, g_end;
    ld_range(g_begin, g_end);
    constexpr int kVAhead = kVStages - 2;
    TileCursor vc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
    vc.open();
    int tv = 0;
    auto load_v = [&]() {
      const int vs = tv % kVStages;
      if (tv >= kVStages) mbar_wait_relaxed(&bars->v_empty[vs], ((tv / kVStages) - 1) & 1);
      if (tc::elect_one()) {
        if (leader) mbar_arrive_expect_tx(&bars->v_full[vs], 2 * kHalfBytes);
        const int y = prow(vc.gv.kh, vc.gv.kv_tok + vc.j * kBN);
        tc::tma_load_2d_pair(smem + kOffV + vs * kHalfBytes, &tmv, 64 * rank, y, &bars->v_full[vs]);
      }
      __syncwarp();
      vc.next();
      ++tv;
    };
    if (!leader) {
      while (!vc.done()) load_v();
    } else {
      while (!vc.done() && tv < kVAhead) load_v();
      constexpr uint32_t idesc_o = tc::idesc_bf16(256, kD, false, true);
      const uint64_t dv = tc::smem_desc(sbase + kOffV, kHalfBytes, 1024);
      TileCursor pc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
      pc.open();
      for (int tp = 0; !pc.done(); ++tp) {
        if (!vc.done()) load_v();  // V(tp + kVAhead)
        const int b = tp % kGroups, vs = tp % kVStages;
        mbar_wait(&bars->p_full[b], (tp / kGroups) & 1);  // P(tp) in both CTAs' TMEM (over S(tp))
        mbar_wait(&bars->v_full[vs], (tp / kVStages) & 1);
        if (pc.j == 0 && pc.n > 0) mbar_wait(&bars->o_free, (pc.n - 1) & 1);  // epilogue read O
        tc::fence_after();
        const uint64_t bv = dv + (uint64_t)((vs * kHalfBytes) >> 4);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kBN / 16; ++k)
            tc::mma2_f16_ts(tmem + kColO, tmem + kColS + b * 128 + k * 8, bv + (uint64_t)((k * 16 * 128) >> 4),
                            idesc_o, (pc.j > 0 || k > 0) ? 1u : 0u);
          tc::commit_pair(&bars->v_empty[vs]);
          tc::commit_pair(&bars->pv_done[tp & 3]);
        }
        __syncwarp();
        pc.next();
      }
    }
  } else if (warp == kQWarp) {
    // ================================================ Q gather (both CTAs)
    int g_begin, g_end;
    ld_range(g_begin, g_end);
    int n = 0;
    int qtma_uses[2] = {0, 0};
    for (int gi = g_begin; gi < g_end; ++gi) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (gv.n_tiles == 0) continue;
      if (n == 0) {
        if (gv.qreq0 >= 0) qtma_uses[0] = 1;
        ++n;
        continue;
      }
      const int qb = n & 1;
      if (n >= 2) {
        mbar_wait_relaxed(&bars->q_empty[qb], ((n - 2) >> 1) & 1);
        mbar_wait_relaxed(&bars->epi_done[qb], ((n - 2) >> 1) & 1);
      }
      uint8_t* qs = smem + kOffQ + qb * kQBytes;
      if (gv.qreq0 >= 0) {
        const int rq = 128 / g;
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars->q_tma[qb], kQBytes);
          tc::tma_load_4d(qs, &tmq, 0, 0, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[qb]);
          tc::tma_load_4d(qs + kQAtom, &tmq, 0, 1, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[qb]);
        }
        mbar_wait(&bars->q_tma[qb], (qtma_uses[qb]++) & 1);
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(&bars->q_full[qb], 0);
        ++n;
        continue;
      }
#pragma unroll 1
      for (int i0 = 0; i0 < 64; i0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = (i0 + i) * 32 + lane, r = e >> 4, c = e & 15;
          const int grow = (int)rank * 128 + r, ridx = grow / g;
          v[i] = make_uint4(0, 0, 0, 0);
          if (ridx < gv.n_req) {
            const int req = __ldg(gv.rows + ridx * kRowInts);
            const uint4* src =
                reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + gv.kh * g + (grow % g)) * kD);
            v[i] = __ldg(src + c);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int e = (i0 + i) * 32 + lane;
          *reinterpret_cast<uint4*>(qs + sw128(e >> 4, e & 15)) = v[i];
        }
      }
      tc::fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(&bars->q_full[qb], 0);
      ++n;
    }
  } else if (warp == kMmaWarp) {
    // ================================================ S issuer (leader only)
    // S(ts) into buffer ts % 3 once PV(ts - 3) has read P(ts - 3) from it
    if (leader) {
      int g_begin, g_end;
      ld_range(g_begin, g_end);
      constexpr uint32_t idesc_s = tc::idesc_bf16(256, kBN, false, false);
      const uint64_t dq = tc::smem_desc(sbase + kOffQ, 16, 1024);
      const uint64_t dk = tc::smem_desc(sbase + kOffK, 16, 1024);
      TileCursor sc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
      sc.open();
      for (int ts = 0; !sc.done(); ++ts) {
        const int s = ts % kKStages, b = ts % kGroups;
        if (ts >= kGroups) mbar_wait(&bars->pv_done[(ts - kGroups) & 3], ((ts - kGroups) >> 2) & 1);
        if (sc.j == 0) mbar_wait(&bars->q_full[sc.n & 1], (sc.n >> 1) & 1);
        mbar_wait(&bars->k_full[s], (ts / kKStages) & 1);
        tc::fence_after();
        const uint64_t aq = dq + (uint64_t)(((sc.n & 1) * kQBytes) >> 4);
        const uint64_t bk = dk + (uint64_t)((s * kHalfBytes) >> 4);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kD / 16; ++k) {
            const uint64_t oa = (uint64_t)((((k >> 2) * kQAtom) + (k & 3) * 32) >> 4);
            const uint64_t ob = (uint64_t)((((k >> 2) * kKAtom) + (k & 3) * 32) >> 4);
            tc::mma2_f16_ss(tmem + kColS + b * 128, aq + oa, bk + ob, idesc_s, k > 0 ? 1u : 0u);
          }
          tc::commit_pair(&bars->s_full[b]);
          tc::commit_pair(&bars->k_empty[s]);
          if (sc.j + 1 == sc.gv.n_tiles) tc::commit_pair(&bars->q_empty[sc.n & 1]);
        }
        __syncwarp();
        sc.next();
      }
    }
  } else {
    // ================================================ softmax warpgroups
    int g_begin, g_end;
    ld_range(g_begin, g_end);
    const int grp = warp >> 2;
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float* mpub = reinterpret_cast<float*>(smem + kOffMpub);
    float2* lx = reinterpret_cast<float2*>(smem + kOffLx);
    const int pub_mine = 1 + grp * 4 + quad, pub_other = 1 + ((grp + kGroups - 1) % kGroups) * 4 + quad;
    const float cscale = 1.4426950408889634f * rsqrtf((float)kD);
    const float2 c2 = make_float2(cscale, cscale);
    const int grow = (int)rank * 128 + r;
    const uint32_t my_s = tmem + lane_addr + kColS + grp * 128;
    auto next_group = [&](int gidx) {
      for (++gidx; gidx < g_end; ++gidx)
        if (group_view(table, off_groups, off_rows, gidx).n_tiles > 0) break;
      return gidx;
    };
    int gi = g_begin;
    while (gi < g_end && group_view(table, off_groups, off_rows, gi).n_tiles == 0) ++gi;
    if (gi < g_end && grp == 0 && group_view(table, off_groups, off_rows, gi).qreq0 >= 0) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (tid == 0) {
        const int rq = 128 / g;
        mbar_arrive_expect_tx(&bars->q_tma[0], kQBytes);
        tc::tma_load_4d(smem + kOffQ, &tmq, 0, 0, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[0]);
        tc::tma_load_4d(smem + kOffQ + kQAtom, &tmq, 0, 1, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[0]);
        mbar_wait(&bars->q_tma[0], 0);
        tc::mbar_arrive_cluster(&bars->q_full[0], 0);
      }
    } else if (gi < g_end && grp == 0) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      const int ridx = grow / g;
      const bool valid = ridx < gv.n_req;
      const int req = valid ? __ldg(gv.rows + ridx * kRowInts) : 0;
      const uint4* src = reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + gv.kh * g + (grow % g)) * kD);
      uint8_t* qs = smem + kOffQ;
#pragma unroll
      for (int c0 = 0; c0 < 16; c0 += 8) {
        uint4 v[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) v[c] = valid ? __ldg(src + c0 + c) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int c = 0; c < 8; ++c) *reinterpret_cast<uint4*>(qs + sw128(r, c0 + c)) = v[c];
      }
      tc::fence_proxy_async_smem();
      named_sync(kBarQ, 128);
      if (tid == 0) tc::mbar_arrive_cluster(&bars->q_full[0], 0);
    }
    int t_total = 0;
    for (int x = gi; x < g_end; ++x) t_total += group_view(table, off_groups, off_rows, x).n_tiles;
    int t = 0, n = 0;
    for (; gi < g_end; gi = next_group(gi), ++n) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      const int ridx = grow / g;
      const bool valid = ridx < gv.n_req;
      const int req = valid ? gv.rows[ridx * kRowInts + 0] : 0;
      const int vis = valid ? gv.rows[ridx * kRowInts + 1] : 0;
      const int slot = valid ? gv.rows[ridx * kRowInts + 2] : 0;
      const int qh = gv.kh * g + (grow % g);
      float l = 0.f, my_m = 0.f;
      bool have = false;
      const bool idle = !__any_sync(0xffffffffu, valid);
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        if (t % kGroups != grp) continue;
        mbar_wait(&bars->s_full[grp], (t / kGroups) & 1);
        tc::fence_after();
        if (idle) {
          // all 32 rows are padding: only the barrier protocol
          if (t > 0) named_sync(pub_other, 64);
          if (t + 1 < t_total) {
            mpub[grp * 128 + r] = 0.f;
            named_arrive(pub_mine, 64);
          }
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_cluster(&bars->p_full[grp], 0);
          continue;
        }
        const int lim = vis - j * kBN;  // visible columns of this tile
        const bool ragged = !__all_sync(0xffffffffu, !valid || lim >= kBN);
        // pass 1: the row max, 64 columns at a time (masked only on a
        // ragged tile: the warp-uniform branch keeps the common path lean)
        float mx = -INFINITY;
#pragma unroll
        for (int c = 0; c < 4; c += 2) {
          uint32_t a[64];
          tc::tmem_ld32(my_s + 32 * c, a);
          tc::tmem_ld32(my_s + 32 * (c + 1), a + 32);
          tc::wait_ld();
          if (ragged) {
#pragma unroll
            for (int i = 0; i < 64; ++i)
              if (32 * c + i >= lim) a[i] = 0xff800000u;  // -inf
          }
          float m8[8];
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = __uint_as_float(a[k]);
#pragma unroll
          for (int i = 8; i < 56; i += 16)
#pragma unroll
            for (int k = 0; k < 8; ++k)
              m8[k] = fmaxf(m8[k], fmaxf(__uint_as_float(a[i + k]), __uint_as_float(a[i + 8 + k])));
#pragma unroll
          for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], __uint_as_float(a[56 + k]));
          mx = fmaxf(mx, fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7]))));
        }
        const float mt = valid ? mx * cscale : 0.f;
        float m_prev = mt;
        if (t > 0) {
          named_sync(pub_other, 64);
          if (j > 0) m_prev = mpub[((grp + kGroups - 1) % kGroups) * 128 + r];
        }
        float mr = m_prev;
        if (j > 0) {
          const bool need = mt > m_prev + kRescaleLog2;
          if (__any_sync(0xffffffffu, need)) {
            // PV(t - 1) must have landed (PV(t) waits for our P); PV(t - 5)
            // is done (S(t) was issued after PV(t - 3)), so the parity is exact
            mbar_wait(&bars->pv_done[(t - 1) & 3], ((t - 1) >> 2) & 1);
            tc::fence_after();
            const float alpha = need ? fast_exp2(m_prev - mt) : 1.f;
            const uint32_t my_o = tmem + lane_addr + kColO;
#pragma unroll 1
            for (int c = 0; c < 8; ++c) {
              uint32_t o[16];
              tc::tmem_ld16(my_o + c * 16, o);
              tc::wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] = __float_as_uint(__uint_as_float(o[i]) * alpha);
              tc::tmem_st16(my_o + c * 16, o);
            }
            tc::wait_st();
            if (need) mr = mt;
          }
        }
        if (t + 1 < t_total) {
          mpub[grp * 128 + r] = mr;
          named_arrive(pub_mine, 64);
        }
        if (!have) {
          my_m = mr;
          have = true;
        } else if (mr != my_m) {
          l *= fast_exp2(my_m - mr);
          my_m = mr;
        }
        // pass 2: P = 2^(S c - m) 32 columns at a time, stored as bf16 over
        // the first half of the tile's S columns (chunk c's P columns
        // [16 c, 16 c + 16) hold S values already read)
        const float2 nm = make_float2(-mr, -mr);
        float2 l2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        uint32_t sa[32];
        tc::tmem_ld32(my_s, sa);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          tc::wait_ld();
          uint32_t sc[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) sc[i] = sa[i];
          if (c + 1 < 4) tc::tmem_ld32(my_s + 32 * (c + 1), sa);  // next chunk in flight
          if (ragged) {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (32 * c + i >= lim) sc[i] = 0xff800000u;  // -inf
          }
          uint32_t pw[16];
#pragma unroll
          for (int w = 0; w < 16; ++w) {
            const float2 y = tc::ffma2(make_float2(__uint_as_float(sc[2 * w]), __uint_as_float(sc[2 * w + 1])), c2, nm);
            const float2 p = make_float2(fast_exp2(y.x), fast_exp2(y.y));
            l2[w & 3] = tc::fadd2(l2[w & 3], p);
            pw[w] = pack_bf16(p.x, p.y);
          }
          tc::tmem_st16(my_s + 16 * c, pw);
        }
        {
          const float2 la = tc::fadd2(l2[0], l2[1]), lb = tc::fadd2(l2[2], l2[3]);
          l += (la.x + la.y) + (lb.x + lb.y);
        }
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(&bars->p_full[grp], 0);
      }
      // ---- unit end: the group that ran the last tile merges the groups'
      // row sums and writes the partial; the others hand over (l, m)
      const int tl = t - 1, last = tl % kGroups, l_bar = 13 + (n & 1);
      if (n > 0) mbar_wait(&bars->epi_done[(n - 1) & 1], ((n - 1) >> 1) & 1);  // lx / staging reuse
      if (grp != last) {
        lx[grp * 128 + r] = make_float2(have ? l : 0.f, my_m);
        named_arrive(l_bar, 32 * kSoftmaxWarps);
      } else {
        named_sync(l_bar, 32 * kSoftmaxWarps);
        float l_run = l;
#pragma unroll
        for (int k = 1; k < kGroups; ++k) {
          const float2 o2 = lx[((grp + k) % kGroups) * 128 + r];
          if (o2.x > 0.f) l_run += o2.x * fast_exp2(o2.y - my_m);
        }
        mbar_wait(&bars->pv_done[tl & 3], (tl >> 2) & 1);  // PV(tl) landed => the unit landed
        tc::fence_after();
        float* dst = nullptr;
        const float inv = 1.f / l_run;
        if (valid) {
          if (slot < 0) {
            dst = out + ((int64_t)req * hq_local + qh) * kD;
          } else {
            const int64_t ei = (int64_t)slot * hq_local + qh;
            dst = part_o + ei * kD;
            part_ml[2 * ei] = my_m * 0.69314718055994530942f;
            part_ml[2 * ei + 1] = l_run;
          }
        }
        // O 32 columns at a time -> this warp's staging rows in the unit's Q
        // buffer -> coalesced 128-byte row-chunk stores; O is released once
        // its last chunk is read
        float4* stg = reinterpret_cast<float4*>(smem + kOffQ + (n & 1) * kQBytes) + quad * 512;
        const uint32_t my_o = tmem + lane_addr + kColO;
#pragma unroll 1
        for (int c = 0; c < 4; ++c) {
          uint32_t ch[32];
          tc::tmem_ld32(my_o + c * 32, ch);
          tc::wait_ld();
          if (c == 3) {
            tc::fence_before();
            __syncwarp();
            if (lane == 0) tc::mbar_arrive_cluster(&bars->o_free, 0);
          }
          float4* sb = stg + (c & 1) * 256;
#pragma unroll
          for (int k = 0; k < 8; ++k)
            sb[lane * 8 + (k ^ (lane & 7))] =
                make_float4(__uint_as_float(ch[4 * k]) * inv, __uint_as_float(ch[4 * k + 1]) * inv,
                            __uint_as_float(ch[4 * k + 2]) * inv, __uint_as_float(ch[4 * k + 3]) * inv);
          __syncwarp();
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int row = 4 * i + (lane >> 3), k = lane & 7;
            float* d = reinterpret_cast<float*>(__shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(dst), row));
            if (d) {
              const float4 v = sb[row * 8 + (k ^ (row & 7))];
              asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                               reinterpret_cast<float4*>(d + c * 32) + k),
                           "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                           : "memory");
            }
          }
        }
        if (cnt) {
          __threadfence();
          named_sync(kBarQ, 128);
          if (valid && slot >= 0) {
            const int e = __ldg(entry_of + (int64_t)req * (hq_local / g) + gv.kh);
            if (e >= 0) atomicAdd(cnt + e, 1);
          }
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars->epi_done[n & 1]);
      }
    }
  }
  // drain: tcgen05.commit arrivals nobody waited for must land before exit
  __threadfence();
  __syncthreads();
  if (tid == 0 && tc_done) atomicAdd(tc_done, 1);
  if (warp == kMmaWarp) {
    int g_begin, g_end;
    ld_range(g_begin, g_end);
    int tiles = 0, units = 0;
    for (int gi = g_begin; gi < g_end; ++gi) {
      const int nt = group_view(table, off_groups, off_rows, gi).n_tiles;
      tiles += nt;
      units += nt > 0;
    }
    auto drain = [&](uint64_t* bar, int stages, bool per_unit) {
      for (int s = 0; s < stages; ++s) {
        const int cnt_s = ((per_unit ? units : tiles) - s + stages - 1) / stages;
        if (cnt_s > 0) mbar_wait(&bar[s], (cnt_s - 1) & 1);
      }
    };
    drain(bars->s_full, kGroups, false);
    drain(bars->k_empty, kKStages, false);
    drain(bars->v_empty, kVStages, false);
    drain(bars->pv_done, 4, false);
    drain(bars->q_empty, 2, true);
  }
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  if (warp == kMmaWarp) tc::tmem_dealloc_pair(tmem, kTmemCols);
}

}  // namespace tc3

int32_t cuda_status(cudaError_t e, const char* what);
int32_t encode_pool_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows);
int32_t encode_pool_halves_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows);
int32_t encode_q_map(CUtensorMap* map, const void* q, int bs, int hq_local, int g);

int32_t launch_tc3(const int32_t* table, const codec_table_info& in, const void* q, const void* k, const void* v,
                   int64_t pool_tokens, int g, int h_local, int bs, void* out, void* part_o, void* part_ml,
                   cudaStream_t st, const int32_t* page_table, int page_shift, int32_t* tc_done,
                   const int32_t* entry_of, int32_t* cnt) {
  if (in.n_tc_groups == 0 || in.n_tc_blocks == 0) return CODEC_OK;
  CUtensorMap mk, mv, mq;
  CODEC_TRY(encode_pool_halves_map(&mk, k, (int64_t)h_local * pool_tokens, 64));
  CODEC_TRY(encode_pool_map(&mv, v, (int64_t)h_local * pool_tokens, tc3::kBN));
  CODEC_TRY(encode_q_map(&mq, q, bs, h_local * g, g));
  cudaError_t e = cudaFuncSetAttribute(tc3::tc3_pac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, tc3::kSmem);
  if (e != cudaSuccess) return cuda_status(e, "tc3 smem attribute");
  dim3 grid(kTcCtasPerBlock * in.n_tc_blocks, 1);
  tc3::tc3_pac_kernel<<<grid, tc3::kThreads, tc3::kSmem, st>>>(
      mk, mv, mq, table, in.off_tc, in.off_rows, in.off_tc_block_ptr, (const __nv_bfloat16*)q, pool_tokens, g,
      h_local * g, (float*)out, (float*)part_o, (float*)part_ml, page_table, page_shift, tc_done, entry_of, cnt);
  return cuda_status(cudaGetLastError(), "tc3 launch");
}

}  // namespace codec
