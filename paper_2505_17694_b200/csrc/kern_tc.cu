// K2: shared-node split attention on the 5th-generation tensor cores,
// one CTA PAIR (cta_group::2) per schedule block.
//
// A group is a KV slice [kv_tok, kv_tok + len) of a shared node and up to
// 256 query-head rows (256/g requests of the node's query set with their g
// query heads: GQA packing turns the per-request GEMVs into one dense
// contraction). The pair runs it as M=256 MMAs: CTA rank c owns rows
// [128c, 128c+128) -- its S, P and O live in its own TMEM, its Q tile in
// its own SMEM -- while each 128-token K/V tile is split between the two
// CTAs' shared memories (K by tokens, V by head-dim columns) and read by
// both through the pair's MMA. Per 128-token KV tile t:
//     S(t) = Q K_t^T       tcgen05.mma.cta_group::2 SS, M256 N128 K128 -> S buffer t%2
//     P(t) = 2^(S c - m)   one softmax thread per row (TMEM lane), bf16 -> P buffer t%2
//     O   += P(t) V_t      tcgen05.mma.cta_group::2 TS (A = P in TMEM), M256 N128 K128
// Per row this is the reference's pac_kernel math (_kernels.pyx:25-54);
// the partial (O/l, m, l) feeds the LSE merge (kern_merge.cu).
//
// Pipeline (why it is shaped like this on B200): S and P are both double-
// buffered in TMEM, so S(t+2) is issued as soon as the softmax has pulled
// S(t) into registers -- the tensor pipe never waits for an exponential.
// Two softmax warpgroups take alternate tiles (A even, B odd) with one
// thread owning a whole 128-column row: no intra-row exchange, and while
// one group waits on TMEM loads the other keeps MUFU/FMA busy. The row's
// running max passes from group to group once per tile through SMEM and a
// named-barrier arrive/sync pair; O is only touched by the lazy rescale
// (row max grew by > 2^8), so the common path has no O traffic at all.
// Cross-CTA signals are per-warp mbarrier arrivals on the leader with
// release.cta semantics (~155 clk one way, tools/ubench_cluster.cu).
//
// TMEM (512 columns per CTA): S0 [0,128) S1 [128,256) P0 [256,320)
// P1 [320,384) O [384,512).
// Warps: 0-3 softmax group A, 4-7 group B (lane quadrant = warp & 3),
// 8 / 10 TMA producers of K / V (both CTAs load their halves; completion on
// the leader's barriers), 9 TMEM allocator + S MMA issuer (leader only),
// 10 also the PV MMA issuer (leader only), 11 Q loads of later units.
#include <cuda.h>
#include <cuda_runtime.h>

#include "common.h"
#include "device_table.h"
#include "device_util.cuh"
#include "mma_sync.cuh"
#include "tc_ptx.cuh"

namespace codec {

// critical-path waits of this kernel (issuers, softmax): plain try_wait loop
// or try_wait with a suspend-time hint (CODEC_TC_WAIT_HINT ns)
__device__ __forceinline__ void tc_wait(uint64_t* bar, uint32_t phase) {
#if defined(CODEC_TC_WAIT_HINT) && !defined(CODEC_HANG_CHECK)
  mbar_wait_hint(bar, phase, CODEC_TC_WAIT_HINT);
#else
  mbar_wait(bar, phase);
#endif
}

constexpr int kTcSoftmaxWarps = 8;           // 2 groups x 4 lane quadrants
constexpr int kTcProducerWarp = kTcSoftmaxWarps;       // K loads
constexpr int kTcMmaWarp = kTcSoftmaxWarps + 1;
constexpr int kTcVProducerWarp = kTcSoftmaxWarps + 2;  // V loads + PV MMAs (K must not queue behind V)
constexpr int kTcQWarp = kTcSoftmaxWarps + 3;          // gathers the next unit's Q rows into SMEM
constexpr int kTcThreads = 32 * (kTcSoftmaxWarps + 4);
constexpr int kTcBN = 128;                   // tokens per KV tile
constexpr int kTcD = 128;                    // head dim
#ifndef CODEC_TC_PREFETCH
#define CODEC_TC_PREFETCH 4
#endif
constexpr int kTcPrefetch = CODEC_TC_PREFETCH;  // tiles ahead the producer warms L2
// K half-tiles as ONE 3-D TMA box (64 d x 64 tokens x 2 halves = both SW128
// atom columns) instead of one 2-D box per atom column: the SM's TMA unit
// pays ~190 clk per op whatever its size
#ifndef CODEC_TC_K3D
#define CODEC_TC_K3D 1
#endif
constexpr int kQBytes = 128 * 128 * 2;       // this CTA's 128-row Q tile (32 KB)
constexpr int kQAtom = kQBytes / 2;          // Q atom column: 128 rows x 64 d (16 KB)
constexpr int kHalfBytes = 64 * 128 * 2;     // this CTA's half of a K or V tile (16 KB)
constexpr int kKAtom = kHalfBytes / 2;       // K-half atom column: 64 tokens x 64 d (8 KB)
// One CTA owns its SM: 384 threads x 168 registers at launch, then
// setmaxnreg moves the role warps' surplus to the softmax warps (per SMSP:
// 2 softmax warps x 200 + 1 role warp x 96 <= 512; the pool the CTA got at
// launch, 384 x 168, must cover it: 256 x 200 + 128 x 96 <= 64512). No other kernel may
// share the SM: the hand-off corrupted the registers of a co-resident CTA
// of another kernel in testing (tools/determinism.py).
constexpr int kTcRegsSoftmax = 200, kTcRegsOther = 96;
static_assert(32 * kTcSoftmaxWarps * kTcRegsSoftmax + (kTcThreads - 32 * kTcSoftmaxWarps) * kTcRegsOther <=
                  kTcThreads * (65536 / kTcThreads / 8 * 8),
              "setmaxnreg.inc would wait forever for registers the CTA does not own");
// K / V ring depths (SMEM: 64 KB of Q + 16 KB per stage); 4 / 4 measured
// 1 % faster than 4 / 6 on cfg2 (tools/ab_rounds.py), 3 / 4 the same
#ifndef CODEC_TC_KSTAGES
#define CODEC_TC_KSTAGES 4
#define CODEC_TC_VSTAGES 4
#endif
constexpr int kTcKStages = CODEC_TC_KSTAGES, kTcVStages = CODEC_TC_VSTAGES;
constexpr int kOffQ = 0;                     // Q0, Q1 (double-buffered across units)
constexpr int kOffK = kOffQ + 2 * kQBytes;
constexpr int kOffV = kOffK + kTcKStages * kHalfBytes;
constexpr int kOffMpub = kOffV + kTcVStages * kHalfBytes;  // [2 groups][128 rows] f32 published row max
constexpr int kOffLx = kOffMpub + 2 * 128 * 4;             // [128 rows] float2 (l, m) at a unit's end
constexpr int kOffBar = kOffLx + 128 * 8;
constexpr int kTcSmem = kOffBar + 512;
static_assert(kTcSmem <= 232448, "exceeds the 227 KB opt-in shared memory");
constexpr uint32_t kTmemCols = 512;
constexpr uint32_t kColS = 0, kColP = 256, kColO = 384;
constexpr float kRescaleLog2 = 8.f;
// of every 4 score pairs, how many take the FMA-pipe polynomial instead of MUFU.EX2
#ifndef CODEC_TC_POLY_PAIRS
#define CODEC_TC_POLY_PAIRS 0
#endif
// epilogue row stores as 256-bit STG (two rows per warp instruction): the
// per-unit global stores 4424 -> 2916 clk, K2 alone 139.9 -> 138.6 us on
// cfg2 (tools/epi_timing.py, tools/ab_rounds.py); =0 restores STG.128
#ifndef CODEC_TC_STG256
#define CODEC_TC_STG256 1
#endif
// epilogue without staging: each thread stores its own row as 16 full
// 32-byte sectors (STG.256), all four warps at once -- stores 2430 clk per
// unit boundary vs 808 + 2921 staged (tools/epi_timing.py), K2 alone 138.7
// -> 137.5 us on cfg2 (tools/ab_rounds.py); =0 restores the staged path
#ifndef CODEC_TC_DIRECT_STORE
#define CODEC_TC_DIRECT_STORE 1
#endif
constexpr int kGroupWarpArrivals = 2 * 4;  // one group's 4 warps in both CTAs

struct TcBars {
  uint64_t k_full[kTcKStages], k_empty[kTcKStages];
  uint64_t v_full[kTcVStages], v_empty[kTcVStages];
  uint64_t q_full[2], q_empty[2], s_full[2], s_free[2], p_full[2];
  uint64_t epi_done[2];  // unit n's epilogue no longer uses Q buffer n % 2 as staging
  uint64_t q_tma[2];     // this CTA's TMA Q load of buffer b landed (local)
  uint64_t pv_done[4];  // PV(t) completes pv_done[t % 4] (parity waits stay within one phase)
  uint64_t o_free;
  uint32_t tmem_slot;
};

// 16-byte chunk c (0..15 along a 128-element row) of row r in a K-major
// SWIZZLE_128B 128-row tile made of two 64-element atom columns
__device__ __forceinline__ uint32_t sw128(int r, int c) {
  return (c >> 3) * kQAtom + r * 128 + (((c & 7) ^ (r & 7)) << 4);
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

// Two lanes of the same polynomial with packed f32x2 arithmetic (FADD2/FFMA2)
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
  v.n_tiles = (grp[kGrpMaxVis] + kTcBN - 1) / kTcBN;
  return v;
}

// Walks the (group, tile) sequence of one schedule block; groups with no
// tiles (cannot occur: every row sees >= 1 token) are skipped.
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


#ifdef CODEC_HANG_CHECK
// per-CTA progress words in host-mapped memory: [role * 2] = tile, [role * 2 + 1] = step
#define PROG(role, tile, step)                                                                      \
  do {                                                                                              \
    if (g_hang_buf && (threadIdx.x & 31) == 0) {                                                  \
      volatile int* pr = g_hang_buf + 8200 + (blockIdx.y * gridDim.x + blockIdx.x) * 8 + (role) * 2; \
      pr[0] = (tile);                                                                               \
      pr[1] = (step);                                                                               \
    }                                                                                               \
  } while (0)
#else
#define PROG(role, tile, step) \
  do {                         \
  } while (0)
#endif

__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void named_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kTcThreads, 1)
    tc_pac_kernel(const __grid_constant__ CUtensorMap tmk, const __grid_constant__ CUtensorMap tmv,
                  const __grid_constant__ CUtensorMap tmq, const int32_t* __restrict__ table, int off_groups, int off_rows, int off_block_ptr,
                  const __nv_bfloat16* __restrict__ q, int64_t pool_tokens, int g, int hq_local,
                  float* __restrict__ out, float* __restrict__ part_o, float* __restrict__ part_ml,
                  long long* __restrict__ trace, int dbg_flags, long long* __restrict__ ctalog,
                  const int32_t* __restrict__ page_table, int page_shift, int32_t* __restrict__ tc_done,
                  const int32_t* __restrict__ entry_of, int32_t* __restrict__ cnt) {
  const long long t_start = ctalog ? global_ns() : 0;
#ifdef CODEC_TC_DEBUG
  // timing-only ablations (tools/tc_ablate.py); compiled out of the product
  // build -- even untaken, their code cost the softmax ~110 register moves
  // per tile
  const int dbg = dbg_flags;
#else
  constexpr int dbg = 0;
#endif
  extern __shared__ __align__(1024) uint8_t smem[];
  const uint32_t sbase = smem_u32(smem);
  if (sbase & 1023) __trap();  // SWIZZLE_128B atoms need 1024-byte alignment
  static_assert(sizeof(TcBars) <= 512, "barrier block");
  TcBars* bars = reinterpret_cast<TcBars*>(smem + kOffBar);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t rank = tc::cluster_rank();
  // pool row of logical token x of kv head kh (paged pool: through the
  // page table; a 64- or 128-token box never crosses a page)
  auto prow = [&](int kh, int x) -> int {
    if (page_shift) x = (__ldg(page_table + (x >> page_shift)) << page_shift) | (x & ((1 << page_shift) - 1));
    return kh * (int)pool_tokens + x;
  };
  const bool leader = rank == 0;
  const int blk = blockIdx.x >> 1;
  // optional timeline of pair (0, 0): trace[(event * 2 + rank) * 64 + tile]
#ifndef CODEC_TC_TRACE_QUAD
#define CODEC_TC_TRACE_QUAD 0  // lane quadrant (warp & 3) whose softmax warp stamps its tiles
#endif
#ifdef CODEC_TC_TRACE
  // debug builds only (CODEC_NVCC_EXTRA=-DCODEC_TC_TRACE): the stamps cost
  // the single-warp MMA issuer ~70 instructions per tile even when off
  const bool tracing = trace != nullptr && blk == 0;
  auto stamp = [&](int ev, int tt) {
    if (tracing && tt < 64) trace[(ev * 2 + rank) * 64 + tt] = clock64();
  };
  // sequential MMA-issuer log after the per-tile stamps: (clock, code << 16 | tile)
  int seq_n = 0;
  auto seq = [&](int code, int tt) {
    // S issuer entries [0, 1024), PV issuer entries [1024, 2048)
    const int base = warp == kTcVProducerWarp ? 1024 : 0;
    if (tracing && seq_n < 1024) {
      trace[17 * 2 * 64 + 2 * (base + seq_n)] = clock64();
      trace[17 * 2 * 64 + 2 * (base + seq_n) + 1] = (code << 16) | (tt & 0xffff);
      ++seq_n;
    }
  };
#else
  (void)trace;
  auto stamp = [](int, int) {};
  auto seq = [](int, int) {};
#endif
  // The block's unit range is re-read inside each role branch (asm loads
  // the compiler cannot hoist): kept live across the setmaxnreg hand-off it
  // was spilled to local memory and reloaded on the issuers' loop paths.
  auto ld_range = [&](int& gb, int& ge) {
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(gb) : "l"(table + off_block_ptr + blk));
    asm volatile("ld.global.nc.b32 %0, [%1];" : "=r"(ge) : "l"(table + off_block_ptr + blk + 1));
    if (dbg_flags & CODEC_FLAG_DBG_NO_TC_UNITS) ge = gb;
  };
#define CODEC_TC_RANGE \
  int g_begin, g_end;  \
  ld_range(g_begin, g_end)

  if (tid == 0) {
    for (int s = 0; s < kTcKStages; ++s) {
      mbar_init(&bars->k_full[s], 1);
      mbar_init(&bars->k_empty[s], 1);
    }
    for (int s = 0; s < kTcVStages; ++s) {
      mbar_init(&bars->v_full[s], 1);
      mbar_init(&bars->v_empty[s], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars->q_full[i], 2);  // the Q warps of both CTAs
      mbar_init(&bars->q_empty[i], 1);
      mbar_init(&bars->epi_done[i], 4);  // the epilogue group's 4 warps (this CTA)
      mbar_init(&bars->q_tma[i], 1);
      mbar_init(&bars->s_full[i], 1);
      mbar_init(&bars->s_free[i], kGroupWarpArrivals);
      mbar_init(&bars->p_full[i], kGroupWarpArrivals);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bars->pv_done[i], 1);
    mbar_init(&bars->o_free, kGroupWarpArrivals);
    fence_barrier_init();
  }
  if (warp == kTcMmaWarp) tc::tmem_alloc_pair(&bars->tmem_slot, kTmemCols);
  if (warp == kTcProducerWarp && lane == 0) {
    tc::prefetch_tmap(&tmk);
    tc::prefetch_tmap(&tmv);
  }
  tc::fence_before();
  // the suffix kernel launched after this one (programmatic dependent
  // launch) may take any SM this grid leaves idle or releases
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  tc::cluster_sync();  // barriers of both CTAs initialised, TMEM allocated
  tc::fence_after();
  const uint32_t tmem = bars->tmem_slot;
  const bool iso = (dbg & CODEC_FLAG_DBG_ISSUER_ONLY) != 0;  // timing experiment
  if (iso && warp != kTcMmaWarp && warp != kTcVProducerWarp) {
    // nothing: only the MMA issuers run
  } else if (warp >= kTcSoftmaxWarps) {
  // producer / MMA warpgroup: hands registers to the softmax warpgroups
#ifndef CODEC_NO_SETMAXNREG
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;" ::"n"(kTcRegsOther));
#endif
  if (warp == kTcProducerWarp) {
    // ================================================ K producer (both CTAs)
    CODEC_TC_RANGE;
    // K half: tokens [64 rank, 64 rank + 64) x all 128 d (two SW128 atom
    // columns), completing on the leader's k_full. Also warms L2 with the
    // K and V tiles kTcPrefetch ahead.
    // L2 warming runs kTcPrefetch tiles ahead of the loads over the block's
    // whole tile sequence -- across unit boundaries, so a new unit's first
    // tiles do not start cold from HBM
    TileCursor pfc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
    pfc.open();
    int t_pf = 0;
    auto prefetch_to = [&](int limit) {
      for (; !pfc.done() && t_pf < limit; ++t_pf, pfc.next()) {
        if (dbg & CODEC_FLAG_DBG_NO_LOADS) continue;
        const int xp = pfc.gv.kv_tok + pfc.j * kTcBN;
        const int ypk = prow(pfc.gv.kh, xp + 64 * rank), ypv = prow(pfc.gv.kh, xp);
        if (tc::elect_one()) {
#if CODEC_TC_K3D
          tc::tma_prefetch_3d(&tmk, 0, ypk, 0);
#else
          tc::tma_prefetch_2d(&tmk, 0, ypk);
          tc::tma_prefetch_2d(&tmk, 64, ypk);
#endif
          tc::tma_prefetch_2d(&tmv, 64 * rank, ypv);
        }
        __syncwarp();
      }
    };
    prefetch_to(kTcPrefetch);
    int t = 0;
    for (int gi = g_begin; gi < g_end; ++gi) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        const int ks = t % kTcKStages;
        PROG(3, t, 1);
        if (t >= kTcKStages) mbar_wait_relaxed(&bars->k_empty[ks], ((t / kTcKStages) - 1) & 1);
        PROG(3, t, 2);
        if (dbg & CODEC_FLAG_DBG_NO_LOADS) {
          if (leader && tc::elect_one()) mbar_arrive(&bars->k_full[ks]);
        } else if (tc::elect_one()) {
          if (leader) mbar_arrive_expect_tx(&bars->k_full[ks], 2 * kHalfBytes);
          uint8_t* kd = smem + kOffK + ks * kHalfBytes;
          const int yk = prow(gv.kh, gv.kv_tok + j * kTcBN + 64 * rank);
#if CODEC_TC_K3D
          tc::tma_load_3d_pair(kd, &tmk, 0, yk, 0, &bars->k_full[ks]);  // both atom columns, one op
#else
          tc::tma_load_2d_pair(kd, &tmk, 0, yk, &bars->k_full[ks]);
          tc::tma_load_2d_pair(kd + kKAtom, &tmk, 64, yk, &bars->k_full[ks]);
#endif
        }
        __syncwarp();
        prefetch_to(t + 1 + kTcPrefetch);
      }
    }
  } else if (warp == kTcVProducerWarp) {
    // ================================================ V producer (both CTAs) + PV issuer (leader)
    // V half: all 128 tokens x d [64 rank, 64 rank + 64), completing on the
    // leader's v_full. The leader's warp interleaves its loads with the PV
    // MMAs, kVAhead tiles ahead: V(tp + 4) reuses the stage of V(tp - 2),
    // free once PV(tp - 2) landed -- which P(tp) waits for anyway, so the
    // load never delays PV(tp). The S and PV MMAs come from two warps: one
    // in-order issuer for both spent ~1800 clk per tile on its own
    // instruction latency (the pipe needs 1024).
    // PV: A = P (TMEM, 8 columns per 16 tokens), B = V half (MN-major SW128,
    // one atom column).
    CODEC_TC_RANGE;
    constexpr int kVAhead = kTcVStages - 2;
    static_assert(kVAhead + 2 <= kTcVStages, "V(tp + kVAhead) must reuse a stage PV(tp - 2) released");
    TileCursor vc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
    vc.open();
    int tv = 0;  // V tiles loaded
    auto load_v = [&]() {
      const int vs = tv % kTcVStages;
      if (tv >= kTcVStages && !iso) mbar_wait_relaxed(&bars->v_empty[vs], ((tv / kTcVStages) - 1) & 1);
      if ((dbg & CODEC_FLAG_DBG_NO_LOADS) || iso) {
        if (leader && tc::elect_one() && !iso) mbar_arrive(&bars->v_full[vs]);
      } else if (tc::elect_one()) {
        if (leader) mbar_arrive_expect_tx(&bars->v_full[vs], 2 * kHalfBytes);
        const int y = prow(vc.gv.kh, vc.gv.kv_tok + vc.j * kTcBN);
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
      constexpr uint32_t idesc_o = tc::idesc_bf16(256, kTcD, false, true);
      const uint64_t dv = tc::smem_desc(sbase + kOffV, kHalfBytes, 1024);
      TileCursor pc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
      pc.open();
      for (int tp = 0; !pc.done(); ++tp) {
        if (!vc.done()) load_v();  // V(tp + kVAhead)
        const int b = tp & 1, vs = tp % kTcVStages;
        if (lane == 0) seq(5, tp);
        if (!iso) tc_wait(&bars->p_full[b], (tp >> 1) & 1);  // P(tp) in both CTAs' TMEM
        if (lane == 0) seq(6, tp);
        if (!iso) tc_wait(&bars->v_full[vs], (tp / kTcVStages) & 1);
        if (lane == 0) seq(7, tp);
        if (pc.j == 0 && pc.n > 0 && !iso) tc_wait(&bars->o_free, (pc.n - 1) & 1);  // epilogue read O
        tc::fence_after();
        const uint64_t bv = dv + (uint64_t)((vs * kHalfBytes) >> 4);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kTcBN / 16; ++k)
            tc::mma2_f16_ts(tmem + kColO, tmem + kColP + b * 64 + k * 8, bv + (uint64_t)((k * 16 * 128) >> 4),
                            idesc_o, (pc.j > 0 || k > 0) ? 1u : 0u);
          tc::commit_pair(&bars->v_empty[vs]);
          tc::commit_pair(&bars->pv_done[tp & 3]);
        }
        __syncwarp();
        if (lane == 0) seq(9, tp);
        pc.next();
      }
    }
  } else if (warp == kTcQWarp) {
    // ================================================ Q gather (both CTAs)
    // this CTA's 128 query-head rows of each unit (row r = request r / g of
    // the unit, q head kv_head * g + r % g) into Q buffer n % 2, K-major
    // SW128; the buffer is reused once the unit two back issued its last S
    CODEC_TC_RANGE;
    const int nq_local = hq_local;
    int n = 0;
    int qtma_uses[2] = {0, 0};  // phases of q_tma[b]
    for (int gi = g_begin; gi < g_end; ++gi) {
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (gv.n_tiles == 0) continue;
      if (n == 0) {  // the first unit's Q is loaded by the softmax warps (lower latency)
        if (gv.qreq0 >= 0) qtma_uses[0] = 1;  // ... through q_tma[0]'s first phase
        ++n;
        continue;
      }
      const int qb = n & 1;
      if (n >= 2) {
        mbar_wait_relaxed(&bars->q_empty[qb], ((n - 2) >> 1) & 1);
        mbar_wait_relaxed(&bars->epi_done[qb], ((n - 2) >> 1) & 1);  // staging of unit n - 2's O
      }
      uint8_t* qs = smem + kOffQ + qb * kQBytes;
      if (gv.qreq0 >= 0) {
        // consecutive requests: two 4D TMA boxes (64 d x g heads x 128/g
        // requests, SW128) -- one round trip instead of a gather
        const int rq = 128 / g;
        if (lane == 0) {
          mbar_arrive_expect_tx(&bars->q_tma[qb], kQBytes);
          tc::tma_load_4d(qs, &tmq, 0, 0, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[qb]);
          tc::tma_load_4d(qs + kQAtom, &tmq, 0, 1, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[qb]);
        }
        tc_wait(&bars->q_tma[qb], (qtma_uses[qb]++) & 1);
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
            const uint4* src = reinterpret_cast<const uint4*>(
                q + ((int64_t)req * nq_local + gv.kh * g + (grow % g)) * kTcD);
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
  } else if (warp == kTcMmaWarp) {
    // ================================================ S issuer (leader only)
    // S(ts) into S buffer ts % 2 once the softmax pulled S(ts - 2) out of it
    // (blocking waits: the issuing thread sleeps in mbarrier.try_wait). A
    // new unit's Q may wait for the epilogue of the unit two back; the PV
    // MMAs come from another warp, so that wait blocks nothing else.
    // A = Q tile (K-major SW128, 16 KB atom columns), B = K half (K-major
    // SW128, 8 KB atom columns).
    if (leader) {
      CODEC_TC_RANGE;
      constexpr uint32_t idesc_s = tc::idesc_bf16(256, kTcBN, false, false);
      const uint64_t dq = tc::smem_desc(sbase + kOffQ, 16, 1024);
      const uint64_t dk = tc::smem_desc(sbase + kOffK, 16, 1024);
      TileCursor sc{table, off_groups, off_rows, g_begin, g_end, 0, 0, {}};
      sc.open();
      for (int ts = 0; !sc.done(); ++ts) {
        const int s = ts % kTcKStages, b = ts & 1;
        if (lane == 0) seq(1, ts);
        if (ts >= 2 && !iso) tc_wait(&bars->s_free[b], ((ts - 2) >> 1) & 1);  // S(ts-2) pulled out by both CTAs
        if (sc.j == 0 && !iso) tc_wait(&bars->q_full[sc.n & 1], (sc.n >> 1) & 1);
        if (lane == 0) seq(2, ts);
        if (!iso) tc_wait(&bars->k_full[s], (ts / kTcKStages) & 1);
        if (lane == 0) seq(3, ts);
        tc::fence_after();
        const uint64_t aq = dq + (uint64_t)(((sc.n & 1) * kQBytes) >> 4);
        const uint64_t bk = dk + (uint64_t)((s * kHalfBytes) >> 4);
        if (tc::elect_one()) {
#pragma unroll
          for (int k = 0; k < kTcD / 16; ++k) {
            const uint64_t oa = (uint64_t)((((k >> 2) * kQAtom) + (k & 3) * 32) >> 4);
            const uint64_t ob = (uint64_t)((((k >> 2) * kKAtom) + (k & 3) * 32) >> 4);
            tc::mma2_f16_ss(tmem + kColS + b * 128, aq + oa, bk + ob, idesc_s, k > 0 ? 1u : 0u);
          }
          tc::commit_pair(&bars->s_full[b]);
          tc::commit_pair(&bars->k_empty[s]);
          if (sc.j + 1 == sc.gv.n_tiles) tc::commit_pair(&bars->q_empty[sc.n & 1]);  // unit's Q no longer read
        }
        __syncwarp();
        if (lane == 0) seq(4, ts);
        sc.next();
      }
      PROG(0, 9999, 7);
    }
  }
  } else {
    // ================================================ softmax warpgroups
#ifndef CODEC_NO_SETMAXNREG
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;" ::"n"(kTcRegsSoftmax));
#endif
    CODEC_TC_RANGE;
    const int grp = warp >> 2;   // 0: even tiles, 1: odd tiles
    const int quad = warp & 3;   // TMEM lane quadrant
    const int r = quad * 32 + lane;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float* mpub = reinterpret_cast<float*>(smem + kOffMpub);
    float2* lx = reinterpret_cast<float2*>(smem + kOffLx);
    const int pub_mine = 1 + grp * 4 + quad, pub_other = 1 + (grp ^ 1) * 4 + quad;
    const float cscale = 1.4426950408889634f * rsqrtf((float)kTcD);
    const float2 c2 = make_float2(cscale, cscale);
    const int grow = (int)rank * 128 + r;  // row of the 256-row group
    auto next_group = [&](int gidx) {
      for (++gidx; gidx < g_end; ++gidx)
        if (group_view(table, off_groups, off_rows, gidx).n_tiles > 0) break;
      return gidx;
    };
    int gi = g_begin;
    while (gi < g_end && group_view(table, off_groups, off_rows, gi).n_tiles == 0) ++gi;
    if (gi < g_end && grp == 0 && group_view(table, off_groups, off_rows, gi).qreq0 >= 0) {
      // first unit's Q, consecutive requests: the two 4D TMA boxes the Q
      // warp uses for later units (q_tma[0]'s first phase)
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      if (tid == 0) {
        const int rq = 128 / g;
        mbar_arrive_expect_tx(&bars->q_tma[0], kQBytes);
        tc::tma_load_4d(smem + kOffQ, &tmq, 0, 0, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[0]);
        tc::tma_load_4d(smem + kOffQ + kQAtom, &tmq, 0, 1, gv.kh * g, gv.qreq0 + (int)rank * rq, &bars->q_tma[0]);
        tc_wait(&bars->q_tma[0], 0);
        tc::mbar_arrive_cluster(&bars->q_full[0], 0);
      }
    } else if (gi < g_end && grp == 0) {
      // first unit's Q: one row per thread of group A, all 16 loads in flight
      const GroupView gv = group_view(table, off_groups, off_rows, gi);
      const int ridx = grow / g;
      const bool valid = ridx < gv.n_req;
      const int req = valid ? __ldg(gv.rows + ridx * kRowInts) : 0;
      const uint4* src = reinterpret_cast<const uint4*>(q + ((int64_t)req * hq_local + gv.kh * g + (grow % g)) * kTcD);
      uint4 v[16];
#pragma unroll
      for (int c = 0; c < 16; ++c) v[c] = valid ? __ldg(src + c) : make_uint4(0, 0, 0, 0);
      uint8_t* qs = smem + kOffQ;
#pragma unroll
      for (int c = 0; c < 16; ++c) *reinterpret_cast<uint4*>(qs + sw128(r, c)) = v[c];
      tc::fence_proxy_async_smem();
      named_sync(11, 128);
      if (tid == 0) tc::mbar_arrive_cluster(&bars->q_full[0], 0);
    }
    // total tiles of the block (the last tile publishes no row max)
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
      float l = 0.f, my_m = 0.f;  // my tiles' row sum, relative to 2^my_m
      bool have = false;          // processed a tile of this group
      if (!__any_sync(0xffffffffu, valid)) {
        // all 32 rows of this warp are padding (a piece with < 256 query-
        // head rows): its P and O rows are never read back, so it only
        // keeps the barrier protocol (S release, row-max hand-off with its
        // equally idle partner warp, P-buffer wait, P release)
        for (int j = 0; j < gv.n_tiles; ++j, ++t) {
          if ((t & 1) != grp) continue;
          const int b = t & 1;
          tc_wait(&bars->s_full[b], (t >> 1) & 1);
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_cluster(&bars->s_free[b], 0);
          if (t > 0) named_sync(pub_other, 64);
          if (t + 1 < t_total) {
            mpub[grp * 128 + r] = 0.f;
            named_arrive(pub_mine, 64);
          }
          if (t >= 2) tc_wait(&bars->pv_done[(t - 2) & 3], ((t - 2) >> 2) & 1);
          __syncwarp();
          if (lane == 0) tc::mbar_arrive_cluster(&bars->p_full[b], 0);
        }
      } else
      for (int j = 0; j < gv.n_tiles; ++j, ++t) {
        if ((t & 1) != grp) continue;
        const int b = t & 1;
        if (quad == 0) PROG(1 + grp, t, 1);
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(14, t);
        tc_wait(&bars->s_full[b], (t >> 1) & 1);
        if (quad == 0) PROG(1 + grp, t, 2);
        tc::fence_after();
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(2, t);
        uint32_t sr[128];
        const uint32_t my_s = tmem + lane_addr + kColS + b * 128;
        if (dbg & CODEC_FLAG_DBG_NO_TMEM) {  // timing experiment: no TMEM S traffic
#pragma unroll
          for (int i = 0; i < 128; ++i) sr[i] = __float_as_uint((float)((i * 37 + lane) & 15) * 0.1f);
        } else {
          tc::tmem_ld32(my_s, sr);
          tc::tmem_ld32(my_s + 32, sr + 32);
          tc::tmem_ld32(my_s + 64, sr + 64);
          tc::tmem_ld32(my_s + 96, sr + 96);
          tc::wait_ld();
        }
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(&bars->s_free[b], 0);  // S buffer b may be overwritten
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(4, t);
        const int lim = vis - j * kTcBN;  // visible columns of this tile
        if (!__all_sync(0xffffffffu, !valid || lim >= kTcBN)) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (i >= lim) sr[i] = 0xff800000u;  // -inf
        }
        // row max as 8 independent 3-input chains (depth 8 instead of 64)
        float m8[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = __uint_as_float(sr[k]);
#pragma unroll
        for (int i = 8; i < 120; i += 16)
#pragma unroll
          for (int k = 0; k < 8; ++k)
            m8[k] = fmaxf(m8[k], fmaxf(__uint_as_float(sr[i + k]), __uint_as_float(sr[i + 8 + k])));
#pragma unroll
        for (int k = 0; k < 8; ++k) m8[k] = fmaxf(m8[k], __uint_as_float(sr[120 + k]));
        const float mx = fmaxf(fmaxf(fmaxf(m8[0], m8[1]), fmaxf(m8[2], m8[3])),
                               fmaxf(fmaxf(m8[4], m8[5]), fmaxf(m8[6], m8[7])));
        const float mt = valid ? mx * cscale : 0.f;
        // the row's exponent reference after tile t-1 (published by the other group)
        float m_prev = mt;
        if (quad == 0) PROG(1 + grp, t, 3);
        if (t > 0) {
          named_sync(pub_other, 64);
          if (j > 0) m_prev = mpub[(grp ^ 1) * 128 + r];
        }
        float mr = m_prev;
        if (j > 0) {
          const bool need = mt > m_prev + kRescaleLog2;
          if (__any_sync(0xffffffffu, need)) {  // tcgen05.ld/st are warp-collective
            // PV(t-1) must have landed (PV(t) waits for our P). pv_done[x]
            // completes for PV(x), PV(x+4), ...: PV(t-5) is done (this group
            // waited for PV(t-4) at tile t-2) and PV(t+3) cannot be, so the
            // parity wait is exact.
            tc_wait(&bars->pv_done[(t - 1) & 3], ((t - 1) >> 2) & 1);
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
#ifndef CODEC_TC_LATE_PUBLISH
        if (t + 1 < t_total) {
          mpub[grp * 128 + r] = mr;
          named_arrive(pub_mine, 64);
        }
#endif
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(5, t);
        // my row sum follows the reference
        if (!have) {
          my_m = mr;
          have = true;
        } else if (mr != my_m) {
          l *= fast_exp2(my_m - mr);
          my_m = mr;
        }
        // P = 2^(S c - m) as bf16 pairs, 16 TMEM columns per 32 scores, all
        // computed into registers before waiting for the P buffer: that wait
        // (PV(t-2) landed) then costs only the TMEM stores on the PV chain
#ifdef CODEC_TC_PWAIT_EARLY
        if (t >= 2) tc_wait(&bars->pv_done[(t - 2) & 3], ((t - 2) >> 2) & 1);
#endif
        const float2 nm = make_float2(-mr, -mr);
        // four independent row-sum chains (a single fadd2 chain would be
        // 64 dependent adds long)
        float2 l2[4] = {make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f), make_float2(0.f, 0.f)};
        const uint32_t my_p = tmem + lane_addr + kColP + b * 64;
        uint32_t pall[64];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          uint32_t* pw = pall + 16 * c;
          if (dbg & CODEC_FLAG_DBG_NO_EXP) {  // timing experiment: no exponentials
#pragma unroll
            for (int w = 0; w < 16; ++w) pw[w] = sr[c * 32 + 2 * w] ^ sr[c * 32 + 2 * w + 1];
          } else
#pragma unroll
          for (int w = 0; w < 16; w += 4) {
            // 8 scores: 6 exponentials on the MUFU (16/clk/SM), 2 as a packed
            // f32x2 polynomial on the FMA pipe: the MUFU share that keeps both
            // the XU pipe and the issue slots below saturation
            float2 x[4], p[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              const int e = c * 32 + 2 * (w + k);
              x[k] = tc::ffma2(make_float2(__uint_as_float(sr[e]), __uint_as_float(sr[e + 1])), c2, nm);
            }
            p[0] = make_float2(fast_exp2(x[0].x), fast_exp2(x[0].y));
            p[1] = make_float2(fast_exp2(x[1].x), fast_exp2(x[1].y));
            // (measured after the issuer split: 8/8 on MUFU 114 us, 6/8 117, 4/8 125)
#if CODEC_TC_POLY_PAIRS >= 2
            p[2] = poly_exp2x2(x[2]);
#else
            p[2] = make_float2(fast_exp2(x[2].x), fast_exp2(x[2].y));
#endif
#if CODEC_TC_POLY_PAIRS >= 1
            p[3] = poly_exp2x2(x[3]);
#else
            p[3] = make_float2(fast_exp2(x[3].x), fast_exp2(x[3].y));
#endif
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              l2[k] = tc::fadd2(l2[k], p[k]);
              pw[w + k] = pack_bf16(p[k].x, p[k].y);
            }
          }
        }
#ifdef CODEC_TC_LATE_PUBLISH
        // (experiment) hand the row's exponent reference to the other group
        // only after this tile's exponentials, so the two groups' MUFU phases
        // alternate: the S period becomes uniform (~1570 clk) but the step
        // is slower (123 vs 115 us on cfg2) -- the groups lose their overlap
        if (t + 1 < t_total) {
          mpub[grp * 128 + r] = mr;
          named_arrive(pub_mine, 64);
        }
#endif
        // P buffer b is free once PV(t-2) landed (PV(t-6) is done: waited
        // for at tile t-4; PV(t+2) cannot be)
        if (quad == 0) PROG(1 + grp, t, 5);
#ifndef CODEC_TC_PWAIT_EARLY
        if (t >= 2 && (dbg & (CODEC_FLAG_DBG_NO_PWAIT | CODEC_FLAG_DBG_NO_TMEM)) !=
                          (CODEC_FLAG_DBG_NO_PWAIT | CODEC_FLAG_DBG_NO_TMEM))
          tc_wait(&bars->pv_done[(t - 2) & 3], ((t - 2) >> 2) & 1);
#endif
        if (quad == 0) PROG(1 + grp, t, 6);
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(12, t);
        tc::fence_after();
        if (!(dbg & CODEC_FLAG_DBG_NO_TMEM)) {
#pragma unroll
          for (int c = 0; c < 4; ++c) tc::tmem_st16(my_p + c * 16, pall + 16 * c);
        } else if (pall[0] == 12345u) {
          sr[0] = pall[1];  // keep the math alive
        }
        {
          const float2 la = tc::fadd2(l2[0], l2[1]), lb = tc::fadd2(l2[2], l2[3]);
          l += (la.x + la.y) + (lb.x + lb.y);
        }
        tc::wait_st();
        tc::fence_before();
        __syncwarp();
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(3, t);
        if (lane == 0 && quad == 3) stamp(7, t);
        if (lane == 0 && quad == 1) stamp(10, t);
        if (lane == 0 && quad == 2) stamp(11, t);
        if (lane == 0) tc::mbar_arrive_cluster(&bars->p_full[b], 0);
      }
      // ---- epilogue: the group that ran the unit's last tile reads all of
      // O out of TMEM into registers, releases the accumulator (o_free: the
      // next unit's first PV may start) and only then writes to global
      // memory. (Both groups waiting for the last PV would deadlock: it is
      // issued after S(tl + 3), which needs the other group's next tile.)
      // The l / m barrier alternates with the unit parity so one epilogue
      // never joins the next.
      const int tl = t - 1, last = tl & 1, l_bar = 9 + (n & 1);
#ifdef CODEC_TC_EPI_TIMING
      const long long epi_t0 = clock64();
#endif
      if (quad == 0) PROG(1 + grp, t, 7);
      if (grp != last) {
        // lx is single-buffered: the previous unit's epilogue group must
        // have read its (l, m) first. Without this wait a short unit let
        // this group overwrite lx while the other group, still finishing
        // its last tile, had not read it yet (wrong l for a few rows at
        // some SM budgets: tests/test_gpu_fuzz.py). epi_done[(n-1) % 2]
        // completes after that epilogue's staging, long after its lx read.
        if (n > 0) tc_wait(&bars->epi_done[(n - 1) & 1], ((n - 1) >> 1) & 1);
        lx[r] = make_float2(have ? l : 0.f, my_m);
        named_arrive(l_bar, 256);
      } else {
        named_sync(l_bar, 256);
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(16, tl);
        const float2 o2 = lx[r];
        const float l_run = l + (o2.x > 0.f ? o2.x * fast_exp2(o2.y - my_m) : 0.f);
        // PV(tl) landed => the whole unit landed (PV(tl - 4) is done)
        tc_wait(&bars->pv_done[tl & 3], (tl >> 2) & 1);
        tc::fence_after();
        uint32_t o[128];
#pragma unroll
        for (int c = 0; c < 4; ++c) tc::tmem_ld32(tmem + lane_addr + kColO + c * 32, o + c * 32);
        tc::wait_ld();
        tc::fence_before();
        __syncwarp();
        if (lane == 0) tc::mbar_arrive_cluster(&bars->o_free, 0);
        if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(15, tl);
#ifdef CODEC_TC_EPI_TIMING
        const long long epi_t1 = clock64();
#endif
        // Write O through this unit's Q buffer (its S MMAs are complete) as a
        // staging area, 64 rows per pass: thread-per-row global stores touch
        // 32 lines per instruction; from SMEM each row goes out as one fully
        // coalesced 512-byte warp store. Chunk c of staging row x lives at
        // c ^ (x % 32): conflict-free both ways.
        {
          float4* stg = reinterpret_cast<float4*>(smem + kOffQ + (n & 1) * kQBytes);
          long long* rdst = reinterpret_cast<long long*>(smem + kOffMpub + grp * 512);  // this group's free mpub half
          float* dst = nullptr;
          const float inv = 1.f / l_run;
          if (valid) {
            if (slot < 0) {
              dst = out + ((int64_t)req * hq_local + qh) * kTcD;
            } else {
              const int64_t ei = (int64_t)slot * hq_local + qh;
              dst = part_o + ei * kTcD;
              part_ml[2 * ei] = my_m * 0.69314718055994530942f;  // natural-log units
              part_ml[2 * ei + 1] = l_run;
            }
          }
          const int wq = warp & 3;
#ifdef CODEC_TC_EPI_SPLIT
          long long t_stage = 0, t_store = 0, t_a = clock64();
#endif
#if CODEC_TC_DIRECT_STORE
          // no staging: every thread writes its own row as 16 full 32-byte
          // sectors (STG.256), all four warps at once
          (void)stg;
          (void)rdst;
          (void)wq;
          if (dst) {
#pragma unroll
            for (int c = 0; c < 16; ++c)
              asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst + 8 * c),
                           "f"(__uint_as_float(o[8 * c]) * inv), "f"(__uint_as_float(o[8 * c + 1]) * inv),
                           "f"(__uint_as_float(o[8 * c + 2]) * inv), "f"(__uint_as_float(o[8 * c + 3]) * inv),
                           "f"(__uint_as_float(o[8 * c + 4]) * inv), "f"(__uint_as_float(o[8 * c + 5]) * inv),
                           "f"(__uint_as_float(o[8 * c + 6]) * inv), "f"(__uint_as_float(o[8 * c + 7]) * inv)
                           : "memory");
          }
#ifdef CODEC_TC_EPI_SPLIT
          t_store = clock64() - t_a;
#endif
#else
#pragma unroll 1
          for (int pass = 0; pass < 2; ++pass) {
            if ((quad >> 1) == pass) {
              const int x = (quad & 1) * 32 + lane;  // staging row
#pragma unroll
              for (int c = 0; c < 32; ++c)
                stg[x * 32 + (c ^ lane)] =
                    make_float4(__uint_as_float(o[4 * c]) * inv, __uint_as_float(o[4 * c + 1]) * inv,
                                __uint_as_float(o[4 * c + 2]) * inv, __uint_as_float(o[4 * c + 3]) * inv);
              rdst[x] = reinterpret_cast<long long>(dst);
            }
            named_sync(12, 128);
#ifdef CODEC_TC_EPI_SPLIT
            { const long long tb = clock64(); t_stage += tb - t_a; t_a = tb; }
#endif
#if CODEC_TC_STG256
            // 256-bit stores (STG.256): one instruction writes two staging
            // rows (a half-warp per row), half the store instructions
#pragma unroll 4
            for (int i = 0; i < 8; ++i) {
              const int x = wq * 16 + 2 * i + (lane >> 4), cp = lane & 15;
              float* d = reinterpret_cast<float*>(rdst[x]);
              if (d) {
                const float4 a = stg[x * 32 + ((2 * cp) ^ (x & 31))];
                const float4 b = stg[x * 32 + ((2 * cp + 1) ^ (x & 31))];
                asm volatile("st.global.L1::no_allocate.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(d + 8 * cp),
                             "f"(a.x), "f"(a.y), "f"(a.z), "f"(a.w), "f"(b.x), "f"(b.y), "f"(b.z), "f"(b.w)
                             : "memory");
              }
            }
#else
#pragma unroll 4
            for (int i = 0; i < 16; ++i) {
              const int x = wq * 16 + i;
              float* d = reinterpret_cast<float*>(rdst[x]);
              if (d) {  // L1::no_allocate: 1.3 % faster TC kernel than a plain store (tools/ab_rounds.py)
                const float4 v = stg[x * 32 + (lane ^ (x & 31))];
                asm volatile("st.global.L1::no_allocate.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(
                                 reinterpret_cast<float4*>(d) + lane),
                             "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w)
                             : "memory");
              }
            }
#endif
            named_sync(12, 128);
#ifdef CODEC_TC_EPI_SPLIT
            { const long long tb = clock64(); t_store += tb - t_a; t_a = tb; }
#endif
          }
#endif  // CODEC_TC_DIRECT_STORE
#ifdef CODEC_TC_EPI_SPLIT
          if (ctalog && tid == grp * 128) {  // [0] staging writes, [3] global stores (debug build only)
            ctalog[4 * (2048 + blockIdx.x) + 0] += t_stage;
            ctalog[4 * (2048 + blockIdx.x) + 3] += t_store;
          }
#endif
          // readiness count of the merge entry of (req, kv head): every
          // thread's stores of the group fenced, then one arrival per row
          if (cnt) {
            __threadfence();
            named_sync(12, 128);
            if (valid && slot >= 0) {
              const int e = __ldg(entry_of + (int64_t)req * (hq_local / g) + gv.kh);
              if (e >= 0) atomicAdd(cnt + e, 1);
            }
          }
          // the staging reads / writes (generic proxy) before the Q warp's
          // next TMA load into this buffer (async proxy)
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) mbar_arrive(&bars->epi_done[n & 1]);
#ifdef CODEC_TC_EPI_TIMING
          if (ctalog && tid == grp * 128) {  // epilogue clocks of this CTA: until O read / after
            ctalog[4 * (2048 + blockIdx.x) + 1] += epi_t1 - epi_t0;
            ctalog[4 * (2048 + blockIdx.x) + 2] += clock64() - epi_t1;
          }
#endif
          if (tid == grp * 128 + 32 * CODEC_TC_TRACE_QUAD) stamp(9, tl);
        }
      }
      if (quad == 0) PROG(1 + grp, t, 8);
    }
#ifndef CODEC_TC_EPI_SPLIT
    if (ctalog && tid == 0) {
      ctalog[4 * (2048 + blockIdx.x)] = global_ns();
      ctalog[4 * (2048 + blockIdx.x) + 3] = t_start;
    }
#endif
  }
  // Drain (both CTAs, once every warp of this CTA is done): tcgen05.commit
  // arrivals land asynchronously, after the MMAs they track. Those nobody
  // waited for (the last S tiles' s_full / k_empty, the last PV tiles'
  // v_empty, the last units' q_empty, ...) must be seen before the CTA
  // exits, or a late arrival hits the shared memory of whatever CTA the SM
  // runs next. After the CTA barrier every such barrier is at most one
  // phase behind its final one, so the parity waits are exact.
  __threadfence();  // this CTA's output / partial writes before the completion count below
  __syncthreads();
  if (tid == 0 && tc_done) atomicAdd(tc_done, 1);  // the merge waits for every TC CTA (launch.cu)
  if (warp == kTcMmaWarp) {
    CODEC_TC_RANGE;
    int tiles = 0, units = 0;
    for (int gi = g_begin; gi < g_end; ++gi) {
      const int nt = group_view(table, off_groups, off_rows, gi).n_tiles;
      tiles += nt;
      units += nt > 0;
    }
    auto drain = [&](uint64_t* bar, int stages, bool per_unit) {
      for (int s = 0; s < stages; ++s) {
        const int n = ((per_unit ? units : tiles) - s + stages - 1) / stages;
        if (n > 0) mbar_wait(&bar[s], (n - 1) & 1);
      }
    };
    drain(bars->s_full, 2, false);
    drain(bars->k_empty, kTcKStages, false);
    drain(bars->v_empty, kTcVStages, false);
    drain(bars->pv_done, 4, false);
    drain(bars->q_empty, 2, true);
  }
  tc::fence_before();
  tc::cluster_sync();  // the leader's MMAs into the peer's TMEM and all remote arrivals are done
  tc::fence_after();
  if (warp == kTcMmaWarp) tc::tmem_dealloc_pair(tmem, kTmemCols);
  cta_log(ctalog, blockIdx.x, t_start);
}

#undef CODEC_TC_RANGE

// ------------------------------------------------------------------ host
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int32_t cuda_status(cudaError_t e, const char* what);

// a [rows][128] bf16 pool viewed as SW128 boxes of 64 head-dim x box_rows tokens
int32_t encode_pool_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows) {
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
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return CODEC_OK;
}

// The pool viewed as [rows][2 halves][64 d] so that ONE box carries
// box_rows whole 256-byte token rows (SW128 per 128-byte half-row "line",
// line = 2 row + half). A TMA op has a large fixed cost in the SM's TMA
// unit (~190 clk per box measured on B200, whatever its size), so the
// HBM-bound suffix stream needs big boxes: 32 rows = 8 KB per op.
int32_t encode_pool_rows_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !p)
      return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[3] = {64, 2, (cuuint64_t)rows};
  cuuint64_t strides[2] = {128, (cuuint64_t)kTcD * 2};
  cuuint32_t box[3] = {64, 2, box_rows};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled (rows) failed (%d)", (int)r);
  return CODEC_OK;
}

// The pool viewed as [2 halves][rows][64 d] (strides 128 B, 256 B): one box
// {64 d, box_rows, 2} lands as the two K-major SW128 atom columns
// [half][row][64] the MMA descriptors expect
int32_t encode_pool_halves_map(CUtensorMap* map, const void* pool, int64_t rows, uint32_t box_rows) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !p)
      return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[3] = {64, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)kTcD * 2, 128};
  cuuint32_t box[3] = {64, box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled (halves) failed (%d)", (int)r);
  return CODEC_OK;
}

constexpr int kTraceLen = 17 * 2 * 64 + 2 * 2048;
static long long* g_trace = nullptr;  // debug timeline (CODEC_FLAG_TRACE), one per process

// Q [bs][hq_local][128] bf16 viewed as [bs][hq_local][2 halves][64 d]: a box
// of 64 d x 1 half x g heads x 128/g requests is one CTA's 128 Q rows of a
// piece with consecutive requests, in the SW128 K-major layout the MMA reads
int32_t encode_q_map(CUtensorMap* map, const void* q, int bs, int hq_local, int g) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult qr;
    void* p = nullptr;
    cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &qr);
    if (e != cudaSuccess || qr != cudaDriverEntryPointSuccess || !p)
      return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    fn = (EncodeTiledFn)p;
  }
  cuuint64_t dims[4] = {64, 2, (cuuint64_t)hq_local, (cuuint64_t)bs};
  cuuint64_t strides[3] = {128, (cuuint64_t)kTcD * 2, (cuuint64_t)hq_local * kTcD * 2};
  cuuint32_t box[4] = {64, 1, (cuuint32_t)g, (cuuint32_t)(128 / g)};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(q), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return fail(CODEC_ERR_CUDA, "cuTensorMapEncodeTiled (q) failed (%d)", (int)r);
  return CODEC_OK;
}

int32_t launch_tc(const int32_t* table, const codec_table_info& in, const void* q, const void* k, const void* v,
                  int64_t pool_tokens, int g, int h_local, int bs, void* out, void* part_o, void* part_ml,
                  cudaStream_t st, int flags, long long* ctalog, const int32_t* page_table, int page_shift,
                  int32_t* tc_done, const int32_t* entry_of, int32_t* cnt) {
  const bool trace = (flags & CODEC_FLAG_TRACE) != 0;
  if (trace && !g_trace) {
    if (cudaMalloc(&g_trace, kTraceLen * sizeof(long long)) != cudaSuccess) return fail(CODEC_ERR_CUDA, "trace alloc");
    cudaMemsetAsync(g_trace, 0, kTraceLen * sizeof(long long), st);
  }
  if (in.n_tc_groups == 0 || in.n_tc_blocks == 0) return CODEC_OK;
  CUtensorMap mk, mv, mq;
#if CODEC_TC_K3D
  CODEC_TRY(encode_pool_halves_map(&mk, k, (int64_t)h_local * pool_tokens, 64));  // K half: 64 tokens, both atoms
#else
  CODEC_TRY(encode_pool_map(&mk, k, (int64_t)h_local * pool_tokens, 64));      // K half: 64 tokens
#endif
  CODEC_TRY(encode_pool_map(&mv, v, (int64_t)h_local * pool_tokens, kTcBN));   // V half: 64 d columns
  CODEC_TRY(encode_q_map(&mq, q, bs, h_local * g, g));
  cudaError_t e = cudaFuncSetAttribute(tc_pac_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kTcSmem);
  if (e != cudaSuccess) return cuda_status(e, "tc smem attribute");
  dim3 grid(kTcCtasPerBlock * in.n_tc_blocks, 1);  // CTA pairs (__cluster_dims__); heads come from the units
  tc_pac_kernel<<<grid, kTcThreads, kTcSmem, st>>>(mk, mv, mq, table, in.off_tc, in.off_rows, in.off_tc_block_ptr,
                                                   (const __nv_bfloat16*)q, pool_tokens, g, h_local * g,
                                                   (float*)out, (float*)part_o, (float*)part_ml,
                                                   trace ? g_trace : nullptr, flags, ctalog, page_table, page_shift,
                                                   tc_done, entry_of, cnt);
  return cuda_status(cudaGetLastError(), "tc launch");
}

#ifdef CODEC_HANG_CHECK
int32_t set_hang_buffer(void* dev_ptr) {
  int* p = static_cast<int*>(dev_ptr);
  return cuda_status(cudaMemcpyToSymbol(g_hang_buf, &p, sizeof(p)), "hang buffer");
}
#else
int32_t set_hang_buffer(void*) { return fail(CODEC_ERR_VALUE, "built without CODEC_HANG_CHECK"); }
#endif

int32_t read_trace(long long* host, int64_t n) {
  if (!g_trace) return fail(CODEC_ERR_VALUE, "no trace recorded");
  if (n > kTraceLen) n = kTraceLen;
  return cuda_status(cudaMemcpy(host, g_trace, n * sizeof(long long), cudaMemcpyDeviceToHost), "trace copy");
}

}  // namespace codec
