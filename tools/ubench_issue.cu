// Microbenchmark: the tensor-core kernel's S -> consumer -> PV hand-off
// chain in isolation (cta_group::2, M256 x N128 x K128 per S and PV, no
// softmax math), to separate MMA pipe time from issuer / barrier latency.
//   mode 0: issuer alone, S and PV back to back, no waits
//   mode 1: + consumer warp per CTA: waits s_full[b], arrives s_free[b] and
//           p_full[b] on the leader; issuer waits s_free(t-2) before S(t)
//           and p_full(t) before PV(t) (the kernel's in-order schedule)
//   mode 2: mode 1 with a one-deeper S lookahead (S(t+1) issued before PV(t))
//   mode 3: the kernel's hand-off: two 4-warp consumer groups per CTA
//           (even / odd tiles) load S from TMEM, free it, wait for PV(t-2)
//           (P buffer reuse), store P (64 columns) to TMEM, arrive p_full;
//           issuer order S(ts) while ts <= tp + 3 (as kern_tc.cu)
//   mode 4: mode 3 without the TMEM loads / stores
//   mode 5: issuer alone with the kernel's commits (3 after S, 2 after PV)
//   mode 6: issuer alone reading rotating K (4) / V (6) stages as the kernel
//   mode 7: issuer alone, S lookahead 3 (S0 S1 S2 S3 PV0 S4 PV1 ...)
//   mode 8: issuer alone, S lookahead 2
// Operand contents are garbage; only time matters.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_17694_b200/csrc -o tools/ubench_issue tools/ubench_issue.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace codec;

struct Bars {
  uint64_t s_full[2], s_free[2], p_full[2], pv_done[4], done, dummy[8];
  uint32_t slot;
};

__global__ void __launch_bounds__(384, 1) k_chain(long long* clk, int iters, int mode, int fill) {
  extern __shared__ __align__(1024) uint8_t smem[];
  // operand contents: zeros or pseudo-random bf16 in (-1, 1) (the tensor
  // pipe's speed may depend on the data through power)
  for (int i = threadIdx.x; i < 224 * 1024 / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + 12345u * blockIdx.x;
    h ^= h >> 13; h *= 0x5bd1e995u; h ^= h >> 15;
    const uint32_t lo = 0x3c00u | (h & 0x807fu), hi = 0x3c00u | ((h >> 16) & 0x807fu);  // |x| in [2^-7, 2^-6)
    reinterpret_cast<uint32_t*>(smem)[i] = fill ? (lo | (hi << 16)) : 0u;
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  __shared__ Bars bars;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = tc::cluster_rank();
  if (threadIdx.x == 0) {
    for (int i = 0; i < 2; ++i) {
      mbar_init(&bars.s_full[i], 1);
      mbar_init(&bars.s_free[i], (mode == 3 || mode == 4) ? 8 : 2);
      mbar_init(&bars.p_full[i], (mode == 3 || mode == 4) ? 8 : 2);
    }
    for (int i = 0; i < 4; ++i) mbar_init(&bars.pv_done[i], 1);
    for (int i = 0; i < 8; ++i) mbar_init(&bars.dummy[i], 1);
    mbar_init(&bars.done, 1);
    fence_barrier_init();
  }
  if (warp == 0) tc::tmem_alloc_pair(&bars.slot, 512);
  tc::fence_before();
  tc::cluster_sync();
  tc::fence_after();
  const uint32_t tmem = bars.slot;
  const uint32_t sb = smem_u32(smem);
  const long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc_s = tc::idesc_bf16(256, 128, false, false);
    constexpr uint32_t idesc_o = tc::idesc_bf16(256, 128, false, true);
    const uint64_t dq = tc::smem_desc(sb, 16, 1024), dk = tc::smem_desc(sb + 65536, 16, 1024);
    const uint64_t dv = tc::smem_desc(sb + (mode == 6 ? 131072 : 98304), 16384, 1024);
    auto issue_s = [&](int t) {
      const int b = t & 1;
      if ((mode >= 1 && mode <= 4) && t >= 2) mbar_wait(&bars.s_free[b], ((t - 2) >> 1) & 1);
      tc::fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t oa = (uint64_t)((((k >> 2) * 16384) + (k & 3) * 32) >> 4);
          const uint64_t ob = (uint64_t)((((k >> 2) * 8192) + (k & 3) * 32) >> 4);
          const uint64_t st = mode == 6 ? (uint64_t)(((t % 4) * 16384) >> 4) : 0;
          tc::mma2_f16_ss(tmem + b * 128, dq + oa, dk + ob + st, idesc_s, k > 0 ? 1u : 0u);
        }
        tc::commit_pair(&bars.s_full[b]);
        if (mode == 5) {
          tc::commit_pair(&bars.dummy[0]);
          tc::commit_pair(&bars.dummy[1]);
        }
      }
      __syncwarp();
    };
    auto issue_pv = [&](int t) {
      const int b = t & 1;
      if (mode >= 1 && mode <= 4) mbar_wait(&bars.p_full[b], (t >> 1) & 1);
      tc::fence_after();
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
          tc::mma2_f16_ts(tmem + 384, tmem + 256 + b * 64 + k * 8,
                          dv + (uint64_t)((k * 16 * 128) >> 4) + (mode == 6 ? (uint64_t)(((t % 6) * 16384) >> 4) : 0),
                          idesc_o, (t > 0 || k > 0) ? 1u : 0u);
        if (mode == 3 || mode == 4) tc::commit_pair(&bars.pv_done[t & 3]);
        if (mode == 5) {
          tc::commit_pair(&bars.dummy[2]);
          tc::commit_pair(&bars.dummy[3]);
        }
      }
      __syncwarp();
    };
    const int ahead = (mode == 2 || mode == 8) ? 2 : (mode == 3 || mode == 4 || mode == 7) ? 3 : 1;
    int ts = 0;
    for (int tp = 0; tp < iters; ++tp) {
      while (ts < iters && ts <= tp + ahead) issue_s(ts++);
      issue_pv(tp);
    }
    if (tc::elect_one()) tc::commit_pair(&bars.done);
    __syncwarp();
  } else if (warp >= 4 && (mode == 3 || mode == 4)) {
    const int grp = (warp - 4) >> 2, quad = warp & 3;
    const uint32_t lane_addr = (uint32_t)(quad * 32) << 16;
    float acc = 0.f;
    for (int t = grp; t < iters; t += 2) {
      const int b = t & 1;
      mbar_wait(&bars.s_full[b], (t >> 1) & 1);
      tc::fence_after();
      uint32_t sr[128];
      if (mode == 3) {
        tc::tmem_ld32(tmem + lane_addr + b * 128, sr);
        tc::tmem_ld32(tmem + lane_addr + b * 128 + 32, sr + 32);
        tc::tmem_ld32(tmem + lane_addr + b * 128 + 64, sr + 64);
        tc::tmem_ld32(tmem + lane_addr + b * 128 + 96, sr + 96);
        tc::wait_ld();
      } else {
#pragma unroll
        for (int i = 0; i < 128; ++i) sr[i] = i * lane;
      }
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(&bars.s_free[b], 0);
      if (t >= 2) mbar_wait(&bars.pv_done[(t - 2) & 3], ((t - 2) >> 2) & 1);
      tc::fence_after();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t pw[16];
#pragma unroll
        for (int w = 0; w < 16; ++w) pw[w] = sr[c * 32 + 2 * w] ^ sr[c * 32 + 2 * w + 1];
        if (mode == 3) tc::tmem_st16(tmem + lane_addr + 256 + b * 64 + c * 16, pw);
        else acc += __uint_as_float(pw[0]);
      }
      if (mode == 3) tc::wait_st();
      tc::fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive_cluster(&bars.p_full[b], 0);
    }
    if (acc == 12345.f) clk[200] = 1;
  } else if (warp == 4 && (mode == 1 || mode == 2)) {
    // consumer: S(t) landed -> release S buffer and publish P (both CTAs)
    for (int t = 0; t < iters; ++t) {
      const int b = t & 1;
      mbar_wait(&bars.s_full[b], (t >> 1) & 1);
      tc::fence_after();
      if (lane == 0) {
        tc::mbar_arrive_cluster(&bars.s_free[b], 0);
        tc::mbar_arrive_cluster(&bars.p_full[b], 0);
      }
      __syncwarp();
    }
  }
  if (warp == 0) mbar_wait(&bars.done, 0);
  const long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) clk[blockIdx.x >> 1] = t1 - t0;
  tc::fence_before();
  tc::cluster_sync();
  if (warp == 0) tc::tmem_dealloc_pair(tmem, 512);
}

int main() {
  long long* clk;
  cudaMalloc(&clk, 256 * 8);
  cudaFuncSetAttribute(k_chain, cudaFuncAttributeMaxDynamicSharedMemorySize, 224 * 1024);
  const int iters = 2000;
  const char* names[9] = {"issuer alone (no waits)", "S->consumer->PV chain", "chain, S lookahead 2",
                          "kernel hand-off + TMEM", "kernel hand-off, no TMEM", "issuer + kernel commits",
                          "issuer + rotating stages", "issuer, lookahead 3", "issuer, lookahead 2"};
  for (int fill = 1; fill < 2; ++fill)
  for (int mode = 0; mode < 9; mode += (mode == 0 ? 7 : 1)) {
    for (int grid : {2, 148}) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(grid);
      cfg.blockDim = dim3(384);
      cfg.dynamicSmemBytes = 224 * 1024;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaLaunchKernelEx(&cfg, k_chain, clk, iters, mode, fill);  // warm
      cudaEventRecord(e0);
      cudaLaunchKernelEx(&cfg, k_chain, clk, iters, mode, fill);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      float ms = 0.f;
      cudaEventElapsedTime(&ms, e0, e1);
      long long h;
      cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
      printf("%-26s %s grid %3d: %.0f clk per tile (S+PV, ideal 1024), %.3f us per tile -> %.0f MHz  [%s]\n",
             names[mode], fill ? "random" : "zeros ", grid, (double)h / iters, ms * 1e3 / iters,
             (double)h / (ms * 1e3), cudaGetErrorString(e));
    }
  }
  return 0;
}
