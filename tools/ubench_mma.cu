// Microbenchmark: tcgen05.mma kind::f16 issue-to-completion throughput for
// the shapes kern_tc.cu uses (M128/M256 x N128 x K16, A from SMEM or TMEM,
// 1-CTA or cta_group::2). Operand contents are garbage; only time matters.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_17694_b200/csrc -o tools/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace codec;

template <bool PAIR, bool TS>
__global__ void __launch_bounds__(128, 1) k_mma(long long* clk, int iters) {
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  const uint32_t rank = PAIR ? tc::cluster_rank() : 0;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    if (PAIR) tc::tmem_alloc_pair(&slot, 512);
    else tc::tmem_alloc(&slot, 512);
  }
  tc::fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  tc::fence_after();
  const uint32_t tmem = slot;
  const uint32_t sb = smem_u32(smem);
  long long t0 = clock64();
  if (warp == 0 && rank == 0) {
    constexpr uint32_t idesc = tc::idesc_bf16(PAIR ? 256 : 128, 128, false, false);
    const uint64_t da = tc::smem_desc(sb, 16, 1024), db = tc::smem_desc(sb + 32768, 16, 1024);
    for (int it = 0; it < iters; ++it) {
      if (tc::elect_one()) {
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          const uint64_t off = (uint64_t)((((k >> 2) * 16384) + (k & 3) * 32) >> 4);
          if (TS) {
            if (PAIR) tc::mma2_f16_ts(tmem + (it & 1) * 128, tmem + 384 + k * 8, db + off, idesc, k > 0);
            else tc::mma_f16_ts(tmem + (it & 1) * 128, tmem + 384 + k * 8, db + off, idesc, k > 0);
          } else {
            if (PAIR) {
              asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                           "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem + (it & 1) * 128),
                           "l"(da + off), "l"(db + off), "r"(idesc), "r"((uint32_t)(k > 0)) : "memory");
            } else {
              tc::mma_f16_ss(tmem + (it & 1) * 128, da + off, db + off, idesc, k > 0);
            }
          }
        }
      }
      __syncwarp();
    }
    if (tc::elect_one()) {
      if (PAIR) tc::commit_pair(&bar); else tc::commit(&bar);
    }
    __syncwarp();
  }
  if (warp == 0) mbar_wait(&bar, 0);
  long long t1 = clock64();
  if (threadIdx.x == 0 && rank == 0) clk[blockIdx.x] = t1 - t0;
  tc::fence_before();
  if (PAIR) tc::cluster_sync(); else __syncthreads();
  if (warp == 0) {
    if (PAIR) tc::tmem_dealloc_pair(tmem, 512); else tc::tmem_dealloc(tmem, 512);
  }
}

template <bool PAIR, bool TS>
void run(const char* name, long long* clk) {
  auto kern = k_mma<PAIR, TS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
  const int iters = 2000, grid = 148;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(128);
  cfg.dynamicSmemBytes = 100 * 1024;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = PAIR ? 2 : 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, clk, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  // per SM: 128 x 128 x 16 MACs per instruction (the pair's M256 is two SMs' worth)
  printf("%-22s %.1f clk per MMA instr (ideal 64)  [%s]\n", name, (double)h / (iters * 8), cudaGetErrorString(e));
}

int main() {
  long long* clk;
  cudaMalloc(&clk, 148 * 8);
  run<false, false>("1cta SS M128N128K16", clk);
  run<false, true>("1cta TS M128N128K16", clk);
  run<true, false>("2cta SS M256N128K16", clk);
  run<true, true>("2cta TS M256N128K16", clk);
  return 0;
}
