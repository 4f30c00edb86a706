// Microbenchmark: mbarrier ping-pong latency inside a 2-CTA cluster
// (remote arrive on the peer's barrier, local wait), for the arrive/wait
// flavours kern_tc.cu can use.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_17694_b200/csrc -o tools/ubench_cluster tools/ubench_cluster.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace codec;

template <int ARRIVE, int WAIT>
__device__ __forceinline__ void ping(uint64_t* bar, uint32_t peer) {
  const uint32_t ra = tc::mapa(smem_u32(bar), peer);
  if (ARRIVE == 0) asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
  if (ARRIVE == 1) asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
  if (ARRIVE == 2) asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
}
template <int WAIT>
__device__ __forceinline__ void waitp(uint64_t* bar, uint32_t ph) {
  if (WAIT == 0)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
  if (WAIT == 1)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.test_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
  if (WAIT == 2)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
  if (WAIT == 4)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
  if (WAIT == 5)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph), "r"(20) : "memory");
  if (WAIT == 3)
    asm volatile("{\n\t.reg .pred p;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n\t}" ::"r"(smem_u32(bar)), "r"(ph) : "memory");
}

template <int ARRIVE, int WAIT>
__global__ void __cluster_dims__(2, 1, 1) k_pp(long long* clk, int iters) {
  __shared__ uint64_t bar;
  const uint32_t rank = tc::cluster_rank();
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  tc::cluster_sync();
  long long t0 = clock64();
  if (threadIdx.x == 0) {
    for (int i = 0; i < iters; ++i) {
      if (rank == 0) {
        ping<ARRIVE, WAIT>(&bar, 1);
        waitp<WAIT>(&bar, i & 1);
      } else {
        waitp<WAIT>(&bar, i & 1);
        ping<ARRIVE, WAIT>(&bar, 0);
      }
    }
  }
  long long t1 = clock64();
  tc::cluster_sync();
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

// fan-in: 4 warps of each CTA arrive on the leader's barrier (count 8); the
// leader's warp 0 waits then releases all 8 warps through both CTAs'
// "go" barriers (count 1) -- one round = signal + response
template <int ARRIVE>
__global__ void __cluster_dims__(2, 1, 1) k_fanin(long long* clk, int iters) {
  __shared__ uint64_t bar, go;
  const uint32_t rank = tc::cluster_rank();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(&bar, 8);
    mbar_init(&go, 1);
    fence_barrier_init();
  }
  tc::cluster_sync();
  long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (warp < 4) {
      if (lane == 0) ping<ARRIVE, 3>(&bar, 0);
      waitp<3>(&go, i & 1);
    } else if (warp == 4 && rank == 0) {
      waitp<3>(&bar, i & 1);
      if (lane == 0) {
        ping<ARRIVE, 3>(&go, 0);
        ping<ARRIVE, 3>(&go, 1);
      }
    }
  }
  long long t1 = clock64();
  tc::cluster_sync();
  if (threadIdx.x == 0 && rank == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

template <int WAIT>
__global__ void k_local(long long* clk, int iters) {
  // warp 0 and warp 1 of one CTA ping-pong through two local barriers
  __shared__ uint64_t bar[2];
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
  }
  __syncthreads();
  long long t0 = clock64();
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < iters; ++i) {
      if (w == 0) {
        mbar_arrive(&bar[1]);
        mbar_wait(&bar[0], i & 1);
      } else {
        mbar_wait(&bar[1], i & 1);
        mbar_arrive(&bar[0]);
      }
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0 && blockIdx.x == 0) clk[0] = t1 - t0;
}

template <int A, int W>
void run(const char* name, long long* clk) {
  const int iters = 2000;
  k_pp<A, W><<<2, 32>>>(clk, iters);
  cudaError_t e = cudaDeviceSynchronize();
  long long h = 0;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("%-44s round trip %.0f clk [%s]\n", name, (double)h / iters, cudaGetErrorString(e));
}

int main() {
  long long* clk;
  cudaMalloc(&clk, 8);
  run<0, 0>("arrive.release.cluster / try_wait.acquire", clk);
  run<0, 1>("arrive.release.cluster / test_wait.acquire", clk);
  run<1, 2>("arrive.relaxed.cluster / try_wait.relaxed", clk);
  run<0, 3>("arrive.release.cluster / try_wait (cta)", clk);
  run<2, 3>("arrive (release.cta) / try_wait (cta)", clk);
  run<1, 3>("arrive.relaxed.cluster / try_wait (cta)", clk);
  run<2, 4>("arrive (release.cta) / test_wait poll (cta)", clk);
  run<2, 5>("arrive (release.cta) / try_wait hint 20ns", clk);
  {
    long long h;
    k_fanin<0><<<2, 160>>>(clk, 2000);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("%-44s round %.0f clk\n", "fan-in 8 warps, release.cluster", (double)h / 2000);
    k_fanin<2><<<2, 160>>>(clk, 2000);
    cudaDeviceSynchronize();
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    printf("%-44s round %.0f clk\n", "fan-in 8 warps, release.cta", (double)h / 2000);
  }
  k_local<0><<<1, 64>>>(clk, 2000);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
  printf("%-44s round trip %.0f clk\n", "local arrive / try_wait (two warps)", (double)h / 2000);
  return 0;
}
