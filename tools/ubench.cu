// Microbenchmarks of the B200 pipes the softmax of kern_tc.cu leans on:
// MUFU.EX2, FFMA2, and tcgen05.ld/st throughput with 16 warps per SM.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void __launch_bounds__(512, 1) k_ex2(float* out, long long* clk, int iters) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f + i;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) k_ffma2(float* out, long long* clk, int iters) {
  unsigned long long a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x + i;
  unsigned long long b = 0x3f8000003f800000ull, c = 0x3f0000003f000000ull;
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) asm volatile("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[i]) : "l"(b), "l"(c));
  }
  __syncthreads();
  long long t1 = clock64();
  unsigned long long s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = (float)s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

__global__ void __launch_bounds__(512, 1) k_tmem(float* out, long long* clk, int iters, int do_st) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        (uint32_t)__cvta_generic_to_shared(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot + ((uint32_t)((warp & 3) * 32) << 16) + (warp >> 2) * 32;
  uint32_t r[32];
  for (int i = 0; i < 32; ++i) r[i] = i;
  float acc = 0;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (do_st) {
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
          "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem),
          "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]),
          "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]),
          "r"(r[17]), "r"(r[18]), "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]),
          "r"(r[25]), "r"(r[26]), "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
          : "memory");
      asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    } else {
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
          "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
            "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]),
            "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]),
            "=r"(r[30]), "=r"(r[31])
          : "r"(tmem));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      acc += __uint_as_float(r[it & 31]);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&clk, 148 * 8);
  long long h[148];
  const int iters = 4096;
  for (int warps : {4, 8, 16}) {
    k_ex2<<<148, warps * 32>>>(out, clk, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    double ops = (double)warps * 32 * 8 * iters;
    printf("ex2   warps=%2d: %.2f ops/clk/SM\n", warps, ops / h[0]);
    k_ffma2<<<148, warps * 32>>>(out, clk, iters);
    cudaDeviceSynchronize();
    cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
    printf("ffma2 warps=%2d: %.2f f32x2-instr lanes/clk/SM\n", warps, ops / h[0]);
    for (int st = 0; st < 2; ++st) {
      k_tmem<<<148, warps * 32>>>(out, clk, 512, st);
      cudaError_t e = cudaDeviceSynchronize();
      cudaMemcpy(h, clk, sizeof h, cudaMemcpyDeviceToHost);
      double bytes = (double)warps * 32 * 32 * 4 * 512;
      printf("tmem %s warps=%2d: %.1f B/clk/SM (%s)\n", st ? "st" : "ld", warps, bytes / h[0], cudaGetErrorString(e));
    }
  }
  return 0;
}
