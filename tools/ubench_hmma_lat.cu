// Dependent-chain latency of mma.sync m16n8k16 bf16 and of movmatrix /
// shfl on sm_100a (1 warp per SM).
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>
__global__ void k_lat(float* out, long long* clk, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  uint32_t b0 = threadIdx.x * 3, b1 = threadIdx.x * 5;
  float c[4] = {0, 0, 0, 0};
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                 : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3]) : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  long long t1 = clock64();
  uint32_t x = threadIdx.x;
  for (int it = 0; it < iters; ++it) asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %0;" : "+r"(x));
  long long t2 = clock64();
  float y = c[0];
  for (int it = 0; it < iters; ++it) y = __shfl_xor_sync(0xffffffffu, y, 4) + 1.f;
  long long t3 = clock64();
  out[threadIdx.x] = c[0] + c[1] + c[2] + c[3] + x + y;
  if (threadIdx.x == 0) { clk[0] = t1 - t0; clk[1] = t2 - t1; clk[2] = t3 - t2; }
}
int main() {
  float* out; long long* clk; cudaMalloc(&out, 4096); cudaMalloc(&clk, 64);
  const int iters = 4096;
  k_lat<<<1, 32>>>(out, clk, iters);
  cudaDeviceSynchronize();
  long long h[3]; cudaMemcpy(h, clk, 24, cudaMemcpyDeviceToHost);
  printf("hmma dep latency %.1f clk, movmatrix %.1f clk, shfl+fadd %.1f clk\n", (double)h[0] / iters, (double)h[1] / iters, (double)h[2] / iters);
  return 0;
}
