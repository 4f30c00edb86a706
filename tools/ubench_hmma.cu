// Throughput of the legacy warp-level tensor-core path (mma.sync
// m16n8k16 bf16 -> f32, HMMA in SASS) on sm_100a, per SM, for 1..16 warps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_hmma tools/ubench_hmma.cu
#include <cstdio>
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_hmma(float* out, long long* clk, int iters) {
  uint32_t a[4] = {threadIdx.x, threadIdx.x + 1, threadIdx.x + 2, threadIdx.x + 3};
  uint32_t b[2] = {threadIdx.x * 3, threadIdx.x * 5};
  float c[8][4] = {};
  __syncthreads();
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
          "{%0,%1,%2,%3};"
          : "+f"(c[i][0]), "+f"(c[i][1]), "+f"(c[i][2]), "+f"(c[i][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  __syncthreads();
  long long t1 = clock64();
  float s = 0;
  for (int i = 0; i < 8; ++i) s += c[i][0] + c[i][1] + c[i][2] + c[i][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;
}

int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 1024 * 4);
  cudaMalloc(&clk, 148 * 8);
  const int iters = 2048;
  for (int warps : {1, 2, 4, 8, 16}) {
    k_hmma<<<148, warps * 32>>>(out, clk, iters);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, clk, 8, cudaMemcpyDeviceToHost);
    double mmas = (double)warps * iters * 8;
    double flops = mmas * 16 * 8 * 16 * 2;
    printf("hmma m16n8k16 warps=%2d: %.3f mma/clk/SM = %.0f flop/clk/SM (tcgen05 dense peak 8192)\n", warps,
           mmas / h, flops / h);
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
