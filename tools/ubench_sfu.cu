// Throughput of the softmax building blocks on sm_100a, 16 warps per SM:
// MUFU ex2 (f32 / bf16x2 / f16x2), the f32->bf16x2 pack, packed f32x2 FMA,
// mixed-precision f32 += bf16 adds.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_sfu tools/ubench_sfu.cu
#include <cstdio>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define KERNEL(NAME, DECL, INIT, BODY, FOLD)                                       \
  __global__ void __launch_bounds__(512, 1) NAME(float* out, long long* clk, int iters) { \
    DECL;                                                                          \
    for (int i = 0; i < 8; ++i) INIT;                                              \
    __syncthreads();                                                               \
    long long t0 = clock64();                                                      \
    for (int it = 0; it < iters; ++it) {                                           \
      _Pragma("unroll") for (int i = 0; i < 8; ++i) BODY;                         \
    }                                                                              \
    __syncthreads();                                                               \
    long long t1 = clock64();                                                      \
    float s = 0;                                                                   \
    for (int i = 0; i < 8; ++i) s += FOLD;                                         \
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;                                \
    if (threadIdx.x == 0) clk[blockIdx.x] = t1 - t0;                               \
  }

KERNEL(k_ex2_f32, float a[8], a[i] = -(threadIdx.x * 1e-3f + i),
       asm volatile("ex2.approx.ftz.f32 %0, %0;" : "+f"(a[i])), a[i])
KERNEL(k_ex2_bf16x2, uint32_t a[8], a[i] = 0xbf80bf80u + i,
       asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(a[i])), (float)a[i])
KERNEL(k_ex2_f16x2, uint32_t a[8], a[i] = 0xbc00bc00u + i,
       asm volatile("ex2.approx.f16x2 %0, %0;" : "+r"(a[i])), (float)a[i])
KERNEL(k_pack, uint32_t a[8], a[i] = 0x3f800000u + i,
       asm volatile("cvt.rn.bf16x2.f32 %0, %0, %0;" : "+r"(a[i])), (float)a[i])
KERNEL(k_ffma2, unsigned long long a[8], a[i] = threadIdx.x + i,
       asm volatile("fma.rn.f32x2 %0, %0, %0, %0;" : "+l"(a[i])), (float)a[i])
KERNEL(k_ffma, float a[8], a[i] = threadIdx.x + i,
       asm volatile("fma.rn.f32 %0, %0, %0, %0;" : "+f"(a[i])), a[i])
KERNEL(k_addmix, float a[8], a[i] = threadIdx.x + i,
       asm volatile("{.reg .b16 h; mov.b16 h, 0x3f80; add.rn.f32.bf16 %0, h, %0;}" : "+f"(a[i])), a[i])
KERNEL(k_fmax3, float a[8], a[i] = threadIdx.x + i,
       asm volatile("max.f32 %0, %0, %0, %0;" : "+f"(a[i])), a[i])

__global__ void check(uint32_t* o) {
  float xs[4] = {-0.5f, -3.25f, -10.f, -0.01f};
  for (int i = 0; i < 4; ++i) {
    __nv_bfloat162 x = __floats2bfloat162_rn(xs[i], xs[i]);
    uint32_t u = *reinterpret_cast<uint32_t*>(&x);
    asm volatile("ex2.approx.ftz.bf16x2 %0, %0;" : "+r"(u));
    o[i] = u;
  }
}

typedef void (*K)(float*, long long*, int);
int main() {
  float* out;
  long long* clk;
  cudaMalloc(&out, 148 * 512 * 4);
  cudaMalloc(&clk, 148 * 8);
  const int iters = 4096;
  struct {
    const char* name;
    K k;
    int elems;
  } ks[] = {{"ex2.f32", k_ex2_f32, 1},   {"ex2.bf16x2", k_ex2_bf16x2, 2}, {"ex2.f16x2", k_ex2_f16x2, 2},
            {"cvt.bf16x2", k_pack, 2},  {"fma.f32x2", k_ffma2, 2},      {"fma.f32", k_ffma, 1},
            {"add.f32.bf16", k_addmix, 1}, {"max3.f32", k_fmax3, 1}};
  for (auto& e : ks) {
    for (int warps : {4, 8, 16}) {
      e.k<<<148, warps * 32>>>(out, clk, iters);
      cudaDeviceSynchronize();
      long long h[1];
      cudaMemcpy(h, clk, 8, cudaMemcpyDeviceToHost);
      double ops = (double)warps * 32 * iters * 8;
      printf("%-14s warps=%2d: %.2f instr/clk/SM (%.2f results/clk/SM)\n", e.name, warps, ops / h[0],
             ops * e.elems / h[0]);
    }
  }
  uint32_t* o;
  cudaMalloc(&o, 16);
  check<<<1, 1>>>(o);
  uint32_t hh[4];
  cudaMemcpy(hh, o, 16, cudaMemcpyDeviceToHost);
  float xs[4] = {-0.5f, -3.25f, -10.f, -0.01f};
  for (int i = 0; i < 4; ++i) {
    uint32_t lo = (hh[i] & 0xffff) << 16;
    float f;
    memcpy(&f, &lo, 4);
    printf("ex2.bf16x2(%g) = %g (exact %g)\n", xs[i], f, exp2f(xs[i]));
  }
  printf("err %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
