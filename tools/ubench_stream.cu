// Microbenchmark: how much HBM bandwidth can N SMs pull with 1-D bulk
// copies (cp.async.bulk, the suffix kernel's data path minus the math)?
// (148 - N) SMs are blocked by a resident spinner kernel (one CTA per SM,
// all its shared memory) so the streaming grid lands on the other N SMs.
// Each streaming CTA walks its own contiguous region with a `stages`-deep
// ring of `box`-byte copies; a consumer warp only waits and releases.
//   ubench_stream N ctas_per_sm stages box_bytes [copies_per_stage]
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2505_17694_b200/csrc -o tools/ubench_stream tools/ubench_stream.cu
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_util.cuh"

using namespace codec;

// pattern 0: SMs with smid < n_block stay blocked; pattern 1: the free SMs
// are spread evenly over the smid range. hammer: blocked SMs read an
// L2-resident buffer in a loop instead of sleeping (L2 / fabric traffic).
__global__ void blocker(volatile int* flag, int n_block, int n_sm, int pattern, int hammer, const uint4* l2buf,
                        unsigned long long* sink) {
  extern __shared__ uint8_t smem[];
  uint32_t smid;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
  const int n_free = n_sm - n_block;
  bool blocked;
  if (pattern == 0) {
    blocked = (int)smid < n_block;
  } else {
    blocked = true;  // free iff smid == floor(i * n_sm / n_free) for some i
    const int i = (int)(((long long)smid * n_free + n_sm - 1) / n_sm);
    if (i < n_free && (int)((long long)i * n_sm / n_free) == (int)smid) blocked = false;
  }
  if (!blocked) return;
  if (!hammer) {
    if (threadIdx.x == 0) {
      smem[0] = 1;
      while (*flag == 0) __nanosleep(1000);
    }
    return;
  }
  uint4 acc = make_uint4(0, 0, 0, 0);
  const int n = (32 << 20) / 16;
  for (int it = 0;; ++it) {
    for (int i = threadIdx.x + blockIdx.x * 64; i < n; i += blockDim.x * 4096) {
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const uint4 v = __ldcg(l2buf + ((i + k * 1024) % n));
        acc.x ^= v.x;
      }
    }
    if ((it & 15) == 0 && *flag) break;
  }
  if (acc.x == 0x12345) *sink = acc.x;
}

__global__ void stream(const uint8_t* __restrict__ src, size_t per_cta, int stages, int box, int copies,
                       unsigned long long* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)stages * box * copies);
  uint64_t* empty = full + stages;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    fence_barrier_init();
  }
  __syncthreads();
  const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
  const size_t stage_bytes = (size_t)box * copies;
  const int n = (int)(per_cta / stage_bytes);
  if (warp == 0) {
    if (lane == 0)
      for (int c = 0; c < n; ++c) {
        const int s = c % stages;
        if (c >= stages) mbar_wait(&empty[s], ((c / stages) - 1) & 1);
        mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
        for (int k = 0; k < copies; ++k)
          bulk_g2s(smem + (size_t)s * stage_bytes + (size_t)k * box, base + (size_t)c * stage_bytes + (size_t)k * box,
                   box, &full[s]);
      }
  } else if (warp == 1) {
    unsigned long long acc = 0;
    for (int c = 0; c < n; ++c) {
      const int s = c % stages;
      mbar_wait(&full[s], (c / stages) & 1);
      acc += smem[(size_t)s * stage_bytes + lane];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
    if (acc == 12345678) *sink = acc;
  }
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 52;
  const int per_sm = argc > 2 ? atoi(argv[2]) : 6;
  const int stages = argc > 3 ? atoi(argv[3]) : 2;
  const int box = argc > 4 ? atoi(argv[4]) : 16384;
  const int copies = argc > 5 ? atoi(argv[5]) : 1;
  const int pattern = argc > 6 ? atoi(argv[6]) : 0;
  const int hammer = argc > 7 ? atoi(argv[7]) : 0;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t total = (size_t)4 << 30;
  uint8_t* buf;
  cudaMalloc(&buf, total);
  cudaMemset(buf, 1, total);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  int* flag;
  cudaHostAlloc(&flag, 4, cudaHostAllocMapped);
  int* dflag;
  cudaHostGetDevicePointer(&dflag, flag, 0);
  const int smem = stages * box * copies + 2 * stages * 8;
  cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int bsmem = 200 * 1024;
  cudaFuncSetAttribute(blocker, cudaFuncAttributeMaxDynamicSharedMemorySize, bsmem);
  cudaStream_t sa, sb;
  cudaStreamCreateWithFlags(&sa, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&sb, cudaStreamNonBlocking);
  const int ctas = N * per_sm;
  const size_t per_cta = (total / ctas) / ((size_t)box * copies) * ((size_t)box * copies);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    *flag = 0;
    blocker<<<sms, hammer ? 512 : 32, bsmem, sa>>>(dflag, sms - N, sms, pattern, hammer, (const uint4*)buf, sink);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("blocker: %s\n", cudaGetErrorString(err)); return 1; }
    // give the blockers time to become resident
    struct timespec ts = {0, 20 * 1000 * 1000};
    nanosleep(&ts, nullptr);
    cudaEventRecord(e0, sb);
    stream<<<ctas, 64, smem, sb>>>(buf, per_cta, stages, box, copies, sink);
    cudaEventRecord(e1, sb);
    err = cudaGetLastError();
    if (err != cudaSuccess) { printf("stream: %s\n", cudaGetErrorString(err)); return 1; }
    cudaEventSynchronize(e1);
    *flag = 1;
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double bytes = (double)per_cta * ctas;
    if (rep) printf("N=%d ctas/SM=%d stages=%d box=%d copies=%d pattern=%d hammer=%d: %.3f ms  %.0f GB/s  %.1f GB/s per SM\n",
                    N, per_sm, stages, box, copies, pattern, hammer, ms, bytes / ms / 1e6, bytes / ms / 1e6 / N);
  }
  return 0;
}
