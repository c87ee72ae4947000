// peaks.cu — measurement infrastructure (not on the render path).
//
// MEASURED_PEAKS.json carries only HBM copy bandwidth and cuBLAS bf16; the
// render kernel is bound by FP32 CUDA-core arithmetic over cache-resident
// gathers, so bench.py measures those two roofs on the box:
//   * FP32 FFMA throughput (register-operand and immediate-operand forms)
//   * L2-resident float4 gather bandwidth (LDG.128 over a 64 MiB working set)
//   * shared-memory RED.ADD.U32 throughput (the sensor deposition's per-pixel
//     operation: the binding roof of the scenes without a medium)
//   * FP64 DFMA throughput (raygen / optics / sensor stages)
#include <cuda_runtime.h>

#include <algorithm>

namespace {

template <bool kImm>
__global__ void __launch_bounds__(256) ffma_kernel(float* out, float b, float c, int iters) {
  float a0 = threadIdx.x * 1e-3f, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5,
        a6 = a0 + 6, a7 = a0 + 7;
#pragma unroll 4
  for (int i = 0; i < iters; ++i) {
    if (kImm) {
      a0 = fmaf(a0, 0.999f, 1e-3f); a1 = fmaf(a1, 0.999f, 1e-3f); a2 = fmaf(a2, 0.999f, 1e-3f);
      a3 = fmaf(a3, 0.999f, 1e-3f); a4 = fmaf(a4, 0.999f, 1e-3f); a5 = fmaf(a5, 0.999f, 1e-3f);
      a6 = fmaf(a6, 0.999f, 1e-3f); a7 = fmaf(a7, 0.999f, 1e-3f);
    } else {
      a0 = fmaf(a0, b, c); a1 = fmaf(a1, b, c); a2 = fmaf(a2, b, c); a3 = fmaf(a3, b, c);
      a4 = fmaf(a4, b, c); a5 = fmaf(a5, b, c); a6 = fmaf(a6, b, c); a7 = fmaf(a7, b, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 12345.678f) out[threadIdx.x] = s;
}

// Packed FP32 pairs (FFMA2, sm_100): 8 independent pairs = 16 FMAs per step.
__global__ void __launch_bounds__(256) ffma2_kernel(float* out, float b, float c, int iters) {
  unsigned long long a[8];
  const unsigned long long bb = ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(b);
  const unsigned long long cc = ((unsigned long long)__float_as_uint(c) << 32) | __float_as_uint(c);
#pragma unroll
  for (int j = 0; j < 8; ++j)
    a[j] = ((unsigned long long)__float_as_uint(threadIdx.x * 1e-3f + j) << 32) |
           __float_as_uint(threadIdx.x * 2e-3f + j);
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) asm("fma.rn.f32x2 %0, %0, %1, %2;" : "+l"(a[j]) : "l"(bb), "l"(cc));
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += __uint_as_float((unsigned)a[j]) + __uint_as_float((unsigned)(a[j] >> 32));
  if (s == 12345.678f) out[threadIdx.x] = s;
}

__global__ void __launch_bounds__(256) gather_kernel(const float4* __restrict__ p, size_t n,
                                                     int reps, float* out) {
  float acc = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (int r = 0; r < reps; ++r)
    for (size_t q = (size_t)blockIdx.x * blockDim.x + threadIdx.x; q < n; q += stride) {
      const float4 v = __ldg(p + q);
      acc += v.x + v.y + v.z + v.w;
    }
  if (acc == 12345.678f) out[0] = acc;
}

// Shared-memory RED.ADD.U32 throughput (the deposition's per-pixel operation,
// render.cuh red_shared): each thread adds to its own words, bank-conflict free.
__global__ void __launch_bounds__(256) red_shared_kernel(float* out, int iters) {
  __shared__ unsigned tile[256 * 8];
  for (int j = 0; j < 8; ++j) tile[j * 256 + threadIdx.x] = 0u;
  __syncthreads();
  const unsigned base = (unsigned)__cvta_generic_to_shared(tile) + 4u * threadIdx.x;
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("red.shared.add.u32 [%0], %1;" ::"r"(base + 1024u * j), "r"(i + j) : "memory");
  __syncthreads();
  unsigned s = 0;
  for (int j = 0; j < 8; ++j) s += tile[j * 256 + threadIdx.x];
  if (s == 0x12345u) out[threadIdx.x] = (float)s;
}

// FP64 DFMA throughput (the FP64 raygen / optics / sensor stages).
__global__ void __launch_bounds__(256) dfma_kernel(double* out, double b, double c, int iters) {
  double a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x * 1e-3 + j;
#pragma unroll 4
  for (int i = 0; i < iters; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == 12345.678) out[threadIdx.x] = s;
}

}  // namespace

extern "C" {

// Best-of-5 shared-memory RED.ADD.U32 throughput in Gop/s.
double rbp_red_shared_gops(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 1 << 12;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    red_shared_kernel<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double ops = 8.0 * iters * (double)blocks * threads;
    if (rep > 0) best = std::max(best, ops / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// Best-of-5 FP64 DFMA throughput in TFLOP/s (2 flops per FMA).
double rbp_dfma_tflops(int device) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  double* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(double));
  const int blocks = sms * 8, threads = 256, iters = 1 << 12;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 0.999, 1e-3, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// Best-of-5 FP32 FFMA throughput in TFLOP/s (2 flops per FMA).  mode 0:
// register operands, 1: immediate operands, 2: packed pairs (FFMA2).
double rbp_ffma_tflops(int device, int mode) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  cudaMalloc(&out, 1024 * sizeof(float));
  const int blocks = sms * 8, threads = 256, iters = 1 << 14;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    if (mode == 2) ffma2_kernel<<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    else if (mode) ffma_kernel<true><<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    else ffma_kernel<false><<<blocks, threads>>>(out, 0.999f, 1e-3f, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * (mode == 2 ? 16.0 : 8.0) * iters * (double)blocks * threads;
    if (rep > 0) best = std::max(best, flops / (ms * 1e-3) / 1e12);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

// Best-of-5 read bandwidth (GB/s) of LDG.128 over an L2-resident working set.
double rbp_l2_gather_gbs(int device, double mib) {
  cudaSetDevice(device);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  const size_t n = (size_t)(mib * 1024 * 1024) / sizeof(float4);
  float4* p = nullptr;
  float* out = nullptr;
  cudaMalloc(&p, n * sizeof(float4));
  cudaMalloc(&out, sizeof(float));
  cudaMemset(p, 0, n * sizeof(float4));
  const int reps = 20;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double best = 0.0;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    gather_kernel<<<sms * 8, 256>>>(p, n, reps, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep > 0) best = std::max(best, (double)n * sizeof(float4) * reps / (ms * 1e-3) / 1e9);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(p);
  cudaFree(out);
  return cudaGetLastError() == cudaSuccess ? best : -1.0;
}

}  // extern "C"
