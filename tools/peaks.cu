// Microbenchmarks for the roofline denominators SURVEY.md §8(d) asks to measure on the box
// (MEASURED_PEAKS.json carries only HBM copy and bf16 GEMM): fp64 and fp32 FMA pipe
// throughput, fp64 add, L2-resident read bandwidth, and a STREAM-style HBM copy for
// reference.  One JSON line on stdout.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/peaks tools/peaks.cu && /tmp/peaks
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                  \
  do {                                                                         \
    cudaError_t e_ = (x);                                                      \
    if (e_ != cudaSuccess) {                                                   \
      std::fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e_));            \
      return 1;                                                                \
    }                                                                          \
  } while (0)

constexpr int kChains = 8;

template <typename T>
__global__ void k_fma(T* out, int iters, T a, T b) {
  T acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = (T)(threadIdx.x + c);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = acc[c] * a + b;  // contracted to FMA
  }
  T s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == (T)12345.678) out[0] = s;
}

__global__ void k_dadd(double* out, int iters, double b) {
  double acc[kChains];
#pragma unroll
  for (int c = 0; c < kChains; ++c) acc[c] = threadIdx.x + c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < kChains; ++c) acc[c] = __dadd_rn(acc[c], b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < kChains; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void k_copy(const float4* __restrict__ in, float4* __restrict__ out, size_t n) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    out[i] = in[i];
}

__global__ void k_l2read(const float4* __restrict__ in, size_t n, int reps, float* out) {
  float s = 0.f;
  for (int r = 0; r < reps; ++r)
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
      const float4 v = __ldcg(in + i);
      s += v.x + v.y + v.z + v.w;
    }
  if (s == 12345.678f) out[0] = s;
}

template <typename F>
static float time_ms(F f, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();  // warm-up
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  return ms / reps;
}

int main() {
  int sms = 0, dev = 0;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  void* scratch;
  CK(cudaMalloc(&scratch, 64));
  const int grid = sms * 8, block = 256, iters = 1 << 14;
  const double fma_ops = (double)grid * block * iters * kChains;
  const float t64 = time_ms([&] { k_fma<double><<<grid, block>>>((double*)scratch, iters, 0.999, 1e-3); }, 5);
  const float t32 = time_ms([&] { k_fma<float><<<grid, block>>>((float*)scratch, iters, 0.999f, 1e-3f); }, 5);
  const float tadd = time_ms([&] { k_dadd<<<grid, block>>>((double*)scratch, iters, 1e-3); }, 5);
  CK(cudaGetLastError());

  const size_t hbm_bytes = (size_t)2 << 30;  // 2 GiB per buffer
  float4 *a = nullptr, *b = nullptr;
  CK(cudaMalloc(&a, hbm_bytes));
  CK(cudaMalloc(&b, hbm_bytes));
  CK(cudaMemset(a, 0, hbm_bytes));
  const size_t n4 = hbm_bytes / sizeof(float4);
  const float tcopy = time_ms([&] { k_copy<<<sms * 16, 512>>>(a, b, n4); }, 10);
  const size_t l2_bytes = (size_t)48 << 20;  // resident in the 126 MB L2
  const size_t l2n = l2_bytes / sizeof(float4);
  const int l2reps = 40;
  const float tl2 = time_ms([&] { k_l2read<<<sms * 8, 512>>>(a, l2n, l2reps, (float*)scratch); }, 5);
  CK(cudaGetLastError());
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
  std::printf(
      "{\"sms\": %d, \"fp64_fma_tflops\": %.2f, \"fp32_fma_tflops\": %.2f, \"fp64_add_tflops\": %.2f, "
      "\"hbm_copy_gbs\": %.1f, \"l2_read_gbs\": %.1f, \"l2_working_set_mb\": %zu, \"clock_attr_mhz\": %d, "
      "\"method\": \"tools/peaks.cu: %d CTAs x %d threads x %d iters x %d independent chains; copy 2 GiB float4; "
      "L2 read 48 MB x %d reps (__ldcg)\"}\n",
      sms, 2.0 * fma_ops / (t64 * 1e-3) / 1e12, 2.0 * fma_ops / (t32 * 1e-3) / 1e12, fma_ops / (tadd * 1e-3) / 1e12,
      2.0 * hbm_bytes / (tcopy * 1e-3) / 1e9, (double)l2_bytes * l2reps / (tl2 * 1e-3) / 1e9, l2_bytes >> 20,
      clk_khz / 1000, grid, block, iters, kChains, l2reps);
  cudaFree(a);
  cudaFree(b);
  cudaFree(scratch);
  return 0;
}
