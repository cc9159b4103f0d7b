// Dependent-chain latency of fp64 add / mul and fp32 add on one thread (clock64), B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 tools/dadd_latency.cu -o /tmp/lat && /tmp/lat
#include <cstdio>
__global__ void k(double* out, float* outf, long long* cyc, int n) {
  double a = out[0], b = out[1];
  float fa = outf[0], fb = outf[1];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = __dadd_rn(a, b);
  long long t1 = clock64();
  for (int i = 0; i < n; ++i) a = __dmul_rn(a, b);
  long long t2 = clock64();
  for (int i = 0; i < n; ++i) fa = __fadd_rn(fa, fb);
  long long t3 = clock64();
  out[2] = a;
  outf[2] = fa;
  cyc[0] = t1 - t0;
  cyc[1] = t2 - t1;
  cyc[2] = t3 - t2;
}
int main() {
  double h[3] = {1.0, 1e-17, 0};
  float hf[3] = {1.f, 1e-9f, 0};
  double* d;
  float* df;
  long long* c;
  cudaMalloc(&d, 24);
  cudaMalloc(&df, 12);
  cudaMalloc(&c, 24);
  cudaMemcpy(d, h, 24, cudaMemcpyHostToDevice);
  cudaMemcpy(df, hf, 12, cudaMemcpyHostToDevice);
  const int n = 1 << 16;
  k<<<1, 1>>>(d, df, c, n);
  k<<<1, 1>>>(d, df, c, n);
  long long hc[3];
  cudaMemcpy(hc, c, 24, cudaMemcpyDeviceToHost);
  printf("{\"dadd_cycles\": %.2f, \"dmul_cycles\": %.2f, \"fadd_cycles\": %.2f}\n", (double)hc[0] / n,
         (double)hc[1] / n, (double)hc[2] / n);
  return 0;
}
