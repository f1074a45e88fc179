// Calibration probe: FP64 dependent-chain latency / throughput and F2F cost on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_probe tools/fp64_probe.cu && ./fp64_probe
#include <cstdio>
#include <cuda_runtime.h>

__global__ void chain_dadd(double* out, long long* cyc, int n, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __dadd_rn(x, a);
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_dfma(double* out, long long* cyc, int n, double a) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = __fma_rn(x, a, a);
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
__global__ void chain_f2f(double* out, long long* cyc, int n, float a) {
  float f = a + threadIdx.x;
  double x = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { x = (double)f; f = (float)x + a; }
  long long t1 = clock64();
  out[threadIdx.x + blockIdx.x * blockDim.x] = x;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}
// throughput: 8 independent chains per thread
__global__ void tput_dfma(double* out, int n, double a) {
  double x[8];
  for (int j = 0; j < 8; ++j) x[j] = a + threadIdx.x + j;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = __fma_rn(x[j], a, a);
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}
__global__ void tput_f2f(double* out, int n, float a) {
  float f[8];
  double x[8];
  for (int j = 0; j < 8; ++j) { f[j] = a + threadIdx.x + j; x[j] = 0; }
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) { x[j] += (double)f[j]; f[j] += 1.0f; }
  double s = 0;
  for (int j = 0; j < 8; ++j) s += x[j];
  out[threadIdx.x + blockIdx.x * blockDim.x] = s;
}

int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 1 << 24); cudaMalloc(&cyc, 8);
  const int n = 4096;
  chain_dadd<<<1, 32>>>(out, cyc, n, 1e-9); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", (double)h / n);
  chain_dfma<<<1, 32>>>(out, cyc, n, 0.999); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)h / n);
  chain_f2f<<<1, 32>>>(out, cyc, n, 1e-3f); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("F2F.F64.F32 + F2F.F32.F64 + FADD round trip: %.2f cycles\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int it = 2048;
  tput_dfma<<<sms * 8, 256>>>(out, it, 0.999);
  cudaEventRecord(e0); tput_dfma<<<sms * 8, 256>>>(out, it, 0.999); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double flops = 2.0 * sms * 8 * 256 * (double)it * 8;
  printf("DFMA throughput: %.1f TFLOP/s (fp64)\n", flops / ms / 1e9);
  cudaEventRecord(e0); tput_f2f<<<sms * 8, 256>>>(out, it, 0.5f); cudaEventRecord(e1); cudaEventSynchronize(e1);
  cudaEventElapsedTime(&ms, e0, e1);
  double conv = (double)sms * 8 * 256 * it * 8;
  printf("F2F.F64.F32 (+DADD) throughput: %.1f Gconv/s = %.1f per clk per SM at 1.9 GHz\n", conv / ms / 1e6,
         conv / ms / 1e6 / sms / 1.9);
  return 0;
}
