// Microbenchmark: FP32 FFMA, packed FFMA2, FP64 DFMA issue/throughput per SM on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_rates tools/fp_rates.cu
#include <cstdio>
#include <cuda_runtime.h>
constexpr int ITERS = 4096;
template <int K> __global__ void k_ffma(float* out, float a, float b) {
  float x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3f + k;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = fmaf(x[k], a, b);
  float s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  if (s == 1234.5f) out[0] = s;
}
template <int K> __global__ void k_ffma2(float* out, float a, float b) {
  float2 x[K];
  float2 A = make_float2(a, a), Bv = make_float2(b, b);
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = make_float2(threadIdx.x * 1e-3f + k, k);
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = __ffma2_rn(x[k], A, Bv);
  float s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k].x + x[k].y;
  if (s == 1234.5f) out[0] = s;
}
template <int K> __global__ void k_dfma(float* out, double a, double b) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  if (s == 1234.5) out[0] = (float)s;
}
template <int K> __global__ void k_mix(float* out, double a, double b, float af, float bf) {
  // one DFMA + two FFMA interleaved: does the fp64 pipe co-issue with fp32?
  double x[K]; float y[2 * K];
#pragma unroll
  for (int k = 0; k < K; ++k) { x[k] = threadIdx.x * 1e-3 + k; y[2*k] = k; y[2*k+1] = k + 1; }
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) { x[k] = fma(x[k], a, b); y[2*k] = fmaf(y[2*k], af, bf); y[2*k+1] = fmaf(y[2*k+1], af, bf); }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k] + y[2*k] + y[2*k+1];
  if (s == 1234.5) out[0] = (float)s;
}
template <int K> __global__ void k_cvt(float* out, float a) {
  // fp32 -> fp64 -> fp32 conversions (cvt.f64.f32 / cvt.rn.f32.f64), volatile so none is folded
  float f[K];
#pragma unroll
  for (int k = 0; k < K; ++k) f[k] = threadIdx.x * 1e-3f + k * a;
  for (int i = 0; i < ITERS; ++i)
#pragma unroll
    for (int k = 0; k < K; ++k) {
      double d;
      asm volatile("cvt.f64.f32 %0, %1;" : "=d"(d) : "f"(f[k]));
      asm volatile("cvt.rn.f32.f64 %0, %1;" : "=f"(f[k]) : "d"(d));
    }
  float s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += f[k];
  if (s == 1234.5f) out[0] = s;
}
int main() {
  int dev = 0, sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  float* out; cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = sms * 8, threads = 256;
  auto run = [&](const char* name, auto launch, double ops_per_thread_iter) {
    launch(); cudaDeviceSynchronize();
    cudaEventRecord(e0); for (int r = 0; r < 5; ++r) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    double ops = double(blocks) * threads * ITERS * ops_per_thread_iter;
    double per_sm_clk = ops / (ms * 1e-3) / sms / (clk * 1e3);
    printf("%-28s %8.3f ms  %10.2f T lane-ops/s  %7.2f lane-ops/clk/SM (at %d MHz nominal)\n", name, ms, ops / (ms * 1e-3) / 1e12, per_sm_clk, clk / 1000);
  };
  run("FFMA (8 chains)", [&] { k_ffma<8><<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 8);
  run("FFMA2 (8 chains, 2 lanes)", [&] { k_ffma2<8><<<blocks, threads>>>(out, 1.0001f, 1e-7f); }, 16);
  run("DFMA (8 chains)", [&] { k_dfma<8><<<blocks, threads>>>(out, 1.0001, 1e-7); }, 8);
  run("DFMA+2 FFMA (4 chains) dfma", [&] { k_mix<4><<<blocks, threads>>>(out, 1.0001, 1e-7, 1.0001f, 1e-7f); }, 4);
  run("F2F f32->f64->f32 (8 chains)", [&] { k_cvt<8><<<blocks, threads>>>(out, 1.0001f); }, 16);
  printf("sms %d\n", sms);
  cudaError_t e = cudaGetLastError(); printf("%s\n", cudaGetErrorString(e));
}
