// Throughput probe: scalar FFMA / FADD vs packed FFMA2 / FADD2 (sm_100a).
// Independent chains per thread, 8 warps per SMSP; prints warp-instructions
// per cycle per SM for each form.  nvcc -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cuda_runtime.h>
typedef unsigned long long u64;
__device__ __forceinline__ u64 fma2(u64 a, u64 b, u64 c) { u64 d; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c)); return d; }
__device__ __forceinline__ u64 add2(u64 a, u64 b) { u64 d; asm volatile("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b)); return d; }
__device__ __forceinline__ float fma1(float a, float b, float c) { float d; asm volatile("fma.rn.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c)); return d; }
__device__ __forceinline__ float add1(float a, float b) { float d; asm volatile("add.rn.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b)); return d; }
constexpr int N = 8, IT = 4096;
__global__ void k_fma1(float* o, float s) { float a[N]; for (int j = 0; j < N; j++) a[j] = threadIdx.x + j;
  for (int i = 0; i < IT; i++) for (int j = 0; j < N; j++) a[j] = fma1(a[j], s, a[(j + 1) % N]);
  float r = 0; for (int j = 0; j < N; j++) r += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = r; }
__global__ void k_add1(float* o, float s) { float a[N]; for (int j = 0; j < N; j++) a[j] = threadIdx.x + j;
  for (int i = 0; i < IT; i++) for (int j = 0; j < N; j++) a[j] = add1(a[j], a[(j + 1) % N]);
  float r = 0; for (int j = 0; j < N; j++) r += a[j]; o[blockIdx.x * blockDim.x + threadIdx.x] = r; }
__global__ void k_fma2(float* o, float s) { u64 a[N]; u64 ss; float2 t = make_float2(s, s); ss = *(u64*)&t;
  for (int j = 0; j < N; j++) { float2 v = make_float2(threadIdx.x + j, j); a[j] = *(u64*)&v; }
  for (int i = 0; i < IT; i++) for (int j = 0; j < N; j++) a[j] = fma2(a[j], ss, a[(j + 1) % N]);
  float r = 0; for (int j = 0; j < N; j++) { float2 v = *(float2*)&a[j]; r += v.x + v.y; } o[blockIdx.x * blockDim.x + threadIdx.x] = r; }
__global__ void k_add2(float* o, float s) { u64 a[N];
  for (int j = 0; j < N; j++) { float2 v = make_float2(threadIdx.x + j, j); a[j] = *(u64*)&v; }
  for (int i = 0; i < IT; i++) for (int j = 0; j < N; j++) a[j] = add2(a[j], a[(j + 1) % N]);
  float r = 0; for (int j = 0; j < N; j++) { float2 v = *(float2*)&a[j]; r += v.x + v.y; } o[blockIdx.x * blockDim.x + threadIdx.x] = r; }
int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* o; cudaMalloc(&o, sms * 4 * 1024 * sizeof(float));
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const char* names[4] = {"FFMA", "FADD", "FFMA2", "FADD2"};
  void (*ks[4])(float*, float) = {k_fma1, k_add1, k_fma2, k_add2};
  for (int w = 0; w < 2; w++)
  for (int k = 0; k < 4; k++) {
    ks[k]<<<sms * 2, 1024>>>(o, 1.0001f);
    cudaEventRecord(a); ks[k]<<<sms * 2, 1024>>>(o, 1.0001f); cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    double winst = (double)sms * 2 * 32 * IT * N;   // warp-instructions
    double cyc = ms * 1e-3 * clk * 1e3;             // at the max clock
    if (w) printf("%-6s %.3f ms  %.2f warp-inst/clk/SM (at %d MHz)\n", names[k], ms, winst / cyc / sms, clk / 1000);
  }
  return 0;
}
