// FMA-pipe forms for the Gaussian taps: which FFMA / FFMA2 operand forms
// issue at what rate on B200 (FMA per clock per SM).  Standalone:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mb2 mb2.cu && ./mb2
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e) { printf("err %s line %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

struct Taps { float2 w2[24]; float w[24]; };

__device__ __forceinline__ unsigned long long f2u(float2 a) { return *reinterpret_cast<unsigned long long*>(&a); }
__device__ __forceinline__ float2 u2f(unsigned long long a) { return *reinterpret_cast<float2*>(&a); }
__device__ __forceinline__ unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}

// MODE 0: FFMA2, tap pair from the kernel parameter (uniform), 20 taps
// MODE 1: FFMA2, tap pair in registers (loaded once)
// MODE 2: scalar FFMA, tap from the kernel parameter
// MODE 3: scalar FFMA, tap an immediate
// MODE 4: half FFMA2 (param taps), half FFMA imm, interleaved
template <int MODE>
__global__ void __launch_bounds__(256) k(float* out, const __grid_constant__ Taps t, int iters) {
  unsigned long long x[8];
  float y[16];
  for (int j = 0; j < 8; ++j) x[j] = f2u(make_float2(threadIdx.x * 1e-7f + j, j));
  for (int j = 0; j < 16; ++j) y[j] = threadIdx.x * 1e-7f + j;
  const unsigned long long v = f2u(make_float2(1.0f + threadIdx.x * 1e-9f, 1.0f));
  const float vs = 1.0f + threadIdx.x * 1e-9f;
  unsigned long long wr[4];
  for (int j = 0; j < 4; ++j) wr[j] = f2u(t.w2[j]);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int tt = 0; tt < 20; ++tt) {
      if (MODE == 0) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = ffma2(v, f2u(t.w2[tt]), x[j]);
      } else if (MODE == 1) {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = ffma2(v, wr[tt & 3], x[j]);
      } else if (MODE == 2) {
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = fmaf(vs, t.w[tt], y[j]);
      } else if (MODE == 3) {
#pragma unroll
        for (int j = 0; j < 16; ++j) y[j] = fmaf(vs, 0.01f * (tt + 1), y[j]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j) x[j] = ffma2(v, f2u(t.w2[tt]), x[j]);
#pragma unroll
        for (int j = 0; j < 8; ++j) y[j] = fmaf(vs, 0.01f * (tt + 1), y[j]);
      }
    }
  }
  float s = 0.f;
  for (int j = 0; j < 8; ++j) { const float2 q = u2f(x[j]); s += q.x + q.y; }
  for (int j = 0; j < 16; ++j) s += y[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const int sms = prop.multiProcessorCount;
  float* out;
  CK(cudaMalloc(&out, size_t(sms) * 8 * 256 * 4));
  Taps t;
  for (int i = 0; i < 24; ++i) { t.w[i] = 1e-3f * i; t.w2[i] = make_float2(1e-3f * i, 2e-3f * i); }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2048, grid = sms * 8;
  const char* names[] = {"FFMA2 param-uniform taps", "FFMA2 register taps", "FFMA param taps",
                         "FFMA immediate taps", "FFMA2 param + FFMA imm"};
  // FMAs per thread per iteration: 20 taps x 16 lanes-of-work
  for (int m = 0; m < 5; ++m) {
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      switch (m) {
        case 0: k<0><<<grid, 256>>>(out, t, iters); break;
        case 1: k<1><<<grid, 256>>>(out, t, iters); break;
        case 2: k<2><<<grid, 256>>>(out, t, iters); break;
        case 3: k<3><<<grid, 256>>>(out, t, iters); break;
        case 4: k<4><<<grid, 256>>>(out, t, iters); break;
      }
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double fmas = double(grid) * 256 * iters * 20 * 16;
    const double per_s = fmas / (best * 1e-3);
    printf("%-28s %.3f ms  %.2f TFMA/s  %.1f FMA/clk/SM (at %d MHz nominal)\n", names[m], best,
           per_s / 1e12, per_s / sms / (clk_khz * 1e3), clk_khz / 1000);
  }
  return 0;
}
