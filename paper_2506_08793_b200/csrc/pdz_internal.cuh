// Internal helpers shared by the libpdz translation units (not part of the ABI).
#pragma once

#include <atomic>
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/pdz.h"

namespace pdz {

// ---------------------------------------------------------------- errors --
void set_error(const char* fmt, ...);
int32_t cuda_status(cudaError_t e, const char* where);

#define PDZ_CHECK_LAUNCH(where)                                        \
  do {                                                                 \
    cudaError_t e_ = cudaGetLastError();                               \
    if (e_ != cudaSuccess) return ::pdz::cuda_status(e_, where);       \
  } while (0)

#define PDZ_CUDA(call, where)                                          \
  do {                                                                 \
    cudaError_t e_ = (call);                                           \
    if (e_ != cudaSuccess) return ::pdz::cuda_status(e_, where);       \
  } while (0)

#define PDZ_REQUIRE(cond, ...)                                         \
  do {                                                                 \
    if (!(cond)) {                                                     \
      ::pdz::set_error(__VA_ARGS__);                                   \
      return PDZ_EINVAL;                                               \
    }                                                                  \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// ------------------------------------------------------------- workspace --
// Bump allocator over a caller-provided device workspace; 256-byte aligned.
struct Carver {
  char* base;
  size_t cap;
  size_t off = 0;
  bool ok = true;
  Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
  template <typename T>
  T* take(size_t count) {
    size_t a = (off + 255) & ~size_t(255);
    size_t bytes = count * sizeof(T);
    if (a + bytes > cap || (base == nullptr && cap != 0)) {
      ok = false;
      off = a + bytes;
      return nullptr;
    }
    off = a + bytes;
    return base ? reinterpret_cast<T*>(base + a) : nullptr;
  }
  // size-only pass (base == nullptr, cap == 0)
  static size_t round(size_t off) { return (off + 255) & ~size_t(255); }
};

// ------------------------------------------------------------ indexing ---
// np.pad(mode="symmetric") source index with repeated reflection
// (solver.py:235): fold modulo 2n, mirror the upper half.
__host__ __device__ __forceinline__ int reflect(int i, int n) {
  if (i >= 0 && i < n) return i;               // fast paths: at most one fold
  if (i < 0 && i >= -n) return -1 - i;
  if (i >= n && i < 2 * n) return 2 * n - 1 - i;
  int m = i % (2 * n);
  if (m < 0) m += 2 * n;
  return m >= n ? 2 * n - 1 - m : m;
}

// Border-truncating clamp (minimum_filter mode="nearest", scattering.py:64).
__host__ __device__ __forceinline__ int clampi(int i, int lo, int hi) {
  return i < lo ? lo : (i > hi ? hi : i);
}

// ----------------------------------------------------- PDL (griddepcontrol)
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Deterministic warp sum (fixed xor tree).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Order-preserving float64 -> uint64 map (-0.0 folded onto +0.0 first).
__host__ __device__ __forceinline__ uint64_t f64_order_key(double v) {
  if (v == 0.0) v = 0.0;
#ifdef __CUDA_ARCH__
  uint64_t b = static_cast<uint64_t>(__double_as_longlong(v));
#else
  uint64_t b;
  memcpy(&b, &v, 8);
#endif
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double f64_from_order_key(uint64_t k) {
  uint64_t b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  memcpy(&d, &b, 8);
  return d;
#endif
}
__host__ __device__ __forceinline__ uint32_t f32_order_key(float v) {
  if (v == 0.0f) v = 0.0f;
#ifdef __CUDA_ARCH__
  uint32_t b = __float_as_uint(v);
#else
  uint32_t b;
  memcpy(&b, &v, 4);
#endif
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float f32_from_order_key(uint32_t k) {
  uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#ifdef __CUDA_ARCH__
  return __uint_as_float(b);
#else
  float f;
  memcpy(&f, &b, 4);
  return f;
#endif
}

constexpr int kMaxDevices = 64;
int current_device();  // cudaGetDevice, clamped to [0, kMaxDevices)
int num_sms();         // SM count of the current device (cached per device)
// True the first time it is called on the current device for this mask:
// per-device one-time setup such as cudaFuncSetAttribute (function
// attributes are per device; a process-wide flag would leave the second GPU
// of a multi-GPU process at the default 48 KB dynamic shared memory limit).
bool first_use_on_device(std::atomic<uint64_t>* mask);

// Gaussian 1-D factor in float64 (host).
int32_t gaussian_taps_host(double sigma, int kernel_size, double* taps);

}  // namespace pdz
