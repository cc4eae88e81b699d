// Image I/O and evaluation helpers around the hot path:
// Netpbm quantisation, the forward haze model and the fidelity metrics.
//
//   pdz_quantize_u8      image.py:128-145 (save_image): clamp to [0, 1] and
//                        floor(v * 255 + 0.5) in float64 -> uint8
//   pdz_synthesize_haze  scattering.py:142-158: J * t + A * (1 - t)
//   pdz_compare          metrics.py:20-37: sums of (x - y)^2 and |x - y|
//
// Float64 throughout with the reference's operation order and no FMA
// contraction (__dmul_rn / __dadd_rn), so quantised bytes and synthesised
// samples are bitwise equal to the reference's.
#include <cmath>

#include "pdz_internal.cuh"

namespace pdz {
namespace {

int io_grid(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8)));
}

__global__ void quantize_kernel(const double* __restrict__ in, int64_t n,
                                uint8_t* __restrict__ out, int32_t* __restrict__ bad) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double v = in[i];
    if (!isfinite(v)) {
      atomicExch(bad, 1);
      out[i] = 0;
      continue;
    }
    const double c = fmin(fmax(v, 0.0), 1.0);
    out[i] = uint8_t(floor(__dadd_rn(__dmul_rn(c, 255.0), 0.5)));
  }
}

__global__ void synthesize_kernel(const double* __restrict__ clean,
                                  const double* __restrict__ t, const double* __restrict__ a,
                                  int64_t hw, int C, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < hw;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double ti = t[i];
    const double om = __dsub_rn(1.0, ti);
    for (int c = 0; c < C; ++c)
      out[i * C + c] = __dadd_rn(__dmul_rn(clean[i * C + c], ti), __dmul_rn(a[c], om));
  }
}

// Fixed-order partial sums: block b sums its grid-stride elements, then one
// block adds the per-block partials in index order (deterministic).
constexpr int kCmpBlocks = 256;

__global__ void compare_partial_kernel(const double* __restrict__ x,
                                       const double* __restrict__ y, int64_t n,
                                       double* __restrict__ part, int32_t* __restrict__ bad) {
  __shared__ double s2[8], s1[8];
  double a2 = 0.0, a1 = 0.0;
  int b = 0;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double xi = x[i], yi = y[i];
    b |= !(isfinite(xi) && xi >= 0.0 && xi <= 1.0) ? 1 : 0;
    b |= !(isfinite(yi) && yi >= 0.0 && yi <= 1.0) ? 2 : 0;
    const double d = __dsub_rn(xi, yi);
    a2 = __dadd_rn(a2, __dmul_rn(d, d));
    a1 = __dadd_rn(a1, fabs(d));
  }
  if (b) atomicOr(bad, b);
  a2 = warp_sum(a2);
  a1 = warp_sum(a1);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    s2[w] = a2;
    s1[w] = a1;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double t2 = 0.0, t1 = 0.0;
    for (int k = 0; k < int(blockDim.x >> 5); ++k) {
      t2 += s2[k];
      t1 += s1[k];
    }
    part[2 * blockIdx.x] = t2;
    part[2 * blockIdx.x + 1] = t1;
  }
}

__global__ void compare_final_kernel(const double* __restrict__ part, int nparts,
                                     double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t2 = 0.0, t1 = 0.0;
    for (int k = 0; k < nparts; ++k) {
      t2 += part[2 * k];
      t1 += part[2 * k + 1];
    }
    out[0] = t2;
    out[1] = t1;
  }
}

}  // namespace
}  // namespace pdz

using namespace pdz;

extern "C" {

int32_t pdz_quantize_u8(const double* image, int64_t n, uint8_t* out, int32_t* flag,
                        void* stream) {
  PDZ_REQUIRE(image && out && flag, "NULL argument");
  PDZ_REQUIRE(n >= 0, "negative sample count");
  cudaStream_t s = as_stream(stream);
  PDZ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), s), "flag reset");
  if (n > 0) {
    quantize_kernel<<<io_grid(n), 256, 0, s>>>(image, n, out, flag);
    PDZ_CHECK_LAUNCH("quantize");
  }
  return PDZ_OK;
}

int32_t pdz_synthesize_haze(const double* clean, const double* transmission,
                            const double* airlight, int64_t pixels, int32_t channels,
                            double* out, void* stream) {
  PDZ_REQUIRE(clean && transmission && airlight && out, "NULL argument");
  PDZ_REQUIRE(channels == 1 || channels == 3, "channels must be 1 or 3, got %d", channels);
  if (pixels > 0) {
    synthesize_kernel<<<io_grid(pixels), 256, 0, as_stream(stream)>>>(clean, transmission,
                                                                      airlight, pixels, channels,
                                                                      out);
    PDZ_CHECK_LAUNCH("synthesize");
  }
  return PDZ_OK;
}

size_t pdz_compare_workspace_bytes(void) { return size_t(kCmpBlocks) * 2 * sizeof(double); }

int32_t pdz_compare(const double* x, const double* y, int64_t n, double* sums, int32_t* flag,
                    void* workspace, size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(x && y && sums && flag && workspace, "NULL argument");
  PDZ_REQUIRE(n > 0, "empty images");
  if (workspace_bytes < pdz_compare_workspace_bytes()) {
    set_error("workspace too small: need %zu bytes, got %zu", pdz_compare_workspace_bytes(),
              workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  PDZ_CUDA(cudaMemsetAsync(flag, 0, sizeof(int32_t), s), "flag reset");
  double* part = static_cast<double*>(workspace);
  compare_partial_kernel<<<kCmpBlocks, 256, 0, s>>>(x, y, n, part, flag);
  PDZ_CHECK_LAUNCH("compare");
  compare_final_kernel<<<1, 32, 0, s>>>(part, kCmpBlocks, sums);
  PDZ_CHECK_LAUNCH("compare final");
  return PDZ_OK;
}

}  // extern "C"
