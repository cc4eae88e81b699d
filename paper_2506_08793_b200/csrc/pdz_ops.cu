// Stand-alone PDE operators behind the API functions divergence_term
// (solver.py:190-210), gaussian_convolve (:225-241) and tau_stability_bound
// (:266-277).  These are probes / one-off diagnostics, not the sweep: they
// are templated on the scalar type so the numpy-facing API can evaluate them
// in float64 exactly like the reference.
#include <type_traits>
#include <algorithm>
#include <cmath>
#include <vector>

#include "pdz_internal.cuh"

namespace pdz {

template <typename T>
struct Face {
  // np.gradient along an axis at position i of n (edge_order 1, unit dx).
  __device__ static T centred(const T* f, int i, int n, ptrdiff_t stride) {
    if (i == 0) return f[stride] - f[0];
    if (i == n - 1) return f[0] - f[-stride];
    return (f[stride] - f[-stride]) / T(2);
  }
  __device__ static T flux(T jump, T along, T eps, bool edge) {
    if (!edge) return jump;
    const T d = T(1) / (sqrt(jump * jump + along * along) + eps);
    return d * jump;
  }
};

// div[y][x] = ((fe(y,x) - fe(y,x-1)) + fs(y,x)) - fs(y-1,x), zero flux outside
// (the accumulation order of divergence_term, solver.py:205-209).
template <typename T>
__global__ void divergence_kernel(const T* __restrict__ u, T* __restrict__ out, int H, int W,
                                  int P, T eps, bool edge) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int p = blockIdx.z;
  if (x >= W || y >= H) return;
  const T* f = u + size_t(p) * H * W;
  auto at = [&](int yy, int xx) { return f + size_t(yy) * W + xx; };
  auto east = [&](int yy, int xx) -> T {  // face between (yy,xx) and (yy,xx+1)
    if (xx < 0 || xx >= W - 1) return T(0);
    const T jump = *at(yy, xx + 1) - *at(yy, xx);
    const T along = T(0.5) * (Face<T>::centred(at(yy, xx + 1), yy, H, W) +
                              Face<T>::centred(at(yy, xx), yy, H, W));
    return Face<T>::flux(jump, along, eps, edge);
  };
  auto south = [&](int yy, int xx) -> T {  // face between (yy,xx) and (yy+1,xx)
    if (yy < 0 || yy >= H - 1) return T(0);
    const T jump = *at(yy + 1, xx) - *at(yy, xx);
    const T along = T(0.5) * (Face<T>::centred(at(yy + 1, xx), xx, W, 1) +
                              Face<T>::centred(at(yy, xx), xx, W, 1));
    return Face<T>::flux(jump, along, eps, edge);
  };
  T acc = T(0);
  if (x < W - 1) acc = acc + east(y, x);
  if (x > 0) acc = acc - east(y, x - 1);
  if (y < H - 1) acc = acc + south(y, x);
  if (y > 0) acc = acc - south(y - 1, x);
  out[size_t(p) * H * W + size_t(y) * W + x] = acc;
}

// One separable Gaussian pass with symmetric reflection (axis 1 = along
// rows, axis 0 = along columns).
template <typename T>
__global__ void gauss_pass_kernel(const T* __restrict__ in, T* __restrict__ out, int H, int W,
                                  const double* __restrict__ taps, int K, int axis) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y * blockDim.y + threadIdx.y;
  const int p = blockIdx.z;
  if (x >= W || y >= H) return;
  const T* f = in + size_t(p) * H * W;
  const int r = K / 2;
  T acc = T(0);
  for (int k = 0; k < K; ++k) {
    const T w = T(taps[k]);
    const T v = axis == 1 ? f[size_t(y) * W + reflect(x - r + k, W)]
                          : f[size_t(reflect(y - r + k, H)) * W + x];
    acc = acc + w * v;
  }
  out[size_t(p) * H * W + size_t(y) * W + x] = acc;
}

// ---- tau_stability_bound: min over faces of |grad|^2 (float64) and max lambda
__device__ __forceinline__ void atomic_min_u64(unsigned long long* a, unsigned long long v) {
  atomicMin(a, v);
}

__global__ void tau_init_kernel(unsigned long long* smin, unsigned long long* lmax, int P) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < P) {
    smin[i] = 0x7ff0000000000000ull;  // +inf
    lmax[i] = 0ull;                   // below every float64 key
  }
}

// u: sample (y, x) of plane p at u[p*ps + (y*W + x)*us] (planar: us = 1,
// ps = H*W; interleaved [H][W][C]: us = C, ps = 1).  lambda planar [P/C][H][W].
template <typename TU, typename TL>
__global__ void tau_scan_kernel(const TU* __restrict__ u, const TL* __restrict__ lam, int H,
                                int W, int C, size_t us, size_t ps, unsigned long long* smin,
                                unsigned long long* lmax) {
  const int p = blockIdx.y;
  const TU* f = u + size_t(p) * ps;
  const TL* lp = lam + size_t(p / C) * H * W;
  double best = INFINITY;
  double lbest = -INFINITY;
  const size_t n = size_t(H) * W;
  auto at = [&](size_t j) -> double { return double(f[j * us]); };
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int y = int(i / W), x = int(i - size_t(y) * W);
    const double c = at(i);
    auto cy = [&](int xx) -> double {
      const size_t j = size_t(y) * W + xx;
      if (y == 0) return at(j + W) - at(j);
      if (y == H - 1) return at(j) - at(j - W);
      return (at(j + W) - at(j - W)) / 2.0;
    };
    auto cx = [&](int yy) -> double {
      const size_t j = size_t(yy) * W + x;
      if (x == 0) return at(j + 1) - at(j);
      if (x == W - 1) return at(j) - at(j - 1);
      return (at(j + 1) - at(j - 1)) / 2.0;
    };
    if (x < W - 1) {
      const double jump = at(i + 1) - c;
      const double along = 0.5 * (cy(x + 1) + cy(x));
      best = fmin(best, jump * jump + along * along);
    }
    if (y < H - 1) {
      const double jump = at(i + W) - c;
      const double along = 0.5 * (cx(y + 1) + cx(y));
      best = fmin(best, jump * jump + along * along);
    }
    if ((p % C) == 0) lbest = fmax(lbest, double(lp[i]));
  }
  // block reduce
  __shared__ double sb[32];
  __shared__ double sl[32];
  for (int o = 16; o > 0; o >>= 1) {
    best = fmin(best, __shfl_xor_sync(0xffffffffu, best, o));
    lbest = fmax(lbest, __shfl_xor_sync(0xffffffffu, lbest, o));
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) {
    sb[warp] = best;
    sl[warp] = lbest;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < int(blockDim.x >> 5); ++w) {
      best = fmin(best, sb[w]);
      lbest = fmax(lbest, sl[w]);
    }
    atomic_min_u64(&smin[p], static_cast<unsigned long long>(__double_as_longlong(best)));
    if ((p % C) == 0)
      atomicMax(&lmax[p / C], static_cast<unsigned long long>(f64_order_key(lbest)));
  }
}

// Interleaved (H, W, C) field, C <= 4: one pass over the pixels with every
// channel handled by the same thread (the per-plane scan read the whole
// interleaved array once per channel).  The same per-face arithmetic as
// tau_scan_kernel; min / max reductions are order-independent, so the bounds
// are bitwise those of the per-plane scan.
template <typename TL>
__global__ void tau_scan_hwc_kernel(const double* __restrict__ u, const TL* __restrict__ lam,
                                    int H, int W, int C, unsigned long long* smin,
                                    unsigned long long* lmax) {
  double best[4] = {INFINITY, INFINITY, INFINITY, INFINITY};
  double lbest = -INFINITY;
  const size_t n = size_t(H) * W;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += size_t(gridDim.x) * blockDim.x) {
    const int y = int(i / W), x = int(i - size_t(y) * W);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      if (c >= C) break;
      auto at = [&](size_t j) -> double { return u[j * C + c]; };
      auto cy = [&](int xx) -> double {
        const size_t j = size_t(y) * W + xx;
        if (y == 0) return at(j + W) - at(j);
        if (y == H - 1) return at(j) - at(j - W);
        return (at(j + W) - at(j - W)) / 2.0;
      };
      auto cx = [&](int yy) -> double {
        const size_t j = size_t(yy) * W + x;
        if (x == 0) return at(j + 1) - at(j);
        if (x == W - 1) return at(j) - at(j - 1);
        return (at(j + 1) - at(j - 1)) / 2.0;
      };
      const double cv = at(i);
      if (x < W - 1) {
        const double jump = at(i + 1) - cv;
        const double along = 0.5 * (cy(x + 1) + cy(x));
        best[c] = fmin(best[c], jump * jump + along * along);
      }
      if (y < H - 1) {
        const double jump = at(i + W) - cv;
        const double along = 0.5 * (cx(y + 1) + cx(y));
        best[c] = fmin(best[c], jump * jump + along * along);
      }
    }
    lbest = fmax(lbest, double(lam[i]));
  }
  __shared__ double sb[4][32];
  __shared__ double sl[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    for (int o = 16; o > 0; o >>= 1) best[c] = fmin(best[c], __shfl_xor_sync(0xffffffffu, best[c], o));
  for (int o = 16; o > 0; o >>= 1) lbest = fmax(lbest, __shfl_xor_sync(0xffffffffu, lbest, o));
  if (lane == 0) {
#pragma unroll
    for (int c = 0; c < 4; ++c) sb[c][warp] = best[c];
    sl[warp] = lbest;
  }
  __syncthreads();
  if (threadIdx.x < C) {
    const int c = threadIdx.x;
    double b = sb[c][0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) b = fmin(b, sb[c][w]);
    atomic_min_u64(&smin[c], static_cast<unsigned long long>(__double_as_longlong(b)));
  }
  if (threadIdx.x == 0) {
    double l = sl[0];
    for (int w = 1; w < int(blockDim.x >> 5); ++w) l = fmax(l, sl[w]);
    atomicMax(&lmax[0], static_cast<unsigned long long>(f64_order_key(l)));
  }
}

__global__ void tau_final_kernel(const unsigned long long* smin, const unsigned long long* lmax,
                                 int P, int C, double eps, double* bound) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const double s = __longlong_as_double(static_cast<long long>(smin[p]));
  const double dmax = 1.0 / (sqrt(s) + eps);
  const double lm = f64_from_order_key(lmax[p / C]);
  bound[p] = 2.0 / (8.0 * dmax + fmax(lm, 0.0));
}

template <typename T>
static int32_t run_divergence(const pdz_solve_params* prm, const T* u, T* out, void* stream) {
  PDZ_REQUIRE(prm && u && out, "NULL argument");
  PDZ_REQUIRE(prm->height >= 2 && prm->width >= 2, "field must be at least 2x2, got (%d, %d)",
              prm->height, prm->width);
  PDZ_REQUIRE(prm->epsilon > 0.0, "epsilon must be > 0");
  PDZ_REQUIRE(prm->planes >= 1, "planes must be >= 1");
  dim3 blk(32, 8);
  dim3 grid((prm->width + 31) / 32, (prm->height + 7) / 8, prm->planes);
  divergence_kernel<T><<<grid, blk, 0, as_stream(stream)>>>(
      u, out, prm->height, prm->width, prm->planes, T(prm->epsilon), prm->edge_preserving != 0);
  PDZ_CHECK_LAUNCH("divergence");
  return PDZ_OK;
}

static size_t gauss_ws(const pdz_solve_params* prm, size_t elem) {
  Carver c(nullptr, 0);
  c.take<double>(prm->kernel_size > 0 ? size_t(prm->kernel_size) : 1);
  c.take<char>(size_t(prm->planes) * prm->height * prm->width * elem);
  return Carver::round(c.off);
}

template <typename T>
static int32_t run_gaussian(const pdz_solve_params* prm, const T* u, T* out, void* ws,
                            size_t ws_bytes, void* stream) {
  PDZ_REQUIRE(prm && u && out, "NULL argument");
  PDZ_REQUIRE(prm->height >= 1 && prm->width >= 1 && prm->planes >= 1, "bad shape");
  std::vector<double> taps(prm->kernel_size > 0 ? prm->kernel_size : 1);
  int32_t rc = gaussian_taps_host(prm->sigma, prm->kernel_size, taps.data());
  if (rc != PDZ_OK) return rc;
  Carver c(ws, ws_bytes);
  double* dtaps = c.take<double>(taps.size());
  T* tmp = c.take<T>(size_t(prm->planes) * prm->height * prm->width);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  PDZ_CUDA(cudaMemcpyAsync(dtaps, taps.data(), taps.size() * 8, cudaMemcpyHostToDevice, s),
           "taps H2D");
  dim3 blk(32, 8);
  dim3 grid((prm->width + 31) / 32, (prm->height + 7) / 8, prm->planes);
  gauss_pass_kernel<T><<<grid, blk, 0, s>>>(u, tmp, prm->height, prm->width, dtaps,
                                            prm->kernel_size, 1);
  gauss_pass_kernel<T><<<grid, blk, 0, s>>>(tmp, out, prm->height, prm->width, dtaps,
                                            prm->kernel_size, 0);
  PDZ_CHECK_LAUNCH("gaussian");
  // taps live in the workspace: the caller must keep it alive until the
  // stream reaches this point (all our Python callers synchronise).
  return cudaStreamSynchronize(s) == cudaSuccess ? PDZ_OK : cuda_status(cudaGetLastError(), "gaussian sync");
}

template <typename TU, typename TL>
static int32_t run_tau(const pdz_solve_params* prm, const TU* u, const TL* lam, double* bound,
                       void* ws, size_t ws_bytes, void* stream, bool interleaved = false) {
  PDZ_REQUIRE(prm && u && lam && bound, "NULL argument");
  PDZ_REQUIRE(prm->height >= 2 && prm->width >= 2, "field must be at least 2x2, got (%d, %d)",
              prm->height, prm->width);
  PDZ_REQUIRE(prm->epsilon > 0.0, "epsilon must be > 0");
  PDZ_REQUIRE(prm->planes >= 1 && prm->channels >= 1 && prm->planes % prm->channels == 0,
              "bad planes/channels");
  Carver c(ws, ws_bytes);
  auto* smin = c.take<unsigned long long>(prm->planes);
  auto* lmax = c.take<unsigned long long>(prm->planes);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, ws_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  const int P = prm->planes;
  tau_init_kernel<<<(P + 255) / 256, 256, 0, s>>>(smin, lmax, P);
  const size_t n = size_t(prm->height) * prm->width;
  const int bx = int(std::min<size_t>((n + 255) / 256, size_t(4 * num_sms())));
  const size_t us = interleaved ? size_t(P) : 1, ps = interleaved ? 1 : n;
  if constexpr (std::is_same<TU, double>::value) {
    if (interleaved && P == prm->channels && P <= 4) {
      tau_scan_hwc_kernel<TL><<<bx, 256, 0, s>>>(u, lam, prm->height, prm->width, P, smin, lmax);
    } else {
      tau_scan_kernel<TU, TL><<<dim3(bx, P), 256, 0, s>>>(u, lam, prm->height, prm->width,
                                                          prm->channels, us, ps, smin, lmax);
    }
  } else {
    tau_scan_kernel<TU, TL><<<dim3(bx, P), 256, 0, s>>>(u, lam, prm->height, prm->width,
                                                        prm->channels, us, ps, smin, lmax);
  }
  tau_final_kernel<<<(P + 255) / 256, 256, 0, s>>>(smin, lmax, P, prm->channels,
                                                   prm->epsilon, bound);
  PDZ_CHECK_LAUNCH("tau bound");
  return PDZ_OK;
}

}  // namespace pdz

using namespace pdz;

extern "C" {

int32_t pdz_divergence(const pdz_solve_params* params, const float* u, float* div,
                       void* stream) {
  return run_divergence<float>(params, u, div, stream);
}
int32_t pdz_divergence_f64(const pdz_solve_params* params, const double* u, double* div,
                           void* stream) {
  return run_divergence<double>(params, u, div, stream);
}

size_t pdz_gaussian_workspace_bytes(const pdz_solve_params* params, int32_t is_f64) {
  if (!params) return 0;
  return gauss_ws(params, is_f64 ? 8 : 4);
}
int32_t pdz_gaussian(const pdz_solve_params* params, const float* u, float* out,
                     void* workspace, size_t workspace_bytes, void* stream) {
  return run_gaussian<float>(params, u, out, workspace, workspace_bytes, stream);
}
int32_t pdz_gaussian_f64(const pdz_solve_params* params, const double* u, double* out,
                         void* workspace, size_t workspace_bytes, void* stream) {
  return run_gaussian<double>(params, u, out, workspace, workspace_bytes, stream);
}

size_t pdz_tau_bound_workspace_bytes(const pdz_solve_params* params) {
  if (!params || params->planes < 1) return 0;
  Carver c(nullptr, 0);
  c.take<unsigned long long>(params->planes);
  c.take<unsigned long long>(params->planes);
  return Carver::round(c.off);
}
int32_t pdz_tau_bound(const pdz_solve_params* params, const float* u, const float* lambda_map,
                      double* bound, void* workspace, size_t workspace_bytes, void* stream) {
  return run_tau<float, float>(params, u, lambda_map, bound, workspace, workspace_bytes, stream);
}
int32_t pdz_tau_bound_f64(const pdz_solve_params* params, const double* u,
                          const double* lambda_map, double* bound, void* workspace,
                          size_t workspace_bytes, void* stream) {
  return run_tau<double, double>(params, u, lambda_map, bound, workspace, workspace_bytes,
                                 stream);
}
int32_t pdz_tau_bound_hwc(const pdz_solve_params* params, const double* u_hwc,
                          const float* lambda_map, double* bound, void* workspace,
                          size_t workspace_bytes, void* stream) {
  if (params && params->planes != params->channels) {
    set_error("pdz_tau_bound_hwc handles one image (planes == channels)");
    return PDZ_EINVAL;
  }
  return run_tau<double, float>(params, u_hwc, lambda_map, bound, workspace, workspace_bytes,
                                stream, true);
}

}  // extern "C"
