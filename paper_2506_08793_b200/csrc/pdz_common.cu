// Library-wide plumbing: error strings, version, Gaussian taps.
#include <atomic>
#include <cmath>
#include <cstring>
#include <mutex>

#include "pdz_internal.cuh"

namespace pdz {

static thread_local char g_last_error[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_last_error, sizeof(g_last_error), fmt, ap);
  va_end(ap);
}

int32_t cuda_status(cudaError_t e, const char* where) {
  set_error("CUDA error in %s: %s", where, cudaGetErrorString(e));
  return PDZ_ECUDA;
}

int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 ? 0 : (dev >= kMaxDevices ? kMaxDevices - 1 : dev);
}

// Per device: SM counts differ between device kinds, and a process may drive
// several GPUs (one thread per device).
int num_sms() {
  static std::atomic<int> cached[kMaxDevices] = {};
  const int dev = current_device();
  int v = cached[dev].load(std::memory_order_relaxed);
  if (v == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    v = n > 0 ? n : 148;
    cached[dev].store(v, std::memory_order_relaxed);
  }
  return v;
}

bool first_use_on_device(std::atomic<uint64_t>* mask) {
  const uint64_t bit = uint64_t(1) << current_device();
  return (mask->fetch_or(bit) & bit) == 0;
}

// g = exp(-d^2 / (2 sigma^2)), d = -K/2..K/2, normalised by its sum.  The
// reference normalises outer(g, g) by its total (solver.py:219-222); that
// equals outer(g/S, g/S) with S = sum(g) up to ~1e-17.
int32_t gaussian_taps_host(double sigma, int kernel_size, double* taps) {
  if (!(sigma > 0.0)) {
    set_error("sigma must be > 0");
    return PDZ_EINVAL;
  }
  if (kernel_size < 1 || kernel_size % 2 == 0) {
    set_error("kernel_size must be odd and >= 1, got %d", kernel_size);
    return PDZ_EINVAL;
  }
  const int r = kernel_size / 2;
  double s = 0.0;
  for (int i = 0; i < kernel_size; ++i) {
    const double d = double(i - r);
    taps[i] = std::exp(-(d * d) / (2.0 * sigma * sigma));
    s += taps[i];
  }
  for (int i = 0; i < kernel_size; ++i) taps[i] /= s;
  return PDZ_OK;
}

}  // namespace pdz

extern "C" {

int32_t pdz_version(void) { return 1; }

const char* pdz_last_error(void) { return pdz::g_last_error; }

int32_t pdz_gaussian_taps(double sigma, int32_t kernel_size, double* taps_host) {
  if (taps_host == nullptr) {
    pdz::set_error("taps_host is NULL");
    return PDZ_EINVAL;
  }
  return pdz::gaussian_taps_host(sigma, kernel_size, taps_host);
}

}  // extern "C"
