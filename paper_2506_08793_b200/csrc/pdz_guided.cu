// Guided-filter refinement of the transmission map (refine.py:21-80) --
// SURVEY 8(f) "next #1": it is on the reference's default dehaze path
// (solver.py:405-408).
//
// Bit-exact with the reference: box_mean builds its integral image with
// cumsum(axis=0) then cumsum(axis=1) (refine.py:28), i.e. two strictly
// sequential float64 scans.  Each scan here runs one thread per line in the
// same order (columns first; rows via a transpose so loads stay coalesced),
// then the window sums are evaluated as ((a - b) - c) + d and divided by the
// integer window area (refine.py:33-40).  All arithmetic avoids FMA
// contraction so every value matches numpy's float64 results exactly.
#include <algorithm>

#include "pdz_internal.cuh"

namespace pdz {

// out[y][x] = sum_{k<=y} in[k][x], sequential per column (thread per column).
__global__ void colscan_kernel(const double* __restrict__ in, double* __restrict__ out, int H,
                               int W) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  if (x >= W) return;
  double s = 0.0;
  int y = 0;
  for (; y + 8 <= H; y += 8) {
    double v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = in[size_t(y + k) * W + x];
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      s = __dadd_rn(s, v[k]);
      out[size_t(y + k) * W + x] = s;
    }
  }
  for (; y < H; ++y) {
    s = __dadd_rn(s, in[size_t(y) * W + x]);
    out[size_t(y) * W + x] = s;
  }
}

__global__ void transpose64_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   int H, int W) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int y = by + j, x = bx + threadIdx.x;
    if (y < H && x < W) t[j][threadIdx.x] = in[size_t(y) * W + x];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int x = bx + j, y = by + threadIdx.x;
    if (y < H && x < W) out[size_t(x) * H + y] = t[threadIdx.x][j];
  }
}

// St is the transposed inclusive 2-D prefix sum: St[x][y] = I[y+1][x+1].
__device__ __forceinline__ double integral_at(const double* St, int H, int i, int j) {
  // I[i][j] with a zero first row / column
  return (i == 0 || j == 0) ? 0.0 : St[size_t(j - 1) * H + (i - 1)];
}

__global__ void box_eval_kernel(const double* __restrict__ St, int H, int W, int r,
                                double* __restrict__ out) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y;
  if (x >= W) return;
  const int lo_r = max(y - r, 0), hi_r = min(y + r, H - 1) + 1;
  const int lo_c = max(x - r, 0), hi_c = min(x + r, W - 1) + 1;
  const double a = integral_at(St, H, hi_r, hi_c);
  const double b = integral_at(St, H, lo_r, hi_c);
  const double c = integral_at(St, H, hi_r, lo_c);
  const double d = integral_at(St, H, lo_r, lo_c);
  const double sum = __dadd_rn(__dsub_rn(__dsub_rn(a, b), c), d);
  const long long cnt = (long long)(hi_r - lo_r) * (long long)(hi_c - lo_c);
  out[size_t(y) * W + x] = __ddiv_rn(sum, double(cnt));
}

struct BoxScratch {
  double* col;  // [H][W]
  double* tr;   // [W][H]
  double* st;   // [W][H]
};

static int32_t box_mean_dev(const double* f, int H, int W, int r, double* out,
                            const BoxScratch& s, cudaStream_t st) {
  colscan_kernel<<<(W + 127) / 128, 128, 0, st>>>(f, s.col, H, W);
  transpose64_kernel<<<dim3((W + 31) / 32, (H + 31) / 32), dim3(32, 8), 0, st>>>(s.col, s.tr, H,
                                                                                W);
  colscan_kernel<<<(H + 127) / 128, 128, 0, st>>>(s.tr, s.st, W, H);
  box_eval_kernel<<<dim3((W + 127) / 128, H), 128, 0, st>>>(s.st, H, W, r, out);
  PDZ_CHECK_LAUNCH("box mean");
  return PDZ_OK;
}

// Elementwise helpers (float64, no contraction).
__global__ void mul_kernel(const double* a, const double* b, double* o, int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    o[i] = __dmul_rn(a[i], b[i]);
}

// var = box(gg) - mg*mg ; cov = box(gp) - mg*mp ; a = cov/(var+reg) ; b = mp - a*mg
__global__ void guided_coef_kernel(const double* mg, const double* mp, const double* bgg,
                                   const double* bgp, double reg, double* a_out, double* b_out,
                                   int64_t n) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double var = __dsub_rn(bgg[i], __dmul_rn(mg[i], mg[i]));
    const double cov = __dsub_rn(bgp[i], __dmul_rn(mg[i], mp[i]));
    const double a = __ddiv_rn(cov, __dadd_rn(var, reg));
    a_out[i] = a;
    b_out[i] = __dsub_rn(mp[i], __dmul_rn(a, mg[i]));
  }
}

// out = ma*g + mb, optionally clipped to [0, 1]
__global__ void guided_out_kernel(const double* ma, const double* g, const double* mb,
                                  double* out, int64_t n, int clip) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double v = __dadd_rn(__dmul_rn(ma[i], g[i]), mb[i]);
    if (clip) v = fmin(fmax(v, 0.0), 1.0);
    out[i] = v;
  }
}

// guide = 0.299 R + 0.587 G + 0.114 B (refine.py:18, :79) or the single channel.
template <typename T>
__global__ void luma_kernel(const void* img, int C, int64_t n, double* out) {
  const T* p = static_cast<const T*>(img);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    if (C == 1) {
      out[i] = double(p[i]);
    } else {
      const double r = double(p[size_t(i) * C]), g = double(p[size_t(i) * C + 1]),
                   b = double(p[size_t(i) * C + 2]);
      out[i] = __dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)),
                         __dmul_rn(0.114, b));
    }
  }
}

static int grid_n(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8)));
}

struct GuidedLayout {
  BoxScratch box;
  double* mg;
  double* mp;
  double* t0;
  double* t1;
  double* t2;
  double* guide;
  size_t bytes;
};

static GuidedLayout carve_guided(int H, int W, void* ws, size_t cap) {
  Carver c(ws, cap);
  const size_t n = size_t(H) * W;
  GuidedLayout L;
  L.box.col = c.take<double>(n);
  L.box.tr = c.take<double>(n);
  L.box.st = c.take<double>(n);
  L.mg = c.take<double>(n);
  L.mp = c.take<double>(n);
  L.t0 = c.take<double>(n);
  L.t1 = c.take<double>(n);
  L.t2 = c.take<double>(n);
  L.guide = c.take<double>(n);
  L.bytes = c.off;
  return L;
}

static int32_t guided_dev(const double* g, const double* p, int H, int W, int r, double reg,
                          double* out, int clip, const GuidedLayout& L, cudaStream_t s) {
  const int64_t n = int64_t(H) * W;
  int32_t rc;
  if ((rc = box_mean_dev(g, H, W, r, L.mg, L.box, s))) return rc;
  if ((rc = box_mean_dev(p, H, W, r, L.mp, L.box, s))) return rc;
  mul_kernel<<<grid_n(n), 256, 0, s>>>(g, g, L.t0, n);
  if ((rc = box_mean_dev(L.t0, H, W, r, L.t1, L.box, s))) return rc;  // box(g*g)
  mul_kernel<<<grid_n(n), 256, 0, s>>>(g, p, L.t0, n);
  if ((rc = box_mean_dev(L.t0, H, W, r, L.t2, L.box, s))) return rc;  // box(g*p)
  // a -> t0, b -> t1
  guided_coef_kernel<<<grid_n(n), 256, 0, s>>>(L.mg, L.mp, L.t1, L.t2, reg, L.t0, L.t1, n);
  if ((rc = box_mean_dev(L.t0, H, W, r, L.t2, L.box, s))) return rc;  // box(a)
  if ((rc = box_mean_dev(L.t1, H, W, r, L.mg, L.box, s))) return rc;  // box(b)
  guided_out_kernel<<<grid_n(n), 256, 0, s>>>(L.t2, g, L.mg, out, n, clip);
  PDZ_CHECK_LAUNCH("guided filter");
  return PDZ_OK;
}

}  // namespace pdz

using namespace pdz;

extern "C" {

size_t pdz_guided_workspace_bytes(int32_t height, int32_t width) {
  if (height < 1 || width < 1) return 0;
  return Carver::round(carve_guided(height, width, nullptr, 0).bytes);
}

int32_t pdz_box_mean(const double* field, int32_t height, int32_t width, int32_t radius,
                     double* out, void* workspace, size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(field && out, "NULL argument");
  PDZ_REQUIRE(height >= 1 && width >= 1, "bad field shape");
  PDZ_REQUIRE(radius >= 1, "radius must be >= 1");
  GuidedLayout L = carve_guided(height, width, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  return box_mean_dev(field, height, width, radius, out, L.box, as_stream(stream));
}

int32_t pdz_guided_filter(const double* guide, const double* target, int32_t height,
                          int32_t width, int32_t radius, double reg, double* out,
                          void* workspace, size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(guide && target && out, "NULL argument");
  PDZ_REQUIRE(height >= 1 && width >= 1, "bad field shape");
  PDZ_REQUIRE(radius >= 1, "radius must be >= 1");
  PDZ_REQUIRE(reg > 0.0, "reg must be > 0");
  GuidedLayout L = carve_guided(height, width, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  return guided_dev(guide, target, height, width, radius, reg, out, 0, L, as_stream(stream));
}

int32_t pdz_refine_transmission(const void* image, int32_t image_is_f64, int32_t height,
                                int32_t width, int32_t channels, const double* t_raw,
                                int32_t radius, double reg, double* t_out, void* workspace,
                                size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(image && t_raw && t_out, "NULL argument");
  PDZ_REQUIRE(channels == 1 || channels == 3, "channels must be 1 or 3");
  PDZ_REQUIRE(radius >= 1, "radius must be >= 1");
  PDZ_REQUIRE(reg > 0.0, "reg must be > 0");
  GuidedLayout L = carve_guided(height, width, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  const int64_t n = int64_t(height) * width;
  if (image_is_f64)
    luma_kernel<double><<<grid_n(n), 256, 0, s>>>(image, channels, n, L.guide);
  else
    luma_kernel<float><<<grid_n(n), 256, 0, s>>>(image, channels, n, L.guide);
  PDZ_CHECK_LAUNCH("luma");
  return guided_dev(L.guide, t_raw, height, width, radius, reg, t_out, 1, L, s);
}

}  // extern "C"
