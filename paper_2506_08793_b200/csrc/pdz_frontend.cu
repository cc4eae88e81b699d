// Dark-channel-prior front end (scattering.py:48-139, solver.py:324-330).
//
// Everything here is float64 and reproduces the reference's operation order,
// so the dark channel, the airlight pixel indices, A and t are bit-exact:
//   * channel min of I_c / A_c with correctly rounded float64 divides   (:60)
//   * (2r+1)^2 window minimum, border-truncated, separable, computed with
//     the van Herk / Gil-Werman prefix/suffix-min scheme in shared memory
//     (scipy minimum_filter mode="nearest", :61-64); min is exact
//   * top ceil(f HW) by (value desc, flat index asc): 8-pass MSD radix select
//     on order-preserving 64-bit keys, index-ordered compaction, rank-by-
//     counting sort (the stable argsort at :105)
//   * float64 sum in numpy's order (sequential rows for C = 3, pairwise for
//     C = 1) in selection order / count, clip [0.05, 1] (picked.mean(axis=0),
//     :106-107)
//   * no FMA contraction anywhere (__dmul_rn / __dadd_rn / __dsub_rn).
#include <algorithm>
#include <cmath>
#include <vector>

#include "pdz_internal.cuh"

namespace pdz {

template <typename T>
__device__ __forceinline__ double load_f64(const void* p, size_t i) {
  return double(static_cast<const T*>(p)[i]);
}

// ---------------------------------------------------------------- dark ---
// Batched kernels: blockIdx.y (blockIdx.z for the transpose) is the image of a
// batch of equal-shaped images stored back to back; the single-image entry
// points launch them with one image.
template <typename T>
__global__ void chanmin_kernel(const void* __restrict__ img, int64_t n, int C,
                               const double* __restrict__ airlight, int a_stride,
                               double* __restrict__ out) {
  const size_t z = blockIdx.y;
  const double* a = airlight + z * a_stride;  // a_stride = 0: one vector for every image
  const size_t ibase = z * size_t(n) * C;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double m = __ddiv_rn(load_f64<T>(img, ibase + size_t(i) * C), a[0]);
    for (int c = 1; c < C; ++c)
      m = fmin(m, __ddiv_rn(load_f64<T>(img, ibase + size_t(i) * C + c), a[c]));
    out[z * size_t(n) + i] = m;
  }
}

// Van Herk / Gil-Werman window minimum along rows: out[y][x] = min of
// in[y][max(0,x-r) .. min(W-1,x+r)].  One block handles a chunk of `span`
// outputs of one row; the chunk plus its r-halo is staged in shared memory,
// padded with +inf outside the row (truncation), split into segments of
// length w = 2r+1 aligned to the staged start; g = running min from each
// segment start, h = running min to each segment end; out = min(h[a], g[a+2r])
// for the window [a, a+2r] in staged coordinates.
__global__ void rowmin_vhgw_kernel(const double* __restrict__ in, double* __restrict__ out,
                                   int H, int W, int r, int span) {
  extern __shared__ double sm[];
  const int y = blockIdx.y + blockIdx.z * gridDim.y;  // (a batch has more rows than grid.y holds)
  if (y >= H) return;
  const int x0 = blockIdx.x * span;
  const int L = span + 2 * r;  // staged length
  double* g = sm;
  double* h = sm + L;
  const double* row = in + size_t(y) * W;
  for (int i = threadIdx.x; i < L; i += blockDim.x) {
    const int x = x0 - r + i;
    const double v = (x >= 0 && x < W) ? row[x] : INFINITY;
    g[i] = v;
    h[i] = v;
  }
  __syncthreads();
  const int w = 2 * r + 1;
  const int nseg = (L + w - 1) / w;
  for (int sgi = threadIdx.x; sgi < nseg; sgi += blockDim.x) {
    const int a = sgi * w, b = min(a + w, L);
    for (int i = a + 1; i < b; ++i) g[i] = fmin(g[i], g[i - 1]);
    for (int i = b - 2; i >= a; --i) h[i] = fmin(h[i], h[i + 1]);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < span; i += blockDim.x) {
    const int x = x0 + i;
    if (x < W) out[size_t(y) * W + x] = fmin(h[i], g[i + 2 * r]);
  }
}

// Direct window minimum along rows for very large radii (rare API edge case).
__global__ void rowmin_direct_kernel(const double* __restrict__ in, double* __restrict__ out,
                                     int H, int W, int r) {
  const int x = blockIdx.x * blockDim.x + threadIdx.x;
  const int y = blockIdx.y + blockIdx.z * gridDim.y;
  if (x >= W || y >= H) return;
  const double* row = in + size_t(y) * W;
  double m = row[x];
  const int lo = max(0, x - r), hi = min(W - 1, x + r);
  for (int i = lo; i <= hi; ++i) m = fmin(m, row[i]);
  out[size_t(y) * W + x] = m;
}

// 32x32 tiled transpose; optionally caps at 1 (np.minimum(dark, 1.0), :65).
__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, int H,
                                 int W, int cap_at_one) {
  __shared__ double t[32][33];
  const int bx = blockIdx.x * 32, by = blockIdx.y * 32;
  in += size_t(blockIdx.z) * H * W;
  out += size_t(blockIdx.z) * H * W;
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int y = by + j, x = bx + threadIdx.x;
    if (y < H && x < W) t[j][threadIdx.x] = in[size_t(y) * W + x];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += blockDim.y) {
    const int x = bx + j, y = by + threadIdx.x;  // out is [W][H]
    if (y < H && x < W) {
      double v = t[threadIdx.x][j];
      if (cap_at_one) v = fmin(v, 1.0);
      out[size_t(x) * H + y] = v;
    }
  }
}

constexpr int kRowGridY = 32768;  // rows per grid.y slab (grid.y <= 65535)

static int32_t rowmin(const double* in, double* out, int H, int W, int r, cudaStream_t s) {
  if (r == 0) {
    PDZ_CUDA(cudaMemcpyAsync(out, in, size_t(H) * W * 8, cudaMemcpyDeviceToDevice, s), "copy");
    return PDZ_OK;
  }
  if (r > 2048) {
    rowmin_direct_kernel<<<dim3((W + 255) / 256, std::min(H, kRowGridY), (H + kRowGridY - 1) / kRowGridY),
                           256, 0, s>>>(in, out, H, W, r);
    PDZ_CHECK_LAUNCH("rowmin direct");
    return PDZ_OK;
  }
  const int span = std::min(W, 2048);
  const size_t smem = size_t(2) * (span + 2 * r) * sizeof(double);
  static std::atomic<uint64_t> raised{0};
  if (first_use_on_device(&raised))
    cudaFuncSetAttribute(rowmin_vhgw_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         2 * (2048 + 2 * 2048) * 8);
  rowmin_vhgw_kernel<<<dim3((W + span - 1) / span, std::min(H, kRowGridY),
                            (H + kRowGridY - 1) / kRowGridY),
                       256, smem, s>>>(in, out, H, W, r, span);
  PDZ_CHECK_LAUNCH("rowmin");
  return PDZ_OK;
}

static int32_t transpose(const double* in, double* out, int H, int W, bool cap, cudaStream_t s,
                         int batch = 1) {
  transpose_kernel<<<dim3((W + 31) / 32, (H + 31) / 32, batch), dim3(32, 8), 0, s>>>(
      in, out, H, W, cap ? 1 : 0);
  PDZ_CHECK_LAUNCH("transpose");
  return PDZ_OK;
}

static size_t dark_ws(int H, int W) {
  Carver c(nullptr, 0);
  c.take<double>(size_t(H) * W);
  c.take<double>(size_t(H) * W);
  c.take<double>(size_t(H) * W);
  return Carver::round(c.off);
}

// `batch` images back to back (tmp_a / tmp_b / dark hold batch * H * W doubles);
// airlight: [batch][C] with a_stride = C, or one [C] vector with a_stride = 0.
// The row pass runs over the batch * H rows of the stacked images, the column
// pass over the batch * W rows of the per-image transposes.
static int32_t dark_channel_impl(const void* img, int is_f64, int H, int W, int C,
                                 const double* airlight, int r, double* dark, double* tmp_a,
                                 double* tmp_b, cudaStream_t s, int batch = 1,
                                 int a_stride = 0) {
  const int64_t n = int64_t(H) * W;
  const int gx = int(std::max<int64_t>(
      1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8 / std::min(batch, 8))));
  const dim3 grid(gx, batch);
  if (is_f64)
    chanmin_kernel<double><<<grid, 256, 0, s>>>(img, n, C, airlight, a_stride, tmp_a);
  else
    chanmin_kernel<float><<<grid, 256, 0, s>>>(img, n, C, airlight, a_stride, tmp_a);
  PDZ_CHECK_LAUNCH("chanmin");
  int32_t rc;
  if ((rc = rowmin(tmp_a, tmp_b, batch * H, W, r, s)) != PDZ_OK) return rc;
  if ((rc = transpose(tmp_b, tmp_a, H, W, false, s, batch)) != PDZ_OK) return rc;  // [W][H]
  if ((rc = rowmin(tmp_a, tmp_b, batch * W, H, r, s)) != PDZ_OK) return rc;
  return transpose(tmp_b, dark, W, H, true, s, batch);
}

// combined = w0*d0 (first) or combined + w*d, float64 without contraction.
__global__ void blend_kernel(const double* __restrict__ d, double* __restrict__ acc, int64_t n,
                             double w, int first) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double t = __dmul_rn(w, d[i]);
    acc[i] = first ? t : __dadd_rn(acc[i], t);
  }
}

// ------------------------------------------------------------- airlight ---
constexpr int kSelThreads = 256;
constexpr int kSelItems = 16;                       // elements per thread (compaction)
constexpr int kSelBlock = kSelThreads * kSelItems;  // elements per block

struct SelectState {
  unsigned long long prefix;
  unsigned long long mask;
  unsigned long long k;        // rank still to place inside the prefix (1-based)
  unsigned long long hist[256];
};

__global__ void select_init_kernel(SelectState* st, unsigned long long count) {
  st += blockIdx.x;  // one state per image of a batch
  const int t = threadIdx.x;
  if (t == 0) {
    st->prefix = 0;
    st->mask = 0;
    st->k = count;
  }
  st->hist[t] = 0;
}

__global__ void select_hist_kernel(const double* __restrict__ dark, int64_t n, SelectState* st,
                                   int shift) {
  __shared__ unsigned int sh[256];
  sh[threadIdx.x] = 0;
  dark += size_t(blockIdx.y) * n;
  st += blockIdx.y;
  __syncthreads();
  const unsigned long long prefix = st->prefix, mask = st->mask;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const unsigned long long key = f64_order_key(dark[i]);
    if ((key & mask) == prefix) atomicAdd(&sh[(key >> shift) & 255ull], 1u);
  }
  __syncthreads();
  if (sh[threadIdx.x]) atomicAdd(&st->hist[threadIdx.x], (unsigned long long)sh[threadIdx.x]);
}

// One block of 256 threads: pick the digit holding the k-th largest key.
__global__ void select_digit_kernel(SelectState* st, int shift) {
  __shared__ unsigned long long cnt[256];
  const int t = threadIdx.x;
  st += blockIdx.x;
  cnt[t] = st->hist[255 - t];  // descending digit order
  __syncthreads();
  if (t == 0) {
    unsigned long long above = 0, k = st->k;
    int d = 0;
    for (; d < 256; ++d) {
      if (above + cnt[d] >= k) break;
      above += cnt[d];
    }
    const unsigned long long digit = 255 - d;
    st->prefix |= digit << shift;
    st->mask |= 255ull << shift;
    st->k = k - above;
  }
  __syncthreads();
  st->hist[t] = 0;
}

// Per-block counts of keys above the threshold and equal to it.
__global__ void select_count_kernel(const double* __restrict__ dark, int64_t n,
                                    const SelectState* st, unsigned int* gt_cnt,
                                    unsigned int* eq_cnt) {
  dark += size_t(blockIdx.y) * n;
  st += blockIdx.y;
  gt_cnt += size_t(blockIdx.y) * gridDim.x;
  eq_cnt += size_t(blockIdx.y) * gridDim.x;
  const unsigned long long T = st->prefix;
  unsigned int gt = 0, eq = 0;
  const int64_t base = int64_t(blockIdx.x) * kSelBlock + int64_t(threadIdx.x) * kSelItems;
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    if (i < n) {
      const unsigned long long key = f64_order_key(dark[i]);
      gt += key > T;
      eq += key == T;
    }
  }
  __shared__ unsigned int sg[kSelThreads / 32], se[kSelThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    gt += __shfl_xor_sync(0xffffffffu, gt, o);
    eq += __shfl_xor_sync(0xffffffffu, eq, o);
  }
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    se[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int a = 0, b = 0;
    for (int w = 0; w < kSelThreads / 32; ++w) {
      a += sg[w];
      b += se[w];
    }
    gt_cnt[blockIdx.x] = a;
    eq_cnt[blockIdx.x] = b;
  }
}

// Exclusive scans of the per-block counts (single block, sequential chunks).
// Exclusive scan of the per-block counts, one block of 1024 threads: each
// thread scans a contiguous run, then the run totals are scanned across the
// block (integer sums: any order is exact).
__global__ void select_scan_kernel(unsigned int* gt_cnt, unsigned int* eq_cnt, int nblocks) {
  __shared__ unsigned int sg[1024], se[1024];
  gt_cnt += size_t(blockIdx.x) * nblocks;
  eq_cnt += size_t(blockIdx.x) * nblocks;
  const int t = threadIdx.x, nt = blockDim.x;
  const int per = (nblocks + nt - 1) / nt;
  const int lo = min(nblocks, t * per), hi = min(nblocks, lo + per);
  unsigned int a = 0, b = 0;
  for (int i = lo; i < hi; ++i) {
    a += gt_cnt[i];
    b += eq_cnt[i];
  }
  sg[t] = a;
  se[t] = b;
  __syncthreads();
  for (int o = 1; o < nt; o <<= 1) {  // Hillis-Steele inclusive scan
    const unsigned int xa = t >= o ? sg[t - o] : 0u, xb = t >= o ? se[t - o] : 0u;
    __syncthreads();
    sg[t] += xa;
    se[t] += xb;
    __syncthreads();
  }
  a = sg[t] - a;  // exclusive start of this thread's run
  b = se[t] - b;
  for (int i = lo; i < hi; ++i) {
    const unsigned int x = gt_cnt[i], y = eq_cnt[i];
    gt_cnt[i] = a;
    eq_cnt[i] = b;
    a += x;
    b += y;
  }
}

// Index-ordered compaction: keys > T in index order, then the first
// (k remaining) keys == T in index order.
__global__ void select_compact_kernel(const double* __restrict__ dark, int64_t n,
                                      const SelectState* st, const unsigned int* gt_off,
                                      const unsigned int* eq_off, unsigned long long count,
                                      unsigned long long* cand_key, int64_t* cand_idx) {
  dark += size_t(blockIdx.y) * n;
  st += blockIdx.y;
  gt_off += size_t(blockIdx.y) * gridDim.x;
  eq_off += size_t(blockIdx.y) * gridDim.x;
  cand_key += size_t(blockIdx.y) * count;
  cand_idx += size_t(blockIdx.y) * count;
  const unsigned long long T = st->prefix;
  const unsigned long long need_eq = st->k;
  const unsigned long long n_gt = count - need_eq;
  const int64_t base = int64_t(blockIdx.x) * kSelBlock + int64_t(threadIdx.x) * kSelItems;
  unsigned long long keys[kSelItems];
  unsigned int gt = 0, eq = 0;
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    keys[j] = i < n ? f64_order_key(dark[i]) : 0ull;
    gt += (i < n) && keys[j] > T;
    eq += (i < n) && keys[j] == T;
  }
  // block-wide exclusive scan of (gt, eq) in thread order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned int ig = gt, ie = eq;
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned int a = __shfl_up_sync(0xffffffffu, ig, o);
    const unsigned int b = __shfl_up_sync(0xffffffffu, ie, o);
    if (lane >= o) {
      ig += a;
      ie += b;
    }
  }
  __shared__ unsigned int wg[kSelThreads / 32], we[kSelThreads / 32];
  if (lane == 31) {
    wg[warp] = ig;
    we[warp] = ie;
  }
  __syncthreads();
  unsigned int pg = 0, pe = 0;
  for (int w = 0; w < warp; ++w) {
    pg += wg[w];
    pe += we[w];
  }
  unsigned long long og = gt_off[blockIdx.x] + pg + ig - gt;
  unsigned long long oe = eq_off[blockIdx.x] + pe + ie - eq;
  for (int j = 0; j < kSelItems; ++j) {
    const int64_t i = base + j;
    if (i >= n) break;
    if (keys[j] > T) {
      cand_key[og] = keys[j];
      cand_idx[og] = i;
      ++og;
    } else if (keys[j] == T) {
      if (oe < need_eq) {
        cand_key[n_gt + oe] = keys[j];
        cand_idx[n_gt + oe] = i;
      }
      ++oe;
    }
  }
}

// Rank of each candidate under (key desc, index asc) by counting; keys are
// unique once the index breaks ties, so ranks form a permutation.
// Rank sort of the m candidates by (key desc, index asc): 4 threads per
// candidate (adjacent lanes) each count a quarter of the comparisons; 64
// candidates per block of 256 threads.
__global__ void select_rank_kernel(const unsigned long long* __restrict__ cand_key,
                                   const int64_t* __restrict__ cand_idx, int64_t m,
                                   int64_t* __restrict__ sorted_idx) {
  __shared__ unsigned long long sk[256];
  __shared__ int64_t si[256];
  cand_key += size_t(blockIdx.y) * m;
  cand_idx += size_t(blockIdx.y) * m;
  sorted_idx += size_t(blockIdx.y) * m;
  const int q = threadIdx.x & 3;
  const int64_t i = int64_t(blockIdx.x) * 64 + (threadIdx.x >> 2);
  const unsigned long long ki = i < m ? cand_key[i] : 0ull;
  const int64_t ii = i < m ? cand_idx[i] : 0;
  int64_t rank = 0;
  for (int64_t j0 = 0; j0 < m; j0 += 256) {
    __syncthreads();
    if (j0 + threadIdx.x < m) {
      sk[threadIdx.x] = cand_key[j0 + threadIdx.x];
      si[threadIdx.x] = cand_idx[j0 + threadIdx.x];
    }
    __syncthreads();
    const int lim = int(m - j0 < 256 ? m - j0 : 256);
    for (int j = q; j < lim; j += 4) {
      const unsigned long long kj = sk[j];
      rank += (kj > ki) || (kj == ki && si[j] < ii);
    }
  }
  rank += __shfl_xor_sync(0xffffffffu, rank, 1);
  rank += __shfl_xor_sync(0xffffffffu, rank, 2);
  if (i < m && q == 0) sorted_idx[rank] = ii;
}

// A = mean of I over the selection, clipped to [0.05, 1] (scattering.py:106-107).
// numpy's picked.mean(axis=0) on the (n, C) gather adds row after row for C = 3
// but, for C = 1, reduces a contiguous axis with its pairwise summation
// (numpy _core/src/umath/loops_utils.h.src); both orders are reproduced.
template <typename T>
__global__ void airlight_gather_kernel(const void* __restrict__ img, int C,
                                       const int64_t* __restrict__ sorted_idx, int64_t m,
                                       double* __restrict__ vals, int64_t n) {
  sorted_idx += size_t(blockIdx.y) * m;
  vals += size_t(blockIdx.y) * 32 * m;
  const size_t ibase = size_t(blockIdx.y) * n * C;
  for (int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < m;
       j += int64_t(gridDim.x) * blockDim.x) {
    const size_t base = ibase + size_t(sorted_idx[j]) * C;
    for (int c = 0; c < C; ++c) vals[size_t(c) * m + j] = load_f64<T>(img, base + c);
  }
}

__device__ double pairwise_sum_dev(const double* a, int64_t n) {
  if (n < 8) {
    double res = 0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    const int64_t top = n - n % 8;
    for (int64_t i = 8; i < top; i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (int64_t i = top; i < n; ++i) res = __dadd_rn(res, a[i]);
    return res;
  }
  int64_t half = n / 2;
  half -= half % 8;
  return __dadd_rn(pairwise_sum_dev(a, half), pairwise_sum_dev(a + half, n - half));
}

// One block per channel; the sequential sum (C = 3) reads the values from
// shared memory, staged in chunks by the whole block (the order is kept).
__global__ void airlight_mean_kernel(const double* __restrict__ vals, int C, int64_t m,
                                     double* __restrict__ airlight) {
  constexpr int kChunk = 2048;
  __shared__ double sv[kChunk];
  const int c = blockIdx.x;
  vals += size_t(blockIdx.y) * 32 * m;
  airlight += size_t(blockIdx.y) * C;
  const double* v = vals + size_t(c) * m;
  double s = 0.0;
  if (C == 1) {
    if (threadIdx.x == 0) s = __dadd_rn(0.0, pairwise_sum_dev(v, m));
  } else {
    for (int64_t j0 = 0; j0 < m; j0 += kChunk) {
      const int cnt = int(m - j0 < kChunk ? m - j0 : kChunk);
      __syncthreads();
      for (int k = threadIdx.x; k < cnt; k += blockDim.x) sv[k] = v[j0 + k];
      __syncthreads();
      if (threadIdx.x == 0)
        for (int k = 0; k < cnt; ++k) s = __dadd_rn(s, sv[k]);
    }
  }
  if (threadIdx.x == 0) {
    const double mean = __ddiv_rn(s, double(m));
    airlight[c] = fmin(fmax(mean, 0.05), 1.0);
  }
}

static int64_t airlight_count(int H, int W, double fraction) {
  return static_cast<int64_t>(std::ceil(fraction * double(int64_t(H) * W)));
}

struct SelectLayout {
  SelectState* st;
  unsigned int* gt;
  unsigned int* eq;
  unsigned long long* ckey;
  int64_t* cidx;
  int64_t* sorted;
  double* vals;  // [C][m] gathered samples (C <= 32)
  size_t bytes;
};

static SelectLayout carve_select(int H, int W, double fraction, void* ws, size_t cap,
                                 int batch = 1) {
  Carver c(ws, cap);
  SelectLayout L;
  const int64_t n = int64_t(H) * W;
  const int64_t m = std::max<int64_t>(1, airlight_count(H, W, fraction));
  const int64_t nb = (n + kSelBlock - 1) / kSelBlock;
  const size_t B = size_t(batch);
  L.st = c.take<SelectState>(B);
  L.gt = c.take<unsigned int>(B * nb);
  L.eq = c.take<unsigned int>(B * nb);
  L.ckey = c.take<unsigned long long>(B * m);
  L.cidx = c.take<int64_t>(B * m);
  L.sorted = c.take<int64_t>(B * m);
  L.vals = c.take<double>(B * size_t(m) * 32);
  L.bytes = c.off;
  return L;
}

// ---------------------------------------------------------- t, Phi, lambda
__global__ void transmission_kernel(const double* __restrict__ dark, int64_t n, double omega,
                                    double* __restrict__ t) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    t[i] = __dsub_rn(1.0, __dmul_rn(omega, dark[i]));
}

template <typename T>
__global__ void fields_kernel(const void* __restrict__ img, int64_t n, int C,
                              const double* __restrict__ t, const double* __restrict__ airlight,
                              double t_floor, int mode, double lambda0, double beta,
                              float* __restrict__ phi, float* __restrict__ lam,
                              double* __restrict__ phi64) {
  const size_t z = blockIdx.y;  // image of a batch
  const size_t ibase = z * size_t(n) * C;
  t += z * size_t(n);
  airlight += z * C;
  if (phi) phi += z * size_t(n) * C;
  if (lam) lam += z * size_t(n);
  if (phi64) phi64 += z * size_t(n) * C;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double ti = t[i];
    const double one_minus_t = __dsub_rn(1.0, ti);
    const double denom = fmax(ti, t_floor);
    for (int c = 0; c < C; ++c) {
      const double v = __ddiv_rn(__dsub_rn(load_f64<T>(img, ibase + size_t(i) * C + c),
                                           __dmul_rn(airlight[c], one_minus_t)),
                                 denom);
      if (phi) phi[size_t(c) * n + i] = float(v);
      if (phi64) phi64[size_t(i) * C + c] = v;
    }
    if (!lam) continue;
    double l;
    switch (mode) {
      case PDZ_LAMBDA_AS_PRINTED: l = __dmul_rn(lambda0, exp(__dmul_rn(-beta, one_minus_t))); break;
      case PDZ_LAMBDA_PROSE: l = __dmul_rn(lambda0, exp(__dmul_rn(-beta, ti))); break;
      case PDZ_LAMBDA_ZERO: l = 0.0; break;
      default: l = lambda0; break;
    }
    lam[i] = float(l);
  }
}

// adaptive_lambda (solver.py:262-263) in float64.
__global__ void lambda_kernel(const double* __restrict__ t, int64_t n, int mode, double lambda0,
                              double beta, double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const double e = mode == PDZ_LAMBDA_PROSE ? t[i] : __dsub_rn(1.0, t[i]);
    out[i] = __dmul_rn(lambda0, exp(__dmul_rn(-beta, e)));
  }
}

// diffusion_coefficient (solver.py:152-164): 1 / (g + eps).
__global__ void dcoef_kernel(const double* __restrict__ g, int64_t n, double eps,
                             double* __restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    out[i] = __ddiv_rn(1.0, __dadd_rn(g[i], eps));
}

__global__ void clamp_interleave_kernel(const float* __restrict__ planes, int64_t n, int C,
                                        void* __restrict__ out, int out_f64) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    for (int c = 0; c < C; ++c) {
      const float v = fminf(fmaxf(planes[size_t(c) * n + i], 0.0f), 1.0f);
      if (out_f64)
        static_cast<double*>(out)[size_t(i) * C + c] = double(v);
      else
        static_cast<float*>(out)[size_t(i) * C + c] = v;
    }
  }
}

static int grid_for(int64_t n) {
  return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, int64_t(num_sms()) * 8)));
}

}  // namespace pdz

using namespace pdz;

extern "C" {

size_t pdz_dark_channel_workspace_bytes(int32_t height, int32_t width) {
  if (height < 1 || width < 1) return 0;
  return dark_ws(height, width);
}

int32_t pdz_dark_channel(const void* image, int32_t image_is_f64, int32_t height,
                         int32_t width, int32_t channels, const double* airlight,
                         int32_t radius, double* dark, void* workspace,
                         size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(image && airlight && dark, "NULL argument");
  PDZ_REQUIRE(height >= 1 && width >= 1 && channels >= 1, "bad image shape");
  PDZ_REQUIRE(radius >= 0, "patch_radius must be >= 0");
  Carver c(workspace, workspace_bytes);
  double* a = c.take<double>(size_t(height) * width);
  double* b = c.take<double>(size_t(height) * width);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  return dark_channel_impl(image, image_is_f64, height, width, channels, airlight, radius, dark,
                           a, b, as_stream(stream));
}

int32_t pdz_multiscale_dark_channel(const void* image, int32_t image_is_f64, int32_t height,
                                    int32_t width, int32_t channels, const double* airlight,
                                    const int32_t* radii_host, const double* weights_host,
                                    int32_t n_radii, double* dark, void* workspace,
                                    size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(image && airlight && dark && radii_host && weights_host, "NULL argument");
  PDZ_REQUIRE(n_radii >= 1, "radii must be nonempty");
  PDZ_REQUIRE(height >= 1 && width >= 1 && channels >= 1, "bad image shape");
  Carver c(workspace, workspace_bytes);
  double* a = c.take<double>(size_t(height) * width);
  double* b = c.take<double>(size_t(height) * width);
  double* d = c.take<double>(size_t(height) * width);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  const int64_t n = int64_t(height) * width;
  for (int k = 0; k < n_radii; ++k) {
    PDZ_REQUIRE(radii_host[k] >= 0, "patch_radius must be >= 0");
    int32_t rc = dark_channel_impl(image, image_is_f64, height, width, channels, airlight,
                                   radii_host[k], d, a, b, s);
    if (rc != PDZ_OK) return rc;
    blend_kernel<<<grid_for(n), 256, 0, s>>>(d, dark, n, weights_host[k], k == 0);
    PDZ_CHECK_LAUNCH("blend");
  }
  return PDZ_OK;
}

int64_t pdz_airlight_count(int32_t height, int32_t width, double fraction) {
  return airlight_count(height, width, fraction);
}

size_t pdz_airlight_workspace_bytes(int32_t height, int32_t width, double fraction) {
  if (height < 1 || width < 1) return 0;
  return Carver::round(carve_select(height, width, fraction, nullptr, 0).bytes);
}

// A of `batch` images (dark: [batch][H][W], airlight out: [batch][C]).
static int32_t airlight_impl(const void* image, int is_f64, int H, int W, int C,
                             const double* dark, double fraction, double* airlight,
                             const SelectLayout& L, cudaStream_t s, int batch) {
  const int64_t n = int64_t(H) * W;
  const int64_t m = airlight_count(H, W, fraction);
  PDZ_REQUIRE(m >= 1 && m <= n, "airlight count %lld out of range", (long long)m);
  select_init_kernel<<<batch, 256, 0, s>>>(L.st, (unsigned long long)m);
  const int hist_gx = std::max(1, grid_for(n) / std::min(batch, 8));
  for (int pass = 7; pass >= 0; --pass) {
    select_hist_kernel<<<dim3(hist_gx, batch), 256, 0, s>>>(dark, n, L.st, pass * 8);
    select_digit_kernel<<<batch, 256, 0, s>>>(L.st, pass * 8);
  }
  PDZ_CHECK_LAUNCH("radix select");
  const int nb = int((n + kSelBlock - 1) / kSelBlock);
  select_count_kernel<<<dim3(nb, batch), kSelThreads, 0, s>>>(dark, n, L.st, L.gt, L.eq);
  select_scan_kernel<<<batch, 1024, 0, s>>>(L.gt, L.eq, nb);
  select_compact_kernel<<<dim3(nb, batch), kSelThreads, 0, s>>>(
      dark, n, L.st, L.gt, L.eq, (unsigned long long)m, L.ckey, L.cidx);
  select_rank_kernel<<<dim3(int((m + 63) / 64), batch), 256, 0, s>>>(L.ckey, L.cidx, m, L.sorted);
  const dim3 gg(grid_for(m), batch);
  if (is_f64)
    airlight_gather_kernel<double><<<gg, 256, 0, s>>>(image, C, L.sorted, m, L.vals, n);
  else
    airlight_gather_kernel<float><<<gg, 256, 0, s>>>(image, C, L.sorted, m, L.vals, n);
  airlight_mean_kernel<<<dim3(C, batch), 256, 0, s>>>(L.vals, C, m, airlight);
  PDZ_CHECK_LAUNCH("airlight");
  return PDZ_OK;
}

int32_t pdz_atmospheric_light(const void* image, int32_t image_is_f64, int32_t height,
                              int32_t width, int32_t channels, const double* dark,
                              double fraction, double* airlight, int64_t* picked,
                              void* workspace, size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(image && dark && airlight, "NULL argument");
  PDZ_REQUIRE(height >= 1 && width >= 1 && channels >= 1 && channels <= 32, "bad image shape");
  PDZ_REQUIRE(fraction > 0.0 && fraction <= 1.0, "fraction must lie in (0, 1]");
  SelectLayout L = carve_select(height, width, fraction, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  const int32_t rc = airlight_impl(image, image_is_f64, height, width, channels, dark, fraction,
                                   airlight, L, s, 1);
  if (rc != PDZ_OK) return rc;
  if (picked)
    PDZ_CUDA(cudaMemcpyAsync(picked, L.sorted,
                             size_t(airlight_count(height, width, fraction)) * 8,
                             cudaMemcpyDeviceToDevice, s),
             "picked copy");
  return PDZ_OK;
}

__global__ void fill_f64_kernel(double* p, int n, double v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

// Workspace of the batched front end: three [batch][H][W] double planes
// (dark + the two min-filter scratch planes), a [C] vector of ones, one more
// plane for the multiscale blend, and the batched selection state.
struct FrontLayout {
  double *dark, *ta, *tb, *blend, *ones;
  SelectLayout sel;
  size_t bytes;
};
static FrontLayout carve_front(int B, int H, int W, int n_radii, double fraction, void* ws,
                               size_t cap) {
  Carver c(ws, cap);
  FrontLayout F;
  const size_t n = size_t(B) * H * W;
  F.dark = c.take<double>(n);
  F.ta = c.take<double>(n);
  F.tb = c.take<double>(n);
  F.blend = n_radii > 1 ? c.take<double>(n) : nullptr;
  F.ones = c.take<double>(32);
  const size_t head = Carver::round(c.off);
  F.sel = carve_select(H, W, fraction, ws ? static_cast<char*>(ws) + head : nullptr,
                       cap > head ? cap - head : 0, B);
  F.bytes = head + Carver::round(F.sel.bytes);
  return F;
}

size_t pdz_front_end_batch_workspace_bytes(int32_t batch, int32_t height, int32_t width,
                                           int32_t n_radii, double fraction) {
  if (batch < 1 || height < 1 || width < 1) return 0;
  return carve_front(batch, height, width, n_radii, fraction, nullptr, 0).bytes;
}

int32_t pdz_front_end_batch(const void* images, int32_t image_is_f64, int32_t batch,
                            int32_t height, int32_t width, int32_t channels,
                            const int32_t* radii_host, const double* weights_host,
                            int32_t n_radii, double fraction, double omega, double t_floor,
                            int32_t lambda_mode, double lambda0, double beta, double* airlight,
                            double* transmission, float* phi, float* lambda_map, double* phi64,
                            void* workspace, size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(images && radii_host && weights_host && airlight && transmission, "NULL argument");
  PDZ_REQUIRE(batch >= 1 && batch <= 65535, "batch must lie in [1, 65535], got %d", batch);
  PDZ_REQUIRE(height >= 1 && width >= 1 && channels >= 1 && channels <= 32, "bad image shape");
  PDZ_REQUIRE(n_radii >= 1, "radii must be nonempty");
  PDZ_REQUIRE(fraction > 0.0 && fraction <= 1.0, "fraction must lie in (0, 1]");
  PDZ_REQUIRE(omega > 0.0 && omega <= 1.0, "omega must lie in (0, 1]");
  PDZ_REQUIRE(t_floor > 0.0, "t_floor must be > 0");
  PDZ_REQUIRE(lambda_mode >= 0 && lambda_mode <= 3, "bad lambda_mode %d", lambda_mode);
  for (int k = 0; k < n_radii; ++k) PDZ_REQUIRE(radii_host[k] >= 0, "patch_radius must be >= 0");
  FrontLayout F = carve_front(batch, height, width, n_radii, fraction, workspace, workspace_bytes);
  if (workspace == nullptr || F.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", F.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  const int64_t n = int64_t(height) * width, nall = n * batch;
  fill_f64_kernel<<<1, 32, 0, s>>>(F.ones, 32, 1.0);
  // (multiscale_)dark_channel of every image for a per-image or shared A
  auto dark_of = [&](const double* a, int a_stride) -> int32_t {
    if (n_radii == 1 && weights_host[0] == 1.0)
      return dark_channel_impl(images, image_is_f64, height, width, channels, a, radii_host[0],
                               F.dark, F.ta, F.tb, s, batch, a_stride);
    for (int k = 0; k < n_radii; ++k) {
      const int32_t rc = dark_channel_impl(images, image_is_f64, height, width, channels, a,
                                           radii_host[k], F.blend, F.ta, F.tb, s, batch,
                                           a_stride);
      if (rc != PDZ_OK) return rc;
      blend_kernel<<<grid_for(nall), 256, 0, s>>>(F.blend, F.dark, nall, weights_host[k], k == 0);
      PDZ_CHECK_LAUNCH("blend");
    }
    return PDZ_OK;
  };
  int32_t rc = dark_of(F.ones, 0);  // scattering.py:88-107 works on the A = 1 dark channel
  if (rc != PDZ_OK) return rc;
  rc = airlight_impl(images, image_is_f64, height, width, channels, F.dark, fraction, airlight,
                     F.sel, s, batch);
  if (rc != PDZ_OK) return rc;
  rc = dark_of(airlight, channels);
  if (rc != PDZ_OK) return rc;
  transmission_kernel<<<grid_for(nall), 256, 0, s>>>(F.dark, nall, omega, transmission);
  PDZ_CHECK_LAUNCH("transmission");
  if (phi || lambda_map || phi64) {
    const dim3 grid(std::max(1, grid_for(n) / std::min<int>(batch, 8)), batch);
    if (image_is_f64)
      fields_kernel<double><<<grid, 256, 0, s>>>(images, n, channels, transmission, airlight,
                                                 t_floor, lambda_mode, lambda0, beta, phi,
                                                 lambda_map, phi64);
    else
      fields_kernel<float><<<grid, 256, 0, s>>>(images, n, channels, transmission, airlight,
                                                t_floor, lambda_mode, lambda0, beta, phi,
                                                lambda_map, phi64);
    PDZ_CHECK_LAUNCH("solver fields");
  }
  return PDZ_OK;
}

int32_t pdz_transmission(const double* dark, int32_t height, int32_t width, double omega,
                         double* transmission, void* stream) {
  PDZ_REQUIRE(dark && transmission, "NULL argument");
  PDZ_REQUIRE(omega > 0.0 && omega <= 1.0, "omega must lie in (0, 1]");
  const int64_t n = int64_t(height) * width;
  transmission_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(dark, n, omega, transmission);
  PDZ_CHECK_LAUNCH("transmission");
  return PDZ_OK;
}

int32_t pdz_solver_fields(const void* image, int32_t image_is_f64, int32_t height,
                          int32_t width, int32_t channels, const double* transmission,
                          const double* airlight, double t_floor, int32_t lambda_mode,
                          double lambda0, double beta, float* phi, float* lambda_map,
                          double* phi64, void* stream) {
  PDZ_REQUIRE(image && transmission && airlight, "NULL argument");
  PDZ_REQUIRE(phi || lambda_map || phi64, "no output requested");
  PDZ_REQUIRE(t_floor > 0.0, "t_floor must be > 0");
  PDZ_REQUIRE(lambda_mode >= 0 && lambda_mode <= 3, "bad lambda_mode %d", lambda_mode);
  const int64_t n = int64_t(height) * width;
  cudaStream_t s = as_stream(stream);
  if (image_is_f64)
    fields_kernel<double><<<grid_for(n), 256, 0, s>>>(image, n, channels, transmission, airlight,
                                                      t_floor, lambda_mode, lambda0, beta, phi,
                                                      lambda_map, phi64);
  else
    fields_kernel<float><<<grid_for(n), 256, 0, s>>>(image, n, channels, transmission, airlight,
                                                     t_floor, lambda_mode, lambda0, beta, phi,
                                                     lambda_map, phi64);
  PDZ_CHECK_LAUNCH("solver fields");
  return PDZ_OK;
}

int32_t pdz_adaptive_lambda(const double* transmission, int64_t n, int32_t mode,
                            double lambda0, double beta, double* out, void* stream) {
  PDZ_REQUIRE(transmission && out, "NULL argument");
  PDZ_REQUIRE(mode == PDZ_LAMBDA_AS_PRINTED || mode == PDZ_LAMBDA_PROSE, "bad mode %d", mode);
  if (n <= 0) return PDZ_OK;
  lambda_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(transmission, n, mode, lambda0,
                                                             beta, out);
  PDZ_CHECK_LAUNCH("adaptive lambda");
  return PDZ_OK;
}

int32_t pdz_diffusion_coefficient(const double* grad_magnitude, int64_t n, double epsilon,
                                  double* out, void* stream) {
  PDZ_REQUIRE(grad_magnitude && out, "NULL argument");
  PDZ_REQUIRE(epsilon > 0.0, "epsilon must be > 0");
  if (n <= 0) return PDZ_OK;
  dcoef_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(grad_magnitude, n, epsilon, out);
  PDZ_CHECK_LAUNCH("diffusion coefficient");
  return PDZ_OK;
}

int32_t pdz_clamp_interleave(const float* planes, int32_t height, int32_t width,
                             int32_t channels, void* out, int32_t out_is_f64, void* stream) {
  PDZ_REQUIRE(planes && out, "NULL argument");
  const int64_t n = int64_t(height) * width;
  clamp_interleave_kernel<<<grid_for(n), 256, 0, as_stream(stream)>>>(planes, n, channels, out,
                                                                      out_is_f64);
  PDZ_CHECK_LAUNCH("clamp");
  return PDZ_OK;
}

}  // extern "C"
