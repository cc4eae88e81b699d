// The relaxed fixed-point sweep -- the hot kernel of the dehazing solve.
//
// One launch = one iteration of fixed_point_solve (solver.py:343-358) for all
// P planes: for every pixel of every plane
//     r  = div(D(grad u) grad u) - lambda * G(u) + Phi        (solver.py:296-300)
//     u' = u + tau * r                                        (solver.py:302)
// plus the per-plane partial sums of r^2 (solver.py:301) and a non-finite flag
// (solver.py:347).  The divergence uses the reference's face discretisation
// (_face_fluxes, solver.py:167-187; divergence_term, :190-210); G is the
// normalised sampled Gaussian with symmetric (edge-inclusive, repeated)
// reflection at the borders (gaussian_convolve, :225-241), applied separably.
//
// Layout: planar float32 [P][H][W]; lambda [P/C][H][W]; ping-pong iterate
// buffers (iteration n reads buf[(n-1)&1], writes buf[n&1]).
//
// Norm reduction is deterministic: every CTA writes one float64 partial per
// iteration; block (0,0,0) of sweep n reduces iteration n-1's partials in a
// fixed order (lane-strided sums + xor tree), applies the stop rule
// (solver.py:353-357) and freezes planes that stopped.  A plane that stops at
// iteration m is still swept (harmlessly, into the other buffer) at m+1 and
// skipped from m+2 on, so its answer in buf[m&1] is never overwritten.
#include <algorithm>
#include <cstdio>
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include <cudaTypedefs.h>

#include "pdz_solver.cuh"
#include "pdz_stream.cuh"

namespace pdz {

constexpr int kTW = 32;           // tile width  (one warp of columns)
constexpr int kTH = 64;           // tile height
constexpr int kThreads = 256;     // 8 warps
constexpr int kRowsPerWarp = kTH / (kThreads / 32);

struct SweepArgs {
  float* buf0;
  float* buf1;
  const float* phi;
  const float* lam;
  Partials pt;           // [2][P][nblk] (tiles = nblk)
  StateView st;          // st.stop_iter == nullptr: single step, no stop rule
  int32_t H, W, P, C, R;
  int32_t tiles_x, nblk;
  int32_t iter_off;      // iteration = (*st.iter_base if set) + iter_off
  int32_t max_iters;
  // Row slab of a larger image (pdz_fixed_point_step_rows): array row y is
  // global row y + y_off of an H_glob-row image; only rows [row_lo, row_hi)
  // are written and counted in the norms.  Whole image: 0, H, 0, H.
  int32_t y_off, H_glob, row_lo, row_hi;
  int32_t cnt_lo, cnt_hi;  // rows counted in the norms (within the row window)
  float eps, tau;
  double rel_tol;
  float w[kMaxTaps];     // 1-D Gaussian taps (kernel params -> constant bank)
};

// ------------------------------------------------------------------------
// Face flux D * jump with D = 1 / (sqrt(jump^2 + along^2) + eps)
// (solver.py:182-187); EDGE == false is the "no-edge" ablation (D == 1).
template <bool EDGE>
__device__ __forceinline__ float face_flux(float jump, float along, float eps) {
  if (!EDGE) return jump;
  const float g = sqrtf(fmaf(jump, jump, along * along));
  return __fdiv_rn(jump, g + eps);
}

// ------------------------------------------------------------------------
// The fused sweep.  RT = compile-time radius (K = 2 RT + 1) or -1 (runtime).
template <int RT, bool EDGE>
__global__ void __launch_bounds__(kThreads) sweep_kernel(const SweepArgs a) {
  extern __shared__ float smem[];
  const int R = RT >= 0 ? RT : a.R;
  const int SH = kTH + 2 * R;
  const int SW = kTW + 2 * R;
  const int PU = SW + 1;  // odd pitch: conflict-free row-group access
  float* s_u = smem;                  // [SH][PU] iterate tile + halo
  float* s_h = smem + ((SH * PU + 3) & ~3);  // [SH][kTW] horizontally blurred rows (16B aligned)
  __shared__ double s_red[kThreads / 32];
  __shared__ int s_nf[kThreads / 32];

  const int tid = threadIdx.x;
  const int p = blockIdx.z;
  const int x0 = blockIdx.x * kTW, y0 = blockIdx.y * kTH;
  const int H = a.H, W = a.W;
  const int blk = blockIdx.y * gridDim.x + blockIdx.x;

  pdl_wait();
  const int iter = (a.st.iter_base ? a.st.iter_base[0] : 0) + a.iter_off;
  if (iter > a.max_iters) return;
  if (a.st.stop_iter) {
    if (iter >= 2 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 &&
        threadIdx.x < 32)
      finalize_iteration_warp(a.st, a.pt, a.P, iter - 1, a.max_iters, a.rel_tol);
    const int s = a.st.stop_iter[p];
    if (s != 0 && s < iter - 1) return;  // stopped at <= iter-2: frozen
  }

  const size_t plane = size_t(H) * W;
  const float* __restrict__ uin = (((iter - 1) & 1) ? a.buf1 : a.buf0) + p * plane;
  float* __restrict__ uout = ((iter & 1) ? a.buf1 : a.buf0) + p * plane;
  const float* __restrict__ phi = a.phi + p * plane;
  const float* __restrict__ lam = a.lam + (p / a.C) * plane;

  // ---- 1. iterate tile + halo -> smem (symmetric reflection at borders)
  const bool interior = (x0 - R >= 0) && (y0 - R >= 0) && (x0 + kTW + R <= W) &&
                        (y0 + kTH + R <= H);
  if (interior) {
    const float* src = uin + size_t(y0 - R) * W + (x0 - R);
    for (int i = tid; i < SH * SW; i += kThreads) {
      const int r = i / SW, c = i - r * SW;
      s_u[r * PU + c] = src[size_t(r) * W + c];
    }
  } else {
    for (int i = tid; i < SH * SW; i += kThreads) {
      const int r = i / SW, c = i - r * SW;
      const int gy = reflect(y0 - R + r, H), gx = reflect(x0 - R + c, W);
      s_u[r * PU + c] = uin[size_t(gy) * W + gx];
    }
  }
  __syncthreads();

  // ---- 2. horizontal Gaussian pass: 4 adjacent outputs per item
  for (int item = tid; item < SH * (kTW / 4); item += kThreads) {
    const int r = item / (kTW / 4), g = item % (kTW / 4);
    const float* row = s_u + r * PU + 4 * g;
    float c0 = 0.f, c1 = 0.f, c2 = 0.f, c3 = 0.f;
    if (RT >= 0) {
      constexpr int NV = 4 + 2 * (RT >= 0 ? RT : 0);
      float v[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = row[k];
#pragma unroll
      for (int k = 0; k <= 2 * (RT >= 0 ? RT : 0); ++k) {
        const float wk = a.w[k];
        c0 = fmaf(wk, v[k], c0);
        c1 = fmaf(wk, v[k + 1], c1);
        c2 = fmaf(wk, v[k + 2], c2);
        c3 = fmaf(wk, v[k + 3], c3);
      }
    } else {
      for (int k = 0; k <= 2 * R; ++k) {
        const float wk = a.w[k];
        c0 = fmaf(wk, row[k], c0);
        c1 = fmaf(wk, row[k + 1], c1);
        c2 = fmaf(wk, row[k + 2], c2);
        c3 = fmaf(wk, row[k + 3], c3);
      }
    }
    *reinterpret_cast<float4*>(s_h + r * kTW + 4 * g) = make_float4(c0, c1, c2, c3);
  }
  __syncthreads();

  // ---- 3. vertical pass, divergence, residual, update (8 rows per thread)
  const int lane = tid & 31, warp = tid >> 5;
  const int j0 = warp * kRowsPerWarp;
  float G[kRowsPerWarp];
  if (RT >= 0) {
    constexpr int NV = kRowsPerWarp + 2 * (RT >= 0 ? RT : 0);
    float hv[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) hv[k] = s_h[(j0 + k) * kTW + lane];
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; ++j) {
      float acc = 0.f;
#pragma unroll
      for (int k = 0; k <= 2 * (RT >= 0 ? RT : 0); ++k) acc = fmaf(a.w[k], hv[j + k], acc);
      G[j] = acc;
    }
  } else {
#pragma unroll
    for (int j = 0; j < kRowsPerWarp; ++j) {
      float acc = 0.f;
      for (int k = 0; k <= 2 * R; ++k) acc = fmaf(a.w[k], s_h[(j0 + j + k) * kTW + lane], acc);
      G[j] = acc;
    }
  }

  // 10 x 3 patch of u around the thread's 8 output rows (rows j0-1 .. j0+8)
  float U[kRowsPerWarp + 2][3];
#pragma unroll
  for (int i = 0; i < kRowsPerWarp + 2; ++i)
#pragma unroll
    for (int d = 0; d < 3; ++d) U[i][d] = s_u[(R + j0 - 1 + i) * PU + (R + lane - 1 + d)];

  const int gx = x0 + lane;
  // np.gradient: centred (f[i+1]-f[i-1])/2 inside, one-sided at the ends.
  // With the symmetric halo the one-sided difference is f[i+1]-f[i-1] at
  // the border (the mirrored sample equals the edge sample), so only the
  // 0.5 factor depends on the position.
  const float sx = (gx == 0 || gx == W - 1) ? 1.0f : 0.5f;
  float cx[kRowsPerWarp + 2];
#pragma unroll
  for (int i = 0; i < kRowsPerWarp + 2; ++i) cx[i] = sx * (U[i][2] - U[i][0]);

  double acc2 = 0.0;
  int nf = 0;
  float fs_up = face_flux<EDGE>(U[1][1] - U[0][1], 0.5f * (cx[0] + cx[1]), a.eps);
#pragma unroll
  for (int j = 0; j < kRowsPerWarp; ++j) {
    const int gy = y0 + j0 + j;
    const int yg = gy + a.y_off;  // global row (np.gradient ends: solver.py:178-179)
    const float sy = (yg == 0 || yg == a.H_glob - 1) ? 1.0f : 0.5f;
    const float cy0 = sy * (U[j + 2][0] - U[j][0]);
    const float cy1 = sy * (U[j + 2][1] - U[j][1]);
    const float cy2 = sy * (U[j + 2][2] - U[j][2]);
    const float fe_r = face_flux<EDGE>(U[j + 1][2] - U[j + 1][1], 0.5f * (cy1 + cy2), a.eps);
    const float fe_l = face_flux<EDGE>(U[j + 1][1] - U[j + 1][0], 0.5f * (cy0 + cy1), a.eps);
    const float fs_dn =
        face_flux<EDGE>(U[j + 2][1] - U[j + 1][1], 0.5f * (cx[j + 1] + cx[j + 2]), a.eps);
    const float div = ((fe_r - fe_l) + fs_dn) - fs_up;
    fs_up = fs_dn;
    if (gy >= a.row_lo && gy < a.row_hi && gx < W) {
      const size_t off = size_t(gy) * W + gx;
      const float r = fmaf(-lam[off], G[j], div) + phi[off];
      const float un = fmaf(a.tau, r, U[j + 1][1]);
      uout[off] = un;
      if (gy >= a.cnt_lo && gy < a.cnt_hi) {
        acc2 = fma(double(r), double(r), acc2);
        nf |= !(isfinite(r) && isfinite(un));
      }
    }
  }

  // ---- 4. deterministic block partial of sum r^2
  acc2 = warp_sum(acc2);
  nf = __any_sync(0xffffffffu, nf);
  if (lane == 0) {
    s_red[warp] = acc2;
    s_nf[warp] = nf;
  }
  __syncthreads();
  if (tid == 0) {
    double s = 0.0;
    int f = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) {
      s += s_red[w];
      f |= s_nf[w];
    }
    const size_t slot = (size_t(iter & 1) * a.P + p) * a.pt.nbmax + blk;
    a.pt.sum[slot] = s;
    a.pt.flag[slot] = f;
  }
  pdl_launch_dependents();
}

__global__ void finalize_kernel(StateView st, Partials pt, int P, int it, int max_iters,
                                double rel_tol) {
  pdl_wait();
  if (threadIdx.x < 32) finalize_iteration_warp(st, pt, P, it, max_iters, rel_tol);
}

// Chunk prologue: iter_base = chunk * kChunk + 1.
__global__ void chunk_base_kernel(StateView st) {
  pdl_wait();
  const int c = st.chunk_ctr[0];
  st.iter_base[0] = c * kChunk + 1;
  st.chunk_ctr[0] = c + 1;
  pdl_launch_dependents();
}

// Solve state and (G > 0: the persistent kernel) its progress counters.
__global__ void init_state_kernel(StateView st, int P, int32_t* done = nullptr,
                                  int32_t* fin = nullptr, int32_t* flags = nullptr, int G = 0) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < G) done[p] = 0;
  if (p == 0 && G > 0) {
    fin[0] = 0;
    flags[0] = 0;
    flags[1] = 0;
  }
  if (p < P) {
    st.stop_iter[p] = 0;
    st.converged[p] = 0;
    st.failed[p] = 0;
    st.iters[p] = 0;
    st.prev_norm[p] = 0.0;
  }
  if (p == 0) {
    st.running[0] = P;
    st.iter_base[0] = 1;
    st.chunk_ctr[0] = 0;
  }
}

// Single fixed_point_step: norms[p] = sqrt(sum of the iteration-1 partials).
__global__ void step_norm_kernel(Partials pt, int P, double* norms, int32_t* nonfinite,
                                 int take_sqrt) {
  for (int p = threadIdx.x; p < P; p += blockDim.x) {
    const size_t base = (size_t(1 % pt.ring) * P + p) * pt.nbmax;
    const int n = partial_count(pt, p);
    double s = 0.0;
    int nf = 0;
    for (int b = 0; b < n; ++b) {
      s += pt.sum[base + b];
      nf |= pt.flag[base + b];
    }
    norms[p] = take_sqrt ? sqrt(s) : s;
    if (nonfinite) nonfinite[p] = nf;
  }
}

// ------------------------------------------------------------------------
// host side

using SweepFn = void (*)(const SweepArgs);

static size_t tile_smem(int R) {
  return size_t(((kTH + 2 * R) * (kTW + 2 * R + 1) + 3 + (kTH + 2 * R) * kTW)) * 4;
}

template <int RT, bool EDGE>
static SweepFn prepared() {
  static std::atomic<uint64_t> done{0};
  if (first_use_on_device(&done))
    cudaFuncSetAttribute(sweep_kernel<RT, EDGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(tile_smem(RT >= 0 ? RT : kMaxFusedRadius)));
  return sweep_kernel<RT, EDGE>;
}

template <bool EDGE>
static SweepFn pick_kernel(int R) {
  switch (R) {
    case 1: return prepared<1, EDGE>();
    case 2: return prepared<2, EDGE>();
    case 3: return prepared<3, EDGE>();
    case 6: return prepared<6, EDGE>();
    case 9: return prepared<9, EDGE>();
    case 12: return prepared<12, EDGE>();
    case 24: return prepared<24, EDGE>();
    default: return prepared<-1, EDGE>();
  }
}

// How a solve is launched: the persistent streaming kernel (width % 4 == 0,
// a compiled radius, S < 2^31) as one cooperative launch, or the tiled
// fallback as graph-replayed per-sweep launches.
struct Plan {
  bool stream = false;
  int R = 1;       // radius the kernel runs (persistent: a compiled radius >= R_taps)
  int R_taps = 1;  // K / 2 of the Gaussian (>= 1)
  int tiles_x = 0, tiles_y = 0, nblk = 0;  // tiled
  int G = 0, nstrips = 0;                   // streaming
  int kps = 0, bonus = 0;                   // per-strip partition (Partials)
  int64_t S = 0, U = 0;
  int nbmax = 0;                            // partial slots per plane
  int pad_r = 0, pad_c = 0;                 // iterate buffer pads (rows, columns)
  int ring = 2;                             // iteration slots of the partials
  int geo = 0;                              // block geometry V (pdz_stream.cuh)
  int ci = 0;                               // channel-inner block order (pdz_stream.cuh)
  size_t smem = 0;
  void* fn = nullptr;
};

static int g_force_tiled = -1;

// Critical-path cost of a persistent partition: every CTA runs each pass over
// its strip segments in blocks of `srb` rows (srb1: the taller geometry, used
// when a segment needs several blocks; 0 = unavailable), each block staging
// 2R halo rows; the slowest CTA sets the sweep time.  Returns the largest
// per-CTA cost in staged rows and the longest segment.
static void partition_cost(const Partials& q, int R, int srb0, int srb1, int64_t* cost,
                           int64_t* max_seg) {
  int64_t worst = 0, mseg = 0;
  for (int64_t i = 0; i < q.G; ++i) {
    const int64_t L0 = part_start(q, i), L1 = part_start(q, i + 1);
    for (int64_t L = L0; L < L1;) {
      const int64_t e = std::min<int64_t>(L1, (L / q.H + 1) * q.H);
      mseg = std::max(mseg, e - L);
      L = e;
    }
  }
  const int64_t srb = (mseg > srb0 && srb1 > 0) ? srb1 : srb0;
  for (int64_t i = 0; i < q.G; ++i) {
    const int64_t L0 = part_start(q, i), L1 = part_start(q, i + 1);
    int64_t c = 0;
    for (int64_t L = L0; L < L1;) {
      const int64_t e = std::min<int64_t>(L1, (L / q.H + 1) * q.H);
      c += (e - L) + 2 * R * ((e - L + srb - 1) / srb);
      L = e;
    }
    worst = std::max(worst, c);
  }
  *cost = worst;
  *max_seg = mseg;
}
#ifdef PDZ_PROFILE
static long long* g_prof = nullptr;  // tools/prof_stream.py
#endif  // PDZ_FORCE_TILED=1 -> always the tiled kernel

static int32_t check_params(const pdz_solve_params* p, Plan* pl, bool allow_stream = true) {
  PDZ_REQUIRE(p != nullptr, "params is NULL");
  PDZ_REQUIRE(p->height >= 2 && p->width >= 2, "field must be at least 2x2, got (%d, %d)",
              p->height, p->width);
  PDZ_REQUIRE(p->planes >= 1 && p->channels >= 1 && p->planes % p->channels == 0,
              "planes (%d) must be a positive multiple of channels (%d)", p->planes,
              p->channels);
  PDZ_REQUIRE(p->kernel_size >= 1 && p->kernel_size % 2 == 1,
              "kernel_size must be odd and >= 1, got %d", p->kernel_size);
  PDZ_REQUIRE(p->kernel_size <= kMaxTaps, "kernel_size %d exceeds the fused limit %d",
              p->kernel_size, kMaxTaps);
  PDZ_REQUIRE(p->sigma > 0.0, "sigma must be > 0");
  PDZ_REQUIRE(p->epsilon > 0.0, "epsilon must be > 0");
  PDZ_REQUIRE(p->max_iters >= 1, "max_iters must be >= 1");
  PDZ_REQUIRE(std::isfinite(p->tau), "tau must be finite");
  if (!pl) return PDZ_OK;
  if (g_force_tiled < 0) {
    const char* e = getenv("PDZ_FORCE_TILED");
    g_force_tiled = (e && e[0] == '1') ? 1 : 0;
  }
  Plan& P = *pl;
  P.R = P.R_taps = std::max(1, p->kernel_size / 2);
  const bool edge = p->edge_preserving != 0;
  size_t smem = 0;
  StreamFn sfn = nullptr;
  const int64_t images = p->planes / p->channels;
  const int64_t strip_rows = int64_t((p->width + kSTW - 1) / kSTW) * p->height * images;
  // The persistent kernel is compiled for a set of radii; any other odd K
  // runs on the next compiled radius with its taps centred between zeros
  // (a zero tap times a finite staged value adds an exact 0, and the border
  // reflection of the wider kernel only feeds zero taps), so every K <= 49
  // takes the fast path (solver.py:225-241 accepts any odd K).
  const int rc = stream_compiled_radius(P.R);
  const int rp = (rc + 3) & ~3;
  if (allow_stream && !g_force_tiled && rc > 0 && p->width % 4 == 0 && p->height >= 2 * rc &&
      p->width >= 2 * rp &&
      strip_rows + p->height < (int64_t(1) << 31)) {
    sfn = edge ? stream_pick<true>(rc, 0, p->rel_tol >= 0.0, &smem)
               : stream_pick<false>(rc, 0, p->rel_tol >= 0.0, &smem);
    if (sfn) P.R = rc;
  }
  int occ = 0;
  if (sfn) {
    const cudaError_t e =
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, sfn, geo_threads(0), smem);
    if (getenv("PDZ_VERBOSE")) {
      cudaFuncAttributes fa = {};
      cudaFuncGetAttributes(&fa, sfn);
      fprintf(stderr,
              "pdz: persistent kernel R=%d smem=%zu occupancy=%d (%s) regs=%d maxthreads=%d "
              "static=%zu maxdyn=%d\n",
              P.R, smem, occ, cudaGetErrorString(e), fa.numRegs, fa.maxThreadsPerBlock,
              fa.sharedSizeBytes, fa.maxDynamicSharedSizeBytes);
    }
  }
  if (!(sfn && int64_t(num_sms()) * occ >= 2)) P.R = P.R_taps;  // tiled kernel: the true radius
  if (sfn && int64_t(num_sms()) * occ >= 2) {
    P.stream = true;
    P.pad_r = P.R;
    P.pad_c = kPadC;
    P.fn = reinterpret_cast<void*>(sfn);
    P.smem = smem;
    P.ring = kRing;
    P.nstrips = (p->width + kSTW - 1) / kSTW;
    P.U = int64_t(P.nstrips) * p->height;  // strip-rows per image
    P.S = P.U * images;                    // the C channels share each range
    // Grid size: all CTAs co-resident (cooperative), and CTA ranges aligned to
    // strip boundaries so every CTA pays the same segment-start halo: k CTAs
    // per strip when strips are fewer than slots, else ~equal strips per CTA.
    const int64_t gmax = int64_t(num_sms()) * occ - 1;  // + 1 finaliser CTA
    const int64_t units = int64_t(P.nstrips) * images;
    int64_t G;
    P.kps = P.bonus = 0;
    if (units <= gmax) {
      // per-strip partition: kps CTAs per strip, one more for each border
      // strip when the budget allows (border rows cost ~15 % more: the
      // mirrored pad stores), rows split evenly within a strip
      int64_t k = std::max<int64_t>(1, std::min<int64_t>(gmax / units, p->height / 16));
      if (const char* e = getenv("PDZ_STREAM_K")) k = std::min<int64_t>(k, atoi(e));  // tuning
      int bonus = (P.nstrips >= 2 && images * (int64_t(P.nstrips) * k + 2) <= gmax &&
                   p->height / (k + 1) >= 16) ? 1 : 0;
      if (const char* e = getenv("PDZ_STREAM_BONUS")) bonus = bonus && atoi(e) != 0;
      P.kps = int(k);
      P.bonus = bonus;
      G = images * (int64_t(P.nstrips) * k + 2 * bonus);
    } else {
      const int64_t m = (units + gmax - 1) / gmax;  // strips per CTA
      G = (units + m - 1) / m;
    }
    P.G = int(std::max<int64_t>(1, G));
    Partials q = {};
    q.S = P.S, q.U = P.U, q.G = P.G, q.kps = P.kps, q.bonus = P.bonus, q.nstr = P.nstrips;
    q.H = p->height;
    // A per-strip partition with an integer number of CTAs per strip can
    // leave SMs idle (configs 4 and 5: 122 of 148).  When CTAs walk several
    // blocks per pass anyway, the even split of all strip-rows over every SM
    // (ranges crossing strip boundaries) may be cheaper despite the extra
    // segment halos: take whichever has the lower critical-path cost.
    const int srb0 = geo_srb(P.R, 0);
    const int srb1 = P.R <= 12 ? geo_srb(P.R, 1) : 0;
    int64_t cost = 0, max_seg = 0;
    partition_cost(q, P.R, srb0, srb1, &cost, &max_seg);
    if ((P.kps > 0 ? P.S / gmax >= 2 * srb0 : P.G < gmax) && !getenv("PDZ_STREAM_K")) {
      Partials f = q;
      f.kps = f.bonus = 0;
      f.G = int(gmax);
      int64_t cf = 0, mf = 0;
      partition_cost(f, P.R, srb0, srb1, &cf, &mf);
      if (cf < cost) {
        q = f;
        P.kps = P.bonus = 0;
        P.G = f.G;
        cost = cf;
        max_seg = mf;
      }
    }
    int nb = 1;
    for (int64_t i = 0; i < images; ++i) {
      const int64_t lo = part_cta_of(q, i * P.U);
      const int64_t hi = part_cta_of(q, (i + 1) * P.U - 1);
      nb = std::max<int>(nb, int(hi - lo + 1));
    }
    P.nbmax = nb;
    // Block geometry: when a CTA's rows of a strip take several 114-row
    // blocks per pass (configs 3 and 4), the taller 120-row / 128-register
    // geometry needs fewer blocks per strip and runs the vertical pass with
    // more registers; a CTA whose rows fit one block (config 2) keeps V = 0.
    P.geo = 0;
    const char* eg = getenv("PDZ_STREAM_GEO");  // tuning / tests: force a geometry
    const int want = eg ? atoi(eg) : (max_seg > srb0 ? 1 : 0);
    if (want == 1) {
      size_t smem1 = 0;
      StreamFn f1 = edge ? stream_pick<true>(P.R, 1, p->rel_tol >= 0.0, &smem1)
                         : stream_pick<false>(P.R, 1, p->rel_tol >= 0.0, &smem1);
      int occ1 = 0;
      if (f1 && cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ1, f1, geo_threads(1), smem1) ==
                    cudaSuccess &&
          occ1 >= occ) {
        P.geo = 1;
        P.fn = reinterpret_cast<void*>(f1);
        P.smem = smem1;
      }
      cudaGetLastError();
    }
    // Block order: CTAs that walk many blocks per pass run the channels of a
    // block position back to back (one lambda tile for the C channel blocks:
    // 14 % less DRAM traffic).  The neighbour dependency is then per sweep,
    // which costs one pipeline refill per sweep: measured +3.2 % on config 3
    // (70 blocks per pass and CTA) but -3 % on config 4 (7 blocks), so the
    // order is used from 24 blocks per pass on, and not for the FP32-bound
    // large radii (config 5, K = 49: 773 vs 771 us).  Everything else keeps
    // the channel-outer order, whose dependencies are C - 1 passes old.
    P.ci = (p->channels >= 2 && p->channels <= 4 && P.R <= 12 &&
            P.S / std::max(1, P.G) >= 24 * int64_t(geo_srb(P.R, P.geo))) ? 1 : 0;
    if (const char* e = getenv("PDZ_STREAM_CI")) P.ci = (atoi(e) != 0 && p->channels >= 2 &&
                                                         p->channels <= 4) ? 1 : 0;
    if (getenv("PDZ_VERBOSE"))
      fprintf(stderr,
              "pdz: plan G=%d kps=%d bonus=%d geometry=%d channel_inner=%d cost=%lld "
              "max_segment=%lld\n",
              P.G, P.kps, P.bonus, P.geo, P.ci, (long long)cost, (long long)max_seg);
  } else {
    cudaGetLastError();  // clear a failed occupancy query
    P.stream = false;
    P.fn = reinterpret_cast<void*>(edge ? pick_kernel<true>(P.R) : pick_kernel<false>(P.R));
    P.smem = tile_smem(P.R);
    P.ring = 2;
    P.tiles_x = (p->width + kTW - 1) / kTW;
    P.tiles_y = (p->height + kTH - 1) / kTH;
    P.nblk = P.tiles_x * P.tiles_y;
    P.nbmax = P.nblk;
  }
  return PDZ_OK;
}

// Kernel arguments for either kernel (the launcher passes the right one).
struct LaunchArgs {
  SweepArgs tile;
  StreamArgs stream;
};

struct Sync {
  int32_t* done;   // [G]
  int32_t* fin;    // [1]
  int32_t* flags;  // [2]
};

// TMA tensor maps of the two padded iterate buffers for the streaming kernel:
// a 3-D tensor [P][H + 2R][W + 2 kPadC] float32, box {64 + 2RP + 4, kSRB + 2R, 1};
// out-of-bounds elements (over-fetch past the last row) zero-fill.
static int32_t encode_stream_maps(const pdz_solve_params* p, const Plan& pl,
                                  float* const* bufs, const float* phi, const float* lam,
                                  StreamArgs* b) {
  static PFN_cuTensorMapEncodeTiled encode = nullptr;
  if (!encode) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    PDZ_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q),
             "cuTensorMapEncodeTiled entry point");
    if (!fn || q != cudaDriverEntryPointSuccess) {
      set_error("cuTensorMapEncodeTiled unavailable");
      return PDZ_ECUDA;
    }
    encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  }
  const int R = pl.R;
  const int pitch = kSTW + 2 * ((R + 3) & ~3) + 4;  // = SGeo<R, V>::PITCH
  const int split = geo_split(pl.geo), srb = geo_srb(R, pl.geo);
  const cuuint64_t wp = cuuint64_t(p->width) + 2 * pl.pad_c;
  const cuuint64_t hp = cuuint64_t(p->height) + 2 * pl.pad_r;
  const cuuint64_t dims[3] = {wp, hp, cuuint64_t(p->planes)};
  const cuuint64_t strides[2] = {wp * 4, wp * hp * 4};
  const cuuint32_t estr[3] = {1, 1, 1};
  for (int bi = 0; bi < kNBuf; ++bi) {
    // two boxes per block: rows [0, split) and [split, 2R + SRB)
    const cuuint32_t box[3] = {cuuint32_t(pitch), cuuint32_t(split), 1};
    const cuuint32_t box2[3] = {cuuint32_t(pitch), cuuint32_t(2 * R + srb - split), 1};
    CUresult r = encode(&b->tm[bi], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, bufs[bi], dims, strides,
                        box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
      r = encode(&b->tm2[bi], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, bufs[bi], dims, strides, box2,
                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                 CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled failed (%d)", int(r));
      return PDZ_ECUDA;
    }
  }
  // Phi [P][H][W] and lambda [P / C][H][W] (dense), box {64, SRB, 1}
  const cuuint64_t ddims[2][3] = {
      {cuuint64_t(p->width), cuuint64_t(p->height), cuuint64_t(p->planes)},
      {cuuint64_t(p->width), cuuint64_t(p->height), cuuint64_t(p->planes / p->channels)}};
  const cuuint64_t dstrides[2] = {cuuint64_t(p->width) * 4,
                                  cuuint64_t(p->width) * p->height * 4};
  const cuuint32_t dbox[3] = {cuuint32_t(kSTW), cuuint32_t(srb), 1};
  const float* dsrc[2] = {phi, lam};
  CUtensorMap* dmap[2] = {&b->tm_phi, &b->tm_lam};
  for (int k = 0; k < 2; ++k) {
    CUresult r = encode(dmap[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float*>(dsrc[k]),
                        ddims[k], dstrides, dbox, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      set_error("cuTensorMapEncodeTiled (Phi / lambda) failed (%d)", int(r));
      return PDZ_ECUDA;
    }
  }
  return PDZ_OK;
}

static int32_t fill_args(const pdz_solve_params* p, const Plan& pl, float* buf0, float* buf1,
                         float* buf2,
                         const float* phi, const float* lam, double* psum, int32_t* pflag,
                         const StateView& st, const Sync& sy, LaunchArgs* la) {
  memset(la, 0, sizeof(*la));
  double taps[kMaxTaps];
  int32_t rc = gaussian_taps_host(p->sigma, p->kernel_size, taps);
  if (rc != PDZ_OK) return rc;
  float w[kMaxTaps] = {0.f};
  const int K = p->kernel_size;
  // taps centred in the kernel radius actually run (pl.R >= K / 2: zeros on
  // both sides; K = 1 is the identity expressed as (0, 1, 0) at R = 1)
  const int shift = pl.R - K / 2;
  for (int i = 0; i < K; ++i) w[i + shift] = float(taps[i]);
  Partials pt;
  pt.sum = psum;
  pt.flag = pflag;
  pt.nbmax = pl.nbmax;
  pt.ring = pl.ring;
  pt.tiles = pl.stream ? 0 : pl.nblk;
  pt.S = pl.S;
  pt.U = pl.U;
  pt.G = pl.G;
  pt.C = pl.stream ? p->channels : 1;
  pt.kps = pl.kps;
  pt.bonus = pl.bonus;
  pt.nstr = pl.nstrips;
  pt.H = p->height;
  SweepArgs& a = la->tile;
  a.buf0 = buf0;
  a.buf1 = buf1;
  a.phi = phi;
  a.lam = lam;
  a.pt = pt;
  a.st = st;
  a.H = p->height;
  a.W = p->width;
  a.P = p->planes;
  a.C = p->channels;
  a.R = pl.R;
  a.tiles_x = pl.tiles_x;
  a.nblk = pl.nblk;
  a.max_iters = p->max_iters;
  a.eps = float(p->epsilon);
  a.tau = float(p->tau);
  a.rel_tol = p->rel_tol;
  a.y_off = 0;
  a.H_glob = p->height;
  a.row_lo = 0;
  a.row_hi = p->height;
  a.cnt_lo = 0;
  a.cnt_hi = p->height;
  memcpy(a.w, w, sizeof(w));
  StreamArgs& b = la->stream;
  b.buf[0] = buf0;
  b.buf[1] = buf1;
  b.buf[2] = buf2;
  b.phi = phi;
  b.lam = lam;
  b.pt = pt;
  b.st = st;
  b.done = sy.done;
  b.fin = sy.fin;
  b.flags = sy.flags;
  b.H = p->height;
  b.W = p->width;
  b.P = p->planes;
  b.C = p->channels;
  b.nstrips = pl.nstrips;
  b.iter_last = p->max_iters;
  b.max_iters = p->max_iters;
  b.stop_rule = (p->rel_tol >= 0.0) ? 1 : 0;
  b.chan_inner = pl.ci;
  b.cnt_lo = 0;
  b.cnt_hi = p->height;
#ifdef PDZ_PROFILE
  if (const char* e = getenv("PDZ_PROF")) {
    if (e[0] == '1' && pl.stream) {
      static long long* prof = nullptr;
      // per-CTA stats rows [0, 8192) + timeline [5][256 CTAs][2048 passes] (ns)
      if (!prof) cudaMalloc(&prof, 16 * 262144 * sizeof(long long));
      if (prof) cudaMemset(prof, 0, 16 * 262144 * sizeof(long long));
      b.prof = prof;
      g_prof = prof;
    }
  }
#endif
  b.eps = float(p->epsilon);
  b.tau = float(p->tau);
  b.rel_tol = p->rel_tol;
  b.srb = geo_srb(pl.R, pl.geo);
  memcpy(b.w, w, sizeof(w));
  for (int i = 0; i < kMaxTaps; ++i) b.w2[i] = make_float2(w[i], w[i]);
  for (int i = 0; i <= kMaxTaps; ++i)
    b.wp[i] = make_float2(i < kMaxTaps ? w[i] : 0.f, i > 0 ? w[i - 1] : 0.f);
  if (pl.stream) return encode_stream_maps(p, pl, b.buf, phi, lam, &b);
  return PDZ_OK;
}

static int32_t launch_tiled(LaunchArgs la, const pdz_solve_params* p, const Plan& pl,
                            int iter_off, cudaStream_t s, bool pdl) {
  cudaLaunchConfig_t cfg = {};
  cfg.stream = s;
  cfg.dynamicSmemBytes = pl.smem;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  la.tile.iter_off = iter_off;
  cfg.gridDim = dim3(pl.tiles_x, pl.tiles_y, p->planes);
  cfg.blockDim = dim3(kThreads);
  PDZ_CUDA(cudaLaunchKernelEx(&cfg, reinterpret_cast<SweepFn>(pl.fn), la.tile),
           "tiled sweep launch");
  return PDZ_OK;
}

// All sweeps of a streaming solve: one cooperative launch (co-residency of the
// G CTAs is what makes the neighbour waits deadlock-free).
static int32_t launch_stream(const LaunchArgs& la, const Plan& pl, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.stream = s;
  cfg.dynamicSmemBytes = pl.smem;
  cfg.gridDim = dim3(pl.G + 1);  // + the finaliser CTA
  cfg.blockDim = dim3(geo_threads(pl.geo));
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PDZ_CUDA(cudaLaunchKernelEx(&cfg, reinterpret_cast<StreamFn>(pl.fn), la.stream),
           "persistent sweep launch");
  return PDZ_OK;
}

// u0 = Phi into a (possibly padded) iterate buffer.  The persistent kernel's
// readers reflect image borders themselves, so the pads of every iterate
// buffer are poisoned with NaN: a read of a pad as data would surface as a
// non-finite result instead of a silent error.
// One CTA per padded row (grid-stride over the P * (H + 2 pr) rows), float4
// columns when every row and the pad width are 16-byte multiples (vec): the
// index arithmetic is per row, not per element (per-element 64-bit divides
// made these copies run at ~1.3 TB/s).
__global__ void pad_init_kernel(const float* __restrict__ phi, float* __restrict__ buf,
                                float* __restrict__ buf1, float* __restrict__ buf2, int H, int W,
                                int P, int pr, int pc, int vec) {
  const int wp = W + 2 * pc, hp = H + 2 * pr;
  const float nan = __int_as_float(0x7fc00000);
#ifdef PDZ_POISON_ALL
  constexpr bool kPoisonAll = true;
#else
  constexpr bool kPoisonAll = false;
#endif
  const int64_t rows = int64_t(P) * hp;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t pl = r / hp;
    const int y = int(r - pl * hp) - pr;
    const bool in_row = y >= 0 && y < H;
    const float* src = phi + (pl * H + (in_row ? y : 0)) * W;
    float* d0 = buf + r * wp;
    float* d1 = buf1 ? buf1 + r * wp : nullptr;
    float* d2 = buf2 ? buf2 + r * wp : nullptr;
    if (vec) {
      const float4 nan4 = make_float4(nan, nan, nan, nan);
      for (int c = threadIdx.x; c < wp / 4; c += blockDim.x) {
        const int x = 4 * c - pc;
        const bool in = in_row && x >= 0 && x < W;
        reinterpret_cast<float4*>(d0)[c] = in ? *reinterpret_cast<const float4*>(src + x) : nan4;
        if (!in || kPoisonAll) {
          if (d1) reinterpret_cast<float4*>(d1)[c] = nan4;
          if (d2) reinterpret_cast<float4*>(d2)[c] = nan4;
        }
      }
    } else {
      for (int c = threadIdx.x; c < wp; c += blockDim.x) {
        const int x = c - pc;
        const bool in = in_row && x >= 0 && x < W;
        d0[c] = in ? src[x] : nan;
        if (!in || kPoisonAll) {
          if (d1) d1[c] = nan;
          if (d2) d2[c] = nan;
        }
      }
    }
  }
}

// Dense final iterate: plane p from buf[iters[p] % nbuf] (the last iteration
// whose norm was recorded; solver.py:359), interior of the padded layout.  One
// CTA per output row, float4 columns when aligned (vec).
__global__ void extract_kernel(const float* __restrict__ buf0, const float* __restrict__ buf1,
                               const float* __restrict__ buf2, int nbuf,
                               const int32_t* __restrict__ iters, float* __restrict__ out, int H,
                               int W, int P, int pr, int pc, int vec) {
  const int wp = W + 2 * pc, hp = H + 2 * pr;
  const int64_t rows = int64_t(P) * H;
  for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
    const int64_t pl = r / H;
    const int y = int(r - pl * H);
    const int k = iters[pl] % nbuf;
    const float* src = (k == 0 ? buf0 : (k == 1 ? buf1 : buf2)) + (pl * hp + y + pr) * wp + pc;
    float* dst = out + r * W;
    if (vec) {
      for (int c = threadIdx.x; c < W / 4; c += blockDim.x)
        reinterpret_cast<float4*>(dst)[c] = reinterpret_cast<const float4*>(src)[c];
    } else {
      for (int c = threadIdx.x; c < W; c += blockDim.x) dst[c] = src[c];
    }
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct SolveLayout {
  float* buf0;  // iterate buffers: tiled ping-pong / persistent triple (padded)
  float* buf1;
  float* buf2;  // persistent kernel only
  float* out;   // dense final iterate [P][H][W] (pdz_fixed_point_sweeps_async)
  double* psum;
  int32_t* pflag;
  StateView st;
  Sync sy;
  size_t bytes;
};

static SolveLayout carve_solve(const pdz_solve_params* p, const Plan& pl, void* ws, size_t cap) {
  Carver c(ws, cap);
  SolveLayout L = {};
  const size_t plane = size_t(p->height) * p->width;
  const size_t plane_pad = size_t(p->height + 2 * pl.pad_r) * (p->width + 2 * pl.pad_c);
  const size_t P = p->planes;
  L.out = c.take<float>(P * plane);  // first: same offset under either plan
  L.buf0 = c.take<float>(P * plane_pad);
  L.buf1 = c.take<float>(P * plane_pad);
  L.buf2 = pl.stream ? c.take<float>(P * plane_pad) : nullptr;
  L.psum = c.take<double>(size_t(pl.ring) * P * pl.nbmax);
  L.pflag = c.take<int32_t>(size_t(pl.ring) * P * pl.nbmax);
  L.st.stop_iter = c.take<int32_t>(P);
  L.st.converged = c.take<int32_t>(P);
  L.st.failed = c.take<int32_t>(P);
  L.st.iters = c.take<int32_t>(P);
  L.st.prev_norm = c.take<double>(P);
  L.st.norms = c.take<double>(size_t(p->max_iters) * P);
  L.st.sums = c.take<double>(size_t(p->max_iters) * P);
  L.st.running = c.take<int32_t>(1);
  L.st.iter_base = c.take<int32_t>(1);
  L.st.chunk_ctr = c.take<int32_t>(1);
  L.sy.done = c.take<int32_t>(std::max(1, pl.G));
  L.sy.fin = c.take<int32_t>(1);
  L.sy.flags = c.take<int32_t>(2);
  L.bytes = c.off;
  return L;
}

// Graph cache for the tiled path: one instantiated chunk graph per
// (args, params, stream).
struct GraphKey {
  std::vector<unsigned char> bytes;
  bool operator<(const GraphKey& o) const { return bytes < o.bytes; }
};
static std::mutex g_graph_mu;
static std::map<GraphKey, cudaGraphExec_t> g_graphs;

static int32_t chunk_graph(const LaunchArgs& la, const pdz_solve_params* p, const Plan& pl,
                           cudaStream_t s, cudaGraphExec_t* out) {
  GraphKey key;
  key.bytes.resize(sizeof(SweepArgs) + sizeof(pdz_solve_params) + sizeof(void*));
  memcpy(key.bytes.data(), &la.tile, sizeof(SweepArgs));
  memcpy(key.bytes.data() + sizeof(SweepArgs), p, sizeof(pdz_solve_params));
  memcpy(key.bytes.data() + sizeof(SweepArgs) + sizeof(pdz_solve_params), &s, sizeof(void*));
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    auto it = g_graphs.find(key);
    if (it != g_graphs.end()) {
      *out = it->second;
      return PDZ_OK;
    }
  }
  cudaStream_t cap;
  PDZ_CUDA(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking), "capture stream");
  cudaGraph_t graph;
  PDZ_CUDA(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal), "begin capture");
  chunk_base_kernel<<<1, 1, 0, cap>>>(la.tile.st);
  int32_t rc = PDZ_OK;
  for (int i = 0; i < kChunk && rc == PDZ_OK; ++i) rc = launch_tiled(la, p, pl, i, cap, true);
  cudaError_t e = cudaStreamEndCapture(cap, &graph);
  cudaStreamDestroy(cap);
  if (rc != PDZ_OK) return rc;
  PDZ_CUDA(e, "end capture");
  cudaGraphExec_t exec;
  PDZ_CUDA(cudaGraphInstantiate(&exec, graph, 0), "graph instantiate");
  cudaGraphDestroy(graph);
  {
    std::lock_guard<std::mutex> lk(g_graph_mu);
    if (g_graphs.size() > 64) {
      for (auto& kv : g_graphs) cudaGraphExecDestroy(kv.second);
      g_graphs.clear();
    }
    g_graphs[key] = exec;
  }
  *out = exec;
  return PDZ_OK;
}

// Queue init + all sweeps on the stream.  Streaming: one persistent launch
// that stops by itself once every plane has stopped.  Tiled: graph chunks;
// with `poll` the host watches the device `running` counter (lagged by one
// chunk) and stops queueing once every plane has stopped.
// Measurement hook (pdz_time_sweep_kernels): events around the sweep launches.
static bool g_time_kernels = false;
// Events are per device (an event recorded on another device's stream
// fails); the last recorded pair is the one pdz_last_sweep_kernel_ms reads.
static cudaEvent_t g_kev[kMaxDevices][2] = {};
static int g_kev_dev = -1;
static std::mutex g_kev_mu;

static void time_mark(int which, cudaStream_t s) {
  if (!g_time_kernels) return;
  std::lock_guard<std::mutex> lk(g_kev_mu);
  const int dev = current_device();
  if (!g_kev[dev][0]) {
    cudaEventCreate(&g_kev[dev][0]);
    cudaEventCreate(&g_kev[dev][1]);
  }
  cudaEventRecord(g_kev[dev][which], s);
  if (which == 1) g_kev_dev = dev;
}

static int32_t queue_extract(const pdz_solve_params* p, const Plan& pl, const SolveLayout& L,
                             float* out, cudaStream_t s) {
  const int64_t rows = int64_t(p->planes) * p->height;
  const int blocks = int(std::min<int64_t>(rows, int64_t(num_sms()) * 16));
  const int vec = p->width % 4 == 0 && pl.pad_c % 4 == 0 && aligned16(out) &&
                  aligned16(L.buf0) && aligned16(L.buf1) && (!L.buf2 || aligned16(L.buf2));
  extract_kernel<<<blocks, 256, 0, s>>>(L.buf0, L.buf1, L.buf2, pl.stream ? kNBuf : 2,
                                        L.st.iters, out, p->height, p->width,
                                        p->planes, pl.pad_r, pl.pad_c, vec);
  PDZ_CHECK_LAUNCH("extract");
  return PDZ_OK;
}

// u_init: the first iterate (nullptr: u0 = Phi, solver.py:333); rows
// [cnt_lo, cnt_hi) are the ones counted in the norms.
// resident_base >= 0 (row-slab blocks, pdz_fixed_point_sweeps_resident): the
// iterate buffers stay in the workspace between calls; the sweeps start from
// buffer `resident_base` (filled from u_init only when that is given), the
// final iterate stays in buffer (resident_base + max_iters) % nbuf and no
// dense copy is made.
static int32_t queue_solve(const pdz_solve_params* p, const Plan& pl, const SolveLayout& L,
                           const float* phi, const float* lam, float* out, cudaStream_t s,
                           bool poll, const float* u_init = nullptr, int cnt_lo = 0,
                           int cnt_hi = -1, int resident_base = -1) {
  LaunchArgs la;
  float* bufs[3] = {L.buf0, L.buf1, L.buf2};
  const int nbuf = pl.stream ? kNBuf : 2;
  const bool resident = resident_base >= 0;
  if (resident) {
    float* all[3] = {L.buf0, L.buf1, L.buf2};
    for (int i = 0; i < nbuf; ++i) bufs[i] = all[(resident_base + i) % nbuf];
  }
  int32_t rc = fill_args(p, pl, bufs[0], bufs[1], bufs[2], phi, lam, L.psum, L.pflag, L.st, L.sy,
                         &la);
  if (rc != PDZ_OK) return rc;
  if (cnt_hi < 0) cnt_hi = p->height;
  la.tile.cnt_lo = la.stream.cnt_lo = cnt_lo;
  la.tile.cnt_hi = la.stream.cnt_hi = cnt_hi;
  if (u_init == nullptr && !resident) u_init = phi;
  if (u_init != nullptr) {
    const int64_t rows = int64_t(p->planes) * (p->height + 2 * pl.pad_r);
    const int blocks = int(std::min<int64_t>(rows, int64_t(num_sms()) * 16));
    const int vec = p->width % 4 == 0 && pl.pad_c % 4 == 0 && aligned16(u_init) &&
                    aligned16(L.buf0) && aligned16(L.buf1) && (!L.buf2 || aligned16(L.buf2));
    pad_init_kernel<<<blocks, 256, 0, s>>>(u_init, bufs[0], pl.stream ? bufs[1] : nullptr,
                                           pl.stream ? bufs[2] : nullptr, p->height, p->width,
                                           p->planes, pl.pad_r, pl.pad_c, vec);
    PDZ_CHECK_LAUNCH("u0 = Phi");
  }
  if (pl.stream) {
    init_state_kernel<<<(std::max<int>(p->planes, pl.G) + 255) / 256, 256, 0, s>>>(
        L.st, p->planes, L.sy.done, L.sy.fin, L.sy.flags, pl.G);
    PDZ_CHECK_LAUNCH("init state");
    time_mark(0, s);
    rc = launch_stream(la, pl, s);
    time_mark(1, s);
    if (rc != PDZ_OK) return rc;
    return resident ? PDZ_OK : queue_extract(p, pl, L, out, s);
  }
  init_state_kernel<<<(p->planes + 255) / 256, 256, 0, s>>>(L.st, p->planes);
  PDZ_CHECK_LAUNCH("init state");

  cudaGraphExec_t exec;
  rc = chunk_graph(la, p, pl, s, &exec);
  if (rc != PDZ_OK) return rc;
  const int n_chunks = (p->max_iters + kChunk - 1) / kChunk;
  // per thread and device: events belong to the device they were created on
  static thread_local int32_t* pinned_dev[kMaxDevices] = {};
  static thread_local cudaEvent_t events_dev[kMaxDevices][2] = {};
  const int dev = current_device();
  int32_t*& pinned = pinned_dev[dev];
  cudaEvent_t* events = events_dev[dev];
  if (poll && pinned == nullptr) {
    PDZ_CUDA(cudaHostAlloc(&pinned, 2 * sizeof(int32_t), cudaHostAllocPortable), "pinned flag");
    PDZ_CUDA(cudaEventCreateWithFlags(&events[0], cudaEventDisableTiming), "event");
    PDZ_CUDA(cudaEventCreateWithFlags(&events[1], cudaEventDisableTiming), "event");
  }
  int launched = 0;
  time_mark(0, s);
  for (int c = 0; c < n_chunks; ++c) {
    if (poll && c >= 2) {
      const int slot = (c - 2) & 1;
      PDZ_CUDA(cudaEventSynchronize(events[slot]), "poll sync");
      if (pinned[slot] == 0) break;
    }
    PDZ_CUDA(cudaGraphLaunch(exec, s), "graph launch");
    launched = std::min(p->max_iters, (c + 1) * kChunk);
    if (poll) {
      const int slot = c & 1;
      PDZ_CUDA(cudaMemcpyAsync(&pinned[slot], L.st.running, sizeof(int32_t),
                               cudaMemcpyDeviceToHost, s),
               "poll copy");
      PDZ_CUDA(cudaEventRecord(events[slot], s), "poll record");
    }
  }
  time_mark(1, s);
  Partials pt = la.tile.pt;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(32);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PDZ_CUDA(cudaLaunchKernelEx(&cfg, finalize_kernel, L.st, pt, int(p->planes), launched,
                              int(p->max_iters), p->rel_tol),
           "finalize launch");
  return resident ? PDZ_OK : queue_extract(p, pl, L, out, s);
}

static int32_t check_abort(const Plan& pl, const Sync& sy) {
  if (!pl.stream) return PDZ_OK;
  int32_t f[2] = {0, 0};
  PDZ_CUDA(cudaMemcpy(f, sy.flags, sizeof(f), cudaMemcpyDeviceToHost), "D2H flags");
  if (f[1]) {
    set_error("persistent sweep aborted: a CTA dependency wait timed out");
    return PDZ_ECUDA;
  }
  return PDZ_OK;
}

}  // namespace pdz

using namespace pdz;

extern "C" {

static size_t step_bytes(const pdz_solve_params* params, const Plan& pl) {
  Carver c(nullptr, 0);
  c.take<double>(size_t(pl.ring) * params->planes * pl.nbmax);
  c.take<int32_t>(size_t(pl.ring) * params->planes * pl.nbmax);
  c.take<int32_t>(std::max(1, pl.G));
  c.take<int32_t>(1);
  c.take<int32_t>(2);
  return Carver::round(c.off);
}

size_t pdz_step_workspace_bytes(const pdz_solve_params* params) {
  Plan pl;
  if (check_params(params, &pl, false) != PDZ_OK) return 0;
  return step_bytes(params, pl);
}

// One tiled sweep over dense caller buffers (shared by the whole-image step
// and the row-slab step).  `out` receives sqrt(sum r^2) (take_sqrt) or the raw
// sum of r^2 over rows [row_lo, row_hi) per plane.
static int32_t step_impl(const pdz_solve_params* params, const float* u, float* u_out,
                         const float* phi, const float* lambda_map, int32_t y_off,
                         int32_t H_glob, int32_t row_lo, int32_t row_hi, double* out,
                         int32_t* nonfinite, int take_sqrt, void* workspace,
                         size_t workspace_bytes, void* stream) {
  Plan pl;
  int32_t rc = check_params(params, &pl, false);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(u && u_out && phi && lambda_map && out, "NULL array argument");
  PDZ_REQUIRE(u != u_out, "u_out must not alias u");
  Carver c(workspace, workspace_bytes);
  double* psum = c.take<double>(size_t(pl.ring) * params->planes * pl.nbmax);
  int32_t* pflag = c.take<int32_t>(size_t(pl.ring) * params->planes * pl.nbmax);
  Sync sy;
  sy.done = c.take<int32_t>(std::max(1, pl.G));
  sy.fin = c.take<int32_t>(1);
  sy.flags = c.take<int32_t>(2);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  pdz_solve_params one = *params;
  one.max_iters = 1;
  LaunchArgs la;
  StateView none = {};
  // iteration 1 reads buf0 (= u), writes buf1 (= u_out)
  rc = fill_args(&one, pl, const_cast<float*>(u), u_out, nullptr, phi, lambda_map, psum, pflag,
                 none, sy, &la);
  if (rc != PDZ_OK) return rc;
  la.tile.y_off = y_off;
  la.tile.H_glob = H_glob;
  la.tile.row_lo = la.tile.cnt_lo = row_lo;
  la.tile.row_hi = la.tile.cnt_hi = row_hi;
  cudaStream_t s = as_stream(stream);
  rc = launch_tiled(la, &one, pl, 1, s, false);
  if (rc != PDZ_OK) return rc;
  step_norm_kernel<<<1, 256, 0, s>>>(la.tile.pt, params->planes, out, nonfinite, take_sqrt);
  PDZ_CHECK_LAUNCH("step norm");
  return PDZ_OK;
}

// A single sweep over dense caller buffers always runs the tiled kernel (the
// persistent kernel's padded layout only pays off over many sweeps).
int32_t pdz_fixed_point_step(const pdz_solve_params* params, const float* u, float* u_out,
                             const float* phi, const float* lambda_map, double* norms,
                             int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                             void* stream) {
  PDZ_REQUIRE(params != nullptr, "params is NULL");
  return step_impl(params, u, u_out, phi, lambda_map, 0, params->height, 0, params->height,
                   norms, nonfinite, 1, workspace, workspace_bytes, stream);
}

int32_t pdz_fixed_point_step_rows(const pdz_solve_params* params, const float* u, float* u_out,
                                  const float* phi, const float* lambda_map, int32_t row_offset,
                                  int32_t global_height, int32_t row_lo, int32_t row_hi,
                                  double* sumsq, int32_t* nonfinite, void* workspace,
                                  size_t workspace_bytes, void* stream) {
  PDZ_REQUIRE(params != nullptr, "params is NULL");
  PDZ_REQUIRE(global_height >= 2, "global_height must be >= 2, got %d", global_height);
  PDZ_REQUIRE(row_lo >= 1 && row_hi <= params->height - 1 && row_lo < row_hi,
              "row window [%d, %d) must leave >= 1 halo row on both sides of %d rows", row_lo,
              row_hi, params->height);
  PDZ_REQUIRE(row_offset + row_lo >= 0 && row_offset + row_hi <= global_height,
              "rows [%d, %d) + offset %d fall outside the %d-row image", row_lo, row_hi,
              row_offset, global_height);
  return step_impl(params, u, u_out, phi, lambda_map, row_offset, global_height, row_lo, row_hi,
                   sumsq, nonfinite, 0, workspace, workspace_bytes, stream);
}

// The plan of a solve: the persistent kernel unless Phi / lambda are not
// 16-byte aligned (TMA), then the tiled kernel.  The workspace covers both.
static int32_t solve_plan(const pdz_solve_params* params, const float* phi, const float* lam,
                          Plan* pl) {
  const bool aligned =
      ((reinterpret_cast<uintptr_t>(phi) | reinterpret_cast<uintptr_t>(lam)) & 15) == 0;
  return check_params(params, pl, aligned);
}

size_t pdz_solve_workspace_bytes(const pdz_solve_params* params) {
  Plan pl, tl;
  if (check_params(params, &pl) != PDZ_OK) return 0;
  if (check_params(params, &tl, false) != PDZ_OK) return 0;
  return Carver::round(std::max(carve_solve(params, pl, nullptr, 0).bytes,
                                carve_solve(params, tl, nullptr, 0).bytes));
}

int32_t pdz_fixed_point_solve(const pdz_solve_params* params, const float* phi,
                              const float* lambda_map, float* u_out, double* norms_host,
                              int32_t* iterations_host, int32_t* converged_host,
                              int32_t* failed_host, void* workspace, size_t workspace_bytes,
                              void* stream) {
  Plan pl;
  int32_t rc = solve_plan(params, phi, lambda_map, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map && u_out, "NULL array argument");
  PDZ_REQUIRE(norms_host && iterations_host && converged_host && failed_host,
              "NULL host output");
  SolveLayout L = carve_solve(params, pl, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  rc = queue_solve(params, pl, L, phi, lambda_map, u_out, s, true);
  if (rc != PDZ_OK) return rc;
  const int P = params->planes;
  PDZ_CUDA(cudaStreamSynchronize(s), "solve sync");
  rc = check_abort(pl, L.sy);
  if (rc != PDZ_OK) return rc;
  PDZ_CUDA(cudaMemcpy(iterations_host, L.st.iters, P * 4, cudaMemcpyDeviceToHost), "D2H iters");
  PDZ_CUDA(cudaMemcpy(converged_host, L.st.converged, P * 4, cudaMemcpyDeviceToHost), "D2H conv");
  PDZ_CUDA(cudaMemcpy(failed_host, L.st.failed, P * 4, cudaMemcpyDeviceToHost), "D2H failed");
  PDZ_CUDA(cudaMemcpy(norms_host, L.st.norms, size_t(params->max_iters) * P * 8,
                      cudaMemcpyDeviceToHost),
           "D2H norms");
  int worst = -1;
  for (int q = 0; q < P && worst < 0; ++q)
    if (failed_host[q] != 0) worst = q;
  if (worst >= 0) {
    set_error("solver produced non-finite values at iteration %d (plane %d)", failed_host[worst],
              worst);
    return PDZ_ENONFINITE;
  }
  return PDZ_OK;
}

size_t pdz_solve_state_bytes(const pdz_solve_params* params) {
  if (params == nullptr || params->planes < 1 || params->max_iters < 1) return 0;
  return size_t(params->max_iters) * params->planes * sizeof(double) +
         (3 * size_t(params->planes) + 1) * sizeof(int32_t);
}

__global__ void abort_flag_kernel(const int32_t* flags, int32_t* out) { out[0] = flags[1]; }

int32_t pdz_fixed_point_solve_async(const pdz_solve_params* params, const float* phi,
                                    const float* lambda_map, float* u_out, void* state,
                                    void* workspace, size_t workspace_bytes, void* stream) {
  Plan pl;
  int32_t rc = solve_plan(params, phi, lambda_map, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map && u_out && state, "NULL array argument");
  SolveLayout L = carve_solve(params, pl, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  // no host polling: the tiled fallback queues every chunk (stopped planes
  // are skipped by the sweeps); the persistent kernel stops by itself
  rc = queue_solve(params, pl, L, phi, lambda_map, u_out, s, false);
  if (rc != PDZ_OK) return rc;
  const size_t P = params->planes;
  char* st = static_cast<char*>(state);
  const size_t nb = size_t(params->max_iters) * P * sizeof(double);
  int32_t* ints = reinterpret_cast<int32_t*>(st + nb);
  PDZ_CUDA(cudaMemcpyAsync(st, L.st.norms, nb, cudaMemcpyDeviceToDevice, s), "state norms");
  PDZ_CUDA(cudaMemcpyAsync(ints, L.st.iters, P * 4, cudaMemcpyDeviceToDevice, s), "state iters");
  PDZ_CUDA(cudaMemcpyAsync(ints + P, L.st.converged, P * 4, cudaMemcpyDeviceToDevice, s),
           "state converged");
  PDZ_CUDA(cudaMemcpyAsync(ints + 2 * P, L.st.failed, P * 4, cudaMemcpyDeviceToDevice, s),
           "state failed");
  if (pl.stream) {
    abort_flag_kernel<<<1, 1, 0, s>>>(L.sy.flags, ints + 3 * P);
    PDZ_CHECK_LAUNCH("abort flag");
  } else {
    PDZ_CUDA(cudaMemsetAsync(ints + 3 * P, 0, 4, s), "abort flag");
  }
  return PDZ_OK;
}

int32_t pdz_fixed_point_sweeps_async(const pdz_solve_params* params, const float* phi,
                                     const float* lambda_map, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  Plan pl;
  int32_t rc = solve_plan(params, phi, lambda_map, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map, "NULL array argument");
  pdz_solve_params fixed = *params;
  fixed.rel_tol = -1.0;  // never stops early
  SolveLayout L = carve_solve(&fixed, pl, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  return queue_solve(&fixed, pl, L, phi, lambda_map, L.out, as_stream(stream), false);
}

int32_t pdz_fixed_point_sweeps_from(const pdz_solve_params* params, const float* u_init,
                                    const float* phi, const float* lambda_map, int32_t count_lo,
                                    int32_t count_hi, float* u_out, double* sumsq,
                                    int32_t* failed, void* workspace, size_t workspace_bytes,
                                    void* stream) {
  Plan pl;
  int32_t rc = solve_plan(params, phi, lambda_map, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(u_init && phi && lambda_map && u_out && sumsq && failed, "NULL array argument");
  PDZ_REQUIRE(u_init != u_out, "u_out must not alias u_init");
  PDZ_REQUIRE(0 <= count_lo && count_lo < count_hi && count_hi <= params->height,
              "count window [%d, %d) outside the %d rows", count_lo, count_hi, params->height);
  pdz_solve_params fixed = *params;
  fixed.rel_tol = -1.0;  // exactly max_iters sweeps: the caller applies the stop rule
  SolveLayout L = carve_solve(&fixed, pl, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  rc = queue_solve(&fixed, pl, L, phi, lambda_map, u_out, s, false, u_init, count_lo, count_hi);
  if (rc != PDZ_OK) return rc;
  const size_t P = params->planes;
  PDZ_CUDA(cudaMemcpyAsync(sumsq, L.st.sums, size_t(params->max_iters) * P * sizeof(double),
                           cudaMemcpyDeviceToDevice, s),
           "sums copy");
  PDZ_CUDA(cudaMemcpyAsync(failed, L.st.failed, P * sizeof(int32_t), cudaMemcpyDeviceToDevice, s),
           "failed copy");
  return PDZ_OK;
}

int32_t pdz_slab_layout(const pdz_solve_params* params, int64_t* info_host, int32_t n) {
  Plan pl;
  int32_t rc = check_params(params, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(info_host && n >= PDZ_SLAB_LAYOUT_LEN, "info buffer too small");
  pdz_solve_params fixed = *params;
  fixed.rel_tol = -1.0;
  SolveLayout L = carve_solve(&fixed, pl, reinterpret_cast<void*>(uintptr_t(256)), ~size_t(0) >> 1);
  const auto off = [&](const float* q) {
    return q ? int64_t(reinterpret_cast<uintptr_t>(q) - uintptr_t(256)) : int64_t(-1);
  };
  info_host[0] = pl.stream ? kNBuf : 2;
  info_host[1] = off(L.buf0);
  info_host[2] = off(L.buf1);
  info_host[3] = off(L.buf2);
  info_host[4] = pl.pad_r;
  info_host[5] = pl.pad_c;
  info_host[6] = int64_t(params->height) + 2 * pl.pad_r;
  info_host[7] = int64_t(params->width) + 2 * pl.pad_c;
  return PDZ_OK;
}

int32_t pdz_fixed_point_sweeps_resident(const pdz_solve_params* params, const float* u_init,
                                        const float* phi, const float* lambda_map,
                                        int32_t count_lo, int32_t count_hi, int32_t base,
                                        double* sumsq, int32_t* failed, void* workspace,
                                        size_t workspace_bytes, void* stream) {
  Plan pl;
  int32_t rc = solve_plan(params, phi, lambda_map, &pl);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map && sumsq && failed, "NULL array argument");
  PDZ_REQUIRE(base >= 0 && base < (pl.stream ? kNBuf : 2), "base buffer %d out of range", base);
  PDZ_REQUIRE(0 <= count_lo && count_lo < count_hi && count_hi <= params->height,
              "count window [%d, %d) outside the %d rows", count_lo, count_hi, params->height);
  pdz_solve_params fixed = *params;
  fixed.rel_tol = -1.0;  // exactly max_iters sweeps: the caller applies the stop rule
  SolveLayout L = carve_solve(&fixed, pl, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  // the finaliser writes the per-sweep sums and the failure record straight
  // into the caller's buffers (same layouts as the state block's)
  L.st.sums = sumsq;
  L.st.failed = failed;
  return queue_solve(&fixed, pl, L, phi, lambda_map, nullptr, as_stream(stream), false, u_init,
                     count_lo, count_hi, base);
}

int64_t pdz_solve_kernel_launches(const pdz_solve_params* params) {
  Plan pl;
  if (check_params(params, &pl) != PDZ_OK) return -1;
  if (pl.stream) return 4;  // pad init + init state + persistent + extract
  const int64_t chunks = (params->max_iters + kChunk - 1) / kChunk;
  return 4 + chunks * (1 + kChunk);  // pad init + init + chunk prologues + sweeps + finalize + extract
}

const float* pdz_solve_result_plane(const pdz_solve_params* params, const void* workspace,
                                    int32_t plane, int32_t iterations) {
  Plan pl;
  if (check_params(params, &pl) != PDZ_OK || workspace == nullptr) return nullptr;
  SolveLayout L = carve_solve(params, pl, const_cast<void*>(workspace), ~size_t(0) >> 1);
  (void)iterations;  // the dense copy already holds each plane's final iterate
  const size_t n = size_t(params->height) * params->width;
  return L.out + plane * n;
}

#ifdef PDZ_PROFILE
// Profiling builds only: per-CTA wait times of the last PDZ_PROF=1 solve.
int32_t pdz_debug_prof(long long* host, int n) {
  if (!g_prof) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_prof, size_t(n) * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  return 1;
}
#endif

void pdz_time_sweep_kernels(int32_t enable) { g_time_kernels = enable != 0; }

float pdz_last_sweep_kernel_ms(void) {
  cudaEvent_t e0, e1;
  {
    std::lock_guard<std::mutex> lk(g_kev_mu);
    if (g_kev_dev < 0) return -1.0f;
    e0 = g_kev[g_kev_dev][0];
    e1 = g_kev[g_kev_dev][1];
  }
  float ms = -1.0f;
  if (cudaEventSynchronize(e1) != cudaSuccess) return -1.0f;
  if (cudaEventElapsedTime(&ms, e0, e1) != cudaSuccess) return -1.0f;
  return ms;
}

int32_t pdz_sweep_kernel_kind(const pdz_solve_params* params) {
  Plan pl;
  if (check_params(params, &pl) != PDZ_OK) return -1;
  return pl.stream ? 2 : 1;
}

int32_t pdz_solve_plan_info(const pdz_solve_params* params, int32_t* info_host, int32_t n) {
  Plan pl;
  const int32_t rc = check_params(params, &pl);
  if (rc != PDZ_OK) return rc;
  const bool rel = params->rel_tol >= 0.0;
  const int32_t v[PDZ_PLAN_INFO_LEN] = {
      pl.stream ? 2 : 1,
      pl.stream ? pl.G : pl.nblk,
      pl.kps,
      pl.bonus,
      pl.geo,
      pl.R,
      pl.nbmax,
      pl.nstrips,
      pl.stream ? geo_srb(pl.R, pl.geo) : kTH,
      pl.stream ? geo_threads(pl.geo) : kThreads,
      rel ? 1 : 0,
      pl.ci,
  };
  for (int i = 0; i < n && i < PDZ_PLAN_INFO_LEN; ++i) info_host[i] = v[i];
  return PDZ_OK;
}

int32_t pdz_solve_kernel_name(const pdz_solve_params* params, char* buf_host, int32_t n) {
  Plan pl;
  const int32_t rc = check_params(params, &pl);
  if (rc != PDZ_OK) return rc;
  if (!buf_host || n <= 0) return PDZ_EINVAL;
  const int edge = params->edge_preserving ? 1 : 0;
  if (pl.stream)
    snprintf(buf_host, size_t(n), "pdz::stream_kernel<%d, %d, %d, %d>", pl.R, pl.geo, edge,
             params->rel_tol >= 0.0 ? 1 : 0);
  else
    snprintf(buf_host, size_t(n), "pdz::sweep_kernel<%d, %d>",
             (pl.R == 1 || pl.R == 2 || pl.R == 3 || pl.R == 6 || pl.R == 9 || pl.R == 12 ||
              pl.R == 24) ? pl.R : -1, edge);
  return PDZ_OK;
}

}  // extern "C"
