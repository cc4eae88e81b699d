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
#include <cmath>
#include <map>
#include <mutex>
#include <vector>

#include "pdz_internal.cuh"

namespace pdz {

constexpr int kTW = 32;           // tile width  (one warp of columns)
constexpr int kTH = 64;           // tile height
constexpr int kThreads = 256;     // 8 warps
constexpr int kRowsPerWarp = kTH / (kThreads / 32);
constexpr int kMaxFusedRadius = 48;
constexpr int kMaxTaps = 2 * kMaxFusedRadius + 1;
constexpr int kChunk = 16;        // sweeps per captured graph chunk

struct StateView {
  int32_t* stop_iter;   // [P] 0 = running, else the iteration it stopped at
  int32_t* converged;   // [P]
  int32_t* failed;      // [P] iteration that went non-finite, 0 = never
  int32_t* iters;       // [P] iterations whose norm is recorded
  double* prev_norm;    // [P]
  double* norms;        // [max_iters][P]
  int32_t* running;     // [1] planes still running after the latest finalize
  int32_t* iter_base;   // [1] first iteration of the current graph chunk
  int32_t* chunk_ctr;   // [1]
};

struct SweepArgs {
  float* buf0;
  float* buf1;
  const float* phi;
  const float* lam;
  double* partials;      // [2][P][nblk]
  int32_t* nf_flags;     // [2][P][nblk]
  StateView st;          // st.stop_iter == nullptr: single step, no stop rule
  int32_t H, W, P, C, R;
  int32_t tiles_x, nblk;
  int32_t iter_off;      // iteration = (*st.iter_base if set) + iter_off
  int32_t max_iters;
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

// Reduce iteration `it`'s partials for every still-running plane and apply
// the stop rule.  Executed by one whole block.
__device__ void finalize_iteration(const SweepArgs& a, int it) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int p = warp; p < a.P; p += nwarps) {
    if (a.st.stop_iter[p] != 0) continue;
    const size_t base = (size_t(it & 1) * a.P + p) * a.nblk;
    double s = 0.0;
    int nf = 0;
    for (int b = lane; b < a.nblk; b += 32) {
      s += a.partials[base + b];
      nf |= a.nf_flags[base + b];
    }
    s = warp_sum(s);
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) {
      if (nf) {
        a.st.failed[p] = it;
        a.st.stop_iter[p] = it;
      } else {
        const double norm = sqrt(s);
        a.st.norms[size_t(it - 1) * a.P + p] = norm;
        a.st.iters[p] = it;
        const double prev = a.st.prev_norm[p];
        if (it >= 2 && fabs(norm - prev) / fmax(prev, 1e-30) <= a.rel_tol) {
          a.st.converged[p] = 1;
          a.st.stop_iter[p] = it;
        } else if (it >= a.max_iters) {
          a.st.stop_iter[p] = it;
        }
        a.st.prev_norm[p] = norm;
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int n = 0;
    for (int p = 0; p < a.P; ++p) n += (a.st.stop_iter[p] == 0);
    a.st.running[0] = n;
  }
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
    if (iter >= 2 && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0)
      finalize_iteration(a, iter - 1);
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
    const float sy = (gy == 0 || gy == H - 1) ? 1.0f : 0.5f;
    const float cy0 = sy * (U[j + 2][0] - U[j][0]);
    const float cy1 = sy * (U[j + 2][1] - U[j][1]);
    const float cy2 = sy * (U[j + 2][2] - U[j][2]);
    const float fe_r = face_flux<EDGE>(U[j + 1][2] - U[j + 1][1], 0.5f * (cy1 + cy2), a.eps);
    const float fe_l = face_flux<EDGE>(U[j + 1][1] - U[j + 1][0], 0.5f * (cy0 + cy1), a.eps);
    const float fs_dn =
        face_flux<EDGE>(U[j + 2][1] - U[j + 1][1], 0.5f * (cx[j + 1] + cx[j + 2]), a.eps);
    const float div = ((fe_r - fe_l) + fs_dn) - fs_up;
    fs_up = fs_dn;
    if (gy < H && gx < W) {
      const size_t off = size_t(gy) * W + gx;
      const float r = fmaf(-lam[off], G[j], div) + phi[off];
      const float un = fmaf(a.tau, r, U[j + 1][1]);
      uout[off] = un;
      acc2 = fma(double(r), double(r), acc2);
      nf |= !(isfinite(r) && isfinite(un));
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
    const size_t slot = (size_t(iter & 1) * a.P + p) * a.nblk + blk;
    a.partials[slot] = s;
    a.nf_flags[slot] = f;
  }
  pdl_launch_dependents();
}

__global__ void finalize_kernel(const SweepArgs a, int it) {
  pdl_wait();
  finalize_iteration(a, it);
}

// Chunk prologue: iter_base = chunk * kChunk + 1.
__global__ void chunk_base_kernel(StateView st) {
  pdl_wait();
  const int c = st.chunk_ctr[0];
  st.iter_base[0] = c * kChunk + 1;
  st.chunk_ctr[0] = c + 1;
  pdl_launch_dependents();
}

__global__ void init_state_kernel(StateView st, int P) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
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

// Single fixed_point_step: norms[p] = sqrt(sum of iteration-1 partials).
__global__ void step_norm_kernel(const SweepArgs a, double* norms, int32_t* nonfinite) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int p = warp; p < a.P; p += blockDim.x >> 5) {
    const size_t base = (size_t(1) * a.P + p) * a.nblk;
    double s = 0.0;
    int nf = 0;
    for (int b = lane; b < a.nblk; b += 32) {
      s += a.partials[base + b];
      nf |= a.nf_flags[base + b];
    }
    s = warp_sum(s);
    nf = __any_sync(0xffffffffu, nf);
    if (lane == 0) {
      norms[p] = sqrt(s);
      if (nonfinite) nonfinite[p] = nf;
    }
  }
}

// ------------------------------------------------------------------------
// host side

using SweepFn = void (*)(const SweepArgs);

template <int RT, bool EDGE>
static SweepFn prepared() {
  static bool done = false;
  if (!done) {
    const int R = RT >= 0 ? RT : kMaxFusedRadius;
    const size_t smem = size_t(((kTH + 2 * R) * (kTW + 2 * R + 1) + 3 + (kTH + 2 * R) * kTW)) * 4;
    cudaFuncSetAttribute(sweep_kernel<RT, EDGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(smem));
    done = true;
  }
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

static size_t sweep_smem(int R) {
  return size_t(((kTH + 2 * R) * (kTW + 2 * R + 1) + 3 + (kTH + 2 * R) * kTW)) * 4;
}

struct Geometry {
  int R;        // fused-kernel radius (>= 1)
  int tiles_x, tiles_y, nblk;
};

static int32_t check_params(const pdz_solve_params* p, Geometry* g) {
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
  if (g) {
    g->R = std::max(1, p->kernel_size / 2);
    g->tiles_x = (p->width + kTW - 1) / kTW;
    g->tiles_y = (p->height + kTH - 1) / kTH;
    g->nblk = g->tiles_x * g->tiles_y;
  }
  return PDZ_OK;
}

static int32_t fill_args(const pdz_solve_params* p, const Geometry& g, SweepArgs* a) {
  memset(a, 0, sizeof(*a));
  double taps[kMaxTaps];
  int32_t st = gaussian_taps_host(p->sigma, p->kernel_size, taps);
  if (st != PDZ_OK) return st;
  const int K = p->kernel_size;
  if (K == 1) {  // identity smoothing expressed as taps (0, 1, 0), R = 1
    a->w[0] = 0.f;
    a->w[1] = float(taps[0]);
    a->w[2] = 0.f;
  } else {
    for (int i = 0; i < K; ++i) a->w[i] = float(taps[i]);
  }
  a->H = p->height;
  a->W = p->width;
  a->P = p->planes;
  a->C = p->channels;
  a->R = g.R;
  a->tiles_x = g.tiles_x;
  a->nblk = g.nblk;
  a->max_iters = p->max_iters;
  a->eps = float(p->epsilon);
  a->tau = float(p->tau);
  a->rel_tol = p->rel_tol;
  return PDZ_OK;
}

static int32_t launch_sweep(const SweepArgs& a, const pdz_solve_params* p, const Geometry& g,
                            cudaStream_t s, bool pdl) {
  SweepFn fn = p->edge_preserving ? pick_kernel<true>(g.R) : pick_kernel<false>(g.R);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(g.tiles_x, g.tiles_y, p->planes);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = sweep_smem(g.R);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  PDZ_CUDA(cudaLaunchKernelEx(&cfg, fn, a), "sweep launch");
  return PDZ_OK;
}

struct SolveLayout {
  float* buf0;
  float* buf1;
  double* partials;
  int32_t* flags;
  StateView st;
  size_t bytes;
};

static SolveLayout carve_solve(const pdz_solve_params* p, const Geometry& g, void* ws,
                               size_t cap) {
  Carver c(ws, cap);
  SolveLayout L = {};
  const size_t plane = size_t(p->height) * p->width;
  const size_t P = p->planes;
  L.buf0 = c.take<float>(P * plane);
  L.buf1 = c.take<float>(P * plane);
  L.partials = c.take<double>(2 * P * g.nblk);
  L.flags = c.take<int32_t>(2 * P * g.nblk);
  L.st.stop_iter = c.take<int32_t>(P);
  L.st.converged = c.take<int32_t>(P);
  L.st.failed = c.take<int32_t>(P);
  L.st.iters = c.take<int32_t>(P);
  L.st.prev_norm = c.take<double>(P);
  L.st.norms = c.take<double>(size_t(p->max_iters) * P);
  L.st.running = c.take<int32_t>(1);
  L.st.iter_base = c.take<int32_t>(1);
  L.st.chunk_ctr = c.take<int32_t>(1);
  L.bytes = c.off;
  return L;
}

// Graph cache: one instantiated chunk graph per (args, stream) signature.
struct GraphKey {
  std::vector<unsigned char> bytes;
  bool operator<(const GraphKey& o) const { return bytes < o.bytes; }
};
static std::mutex g_graph_mu;
static std::map<GraphKey, cudaGraphExec_t> g_graphs;

static int32_t chunk_graph(const SweepArgs& base, const pdz_solve_params* p, const Geometry& g,
                           cudaStream_t s, cudaGraphExec_t* out) {
  GraphKey key;
  key.bytes.resize(sizeof(SweepArgs) + sizeof(pdz_solve_params) + sizeof(void*));
  memcpy(key.bytes.data(), &base, sizeof(SweepArgs));
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
  chunk_base_kernel<<<1, 1, 0, cap>>>(base.st);
  int32_t rc = PDZ_OK;
  for (int i = 0; i < kChunk && rc == PDZ_OK; ++i) {
    SweepArgs a = base;
    a.iter_off = i;
    rc = launch_sweep(a, p, g, cap, true);
  }
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

// Queue init + all sweeps (graph chunks) on the stream.  If `poll` is set the
// host watches the device `running` counter (lagged by one chunk) and stops
// queueing once every plane has stopped.  Returns the last iteration queued.
static int32_t queue_solve(const pdz_solve_params* p, const Geometry& g, const SolveLayout& L,
                           const float* phi, const float* lam, cudaStream_t s, bool poll,
                           int* last_iter) {
  SweepArgs a;
  int32_t rc = fill_args(p, g, &a);
  if (rc != PDZ_OK) return rc;
  a.buf0 = L.buf0;
  a.buf1 = L.buf1;
  a.phi = phi;
  a.lam = lam;
  a.partials = L.partials;
  a.nf_flags = L.flags;
  a.st = L.st;

  const size_t plane_bytes = size_t(p->height) * p->width * sizeof(float);
  PDZ_CUDA(cudaMemcpyAsync(L.buf0, phi, plane_bytes * p->planes, cudaMemcpyDeviceToDevice, s),
           "u0 = Phi");
  init_state_kernel<<<(p->planes + 255) / 256, 256, 0, s>>>(L.st, p->planes);
  PDZ_CHECK_LAUNCH("init state");

  cudaGraphExec_t exec;
  rc = chunk_graph(a, p, g, s, &exec);
  if (rc != PDZ_OK) return rc;

  const int n_chunks = (p->max_iters + kChunk - 1) / kChunk;
  static thread_local int32_t* pinned = nullptr;
  static thread_local cudaEvent_t events[2] = {nullptr, nullptr};
  if (poll && pinned == nullptr) {
    PDZ_CUDA(cudaHostAlloc(&pinned, 2 * sizeof(int32_t), cudaHostAllocDefault), "pinned flag");
    PDZ_CUDA(cudaEventCreateWithFlags(&events[0], cudaEventDisableTiming), "event");
    PDZ_CUDA(cudaEventCreateWithFlags(&events[1], cudaEventDisableTiming), "event");
  }
  int launched = 0;
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
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(1);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PDZ_CUDA(cudaLaunchKernelEx(&cfg, finalize_kernel, a, launched), "finalize launch");
  *last_iter = launched;
  return PDZ_OK;
}

}  // namespace pdz

using namespace pdz;

extern "C" {

size_t pdz_step_workspace_bytes(const pdz_solve_params* params) {
  Geometry g;
  if (check_params(params, &g) != PDZ_OK) return 0;
  Carver c(nullptr, 0);
  c.take<double>(2 * size_t(params->planes) * g.nblk);
  c.take<int32_t>(2 * size_t(params->planes) * g.nblk);
  return Carver::round(c.off);
}

int32_t pdz_fixed_point_step(const pdz_solve_params* params, const float* u, float* u_out,
                             const float* phi, const float* lambda_map, double* norms,
                             int32_t* nonfinite, void* workspace, size_t workspace_bytes,
                             void* stream) {
  Geometry g;
  int32_t rc = check_params(params, &g);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(u && u_out && phi && lambda_map && norms, "NULL array argument");
  PDZ_REQUIRE(u != u_out, "u_out must not alias u");
  Carver c(workspace, workspace_bytes);
  double* partials = c.take<double>(2 * size_t(params->planes) * g.nblk);
  int32_t* flags = c.take<int32_t>(2 * size_t(params->planes) * g.nblk);
  if (!c.ok) {
    set_error("workspace too small: need %zu bytes, got %zu", c.off, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  SweepArgs a;
  rc = fill_args(params, g, &a);
  if (rc != PDZ_OK) return rc;
  a.buf0 = const_cast<float*>(u);  // iteration 1 reads buf0, writes buf1
  a.buf1 = u_out;
  a.phi = phi;
  a.lam = lambda_map;
  a.partials = partials;
  a.nf_flags = flags;
  a.iter_off = 1;
  a.max_iters = 1;
  cudaStream_t s = as_stream(stream);
  rc = launch_sweep(a, params, g, s, false);
  if (rc != PDZ_OK) return rc;
  step_norm_kernel<<<1, 256, 0, s>>>(a, norms, nonfinite);
  PDZ_CHECK_LAUNCH("step norm");
  return PDZ_OK;
}

size_t pdz_solve_workspace_bytes(const pdz_solve_params* params) {
  Geometry g;
  if (check_params(params, &g) != PDZ_OK) return 0;
  return Carver::round(carve_solve(params, g, nullptr, 0).bytes);
}

int32_t pdz_fixed_point_solve(const pdz_solve_params* params, const float* phi,
                              const float* lambda_map, float* u_out, double* norms_host,
                              int32_t* iterations_host, int32_t* converged_host,
                              int32_t* failed_host, void* workspace, size_t workspace_bytes,
                              void* stream) {
  Geometry g;
  int32_t rc = check_params(params, &g);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map && u_out, "NULL array argument");
  PDZ_REQUIRE(norms_host && iterations_host && converged_host && failed_host,
              "NULL host output");
  SolveLayout L = carve_solve(params, g, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  cudaStream_t s = as_stream(stream);
  int last = 0;
  rc = queue_solve(params, g, L, phi, lambda_map, s, true, &last);
  if (rc != PDZ_OK) return rc;
  const int P = params->planes;
  PDZ_CUDA(cudaStreamSynchronize(s), "solve sync");
  std::vector<int32_t> stop(P);
  PDZ_CUDA(cudaMemcpy(iterations_host, L.st.iters, P * 4, cudaMemcpyDeviceToHost), "D2H iters");
  PDZ_CUDA(cudaMemcpy(converged_host, L.st.converged, P * 4, cudaMemcpyDeviceToHost), "D2H conv");
  PDZ_CUDA(cudaMemcpy(failed_host, L.st.failed, P * 4, cudaMemcpyDeviceToHost), "D2H failed");
  PDZ_CUDA(cudaMemcpy(norms_host, L.st.norms, size_t(params->max_iters) * P * 8,
                      cudaMemcpyDeviceToHost),
           "D2H norms");
  const size_t plane = size_t(params->height) * params->width;
  int worst = -1;
  for (int p = 0; p < P; ++p) {
    const int it = iterations_host[p];
    const float* src = (it & 1) ? L.buf1 : L.buf0;
    PDZ_CUDA(cudaMemcpyAsync(u_out + p * plane, src + p * plane, plane * 4,
                             cudaMemcpyDeviceToDevice, s),
             "final iterate");
    if (failed_host[p] != 0 && worst < 0) worst = p;
  }
  PDZ_CUDA(cudaStreamSynchronize(s), "solve sync");
  if (worst >= 0) {
    set_error("solver produced non-finite values at iteration %d (plane %d)", failed_host[worst],
              worst);
    return PDZ_ENONFINITE;
  }
  return PDZ_OK;
}

int32_t pdz_fixed_point_sweeps_async(const pdz_solve_params* params, const float* phi,
                                     const float* lambda_map, void* workspace,
                                     size_t workspace_bytes, void* stream) {
  Geometry g;
  int32_t rc = check_params(params, &g);
  if (rc != PDZ_OK) return rc;
  PDZ_REQUIRE(phi && lambda_map, "NULL array argument");
  pdz_solve_params fixed = *params;
  fixed.rel_tol = -1.0;  // never stops early
  SolveLayout L = carve_solve(&fixed, g, workspace, workspace_bytes);
  if (workspace == nullptr || L.bytes > workspace_bytes) {
    set_error("workspace too small: need %zu bytes, got %zu", L.bytes, workspace_bytes);
    return PDZ_EWORKSPACE;
  }
  int last = 0;
  return queue_solve(&fixed, g, L, phi, lambda_map, as_stream(stream), false, &last);
}

int64_t pdz_solve_kernel_launches(const pdz_solve_params* params) {
  Geometry g;
  if (check_params(params, &g) != PDZ_OK) return -1;
  const int64_t chunks = (params->max_iters + kChunk - 1) / kChunk;
  return 2 + chunks * (1 + kChunk);  // init + chunk prologues + sweeps + finalize
}

const float* pdz_solve_result_plane(const pdz_solve_params* params, const void* workspace,
                                    int32_t plane, int32_t iterations) {
  Geometry g;
  if (check_params(params, &g) != PDZ_OK || workspace == nullptr) return nullptr;
  SolveLayout L = carve_solve(params, g, const_cast<void*>(workspace), ~size_t(0) >> 1);
  const size_t n = size_t(params->height) * params->width;
  return ((iterations & 1) ? L.buf1 : L.buf0) + plane * n;
}

}  // extern "C"
