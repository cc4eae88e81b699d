// Streaming, persistent relaxed fixed-point solve -- the production hot kernel.
//
// Same mathematics as the tiled sweep (pdz_sweep.cu; solver.py:280-302), laid
// out for B200:
//  * ONE cooperative launch runs all sweeps of a solve.  CTA i owns the same
//    exactly balanced range [floor(iS/G), floor((i+1)S/G)) of the S = planes x
//    strips x H "strip-rows" (strip = 64 output columns) in every sweep, so
//    every SM gets the same pixels (+-1 row) -- no wave quantisation on 148
//    SMs, no per-sweep launch, no grid-wide barrier: before sweep n a CTA only
//    waits (acquire loads of per-CTA progress counters) for the CTAs whose
//    rows its stencil reads -- its strip and the two neighbouring strips,
//    +-R rows -- to have published sweep n-1.  The same wait protects the
//    ping-pong buffer it overwrites (those CTAs were its readers).
//  * inside a sweep the CTA streams down its range in blocks of 32 rows:
//    input rows (64 + 2*ceil4(R) columns) arrive by cp.async.bulk (TMA bulk
//    copies, UBLKCP) into a double buffer signalled by an mbarrier while the
//    previous block computes; horizontally blurred rows of the 2R-row overlap
//    are carried between blocks (only range/strip starts pay the halo);
//  * horizontal Gaussian from shared memory (8 outputs per item), vertical
//    pass with packed FFMA2 over column pairs, MUFU sqrt/rcp face fluxes,
//    residual, update and r^2 fused in registers;
//  * warps 0-3 compute; warp 4 of CTA 0 is the service warp: it waits for
//    every CTA to publish sweep m, reduces the r^2 partials of m in a fixed
//    order (bitwise reproducible), applies the stop rule (solver.py:347-358)
//    and publishes `fin = m`.  Partials live in a ring of kRing slots; a CTA
//    writing slot n % kRing first waits for fin >= n - kRing, and with the
//    stop rule active it waits for fin >= n - 2 so planes stopped at <= n-2
//    are skipped (their answer stays in buf[stop & 1]).
// Border handling: rows are reflected (np.pad "symmetric", solver.py:235) at
// load time; out-of-image columns are fixed up in shared memory from their
// reflected in-window sources; the centred differences use the one-sided
// form at the first/last row/column (np.gradient, solver.py:178-179).
// Requirements: width % 4 == 0 (16-byte bulk copies), a compiled radius, and
// all G CTAs co-resident (cooperative launch); otherwise the tiled kernel.
// Every spin has a 10 s timeout that sets an abort flag instead of hanging.
#pragma once
#include <algorithm>
#include <cmath>

#include "pdz_solver.cuh"

namespace pdz {

constexpr int kSTW = 64;                    // strip width (output columns)
constexpr int kSRB = 32;                    // output rows per block (4 warps x 8)
constexpr int kSCW = 4;                     // compute warps
constexpr int kSThreads = (kSCW + 1) * 32;  // + service warp
constexpr int kComputeThreads = kSCW * 32;
constexpr int kRing = 4;                    // partial-sum slots (iterations in flight)
constexpr long long kSpinTimeoutNs = 10000000000ll;

template <int R>
struct SGeo {
  static constexpr int RP = (R + 3) & ~3;  // column halo rounded to float4
  static constexpr int PWD = kSTW + 2 * RP;  // staged floats per row
  static constexpr int PITCH = PWD;          // 16-byte aligned smem rows
  static constexpr int ROWS = kSRB + 2 * R;  // staged input rows / H rows
  static constexpr int IN_FLOATS = ROWS * PITCH;
  static constexpr int H_FLOATS = ROWS * kSTW;
  static constexpr size_t SMEM = size_t(2 * IN_FLOATS + 2 * H_FLOATS) * 4 + 128;
};

struct StreamArgs {
  float* buf0;
  float* buf1;
  const float* phi;
  const float* lam;
  Partials pt;          // ring of kRing slots
  StateView st;         // st.stop_iter == nullptr: single step (no service warp)
  int32_t* done;        // [G] last sweep each CTA has published
  int32_t* fin;         // [1] last iteration the service warp finalised
  int32_t* flags;       // [0] every plane stopped, [1] abort (spin timeout)
  int32_t H, W, P, C, nstrips;
  int32_t iter_first, iter_last, max_iters;
  int32_t stop_rule;    // rel_tol active: sweep n needs fin >= n - 2
  float eps, tau;
  double rel_tol;
  float w[kMaxTaps];
};

// ------------------------------------------------------------ primitives --
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_fence_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// Bulk global -> shared copy (TMA engine), completion counted on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
// Order this thread's earlier generic-proxy global accesses (as observed via
// the acquire) before its later async-proxy (bulk copy) accesses.
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ int ld_acquire(const int32_t* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// Polling load: relaxed (no L1 invalidation per poll); the caller issues one
// acquire fence once the condition holds.
__device__ __forceinline__ int ld_relaxed(const int32_t* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acquire_gpu() {
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
__device__ __forceinline__ void st_release(int32_t* p, int v) {
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ long long global_ns() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void compute_bar() {
  asm volatile("bar.sync 1, %0;" ::"n"(kComputeThreads) : "memory");
}
__device__ __forceinline__ float sqrt_approx(float x) {
  float y;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float y;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
// d = a * b + c on packed float pairs (FFMA2).
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long*>(&a)),
        "l"(*reinterpret_cast<unsigned long long*>(&b)),
        "l"(*reinterpret_cast<unsigned long long*>(&c)));
  return *reinterpret_cast<float2*>(&d);
}

template <bool EDGE>
__device__ __forceinline__ float sflux(float jump, float along, float eps) {
  if (!EDGE) return jump;
  const float s = fmaf(jump, jump, along * along);
  return jump * rcp_approx(sqrt_approx(s) + eps);
}

struct SBlock {
  int p, x0, yb, n, first;
};

// Walks a CTA's range [L0, L1) of strip-rows block by block: (plane p, strip
// s, row y) advance incrementally, so only the start needs divisions.  Planes
// frozen at <= iter-2 are skipped.  (32-bit: the host only selects this
// kernel when S < 2^31.)
struct RangeIter {
  int L, L0, L1, p, s, y;
  __device__ __forceinline__ void init(int l0, int l1, const StreamArgs& a) {
    L = L0 = l0;
    L1 = l1;
    const int u = l0 / a.H;
    y = l0 - u * a.H;
    p = u / a.nstrips;
    s = u - p * a.nstrips;
  }
  __device__ __forceinline__ void wrap(const StreamArgs& a) {
    y = 0;
    if (++s == a.nstrips) {
      s = 0;
      ++p;
    }
  }
  __device__ __forceinline__ bool next(const StreamArgs& a, int iter, SBlock& b) {
    while (L < L1) {
      const int seg_end = min(L1, L - y + a.H);
      if (a.st.stop_iter) {
        const int st = a.st.stop_iter[p];
        if (st != 0 && st < iter - 1) {
          L = seg_end;
          wrap(a);
          continue;
        }
      }
      b.p = p;
      b.x0 = s * kSTW;
      b.yb = y;
      b.n = min(kSRB, seg_end - L);
      b.first = (L == L0) || (y == 0);
      L += b.n;
      y += b.n;
      if (y == a.H) wrap(a);
      return true;
    }
    return false;
  }
};

// Warp 0 of the compute warps: queue the bulk copies of the block's new input
// rows (reflected row indices, in-image column span) into `in`.
template <int R>
__device__ __forceinline__ void issue_rows(const SBlock& b, const float* __restrict__ uin,
                                           float* in, uint64_t* bar, int H, int W, int lane) {
  using Gm = SGeo<R>;
  const int r0 = b.first ? b.yb - R : b.yb + R;
  const int nrows = b.first ? b.n + 2 * R : b.n;
  const int idx0 = b.first ? 0 : R + 1;
  const int gc0 = max(0, b.x0 - Gm::RP);
  const int gc1 = min(W, b.x0 + kSTW + Gm::RP);
  const uint32_t bytes = uint32_t(gc1 - gc0) * 4u;
  if (lane == 0) mbar_expect_tx(bar, bytes * uint32_t(nrows));
  __syncwarp();
  const int dcol = gc0 - (b.x0 - Gm::RP);
  for (int i = lane; i < nrows; i += 32) {
    const int gy = reflect(r0 + i, H);
    bulk_g2s(in + (idx0 + i) * Gm::PITCH + dcol, uin + size_t(gy) * W + gc0, bytes, bar);
  }
}

// One warp: spin until done[lo..hi] >= need and the fin conditions hold.
// Returns false on stop-all or abort (timeout).
__device__ bool wait_deps(const StreamArgs& a, int lo, int hi, int need_done, int need_fin) {
  const int lane = threadIdx.x & 31;
  const long long t0 = global_ns();
  unsigned ns = 32;
  while (true) {
    bool ok = true;
    for (int j = lo + lane; j <= hi; j += 32) ok &= ld_relaxed(a.done + j) >= need_done;
    if (lane == 0 && need_fin > 0) ok &= ld_relaxed(a.fin) >= need_fin;
    ok = __all_sync(0xffffffffu, ok);
    const int stop = ld_relaxed(a.flags) | ld_relaxed(a.flags + 1);
    if (__any_sync(0xffffffffu, stop != 0)) return false;
    if (ok) {
      fence_acquire_gpu();
      return true;
    }
    if (global_ns() - t0 > kSpinTimeoutNs) {
      if (lane == 0) atomicExch(a.flags + 1, 1);
      return false;
    }
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
  }
}

// CTA 0 / warp kSCW: finalise iterations as soon as every CTA published them.
__device__ void service_loop(const StreamArgs& a) {
  const int lane = threadIdx.x & 31;
  const int G = gridDim.x;
  for (int m = a.iter_first; m <= a.iter_last; ++m) {
    const long long t0 = global_ns();
    unsigned ns = 64;
    while (true) {
      bool ok = true;
      for (int j = lane; j < G; j += 32) ok &= ld_relaxed(a.done + j) >= m;
      ok = __all_sync(0xffffffffu, ok);
      if (ok) {
        fence_acquire_gpu();
        break;
      }
      if (__any_sync(0xffffffffu, ld_relaxed(a.flags + 1) != 0)) return;
      if (global_ns() - t0 > kSpinTimeoutNs) {
        if (lane == 0) atomicExch(a.flags + 1, 1);
        return;
      }
      __nanosleep(ns);
      if (ns < 1024) ns <<= 1;
    }
    finalize_iteration_warp(a.st, a.pt, a.P, m, a.max_iters, a.rel_tol);
    __syncwarp();
    __threadfence();
    const int running = a.st.running[0];
    if (lane == 0) {
      if (running == 0) atomicExch(a.flags, 1);
      st_release(a.fin, m);
    }
    if (running == 0) return;
  }
}

template <int R, bool EDGE>
__global__ void __launch_bounds__(kSThreads, 3) stream_kernel(const StreamArgs a) {
  using Gm = SGeo<R>;
  extern __shared__ __align__(128) float smem[];
  float* const in0 = smem;
  float* const in1 = smem + Gm::IN_FLOATS;
  float* const h0 = smem + 2 * Gm::IN_FLOATS;
  float* const h1 = h0 + Gm::H_FLOATS;
  uint64_t* const bars = reinterpret_cast<uint64_t*>(h1 + Gm::H_FLOATS);
  __shared__ double s_red[kSCW];
  __shared__ int s_nf[kSCW];
  __shared__ int s_go;

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    mbar_init(&bars[0], 1);
    mbar_init(&bars[1], 1);
    mbar_fence_init();
  }
  __syncthreads();

  if (warp == kSCW) {  // service warp
    if (a.st.stop_iter && blockIdx.x == 0) service_loop(a);
    return;
  }

  const int H = a.H, W = a.W;
  const size_t plane = size_t(H) * W;
  const int S = int(a.pt.S), G = a.pt.G;
  const int L0 = int(cta_start(blockIdx.x, S, G));
  const int L1 = int(cta_start(blockIdx.x + 1, S, G));
  // CTAs whose output rows this CTA's stencil reads: same strip +-R rows and
  // the neighbouring strips (a superset: one interval of the linear order).
  const int dep_lo = int(cta_of(max(0, L0 - H - R), S, G));
  const int dep_hi = int(cta_of(min(S - 1, L1 - 1 + H + R), S, G));

  // thread roles for the vertical pass / update: column pair, 8-row group
  const int c = 2 * lane;   // strip-local output column of the pair
  const int j0 = warp * 8;  // block-local first row
  uint32_t phase0 = 0, phase1 = 0;
  int ib = 0;

  for (int iter = a.iter_first; iter <= a.iter_last; ++iter) {
    // ---- dependencies: neighbours published iter-1; ring slot / stop state
    if (warp == 0) {
      int need_fin = iter - kRing;
      if (a.stop_rule) need_fin = max(need_fin, iter - 2);
      const bool go = wait_deps(a, dep_lo, dep_hi, iter - 1, a.st.stop_iter ? need_fin : 0);
      if (lane == 0) s_go = go ? 1 : 0;
      fence_proxy_async_global();
    }
    compute_bar();
    if (!s_go) return;

    const float* __restrict__ uin_all = ((iter - 1) & 1) ? a.buf1 : a.buf0;
    float* __restrict__ uout_all = (iter & 1) ? a.buf1 : a.buf0;
    RangeIter it;
    it.init(L0, L1, a);
    SBlock cur, nxt;
    bool have = it.next(a, iter, cur);
    if (have && warp == 0)
      issue_rows<R>(cur, uin_all + cur.p * plane, ib ? in1 : in0, &bars[ib], H, W, lane);
    double acc_r2 = 0.0;
    float acc_nf = 0.0f;
    int acc_p = have ? cur.p : -1;

    // One CTA barrier per block:
    //   wait IN(b) [+ border fix-up + barrier, border strips only]
    //   -> carry H overlap, blur the new rows into H(b)
    //   -> barrier
    //   -> carry the IN overlap into the other buffer, queue IN(b+1),
    //      vertical pass + divergence + update of block b.
    // H(b) is written while only H(b-1) is read; IN(b+1) overwrites the
    // buffer last read by block b-1, which every thread finished before the
    // barrier.
    while (have) {
      const bool have_nxt = it.next(a, iter, nxt);
      float* const in_cur = ib ? in1 : in0;
      float* const in_nxt = ib ? in0 : in1;
      float* const h_cur = ib ? h1 : h0;
      float* const h_prev = ib ? h0 : h1;
      uint64_t* const bar_cur = &bars[ib];
      uint64_t* const bar_nxt = &bars[ib ^ 1];
      const int gx = cur.x0 + c;
      const bool col_ok = gx < W;

      // ---- prefetch Phi / lambda for this thread's outputs into registers
      float2 phv[8], lmv[8];
      {
        const size_t off0 = size_t(cur.yb + j0) * W + gx;
        const float2* __restrict__ ph =
            reinterpret_cast<const float2*>(a.phi + cur.p * plane + off0);
        const float2* __restrict__ lm =
            reinterpret_cast<const float2*>(a.lam + (cur.p / a.C) * plane + off0);
        const int rows_here = col_ok ? min(8, cur.n - j0) : 0;
        const int w2 = W >> 1;  // row stride in float2
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (j < rows_here) {
            phv[j] = __ldg(ph + j * w2);
            lmv[j] = __ldg(lm + j * w2);
          } else {
            phv[j] = make_float2(0.f, 0.f);
            lmv[j] = make_float2(0.f, 0.f);
          }
        }
      }

      // ---- wait for this block's input rows; mirror out-of-image columns
      if (ib) {
        mbar_wait(bar_cur, phase1);
        phase1 ^= 1;
      } else {
        mbar_wait(bar_cur, phase0);
        phase0 ^= 1;
      }
      const int xbase = cur.x0 - Gm::RP;  // global column of staged column 0
      if (xbase < 0 || xbase + Gm::PWD > W) {  // border strip (CTA-uniform)
        const int new0 = cur.first ? 0 : R + 1;
        const int nnew = cur.first ? cur.n + 2 * R : cur.n;
        // only the out-of-image staged columns: [0, nl) left, [cr, PWD) right
        const int nl = xbase < 0 ? -xbase : 0;
        const int cr = min(Gm::PWD, max(nl, W - xbase));
        const int nh = nl + (Gm::PWD - cr);
        for (int k = tid; k < nnew * nh; k += kComputeThreads) {
          const int i = k / nh, h = k - i * nh;
          const int ci = h < nl ? h : cr + (h - nl);
          const int src = reflect(xbase + ci, W) - xbase;
          if (src >= 0 && src < Gm::PWD)
            in_cur[(new0 + i) * Gm::PITCH + ci] = in_cur[(new0 + i) * Gm::PITCH + src];
        }
        compute_bar();
      }

      // ---- H rows: carry the 2R overlap, blur the new rows
      int hnew0, hn, in0row;
      if (cur.first) {
        hnew0 = 0;
        hn = cur.n + 2 * R;
        in0row = 0;
      } else {
        for (int k = tid; k < 2 * R * (kSTW / 4); k += kComputeThreads)
          reinterpret_cast<float4*>(h_cur)[k] =
              reinterpret_cast<const float4*>(h_prev + kSRB * kSTW)[k];
        hnew0 = 2 * R;
        hn = cur.n;
        in0row = R + 1;
      }
      // 8 adjacent outputs per item: 8 independent FMA chains, (8 + 2R)
      // staged values per 8 outputs.
      for (int item = tid; item < hn * (kSTW / 8); item += kComputeThreads) {
        const int i = item >> 3, g = item & 7;
        const float* row = in_cur + (in0row + i) * Gm::PITCH + 8 * g;
        constexpr int OFF = Gm::RP - R;
        constexpr int NQ = (OFF + 2 * R + 8 + 3) / 4;
        float v[4 * NQ];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
          const float4 t = reinterpret_cast<const float4*>(row)[q];
          v[4 * q] = t.x;
          v[4 * q + 1] = t.y;
          v[4 * q + 2] = t.z;
          v[4 * q + 3] = t.w;
        }
        float o[8];
#pragma unroll
        for (int m = 0; m < 8; ++m) o[m] = 0.f;
#pragma unroll
        for (int k = 0; k <= 2 * R; ++k) {
          const float wk = a.w[k];
#pragma unroll
          for (int m = 0; m < 8; ++m) o[m] = fmaf(wk, v[OFF + k + m], o[m]);
        }
        float4* dst = reinterpret_cast<float4*>(h_cur + (hnew0 + i) * kSTW + 8 * g);
        dst[0] = make_float4(o[0], o[1], o[2], o[3]);
        dst[1] = make_float4(o[4], o[5], o[6], o[7]);
      }
      compute_bar();

      // ---- queue the next block's rows (+ carry of the R+1 overlap rows)
      if (have_nxt) {
        if (!nxt.first) {
          // rows [nxt.yb - 1, nxt.yb + R) live in in_cur at idx (row - cur_base)
          const int cur_base = cur.first ? cur.yb - R : cur.yb - 1;
          const int s0 = (nxt.yb - 1) - cur_base;
          constexpr int Q = Gm::PWD / 4;
          for (int k = tid; k < (R + 1) * Q; k += kComputeThreads) {
            const int i = k / Q, q = k - i * Q;
            reinterpret_cast<float4*>(in_nxt + i * Gm::PITCH)[q] =
                reinterpret_cast<const float4*>(in_cur + (s0 + i) * Gm::PITCH)[q];
          }
        }
        if (warp == 0)
          issue_rows<R>(nxt, uin_all + nxt.p * plane, in_nxt, bar_nxt, H, W, lane);
      }

      // ---- vertical pass (FFMA2 over the column pair), divergence, update
      if (j0 < cur.n) {
        float2 G2[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) G2[j] = make_float2(0.f, 0.f);
#pragma unroll
        for (int k = 0; k < 8 + 2 * R; ++k) {
          const float2 hv = *reinterpret_cast<const float2*>(h_cur + (j0 + k) * kSTW + c);
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const int t = k - j;
            if (t >= 0 && t <= 2 * R) G2[j] = ffma2(make_float2(a.w[t], a.w[t]), hv, G2[j]);
          }
        }

        // rolling window of u rows (A = y-1, B = y, C = y+1) at columns c-1 .. c+2
        // (staged column RP + c is 8-byte aligned)
        const float* urow = in_cur + ((cur.first ? R : 1) + j0 - 1) * Gm::PITCH + Gm::RP + c;
        const float sx0 = (gx == 0) ? 1.0f : 0.5f;          // column c   (c >= 0)
        const float sx1 = (gx + 1 == W - 1) ? 1.0f : 0.5f;  // column c+1
        float lA = urow[-1], rA = urow[2];
        float2 cA = *reinterpret_cast<const float2*>(urow);
        urow += Gm::PITCH;
        float lB = urow[-1], rB = urow[2];
        float2 cB = *reinterpret_cast<const float2*>(urow);
        float2 xA = make_float2(sx0 * (cA.y - lA), sx1 * (rA - cA.x));
        float2 xB = make_float2(sx0 * (cB.y - lB), sx1 * (rB - cB.x));
        // south flux of the row above the first output row
        float2 fs_up = make_float2(sflux<EDGE>(cB.x - cA.x, 0.5f * (xA.x + xB.x), a.eps),
                                   sflux<EDGE>(cB.y - cA.y, 0.5f * (xA.y + xB.y), a.eps));
        float r2 = 0.f;
        float* __restrict__ uout = uout_all + cur.p * plane;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          urow += Gm::PITCH;
          const float lC = urow[-1], rC = urow[2];
          const float2 cC = *reinterpret_cast<const float2*>(urow);
          const float2 xC = make_float2(sx0 * (cC.y - lC), sx1 * (rC - cC.x));
          const int y = cur.yb + j0 + j;
          const float sy = (y == 0 || y == H - 1) ? 1.0f : 0.5f;
          // centred vertical differences at columns c-1, c, c+1, c+2
          const float dl = sy * (lC - lA);
          const float d0 = sy * (cC.x - cA.x);
          const float d1 = sy * (cC.y - cA.y);
          const float dr = sy * (rC - rA);
          const float u0 = cB.x, u1 = cB.y;
          const float fw = sflux<EDGE>(u0 - lB, 0.5f * (dl + d0), a.eps);  // face c-1|c
          const float fm = sflux<EDGE>(u1 - u0, 0.5f * (d0 + d1), a.eps);  // face c|c+1
          const float fe = sflux<EDGE>(rB - u1, 0.5f * (d1 + dr), a.eps);  // face c+1|c+2
          const float2 fs_dn = make_float2(sflux<EDGE>(cC.x - u0, 0.5f * (xB.x + xC.x), a.eps),
                                           sflux<EDGE>(cC.y - u1, 0.5f * (xB.y + xC.y), a.eps));
          const float div0 = ((fm - fw) + fs_dn.x) - fs_up.x;
          const float div1 = ((fe - fm) + fs_dn.y) - fs_up.y;
          fs_up = fs_dn;
          lA = lB;
          rA = rB;
          cA = cB;
          xA = xB;
          lB = lC;
          rB = rC;
          cB = cC;
          xB = xC;
          const float r0 = fmaf(-lmv[j].x, G2[j].x, div0) + phv[j].x;
          const float r1 = fmaf(-lmv[j].y, G2[j].y, div1) + phv[j].y;
          const float n0 = fmaf(a.tau, r0, u0);
          const float n1 = fmaf(a.tau, r1, u1);
          if (col_ok && j0 + j < cur.n) {
            *reinterpret_cast<float2*>(uout + size_t(y) * W + gx) = make_float2(n0, n1);
            r2 = fmaf(r0, r0, fmaf(r1, r1, r2));
            acc_nf = fmaf(n0, 0.0f, fmaf(n1, 0.0f, acc_nf));  // NaN iff non-finite update
          }
        }
        acc_r2 += double(r2);
      }

      // ---- flush the plane partial when the plane changes / at the end
      const bool flush = !have_nxt || nxt.p != acc_p;
      if (flush) {
        double s = warp_sum(acc_r2);
        const int nfw = __any_sync(0xffffffffu, !(acc_nf == 0.0f));
        if (lane == 0) {
          s_red[warp] = s;
          s_nf[warp] = nfw;
        }
        compute_bar();
        if (tid == 0) {
          double t = 0.0;
          int f = 0;
#pragma unroll
          for (int w2 = 0; w2 < kSCW; ++w2) {
            t += s_red[w2];
            f |= s_nf[w2];
          }
          const int k = int(blockIdx.x - cta_of(int64_t(acc_p) * a.pt.U, S, G));
          const size_t slot = (size_t(iter % a.pt.ring) * a.P + acc_p) * a.pt.nbmax + k;
          a.pt.sum[slot] = t;
          a.pt.flag[slot] = f;
        }
        acc_r2 = 0.0;
        acc_nf = 0.0f;
        acc_p = have_nxt ? nxt.p : -1;
      }
      cur = nxt;
      have = have_nxt;
      ib ^= 1;
    }
    // ---- publish: every output row and partial of this sweep is written
    // (barrier orders the CTA's writes before thread 0's cumulative fence)
    compute_bar();
    if (tid == 0) {
      __threadfence();
      st_release(a.done + blockIdx.x, iter);
    }
  }
}

// ------------------------------------------------------------------- host --
using StreamFn = void (*)(const StreamArgs);

template <int R, bool EDGE>
static StreamFn stream_prepared(size_t* smem) {
  static bool done = false;
  *smem = SGeo<R>::SMEM;
  if (!done) {
    cudaFuncSetAttribute(stream_kernel<R, EDGE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(SGeo<R>::SMEM));
    done = true;
  }
  return stream_kernel<R, EDGE>;
}

template <bool EDGE>
static StreamFn stream_pick(int R, size_t* smem) {
  switch (R) {
    case 1: return stream_prepared<1, EDGE>(smem);
    case 2: return stream_prepared<2, EDGE>(smem);
    case 3: return stream_prepared<3, EDGE>(smem);
    case 6: return stream_prepared<6, EDGE>(smem);
    case 9: return stream_prepared<9, EDGE>(smem);
    case 12: return stream_prepared<12, EDGE>(smem);
    case 24: return stream_prepared<24, EDGE>(smem);
    default: return nullptr;
  }
}

}  // namespace pdz
