/* CPU oracle for the relaxed fixed-point solve -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, float64, OpenMP restatement of the reference's per-channel
 * solve (/root/reference/pkg/src/pdehaze/solver.py:305-359) so the parity
 * tests can check the GPU solve at BASELINE sizes (config 2 at 1024^2 for
 * 200 sweeps, a config-4 crop for 500 sweeps, the config-5 stop rule) in
 * seconds, on the GPU box's host cores.  It is compiled by
 * __graft_entry__.build() into oracle/_build/liboracle_solve.so and loaded
 * only by tests/, smoke() and bench.py's CPU legs, never by the product.
 *
 * Pinning: tests/test_oracle_golden.py checks it against the numpy oracle
 * (oracle/pdz_oracle.py, itself pinned bit-for-bit to fixtures produced by
 * the real reference) and against the reference's golden fixtures, to
 * 1e-12: the arithmetic is the reference's except for summation order
 * (separable Gaussian; row-blocked norm sum instead of numpy's
 * pairwise sum), which moves results by ~1e-16 relative.
 *
 * Per sweep (solver.py:280-302):
 *   gy, gx   = np.gradient(u) centred, one-sided at the ends  (solver.py:178-179)
 *   east  face (y, x|x+1): jump = u[y][x+1]-u[y][x], tang = (gy[y][x]+gy[y][x+1])/2
 *   south face (y|y+1, x): jump = u[y+1][x]-u[y][x], tang = (gx[y][x]+gx[y+1][x])/2
 *   D = 1/(sqrt(jump^2+tang^2)+eps) (D = 1 for no-edge),  flux = D*jump (:175-187)
 *   div = sum of outgoing minus incoming fluxes, zero flux at the border (:205-209)
 *   G   = separable normalised Gaussian, np.pad "symmetric" reflection  (:225-241)
 *   r   = div - lambda*G + Phi;  u' = u + tau*r;  ||r|| = sqrt(sum r^2)  (:296-302)
 * Solve (solver.py:333-358): u0 = Phi; stop when |n - p| / max(p, 1e-30) <= rel_tol
 * from iteration 2 on; non-finite u or norm aborts (returns the iteration).
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#ifdef _OPENMP
#include <omp.h>
#endif

/* np.pad(mode="symmetric") source index, repeated for pads >= n (solver.py:235) */
static int reflect(int i, int n) {
  int m = i % (2 * n);
  if (m < 0) m += 2 * n;
  return m >= n ? 2 * n - 1 - m : m;
}

/* g / sum(g), g = exp(-d^2 / (2 sigma^2)), d = -K//2 .. K//2 (solver.py:219-222) */
static void taps_1d(double sigma, int K, double* w) {
  double s = 0.0;
  for (int i = 0; i < K; ++i) {
    const double d = (double)(i - K / 2);
    w[i] = exp(-(d * d) / (2.0 * sigma * sigma));
    s += w[i];
  }
  for (int i = 0; i < K; ++i) w[i] /= s;
}

typedef struct {
  int H, W, K, edge;
  double eps, tau;
  const double* w;
  const int* rx;  /* [W + 2r] reflected column index */
  const int* ry;  /* [H + 2r] reflected row index */
  double* tmp;    /* [H][W] horizontal pass */
  double* gy;     /* [H][W] */
  double* gx;     /* [H][W] */
  double* rowsum; /* [H] sum of r^2 per row */
} Work;

/* One sweep: u -> un, returns sum of r^2 (row-blocked). */
static double sweep(const Work* k, const double* u, const double* src, const double* lam,
                    double* un, int threads) {
  const int H = k->H, W = k->W, K = k->K, R = K / 2;
  (void)threads;
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int y = 0; y < H; ++y) {
    const double* row = u + (size_t)y * W;
    double* t = k->tmp + (size_t)y * W;
    for (int x = 0; x < W; ++x) {
      double acc = 0.0;
      for (int b = 0; b < K; ++b) acc += k->w[b] * row[k->rx[x + b]];
      t[x] = acc;
    }
    if (k->edge) {
      double* gyr = k->gy + (size_t)y * W;
      double* gxr = k->gx + (size_t)y * W;
      const double* up = u + (size_t)(y > 0 ? y - 1 : y) * W;
      const double* dn = u + (size_t)(y < H - 1 ? y + 1 : y) * W;
      const double fy = (y == 0 || y == H - 1) ? 1.0 : 0.5;
      for (int x = 0; x < W; ++x) gyr[x] = (dn[x] - up[x]) * fy;
      gxr[0] = row[1] - row[0];
      for (int x = 1; x < W - 1; ++x) gxr[x] = (row[x + 1] - row[x - 1]) / 2.0;
      gxr[W - 1] = row[W - 1] - row[W - 2];
    }
  }
#pragma omp parallel for schedule(static) num_threads(threads)
  for (int y = 0; y < H; ++y) {
    const double* row = u + (size_t)y * W;
    double s2 = 0.0;
    for (int x = 0; x < W; ++x) {
      double g = 0.0;
      for (int a = 0; a < K; ++a) g += k->w[a] * k->tmp[(size_t)k->ry[y + a] * W + x];
      /* divergence: + east(x) - east(x-1) + south(y) - south(y-1) */
      double div = 0.0;
      if (x < W - 1) {
        const double j = row[x + 1] - row[x];
        double d = 1.0;
        if (k->edge) {
          const double tg = 0.5 * (k->gy[(size_t)y * W + x + 1] + k->gy[(size_t)y * W + x]);
          d = 1.0 / (sqrt(j * j + tg * tg) + k->eps);
        }
        div += d * j;
      }
      if (x > 0) {
        const double j = row[x] - row[x - 1];
        double d = 1.0;
        if (k->edge) {
          const double tg = 0.5 * (k->gy[(size_t)y * W + x] + k->gy[(size_t)y * W + x - 1]);
          d = 1.0 / (sqrt(j * j + tg * tg) + k->eps);
        }
        div -= d * j;
      }
      if (y < H - 1) {
        const double j = u[(size_t)(y + 1) * W + x] - row[x];
        double d = 1.0;
        if (k->edge) {
          const double tg = 0.5 * (k->gx[(size_t)(y + 1) * W + x] + k->gx[(size_t)y * W + x]);
          d = 1.0 / (sqrt(j * j + tg * tg) + k->eps);
        }
        div += d * j;
      }
      if (y > 0) {
        const double j = row[x] - u[(size_t)(y - 1) * W + x];
        double d = 1.0;
        if (k->edge) {
          const double tg = 0.5 * (k->gx[(size_t)y * W + x] + k->gx[(size_t)(y - 1) * W + x]);
          d = 1.0 / (sqrt(j * j + tg * tg) + k->eps);
        }
        div -= d * j;
      }
      const size_t i = (size_t)y * W + x;
      const double r = div - lam[i] * g + src[i];
      un[i] = row[x] + k->tau * r;
      s2 += r * r;
    }
    k->rowsum[y] = s2;
  }
  double s = 0.0;
  for (int y = 0; y < H; ++y) s += k->rowsum[y];
  return s;
}

/* Solve P planes of H x W (plane p uses src + p*H*W and lam + (p / lam_div)*H*W)
 * for at most max_iters sweeps.  u_out [P][H][W], norms [max_iters][P]
 * (residual norm of plane p at iteration n in norms[(n-1)*P + p]), iters[P],
 * converged[P].  Returns 0, or the (1-based) iteration at which a plane went
 * non-finite (FloatingPointError in the reference), or -1 on bad arguments. */
int oracle_relaxed_solve(const double* src, const double* lam, int P, int lam_div, int H, int W,
                         int K, double sigma, double eps, double tau, int edge, int max_iters,
                         double rel_tol, double* u_out, double* norms, int* iters, int* converged,
                         int threads) {
  if (H < 2 || W < 2 || K < 1 || (K % 2) == 0 || P < 1 || lam_div < 1 || max_iters < 1)
    return -1;
  if (threads < 1) threads = 1;
  const int R = K / 2;
  const size_t n = (size_t)H * W;
  double* w = malloc(sizeof(double) * K);
  int* rx = malloc(sizeof(int) * (W + 2 * R));
  int* ry = malloc(sizeof(int) * (H + 2 * R));
  double* buf = malloc(sizeof(double) * n * 4 + sizeof(double) * H);
  double* alt = malloc(sizeof(double) * n);
  if (!w || !rx || !ry || !buf || !alt) return -1;
  taps_1d(sigma, K, w);
  for (int i = 0; i < W + 2 * R; ++i) rx[i] = reflect(i - R, W);
  for (int i = 0; i < H + 2 * R; ++i) ry[i] = reflect(i - R, H);
  Work k = {H, W, K, edge, eps, tau, w, rx, ry, buf, buf + n, buf + 2 * n, buf + 4 * n};
  int rc = 0;
  for (int p = 0; p < P && rc == 0; ++p) {
    const double* s = src + (size_t)p * n;
    const double* l = lam + (size_t)(p / lam_div) * n;
    double* u = u_out + (size_t)p * n;
    memcpy(u, s, sizeof(double) * n); /* u0 = Phi (solver.py:333) */
    double prev = -1.0;
    iters[p] = 0;
    converged[p] = 0;
    for (int it = 1; it <= max_iters; ++it) {
      const double s2 = sweep(&k, u, s, l, alt, threads);
      const double nrm = sqrt(s2);
      int finite = isfinite(nrm);
      for (size_t i = 0; i < n && finite; ++i) finite = isfinite(alt[i]);
      if (!finite) {
        rc = it;
        break;
      }
      memcpy(u, alt, sizeof(double) * n);
      norms[(size_t)(it - 1) * P + p] = nrm;
      iters[p] = it;
      if (prev >= 0.0 && fabs(nrm - prev) / fmax(prev, 1e-30) <= rel_tol) {
        converged[p] = 1;
        break;
      }
      prev = nrm;
    }
  }
  free(w);
  free(rx);
  free(ry);
  free(buf);
  free(alt);
  return rc;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}
