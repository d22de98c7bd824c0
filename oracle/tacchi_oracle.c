/* oracle/tacchi_oracle.c — TEST INFRASTRUCTURE ONLY (parity checker).
 *
 * Serial plain-C restatement of the reference hot path. Every function cites
 * the reference file:line it restates (paths relative to
 * /root/reference/proj). Arithmetic follows the reference expression order,
 * with the Eigen-subset conventions documented in oracle/eigen_shim/Eigen/Core
 * (left-to-right 3-term sums, Eigen's 3x3 determinant expansion). Compiled
 * with -ffp-contract=off so no FMA contraction changes the rounding.
 *
 * Pinned by tests/test_oracle_pin.py against the unmodified reference compiled
 * in oracle/_ref and against the committed fixtures in tests/golden/.
 * Never linked or called by the product path.
 */
#include "tacchi_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ERR_EMPTY_SCENE 2
#define ERR_OUT_OF_GRID 3
#define ERR_DEGENERATE_F 4
#define ERR_CONFIG 5
#define ERR_NO_SURFACE 6
#define ERR_CROP_OOB 7

static double det3(const double* m) { /* Eigen bruteforce_det3 order */
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

static void matmul(const double* a, const double* b, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = a[3 * i + 0] * b[0 + j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
  memcpy(o, t, sizeof t);
}

static void transpose(const double* a, double* o) {
  double t[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) t[3 * j + i] = a[3 * i + j];
  memcpy(o, t, sizeof t);
}

/* --- polar decomposition ------------------------------------------------ */

/* One-sided Jacobi SVD, singular values descending (the shim's JacobiSVD). */
static void svd3(const double* F, double* U, double* V) {
  double A[9], W[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
  memcpy(A, F, sizeof A);
#define COLDOT(M, p, q) (M[0 + (p)] * M[0 + (q)] + M[3 + (p)] * M[3 + (q)] + M[6 + (p)] * M[6 + (q)])
  static const int ps[3] = {0, 0, 1}, qs[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 60; ++sweep) {
    int rotated = 0;
    for (int r = 0; r < 3; ++r) {
      const int p = ps[r], q = qs[r];
      const double alpha = COLDOT(A, p, p), beta = COLDOT(A, q, q), gamma = COLDOT(A, p, q);
      if (gamma == 0.0 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
      rotated = 1;
      const double zeta = (beta - alpha) / (2.0 * gamma);
      const double t = (zeta >= 0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
      const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
      for (int i = 0; i < 3; ++i) {
        const double ap = A[3 * i + p], aq = A[3 * i + q];
        A[3 * i + p] = c * ap - s * aq;
        A[3 * i + q] = s * ap + c * aq;
        const double vp = W[3 * i + p], vq = W[3 * i + q];
        W[3 * i + p] = c * vp - s * vq;
        W[3 * i + q] = s * vp + c * vq;
      }
    }
    if (!rotated) break;
  }
  double sig[3];
  for (int k = 0; k < 3; ++k) sig[k] = sqrt(COLDOT(A, k, k));
#undef COLDOT
  int order[3] = {0, 1, 2};
  for (int a = 0; a < 3; ++a) /* stable insertion sort, descending */
    for (int b = a + 1; b < 3; ++b)
      if (sig[order[b]] > sig[order[a]]) { int t = order[a]; order[a] = order[b]; order[b] = t; }
  double s_sorted[3];
  for (int k = 0; k < 3; ++k) {
    const int o = order[k];
    s_sorted[k] = sig[o];
    for (int i = 0; i < 3; ++i) {
      V[3 * i + k] = W[3 * i + o];
      U[3 * i + k] = sig[o] > 1e-300 ? A[3 * i + o] / sig[o] : 0.0;
    }
  }
  for (int k = 0; k < 3; ++k) {
    if (s_sorted[k] > 1e-300) continue;
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    double c[3] = {U[3 + a] * U[6 + b] - U[6 + a] * U[3 + b], U[6 + a] * U[0 + b] - U[0 + a] * U[6 + b],
                   U[0 + a] * U[3 + b] - U[3 + a] * U[0 + b]};
    double n2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    if (n2 == 0.0) { c[0] = k == 0; c[1] = k == 1; c[2] = k == 2; n2 = 1.0; }
    const double n = sqrt(n2);
    for (int i = 0; i < 3; ++i) U[3 * i + k] = c[i] / n;
  }
}

/* material.cpp:18-25 */
int to_polar_rotation_svd(const double F[9], double R[9]) {
  if (!(det3(F) > 0.0)) return ERR_DEGENERATE_F;
  double U[9], V[9], Vt[9], UVt[9];
  svd3(F, U, V);
  transpose(V, Vt);
  matmul(U, Vt, UVt);
  if (det3(UVt) < 0.0)
    for (int i = 0; i < 3; ++i) U[3 * i + 2] *= -1.0;
  matmul(U, Vt, R);
  return 0;
}

/* material.cpp:27-81 — scaled Newton iteration with cofactor inverse. */
int to_polar_rotation(const double F[9], double R[9]) {
  const double det = det3(F);
  if (!(det > 0.0)) return ERR_DEGENERATE_F;
  double r00 = F[0], r01 = F[1], r02 = F[2];
  double r10 = F[3], r11 = F[4], r12 = F[5];
  double r20 = F[6], r21 = F[7], r22 = F[8];
  for (int it = 0; it < 40; ++it) {
    const double c00 = r11 * r22 - r12 * r21;
    const double c01 = r12 * r20 - r10 * r22;
    const double c02 = r10 * r21 - r11 * r20;
    const double c10 = r02 * r21 - r01 * r22;
    const double c11 = r00 * r22 - r02 * r20;
    const double c12 = r01 * r20 - r00 * r21;
    const double c20 = r01 * r12 - r02 * r11;
    const double c21 = r02 * r10 - r00 * r12;
    const double c22 = r00 * r11 - r01 * r10;
    const double d = r00 * c00 + r01 * c01 + r02 * c02;
    if (!(fabs(d) > 1e-300)) return to_polar_rotation_svd(F, R);
    const double g = fabs(d - 1.0) > 1e-2 ? 1.0 / cbrt(fabs(d)) : 1.0;
    const double hg = 0.5 * g;
    const double hd = 0.5 / (g * d);
    const double n00 = hg * r00 + hd * c00, n01 = hg * r01 + hd * c01, n02 = hg * r02 + hd * c02;
    const double n10 = hg * r10 + hd * c10, n11 = hg * r11 + hd * c11, n12 = hg * r12 + hd * c12;
    const double n20 = hg * r20 + hd * c20, n21 = hg * r21 + hd * c21, n22 = hg * r22 + hd * c22;
    double step = fabs(n00 - r00);
    step = fmax(step, fabs(n01 - r01));
    step = fmax(step, fabs(n02 - r02));
    step = fmax(step, fabs(n10 - r10));
    step = fmax(step, fabs(n11 - r11));
    step = fmax(step, fabs(n12 - r12));
    step = fmax(step, fabs(n20 - r20));
    step = fmax(step, fabs(n21 - r21));
    step = fmax(step, fabs(n22 - r22));
    r00 = n00; r01 = n01; r02 = n02;
    r10 = n10; r11 = n11; r12 = n12;
    r20 = n20; r21 = n21; r22 = n22;
    if (step < 1e-13) {
      R[0] = r00; R[1] = r01; R[2] = r02;
      R[3] = r10; R[4] = r11; R[5] = r12;
      R[6] = r20; R[7] = r21; R[8] = r22;
      return 0;
    }
  }
  return to_polar_rotation_svd(F, R);
}

/* engine.cpp:137-138 / material.cpp:83-89:
 * S = 2 mu (F - R) F^T + lambda (J - 1) J I. */
static void stress_from(const double* F, const double* R, double J, double mu, double lambda,
                        double* S) {
  double A[9], Ft[9];
  const double s2mu = 2.0 * mu;
  for (int i = 0; i < 9; ++i) A[i] = s2mu * (F[i] - R[i]);
  transpose(F, Ft);
  matmul(A, Ft, S);
  const double sl = lambda * (J - 1.0) * J;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) S[3 * i + j] = S[3 * i + j] + sl * (i == j ? 1.0 : 0.0);
}

int to_corotated_stress(const double F[9], double mu, double lambda, double S[9]) {
  const double J = det3(F);
  if (!(J > 0.0)) return ERR_DEGENERATE_F;
  double R[9];
  const int rc = to_polar_rotation(F, R);
  if (rc) return rc;
  stress_from(F, R, J, mu, lambda, S);
  return 0;
}

/* --- stencil -------------------------------------------------------------- */

/* bspline.hpp:26-45 */
void to_stencil(const double x[3], const double origin[3], double inv_dx, int base[3],
                double w[3][3], double fx[3]) {
  for (int a = 0; a < 3; ++a) {
    const double xn = (x[a] - origin[a]) * inv_dx;
    const double b = floor(xn - 0.5);
    base[a] = (int)b;
    fx[a] = xn - b;
    w[a][0] = 0.5 * (1.5 - fx[a]) * (1.5 - fx[a]);
    w[a][1] = 0.75 - (fx[a] - 1.0) * (fx[a] - 1.0);
    w[a][2] = 0.5 * (fx[a] - 0.5) * (fx[a] - 0.5);
  }
}

/* --- the six phases --------------------------------------------------------- */

static int base_index(double x, double origin, double inv_dx) { /* engine.cpp:47-49 */
  return (int)floor((x - origin) * inv_dx - 0.5);
}

/* engine.cpp:31-45 + 53-68 */
int to_window(const to_params* p, long n, const double* x, int lo[3], int hi[3]) {
  if (n <= 0) return ERR_EMPTY_SCENE;
  const double inv_dx = 1.0 / p->dx;
  for (int a = 0; a < 3; ++a) {
    double l = x[a], h = x[a];
    for (long q = 0; q < n; ++q) {
      l = fmin(l, x[3 * q + a]);
      h = fmax(h, x[3 * q + a]);
    }
    const int b0 = base_index(l, p->origin[a], inv_dx);
    const int b1 = base_index(h, p->origin[a], inv_dx);
    if (b0 < 0 || b1 + 2 >= p->res[a]) return ERR_OUT_OF_GRID;
    lo[a] = b0;
    hi[a] = b1 + 3;
  }
  return 0;
}

#define WIDX(lo, hi, i, j, k) \
  ((((size_t)((i) - (lo)[0])) * ((hi)[1] - (lo)[1]) + ((j) - (lo)[1])) * ((hi)[2] - (lo)[2]) + ((k) - (lo)[2]))

/* engine.cpp:107-178 (serial; the reference's slab order only changes the
 * summation order, which is bit-deterministic there and tolerance-level here). */
int to_p2g(const to_params* p, long n, const double* x, const double* v, const double* C,
           const double* F, const double* mass, const double* vol0, const uint8_t* tag,
           const int lo[3], const int hi[3], double* gmass, double* gmom, double* min_det_f) {
  const double inv_dx = 1.0 / p->dx;
  const double dx = p->dx;
  const double stress_scale = -p->dt * 4.0 * inv_dx * inv_dx;
  double mdf = 1.0;
  for (long q = 0; q < n; ++q) {
    int base[3];
    double w[3][3], fx[3];
    to_stencil(x + 3 * q, p->origin, inv_dx, base, w, fx);
    const double m = mass[q];
    double A[9];
    for (int i = 0; i < 9; ++i) A[i] = m * C[9 * q + i];
    if (tag[q] != TO_INDENTER) {
      const double* Fq = F + 9 * q;
      const double J = det3(Fq);
      if (!(J > 0.0)) return ERR_DEGENERATE_F;
      mdf = fmin(mdf, J);
      double R[9], S[9];
      const int rc = to_polar_rotation(Fq, R);
      if (rc) return rc;
      stress_from(Fq, R, J, p->mu, p->lambda, S);
      const double k = stress_scale * vol0[q];
      for (int i = 0; i < 9; ++i) A[i] = A[i] + k * S[i];
    }
    const double mv0 = m * v[3 * q], mv1 = m * v[3 * q + 1], mv2 = m * v[3 * q + 2];
    for (int a = 0; a < 3; ++a) {
      const double wa = w[0][a];
      const double dxa = (a - fx[0]) * dx;
      for (int b = 0; b < 3; ++b) {
        const double wab = wa * w[1][b];
        const double dxb = (b - fx[1]) * dx;
        const double m0 = mv0 + A[0] * dxa + A[1] * dxb;
        const double m1 = mv1 + A[3] * dxa + A[4] * dxb;
        const double m2 = mv2 + A[6] * dxa + A[7] * dxb;
        for (int c = 0; c < 3; ++c) {
          const double wt = wab * w[2][c];
          const double dxc = (c - fx[2]) * dx;
          const size_t node = WIDX(lo, hi, base[0] + a, base[1] + b, base[2] + c);
          gmass[node] += wt * m;
          gmom[3 * node + 0] += wt * (m0 + A[2] * dxc);
          gmom[3 * node + 1] += wt * (m1 + A[5] * dxc);
          gmom[3 * node + 2] += wt * (m2 + A[8] * dxc);
        }
      }
    }
  }
  *min_det_f = mdf;
  return 0;
}

/* engine.cpp:180-205 */
void to_grid_update(const to_params* p, const int lo[3], const int hi[3], const double* gmass,
                    const double* gmom, double* gvel) {
  const double gdt[3] = {p->gravity[0] * p->dt, p->gravity[1] * p->dt, p->gravity[2] * p->dt};
  const int with_g = (p->gravity[0] * p->gravity[0] + p->gravity[1] * p->gravity[1] +
                      p->gravity[2] * p->gravity[2]) > 0.0;
  for (int i = lo[0]; i < hi[0]; ++i)
    for (int j = lo[1]; j < hi[1]; ++j)
      for (int k = lo[2]; k < hi[2]; ++k) {
        const size_t nd = WIDX(lo, hi, i, j, k);
        double* vel = gvel + 3 * nd;
        if (gmass[nd] > 0.0) {
          for (int a = 0; a < 3; ++a) vel[a] = gmom[3 * nd + a] / gmass[nd];
          if (with_g)
            for (int a = 0; a < 3; ++a) vel[a] = vel[a] + gdt[a];
          if (i == 0 || i == p->res[0] - 1) vel[0] = 0.0;
          if (j == 0 || j == p->res[1] - 1) vel[1] = 0.0;
          if (k == 0 || k == p->res[2] - 1) vel[2] = 0.0;
        } else {
          vel[0] = vel[1] = vel[2] = 0.0;
        }
      }
}

/* engine.cpp:207-252 */
void to_g2p(const to_params* p, long n, const double* x, double* v, double* C, double* F,
            const uint8_t* tag, const int lo[3], const int hi[3], const double* gvel) {
  const double inv_dx = 1.0 / p->dx;
  const double dt = p->dt;
  for (long q = 0; q < n; ++q) {
    if (tag[q] == TO_INDENTER) continue;
    int base[3];
    double w[3][3], fx[3];
    to_stencil(x + 3 * q, p->origin, inv_dx, base, w, fx);
    double v0 = 0, v1 = 0, v2 = 0;
    double b00 = 0, b01 = 0, b02 = 0, b10 = 0, b11 = 0, b12 = 0, b20 = 0, b21 = 0, b22 = 0;
    for (int a = 0; a < 3; ++a) {
      const double wa = w[0][a];
      const double da = a - fx[0];
      for (int b = 0; b < 3; ++b) {
        const double wab = wa * w[1][b];
        const double db = b - fx[1];
        for (int c = 0; c < 3; ++c) {
          const double wt = wab * w[2][c];
          const double dc = c - fx[2];
          const double* vel = gvel + 3 * WIDX(lo, hi, base[0] + a, base[1] + b, base[2] + c);
          const double wv0 = wt * vel[0], wv1 = wt * vel[1], wv2 = wt * vel[2];
          v0 += wv0; v1 += wv1; v2 += wv2;
          b00 += wv0 * da; b01 += wv0 * db; b02 += wv0 * dc;
          b10 += wv1 * da; b11 += wv1 * db; b12 += wv1 * dc;
          b20 += wv2 * da; b21 += wv2 * db; b22 += wv2 * dc;
        }
      }
    }
    v[3 * q] = v0; v[3 * q + 1] = v1; v[3 * q + 2] = v2;
    const double k = 4.0 * inv_dx;
    double* Cq = C + 9 * q;
    Cq[0] = k * b00; Cq[1] = k * b01; Cq[2] = k * b02;
    Cq[3] = k * b10; Cq[4] = k * b11; Cq[5] = k * b12;
    Cq[6] = k * b20; Cq[7] = k * b21; Cq[8] = k * b22;
    double G[9];
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j) G[3 * i + j] = (i == j ? 1.0 : 0.0) + dt * Cq[3 * i + j];
    matmul(G, F + 9 * q, F + 9 * q);
  }
}

/* engine.cpp:254-266 */
void to_apply_boundary(long n, double* v, const uint8_t* tag, const double vind[3]) {
  for (long q = 0; q < n; ++q) {
    if (tag[q] == TO_INDENTER) {
      v[3 * q] = vind[0]; v[3 * q + 1] = vind[1]; v[3 * q + 2] = vind[2];
    } else if (tag[q] == TO_ELASTOMER_BOTTOM) {
      v[3 * q] = v[3 * q + 1] = v[3 * q + 2] = 0.0;
    }
  }
}

/* grid.cpp:29-36 (note: divides by dx, unlike base_index) */
static int in_range(const to_params* p, const double* x) {
  for (int a = 0; a < 3; ++a) {
    const double xn = (x[a] - p->origin[a]) / p->dx;
    const int b = (int)floor(xn - 0.5);
    if (b < 0 || b + 2 >= p->res[a]) return 0;
  }
  return 1;
}

/* engine.cpp:268-286 */
int to_advect(const to_params* p, long n, double* x, const double* v, double* max_speed) {
  double max_v2 = 0.0;
  for (long q = 0; q < n; ++q) {
    for (int a = 0; a < 3; ++a) x[3 * q + a] = x[3 * q + a] + p->dt * v[3 * q + a];
    const double s2 = v[3 * q] * v[3 * q] + v[3 * q + 1] * v[3 * q + 1] + v[3 * q + 2] * v[3 * q + 2];
    max_v2 = fmax(max_v2, s2);
  }
  *max_speed = sqrt(max_v2);
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = x[a];
    hi[a] = x[a];
    for (long q = 0; q < n; ++q) {
      lo[a] = fmin(lo[a], x[3 * q + a]);
      hi[a] = fmax(hi[a], x[3 * q + a]);
    }
  }
  if (!in_range(p, lo) || !in_range(p, hi)) return ERR_OUT_OF_GRID;
  return 0;
}

/* engine.cpp:288-297 */
int to_step(const to_params* p, long n, double* x, double* v, double* C, double* F,
            const double* mass, const double* vol0, const uint8_t* tag, const double vind[3],
            int n_substeps, to_diag* diag) {
  for (int s = 0; s < n_substeps; ++s) {
    int lo[3], hi[3];
    int rc = to_window(p, n, x, lo, hi);
    if (rc) return rc;
    const size_t nn = (size_t)(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
    double* gm = (double*)calloc(nn, sizeof(double));
    double* gp = (double*)calloc(3 * nn, sizeof(double));
    double* gv = (double*)calloc(3 * nn, sizeof(double));
    double mdf;
    rc = to_p2g(p, n, x, v, C, F, mass, vol0, tag, lo, hi, gm, gp, &mdf);
    if (!rc) {
      diag->min_det_f = mdf;
      to_grid_update(p, lo, hi, gm, gp, gv);
      to_g2p(p, n, x, v, C, F, tag, lo, hi, gv);
      to_apply_boundary(n, v, tag, vind);
      ++diag->step_count;
      rc = to_advect(p, n, x, v, &diag->max_speed);
    }
    free(gm);
    free(gp);
    free(gv);
    if (rc) return rc;
  }
  return 0;
}

/* --- render ------------------------------------------------------------------ */

/* depth_extract.cpp:10-49; geom = {x0, y0, sx, sy, z0}. */
int to_extract_depth(int nx, int ny, const double geom[5], const uint32_t* surf_idx,
                     const double* x, int w, int h, double r, double* out) {
  if (nx < 2 || ny < 2 || !surf_idx) return ERR_NO_SURFACE;
  if (w < 2 || h < 2 || !(r > 0.0)) return ERR_CONFIG;
  const double x0 = geom[0], y0 = geom[1], sx = geom[2], sy = geom[3], z0 = geom[4];
  double* dg = (double*)malloc(sizeof(double) * (size_t)nx * ny);
  for (size_t s = 0; s < (size_t)nx * ny; ++s) dg[s] = z0 - x[3 * (size_t)surf_idx[s] + 2];
  const double cx = x0 + 0.5 * (nx - 1) * sx;
  const double cy = y0 + 0.5 * (ny - 1) * sy;
  for (int v = 0; v < h; ++v) {
    const double y = cy + (v - 0.5 * (h - 1)) * r;
    double gj = (y - y0) / sy;
    gj = gj < 0.0 ? 0.0 : (gj > ny - 1.0 ? ny - 1.0 : gj);
    int j0 = (int)gj;
    if (j0 > ny - 2) j0 = ny - 2;
    const double fj = gj - j0;
    for (int u = 0; u < w; ++u) {
      const double xx = cx + (u - 0.5 * (w - 1)) * r;
      double gi = (xx - x0) / sx;
      gi = gi < 0.0 ? 0.0 : (gi > nx - 1.0 ? nx - 1.0 : gi);
      int i0 = (int)gi;
      if (i0 > nx - 2) i0 = nx - 2;
      const double fi = gi - i0;
      const double d00 = dg[(size_t)i0 * ny + j0];
      const double d10 = dg[(size_t)(i0 + 1) * ny + j0];
      const double d01 = dg[(size_t)i0 * ny + j0 + 1];
      const double d11 = dg[(size_t)(i0 + 1) * ny + j0 + 1];
      out[(size_t)v * w + u] = (1 - fj) * ((1 - fi) * d00 + fi * d10) + fj * ((1 - fi) * d01 + fi * d11);
    }
  }
  free(dg);
  return 0;
}

/* depth_extract.cpp:51-57 */
void to_full_depth_size(int nx, int ny, const double geom[5], double r, int* w, int* h) {
  *w = (int)ceil((nx - 1) * geom[2] / r) + 1;
  *h = (int)ceil((ny - 1) * geom[3] / r) + 1;
}

/* depth_map.cpp:62-101 */
int to_crop_align(const double* src, int sw, int sh, double off_x, double off_y, double scale,
                  int ow, int oh, double* out) {
  if (!(scale > 0.0)) return ERR_CONFIG;
  const double cx_src = 0.5 * (sw - 1), cy_src = 0.5 * (sh - 1);
  const double cx_out = 0.5 * (ow - 1), cy_out = 0.5 * (oh - 1);
  for (int corner = 0; corner < 4; ++corner) {
    const double u = (corner & 1) ? ow - 1 : 0;
    const double v = (corner & 2) ? oh - 1 : 0;
    const double sx = cx_src + scale * (u - cx_out) + off_x;
    const double sy = cy_src + scale * (v - cy_out) + off_y;
    if (sx < -1e-9 || sx > sw - 1 + 1e-9 || sy < -1e-9 || sy > sh - 1 + 1e-9) return ERR_CROP_OOB;
  }
  for (int v = 0; v < oh; ++v) {
    double sy = cy_src + scale * (v - cy_out) + off_y;
    sy = sy < 0.0 ? 0.0 : (sy > (double)(sh - 1) ? (double)(sh - 1) : sy);
    int y0 = (int)sy;
    if (y0 > sh - 2) y0 = sh - 2;
    const double fy = sy - y0;
    for (int u = 0; u < ow; ++u) {
      double sx = cx_src + scale * (u - cx_out) + off_x;
      sx = sx < 0.0 ? 0.0 : (sx > (double)(sw - 1) ? (double)(sw - 1) : sx);
      int x0 = (int)sx;
      if (x0 > sw - 2) x0 = sw - 2;
      const double fx = sx - x0;
      const double d00 = src[(size_t)y0 * sw + x0], d01 = src[(size_t)y0 * sw + x0 + 1];
      const double d10 = src[(size_t)(y0 + 1) * sw + x0], d11 = src[(size_t)(y0 + 1) * sw + x0 + 1];
      out[(size_t)v * ow + u] = (1 - fy) * ((1 - fx) * d00 + fx * d01) + fy * ((1 - fx) * d10 + fx * d11);
    }
  }
  return 0;
}

/* phong.cpp:10-41 */
int to_surface_normals(const double* d, int w, int h, double r, double* out) {
  if (!(r > 0.0)) return ERR_CONFIG;
  const double inv_2r = 1.0 / (2.0 * r);
  const double inv_r = 1.0 / r;
#define H(row, col) (-d[(size_t)(row) * w + (col)])
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      double gx, gy;
      if (u == 0) gx = (H(v, 1) - H(v, 0)) * inv_r;
      else if (u == w - 1) gx = (H(v, u) - H(v, u - 1)) * inv_r;
      else gx = (H(v, u + 1) - H(v, u - 1)) * inv_2r;
      if (v == 0) gy = (H(1, u) - H(0, u)) * inv_r;
      else if (v == h - 1) gy = (H(v, u) - H(v - 1, u)) * inv_r;
      else gy = (H(v + 1, u) - H(v - 1, u)) * inv_2r;
      const double nrm = sqrt(gx * gx + gy * gy + (-1.0) * (-1.0));
      double* o = out + 3 * ((size_t)v * w + u);
      o[0] = gx / nrm;
      o[1] = gy / nrm;
      o[2] = -1.0 / nrm;
    }
#undef H
  return 0;
}

static void normalize3(double* v) {
  const double n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (n2 > 0.0) {
    const double n = sqrt(n2);
    v[0] /= n; v[1] /= n; v[2] /= n;
  }
}

/* phong.cpp:43-84 */
int to_phong(const double* depth, int w, int h, double r, const double* lights, int n_lights,
             const double rp[10], const uint8_t* bg, uint8_t* out) {
  if (n_lights < 1) return ERR_CONFIG;
  double* nm = (double*)malloc(sizeof(double) * 3 * (size_t)w * h);
  int rc = to_surface_normals(depth, w, h, r, nm);
  if (rc) { free(nm); return rc; }
  const double ka = rp[0], kd = rp[1], ks = rp[2], alpha = rp[3];
  double view[3] = {rp[7], rp[8], rp[9]};
  normalize3(view);
  double* L = (double*)malloc(sizeof(double) * 9 * n_lights);
  memcpy(L, lights, sizeof(double) * 9 * n_lights);
  for (int l = 0; l < n_lights; ++l) normalize3(L + 9 * l);
  for (int v = 0; v < h; ++v)
    for (int u = 0; u < w; ++u) {
      const size_t px = (size_t)v * w + u;
      const double* n = nm + 3 * px;
      double col[3];
      for (int c = 0; c < 3; ++c)
        col[c] = bg ? ka * (bg[3 * px + c] / 255.0) : ka * rp[4 + c];
      for (int l = 0; l < n_lights; ++l) {
        const double* dir = L + 9 * l;
        const double ln = dir[0] * n[0] + dir[1] * n[1] + dir[2] * n[2];
        if (ln <= 0.0) continue;
        const double kdl = kd * ln;
        for (int c = 0; c < 3; ++c) col[c] = col[c] + kdl * dir[3 + c];
        const double t = 2.0 * ln;
        const double rr[3] = {t * n[0] - dir[0], t * n[1] - dir[1], t * n[2] - dir[2]};
        const double rv = rr[0] * view[0] + rr[1] * view[1] + rr[2] * view[2];
        if (rv > 0.0) {
          const double sp = ks * pow(rv, alpha);
          for (int c = 0; c < 3; ++c) col[c] = col[c] + sp * dir[6 + c];
        }
      }
      for (int c = 0; c < 3; ++c) {
        const double cc = col[c] < 0.0 ? 0.0 : (col[c] > 1.0 ? 1.0 : col[c]);
        out[3 * px + c] = (uint8_t)lround(cc * 255.0);
      }
    }
  free(L);
  free(nm);
  return 0;
}
