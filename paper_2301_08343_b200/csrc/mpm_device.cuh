// Device-side building blocks of the MLS-MPM substep (sm_100a).
//
// Each function restates one reference routine; file:line refer to
// /root/reference/proj. Matrices are row-major 3x3 (M(i,j) = m[3*i + j]).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace tacchi_b200 {

// Error codes; identical to include/tacchi_cuda.h TG_ERR_*.
enum : int {
  kOk = 0,
  kErrGridTooSmall = 1,
  kErrEmptyScene = 2,
  kErrOutOfGrid = 3,
  kErrDegenerateF = 4,
  kErrConfig = 5,
  kErrNoSurface = 6,
  kErrCropOutOfBounds = 7,
  kErrShapeMismatch = 8,
};

// Internal: a scatter would write outside the node arrays' allocation box;
// the host grows the allocation and re-runs from that substep (engine.cu).
constexpr int kErrRegrow = 250;
// Internal: a deterministic-mode node sum left the fixed-point range.
constexpr int kErrFixedRange = 249;
constexpr unsigned long long kNoError = ~0ull;
__host__ __device__ __forceinline__ unsigned long long err_key(int substep, int code) {
  return (static_cast<unsigned long long>(substep) << 8) | static_cast<unsigned>(code & 0xff);
}
__host__ __device__ __forceinline__ int err_code_of(unsigned long long k) {
  return k == kNoError ? 0 : static_cast<int>(k & 0xff);
}
__host__ __device__ __forceinline__ int err_substep_of(unsigned long long k) {
  return static_cast<int>(k >> 8);
}

// Particle tags (geo/particle_set.hpp:12).
enum : uint8_t { kElastomer = 0, kElastomerBottom = 1, kIndenter = 2 };

// Exact-rounding helpers: the reference is compiled without FMA contraction,
// so wherever a result feeds an integer decision (stencil base, window,
// in_range) or must be bit-identical (capture path) we spell the operations
// with the _rn intrinsics, which nvcc never fuses.
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// bspline.hpp:26-45 — quadratic B-spline stencil, node-centred convention.
struct Stencil {
  int base[3];
  double w[3][3];
  double fx[3];
};

__device__ __forceinline__ void make_stencil(double x0, double x1, double x2, const double* origin,
                                             double inv_dx, Stencil& st) {
  const double xs[3] = {x0, x1, x2};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double xn = mul_rn(sub_rn(xs[a], origin[a]), inv_dx);
    const double b = floor(sub_rn(xn, 0.5));
    st.base[a] = static_cast<int>(b);
    const double f = sub_rn(xn, b);
    st.fx[a] = f;
    const double t0 = sub_rn(1.5, f), t1 = sub_rn(f, 1.0), t2 = sub_rn(f, 0.5);
    st.w[a][0] = mul_rn(mul_rn(0.5, t0), t0);
    st.w[a][1] = sub_rn(0.75, mul_rn(t1, t1));
    st.w[a][2] = mul_rn(mul_rn(0.5, t2), t2);
  }
}

// Eigen's bruteforce 3x3 determinant expansion (engine.cpp:133 via Eigen).
__device__ __forceinline__ double det3(const double* m) {
  return m[0] * (m[4] * m[8] - m[5] * m[7]) - m[1] * (m[3] * m[8] - m[5] * m[6]) +
         m[2] * (m[3] * m[7] - m[4] * m[6]);
}

__device__ __forceinline__ void matmul3(const double* a, const double* b, double* o) {
  double t[9];
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      t[3 * i + j] = a[3 * i + 0] * b[0 + j] + a[3 * i + 1] * b[3 + j] + a[3 * i + 2] * b[6 + j];
#pragma unroll
  for (int i = 0; i < 9; ++i) o[i] = t[i];
}

// Rotation of the polar decomposition via a one-sided Jacobi SVD with the
// reflection fix (material.cpp:18-25). Only reached when the Newton iteration
// below fails, i.e. essentially never for a well-posed press.
static __device__ __noinline__ void polar_rotation_svd(const double* F, double* R) {
  double A[9], W[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
#pragma unroll
  for (int i = 0; i < 9; ++i) A[i] = F[i];
  const int ps[3] = {0, 0, 1}, qs[3] = {1, 2, 2};
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int r = 0; r < 3; ++r) {
      const int p = ps[r], q = qs[r];
      const double alpha = A[p] * A[p] + A[3 + p] * A[3 + p] + A[6 + p] * A[6 + p];
      const double beta = A[q] * A[q] + A[3 + q] * A[3 + q] + A[6 + q] * A[6 + q];
      const double gamma = A[p] * A[q] + A[3 + p] * A[3 + q] + A[6 + p] * A[6 + q];
      if (gamma == 0.0 || fabs(gamma) <= 1e-17 * sqrt(alpha * beta)) continue;
      rotated = true;
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
  for (int k = 0; k < 3; ++k) sig[k] = sqrt(A[k] * A[k] + A[3 + k] * A[3 + k] + A[6 + k] * A[6 + k]);
  int order[3] = {0, 1, 2};
  for (int a = 0; a < 3; ++a)
    for (int b = a + 1; b < 3; ++b)
      if (sig[order[b]] > sig[order[a]]) { const int t = order[a]; order[a] = order[b]; order[b] = t; }
  double U[9], V[9], ss[3];
  for (int k = 0; k < 3; ++k) {
    const int o = order[k];
    ss[k] = sig[o];
    for (int i = 0; i < 3; ++i) {
      V[3 * i + k] = W[3 * i + o];
      U[3 * i + k] = sig[o] > 1e-300 ? A[3 * i + o] / sig[o] : 0.0;
    }
  }
  for (int k = 0; k < 3; ++k) {
    if (ss[k] > 1e-300) continue;
    const int a = (k + 1) % 3, b = (k + 2) % 3;
    double c[3] = {U[3 + a] * U[6 + b] - U[6 + a] * U[3 + b], U[6 + a] * U[b] - U[a] * U[6 + b],
                   U[a] * U[3 + b] - U[3 + a] * U[b]};
    double n2 = c[0] * c[0] + c[1] * c[1] + c[2] * c[2];
    if (n2 == 0.0) { c[0] = k == 0; c[1] = k == 1; c[2] = k == 2; n2 = 1.0; }
    const double n = sqrt(n2);
    for (int i = 0; i < 3; ++i) U[3 * i + k] = c[i] / n;
  }
  double Vt[9], UVt[9];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) Vt[3 * i + j] = V[3 * j + i];
  matmul3(U, Vt, UVt);
  if (det3(UVt) < 0.0)
    for (int i = 0; i < 3; ++i) U[3 * i + 2] *= -1.0;
  matmul3(U, Vt, R);
}

// The SVD fallback through private copies: the caller's F and R arrays never
// have their address taken, so they stay in registers on the hot path (a
// noinline callee taking them directly forced both into local memory for
// every particle).
__device__ __forceinline__ void polar_svd_fallback(const double* F, double* R) {
  double f[9], r[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) f[i] = F[i];
  polar_rotation_svd(f, r);
#pragma unroll
  for (int i = 0; i < 9; ++i) R[i] = r[i];
}

// material.cpp:27-81 — scaled Newton iteration R <- (g R + R^-T / g) / 2 with
// the cofactor inverse; <= 40 iterations, stop when the max step < 1e-13;
// SVD fallback for a vanishing determinant or no convergence. Caller has
// already checked det(F) > 0.
__device__ __forceinline__ void polar_rotation(const double* F, double* R) {
  double r00 = F[0], r01 = F[1], r02 = F[2];
  double r10 = F[3], r11 = F[4], r12 = F[5];
  double r20 = F[6], r21 = F[7], r22 = F[8];
  // the SVD fallback is called once, after the loop (a call inside the loop
  // made every Newton value live across it)
  bool converged = false;
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
    if (!(fabs(d) > 1e-300)) break;  // vanishing determinant: SVD below
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
      converged = true;
      break;
    }
  }
  if (converged) {
    R[0] = r00; R[1] = r01; R[2] = r02;
    R[3] = r10; R[4] = r11; R[5] = r12;
    R[6] = r20; R[7] = r21; R[8] = r22;
    return;
  }
  polar_svd_fallback(F, R);
}

// corotated_stress (material.cpp:83-89) given R = polar_rotation(F) and
// J = det F: S = 2 mu (F - R) F^T + lambda (J - 1) J I.
__device__ __forceinline__ void corotated_stress(const double* F, const double* R, double J,
                                                 double mu, double lambda, double* S) {
  double A[9];
  const double s2mu = 2.0 * mu;
#pragma unroll
  for (int i = 0; i < 9; ++i) A[i] = s2mu * (F[i] - R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      S[3 * i + j] = A[3 * i] * F[3 * j] + A[3 * i + 1] * F[3 * j + 1] + A[3 * i + 2] * F[3 * j + 2];
  const double sl = lambda * (J - 1.0) * J;
  S[0] += sl;
  S[4] += sl;
  S[8] += sl;
}

// Order-preserving u64 encodings for atomicMin/atomicMax on doubles.
__device__ __forceinline__ unsigned long long order_key(double v) {
  const unsigned long long b = __double_as_longlong(v);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__host__ __device__ __forceinline__ double order_val(unsigned long long k) {
  const unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double(static_cast<long long>(b));
#else
  double d;
  __builtin_memcpy(&d, &b, sizeof d);
  return d;
#endif
}

}  // namespace tacchi_b200
