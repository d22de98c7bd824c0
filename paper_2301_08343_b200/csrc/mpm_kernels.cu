// MLS-MPM substep kernels for sm_100a.
//
// One substep (mpm::step body, engine.cpp:289-296) is launched as
//   k_clear      zero_grid's clear of prev ∪ new window (engine.cpp:70-85)
//   k_p2g_gel    particle_to_grid for elastomer particles: det F, Newton polar,
//                corotated stress, APIC affine, 27-node RED.F64 scatter
//                (engine.cpp:107-178, material.cpp:27-89)
//   k_p2g_ind    particle_to_grid for the rigid indenter cloud (C = 0, no
//                stress, engine.cpp:131)
//   k_grid_update  v = p / m (+ g dt), zero normal velocity on the domain
//                faces, 0 where m = 0 (engine.cpp:180-205)
//   k_g2p_gel    grid_to_particle + apply_boundary + advect for elastomer
//                particles (engine.cpp:207-252, 254-266, 268-279), fused, with
//                the bbox / max-speed reductions of advect
//   k_ind_move   apply_boundary + advect for the indenter (engine.cpp:260-261)
//   k_finalize   advect's in_range check and step_count, then the next
//                substep's zero_grid window (engine.cpp:53-68, 280-285)
// Errors are latched in Ctl::err_code and every later kernel of the substep
// exits early, which reproduces the reference's "state at the throwing phase".
#include "engine.cuh"

namespace tacchi_b200 {

namespace {

__device__ __forceinline__ void raise(Ctl* ctl, int code, int substep) {
  if (atomicCAS(&ctl->err_code, 0, code) == 0) ctl->err_substep = substep;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// advect's reductions: max |v|^2 and the bbox of x (engine.cpp:273-282).
// Warp shuffles, then one shared-memory pass per block, then 7 atomics per
// block (a per-warp atomic on 7 hot words serialises badly at 1e6 particles).
// Every thread of the block must call this (no early exits before it).
__device__ __forceinline__ void reduce_motion(Ctl* ctl, bool active, double v2, double x0,
                                              double x1, double x2) {
  __shared__ double red[7][32];
  double r[7];
  r[0] = active ? v2 : 0.0;
  r[1] = active ? x0 : INFINITY;
  r[2] = active ? x1 : INFINITY;
  r[3] = active ? x2 : INFINITY;
  r[4] = active ? x0 : -INFINITY;
  r[5] = active ? x1 : -INFINITY;
  r[6] = active ? x2 : -INFINITY;
  r[0] = warp_max(r[0]);
#pragma unroll
  for (int a = 1; a < 4; ++a) r[a] = warp_min(r[a]);
#pragma unroll
  for (int a = 4; a < 7; ++a) r[a] = warp_max(r[a]);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = (blockDim.x + 31) >> 5;
  if (lane == 0)
#pragma unroll
    for (int a = 0; a < 7; ++a) red[a][warp] = r[a];
  __syncthreads();
  if (warp == 0) {
#pragma unroll
    for (int a = 0; a < 7; ++a) {
      const double ident = a == 0 ? 0.0 : (a < 4 ? INFINITY : -INFINITY);
      r[a] = lane < nwarps ? red[a][lane] : ident;
    }
    r[0] = warp_max(r[0]);
#pragma unroll
    for (int a = 1; a < 4; ++a) r[a] = warp_min(r[a]);
#pragma unroll
    for (int a = 4; a < 7; ++a) r[a] = warp_max(r[a]);
    if (lane == 0 && r[1] <= r[4]) {
      atomicMax(&ctl->max_v2, static_cast<unsigned long long>(__double_as_longlong(r[0])));
      atomicMin(&ctl->bb_lo[0], order_key(r[1]));
      atomicMin(&ctl->bb_lo[1], order_key(r[2]));
      atomicMin(&ctl->bb_lo[2], order_key(r[3]));
      atomicMax(&ctl->bb_hi[0], order_key(r[4]));
      atomicMax(&ctl->bb_hi[1], order_key(r[5]));
      atomicMax(&ctl->bb_hi[2], order_key(r[6]));
    }
  }
}

__device__ __forceinline__ size_t node_index(const Geometry& g, int i, int j, int k) {
  return (static_cast<size_t>(i) * g.res[1] + j) * g.res[2] + k;
}

__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

}  // namespace

// bbox of all positions (particle_bbox, engine.cpp:31-45), for a fresh window.
__global__ void k_bbox(const double* __restrict__ x, int64_t n, Ctl* ctl) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n;
  reduce_motion(ctl, active, 0.0, active ? x[p] : 0.0, active ? x[n + p] : 0.0,
                active ? x[2 * n + p] : 0.0);
}

__global__ void k_reset(Ctl* ctl) {
  for (int a = 0; a < 3; ++a) {
    ctl->bb_lo[a] = order_key(INFINITY);
    ctl->bb_hi[a] = order_key(-INFINITY);
  }
  ctl->max_v2 = 0ull;
  ctl->min_detf = order_key(1.0);
}

enum : int { kFinAdvect = 1, kFinWindow = 2, kFinDiag = 4 };

// grid.cpp:29-36: in_range divides by dx.
__device__ bool in_range(const Geometry& g, const double* x) {
  for (int a = 0; a < 3; ++a) {
    const double xn = div_rn(sub_rn(x[a], g.origin[a]), g.dx);
    const int b = static_cast<int>(floor(sub_rn(xn, 0.5)));
    if (b < 0 || b + 2 >= g.res[a]) return false;
  }
  return true;
}

__global__ void k_finalize(Ctl* ctl, Geometry g, int mode) {
  if (ctl->err_code) return;
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = order_val(ctl->bb_lo[a]);
    hi[a] = order_val(ctl->bb_hi[a]);
  }
  if (mode & kFinDiag) {  // particle_to_grid's min_det_f (engine.cpp:177)
    ctl->diag_min_det_f = order_val(ctl->min_detf);
    ctl->min_detf = order_key(1.0);
  }
  if (mode & kFinAdvect) {
    // engine.cpp:279-285
    ctl->diag_max_speed = sqrt(__longlong_as_double(static_cast<long long>(ctl->max_v2)));
    ctl->step_count += 1;
    const int s = ctl->substep;
    ctl->substep = s + 1;
    if (!in_range(g, lo) || !in_range(g, hi)) {
      raise(ctl, kErrOutOfGrid, s);
      return;
    }
  }
  if (mode & kFinWindow) {
    // engine.cpp:60-85 — window [base(lo), base(hi) + 3); clear prev ∪ new.
    int wlo[3], whi[3];
    for (int a = 0; a < 3; ++a) {
      const int b0 = static_cast<int>(floor(sub_rn(mul_rn(sub_rn(lo[a], g.origin[a]), g.inv_dx), 0.5)));
      const int b1 = static_cast<int>(floor(sub_rn(mul_rn(sub_rn(hi[a], g.origin[a]), g.inv_dx), 0.5)));
      if (b0 < 0 || b1 + 2 >= g.res[a]) {
        raise(ctl, kErrOutOfGrid, ctl->substep);
        return;
      }
      wlo[a] = b0;
      whi[a] = b1 + 3;
    }
    int pmin = 1 << 30;
    for (int a = 0; a < 3; ++a) pmin = min(pmin, ctl->prev_hi[a] - ctl->prev_lo[a]);
    for (int a = 0; a < 3; ++a) {
      ctl->clr_lo[a] = pmin <= 0 ? wlo[a] : min(wlo[a], ctl->prev_lo[a]);
      ctl->clr_hi[a] = pmin <= 0 ? whi[a] : max(whi[a], ctl->prev_hi[a]);
      ctl->win_lo[a] = ctl->prev_lo[a] = wlo[a];
      ctl->win_hi[a] = ctl->prev_hi[a] = whi[a];
    }
  }
  for (int a = 0; a < 3; ++a) {
    ctl->bb_lo[a] = order_key(INFINITY);
    ctl->bb_hi[a] = order_key(-INFINITY);
  }
  ctl->max_v2 = 0ull;
}

// Clear of Grid::mass / momentum over Ctl::clr box (engine.cpp:72-83).
__global__ void k_clear(double4* __restrict__ grid, Ctl* ctl, Geometry g) {
  if (ctl->err_code) return;
  const int lx = ctl->clr_lo[0], ly = ctl->clr_lo[1], lz = ctl->clr_lo[2];
  const int ny = ctl->clr_hi[1] - ly, nz = ctl->clr_hi[2] - lz;
  const int64_t total = static_cast<int64_t>(ctl->clr_hi[0] - lx) * ny * nz;
  const double4 z = make_double4(0, 0, 0, 0);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(t % nz);
    const int64_t r = t / nz;
    const int j = static_cast<int>(r % ny);
    const int i = static_cast<int>(r / ny);
    grid[node_index(g, lx + i, ly + j, lz + k)] = z;
  }
}

// particle_to_grid for elastomer particles (engine.cpp:126-168).
__global__ void __launch_bounds__(256) k_p2g_gel(const double* __restrict__ x,
                                                 const double* __restrict__ v,
                                                 const double* __restrict__ Cm,
                                                 const double* __restrict__ Fm, int64_t n,
                                                 int64_t n_el, Ctl* ctl, Geometry g,
                                                 double4* __restrict__ grid, double m,
                                                 double vol0) {
  if (ctl->err_code) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n_el;
  double F[9];
  double J = 1.0;
  if (active) {
#pragma unroll
    for (int i = 0; i < 9; ++i) F[i] = Fm[i * n_el + p];
    J = det3(F);
  }
  // StepDiagnostics::min_det_f, seeded with 1.0 (engine.cpp:119,135).
  const bool bad = active && !(J > 0.0);
  if (__any_sync(0xffffffffu, bad)) {
    if (bad) raise(ctl, kErrDegenerateF, ctl->substep);
    return;
  }
  const double wmin = warp_min(active ? J : 1.0);
  if ((threadIdx.x & 31) == 0) atomicMin(&ctl->min_detf, order_key(wmin));
  if (!active) return;

  Stencil st;
  make_stencil(x[p], x[n + p], x[2 * n + p], g.origin, g.inv_dx, st);
  double R[9];
  polar_rotation(F, R);
  // S = 2 mu (F - R) F^T + lambda (J - 1) J I   (engine.cpp:137-138)
  double A[9], S[9];
  const double s2mu = 2.0 * g.mu;
#pragma unroll
  for (int i = 0; i < 9; ++i) A[i] = s2mu * (F[i] - R[i]);
#pragma unroll
  for (int i = 0; i < 3; ++i)
#pragma unroll
    for (int j = 0; j < 3; ++j)
      S[3 * i + j] = A[3 * i] * F[3 * j] + A[3 * i + 1] * F[3 * j + 1] + A[3 * i + 2] * F[3 * j + 2];
  const double sl = g.lambda * (J - 1.0) * J;
  S[0] += sl; S[4] += sl; S[8] += sl;
  // affine = m C + (-dt 4/dx^2 V0) S   (engine.cpp:130,139)
  const double ks = g.stress_scale * vol0;
  double aff[9];
#pragma unroll
  for (int i = 0; i < 9; ++i) aff[i] = m * Cm[i * n_el + p] + ks * S[i];
  const double mv0 = m * v[p], mv1 = m * v[n + p], mv2 = m * v[2 * n + p];
  const double dx = g.dx;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double wa = st.w[0][a];
    const double dxa = (a - st.fx[0]) * dx;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double wab = wa * st.w[1][b];
      const double dxb = (b - st.fx[1]) * dx;
      const double m0 = mv0 + aff[0] * dxa + aff[1] * dxb;
      const double m1 = mv1 + aff[3] * dxa + aff[4] * dxb;
      const double m2 = mv2 + aff[6] * dxa + aff[7] * dxb;
      double* row = reinterpret_cast<double*>(
          grid + node_index(g, st.base[0] + a, st.base[1] + b, st.base[2]));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = wab * st.w[2][c];
        const double dxc = (c - st.fx[2]) * dx;
        red_add(row + 4 * c + 0, w * m);
        red_add(row + 4 * c + 1, w * (m0 + aff[2] * dxc));
        red_add(row + 4 * c + 2, w * (m1 + aff[5] * dxc));
        red_add(row + 4 * c + 3, w * (m2 + aff[8] * dxc));
      }
    }
  }
}

// particle_to_grid for the rigid indenter (engine.cpp:126-168 with C = 0 and
// no stress, engine.cpp:131): affine = m C = 0, so each node receives
// w m and w m v. Direct RED.F64 scatter (baseline variant).
__global__ void __launch_bounds__(256) k_p2g_ind(const double* __restrict__ x,
                                                 const double* __restrict__ v, int64_t n,
                                                 int64_t n_el, Ctl* ctl, Geometry g,
                                                 double4* __restrict__ grid, double m) {
  if (ctl->err_code) return;
  const int64_t p = n_el + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  Stencil st;
  make_stencil(x[p], x[n + p], x[2 * n + p], g.origin, g.inv_dx, st);
  const double mv0 = m * v[p], mv1 = m * v[n + p], mv2 = m * v[2 * n + p];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double wa = st.w[0][a];
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double wab = wa * st.w[1][b];
      double* row = reinterpret_cast<double*>(
          grid + node_index(g, st.base[0] + a, st.base[1] + b, st.base[2]));
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = wab * st.w[2][c];
        red_add(row + 4 * c + 0, w * m);
        red_add(row + 4 * c + 1, w * mv0);
        red_add(row + 4 * c + 2, w * mv1);
        red_add(row + 4 * c + 3, w * mv2);
      }
    }
  }
}

// particle_to_grid for the rigid indenter when every indenter particle carries
// the same velocity (always true after the first apply_boundary,
// engine.cpp:260-261). Each node then receives (sum_p w_p m) (1, v): the
// scatter reduces to one weight sum per node. Particles are ordered by base
// cell (bx, by) then z at creation, so a thread walking kChunk consecutive
// particles sees long runs of one base cell; it accumulates the 27 weight
// sums in registers and issues the 27 x 4 REDs only when the base changes.
// This cuts the RED.F64 count by ~the particles-per-cell density (~19 for the
// 1e6-point sphere).
template <int kChunk>
__global__ void __launch_bounds__(256) k_p2g_ind_chunk(const double* __restrict__ x, int64_t n,
                                                       int64_t n_el, Ctl* ctl, Geometry g,
                                                       double4* __restrict__ grid, double m) {
  if (ctl->err_code) return;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t p0 = n_el + t * kChunk;
  if (p0 >= n) return;
  const int64_t p1 = p0 + kChunk < n ? p0 + kChunk : n;
  const double mv0 = m * ctl->ind_v[0], mv1 = m * ctl->ind_v[1], mv2 = m * ctl->ind_v[2];
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0.0;
  int cb0 = 0, cb1 = 0, cb2 = 0;
  bool have = false;
  auto flush = [&]() {
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        double* row = reinterpret_cast<double*>(grid + node_index(g, cb0 + a, cb1 + b, cb2));
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double w = acc[9 * a + 3 * b + c];
          if (w != 0.0) {
            red_add(row + 4 * c + 0, w * m);
            red_add(row + 4 * c + 1, w * mv0);
            red_add(row + 4 * c + 2, w * mv1);
            red_add(row + 4 * c + 3, w * mv2);
          }
          acc[9 * a + 3 * b + c] = 0.0;
        }
      }
  };
  for (int64_t p = p0; p < p1; ++p) {
    Stencil st;
    make_stencil(x[p], x[n + p], x[2 * n + p], g.origin, g.inv_dx, st);
    if (have && (st.base[0] != cb0 || st.base[1] != cb1 || st.base[2] != cb2)) flush();
    cb0 = st.base[0];
    cb1 = st.base[1];
    cb2 = st.base[2];
    have = true;
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double wab = st.w[0][a] * st.w[1][b];
#pragma unroll
        for (int c = 0; c < 3; ++c) acc[9 * a + 3 * b + c] += wab * st.w[2][c];
      }
  }
  flush();
}

// grid_update over the active window (engine.cpp:180-205).
__global__ void k_grid_update(const double4* __restrict__ mp, double4* __restrict__ vel, Ctl* ctl,
                              Geometry g) {
  if (ctl->err_code) return;
  const int lx = ctl->win_lo[0], ly = ctl->win_lo[1], lz = ctl->win_lo[2];
  const int ny = ctl->win_hi[1] - ly, nz = ctl->win_hi[2] - lz;
  const int64_t total = static_cast<int64_t>(ctl->win_hi[0] - lx) * ny * nz;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = lz + static_cast<int>(t % nz);
    const int64_t r = t / nz;
    const int j = ly + static_cast<int>(r % ny);
    const int i = lx + static_cast<int>(r / ny);
    const size_t nd = node_index(g, i, j, k);
    const double4 q = mp[nd];
    double4 o = make_double4(0, 0, 0, 0);
    if (q.x > 0.0) {
      o.x = q.y / q.x;
      o.y = q.z / q.x;
      o.z = q.w / q.x;
      if (g.with_gravity) {
        o.x = o.x + g.gdt[0];
        o.y = o.y + g.gdt[1];
        o.z = o.z + g.gdt[2];
      }
      if (i == 0 || i == g.res[0] - 1) o.x = 0.0;
      if (j == 0 || j == g.res[1] - 1) o.y = 0.0;
      if (k == 0 || k == g.res[2] - 1) o.z = 0.0;
    }
    vel[nd] = o;
  }
}

// grid_to_particle (engine.cpp:217-251), optionally fused with
// apply_boundary's bottom pin (engine.cpp:262-263) and advect
// (engine.cpp:275-279).
template <bool kBoundary, bool kAdvect>
__global__ void __launch_bounds__(256) k_g2p_gel(double* __restrict__ x, double* __restrict__ v,
                                                 double* __restrict__ Cm, double* __restrict__ Fm,
                                                 const uint8_t* __restrict__ tag, int64_t n,
                                                 int64_t n_el, Ctl* ctl, Geometry g,
                                                 const double4* __restrict__ vel) {
  if (ctl->err_code) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n_el;
  double px0 = 0, px1 = 0, px2 = 0, v2 = 0;
  if (active) {
    px0 = x[p];
    px1 = x[n + p];
    px2 = x[2 * n + p];
    Stencil st;
    make_stencil(px0, px1, px2, g.origin, g.inv_dx, st);
    double v0 = 0, v1 = 0, vz = 0;
    double b00 = 0, b01 = 0, b02 = 0, b10 = 0, b11 = 0, b12 = 0, b20 = 0, b21 = 0, b22 = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double wa = st.w[0][a];
      const double da = a - st.fx[0];
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double wab = wa * st.w[1][b];
        const double db = b - st.fx[1];
        const double4* row = vel + node_index(g, st.base[0] + a, st.base[1] + b, st.base[2]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
          const double w = wab * st.w[2][c];
          const double dc = c - st.fx[2];
          const double2* q2 = reinterpret_cast<const double2*>(row + c);
          const double2 qa = __ldg(q2), qb = __ldg(q2 + 1);
          const double wv0 = w * qa.x, wv1 = w * qa.y, wv2 = w * qb.x;
          v0 += wv0; v1 += wv1; vz += wv2;
          b00 += wv0 * da; b01 += wv0 * db; b02 += wv0 * dc;
          b10 += wv1 * da; b11 += wv1 * db; b12 += wv1 * dc;
          b20 += wv2 * da; b21 += wv2 * db; b22 += wv2 * dc;
        }
      }
    }
    const double k = 4.0 * g.inv_dx;
    const double Cn[9] = {k * b00, k * b01, k * b02, k * b10, k * b11, k * b12,
                          k * b20, k * b21, k * b22};
    double F[9];
#pragma unroll
    for (int i = 0; i < 9; ++i) F[i] = Fm[i * n_el + p];
    double G[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) G[3 * i + j] = (i == j ? 1.0 : 0.0) + g.dt * Cn[3 * i + j];
    double Fn[9];
    matmul3(G, F, Fn);
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      Cm[i * n_el + p] = Cn[i];
      Fm[i * n_el + p] = Fn[i];
    }
    if (kBoundary && tag[p] == kElastomerBottom) { v0 = 0.0; v1 = 0.0; vz = 0.0; }
    v[p] = v0;
    v[n + p] = v1;
    v[2 * n + p] = vz;
    if (kAdvect) {
      px0 = px0 + g.dt * v0;
      px1 = px1 + g.dt * v1;
      px2 = px2 + g.dt * vz;
      x[p] = px0;
      x[n + p] = px1;
      x[2 * n + p] = px2;
      v2 = v0 * v0 + v1 * v1 + vz * vz;
    }
  }
  if (kAdvect) reduce_motion(ctl, active, v2, px0, px1, px2);
}

// apply_boundary + advect for the indenter (engine.cpp:260-261, 275-279).
// kUniform: all indenter velocities equal Ctl::ind_v (the per-particle v array
// is not read or written; tg_download fills it in). apply_boundary makes the
// velocity uniform, so after it the indenter is always in this mode.
template <bool kBoundary, bool kAdvect, bool kUniform>
__global__ void __launch_bounds__(256) k_ind_move(double* __restrict__ x, double* __restrict__ v,
                                                  int64_t n, int64_t n_el, Ctl* ctl, Geometry g) {
  if (ctl->err_code) return;
  const int64_t p = n_el + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n;
  double v0, v1, vz;
  if (kBoundary) {
    v0 = ctl->vind[0];
    v1 = ctl->vind[1];
    vz = ctl->vind[2];
  } else if (kUniform) {
    v0 = ctl->ind_v[0];
    v1 = ctl->ind_v[1];
    vz = ctl->ind_v[2];
  } else {
    v0 = active ? v[p] : 0.0;
    v1 = active ? v[n + p] : 0.0;
    vz = active ? v[2 * n + p] : 0.0;
  }
  if (kBoundary && blockIdx.x == 0 && threadIdx.x == 0) {
    // every thread read vind above; Ctl::ind_v is only read by later kernels
    ctl->ind_v[0] = v0;
    ctl->ind_v[1] = v1;
    ctl->ind_v[2] = vz;
  }
  double px0 = 0, px1 = 0, px2 = 0, v2 = 0;
  if (active && kAdvect) {
    px0 = x[p] + g.dt * v0;
    px1 = x[n + p] + g.dt * v1;
    px2 = x[2 * n + p] + g.dt * vz;
    x[p] = px0;
    x[n + p] = px1;
    x[2 * n + p] = px2;
    v2 = v0 * v0 + v1 * v1 + vz * vz;
  }
  if (kAdvect) reduce_motion(ctl, active, v2, px0, px1, px2);
}

// Phase-API pieces (engine.cpp:254-286) that the fused step path folds into
// k_g2p_gel / k_ind_move.
__global__ void k_gel_boundary(double* __restrict__ v, const uint8_t* __restrict__ tag, int64_t n,
                               int64_t n_el, Ctl* ctl) {
  if (ctl->err_code) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n_el && tag[p] == kElastomerBottom) {
    v[p] = 0.0;
    v[n + p] = 0.0;
    v[2 * n + p] = 0.0;
  }
}

__global__ void k_gel_advect(double* __restrict__ x, const double* __restrict__ v, int64_t n,
                             int64_t n_el, Ctl* ctl, Geometry g) {
  if (ctl->err_code) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n_el;
  double px0 = 0, px1 = 0, px2 = 0, v2 = 0;
  if (active) {
    const double v0 = v[p], v1 = v[n + p], vz = v[2 * n + p];
    px0 = x[p] + g.dt * v0;
    px1 = x[n + p] + g.dt * v1;
    px2 = x[2 * n + p] + g.dt * vz;
    x[p] = px0;
    x[n + p] = px1;
    x[2 * n + p] = px2;
    v2 = v0 * v0 + v1 * v1 + vz * vz;
  }
  reduce_motion(ctl, active, v2, px0, px1, px2);
}

// End of particle_to_grid: publish StepDiagnostics::min_det_f (engine.cpp:177).
__global__ void k_p2g_done(Ctl* ctl) {
  if (ctl->err_code) return;
  ctl->diag_min_det_f = order_val(ctl->min_detf);
  ctl->min_detf = order_key(1.0);
}

// Copies a node box [lo, hi) into dense staging buffers (tg_download_grid).
__global__ void k_gather_box(const double4* __restrict__ mp, const double4* __restrict__ vel,
                             Geometry g, int3 lo, int3 hi, double* __restrict__ mass,
                             double* __restrict__ mom, double* __restrict__ velo) {
  const int ny = hi.y - lo.y, nz = hi.z - lo.z;
  const int64_t total = static_cast<int64_t>(hi.x - lo.x) * ny * nz;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = lo.z + static_cast<int>(t % nz);
    const int64_t r = t / nz;
    const int j = lo.y + static_cast<int>(r % ny);
    const int i = lo.x + static_cast<int>(r / ny);
    const size_t nd = node_index(g, i, j, k);
    const double4 q = mp[nd];
    const double4 u = vel[nd];
    mass[t] = q.x;
    mom[3 * t] = q.y; mom[3 * t + 1] = q.z; mom[3 * t + 2] = q.w;
    velo[3 * t] = u.x; velo[3 * t + 1] = u.y; velo[3 * t + 2] = u.z;
  }
}

// ---------------------------------------------------------------------------
// Launch helpers (host).
// ---------------------------------------------------------------------------

namespace {
constexpr int kThreads = 256;
inline unsigned blocks_for(int64_t n) {
  return static_cast<unsigned>((n + kThreads - 1) / kThreads > 0 ? (n + kThreads - 1) / kThreads : 1);
}
}  // namespace

int launch_window(DeviceSim& s) {
  k_reset<<<1, 1, 0, s.stream>>>(s.ctl);
  k_bbox<<<blocks_for(s.n), kThreads, 0, s.stream>>>(s.x, s.n, s.ctl);
  k_finalize<<<1, 1, 0, s.stream>>>(s.ctl, s.geo, kFinWindow);
  s.kernel_launches += 3;
  return 3;
}

static unsigned window_blocks(int sm_count) { return static_cast<unsigned>(sm_count * 8); }

int launch_clear(DeviceSim& s, int sms) {
  k_clear<<<window_blocks(sms), kThreads, 0, s.stream>>>(s.grid_mp, s.ctl, s.geo);
  s.kernel_launches += 1;
  return 1;
}

int launch_p2g_gel(DeviceSim& s) {
  if (s.n_el <= 0) return 0;
  k_p2g_gel<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.x, s.v, s.C, s.F, s.n, s.n_el, s.ctl,
                                                           s.geo, s.grid_mp, s.m_el, s.vol_el);
  s.kernel_launches += 1;
  return 1;
}

constexpr int kIndChunk = 16;

int launch_p2g_ind(DeviceSim& s) {
  if (s.n_ind <= 0) return 0;
  if (s.ind_v_uniform)
    k_p2g_ind_chunk<kIndChunk><<<blocks_for((s.n_ind + kIndChunk - 1) / kIndChunk), kThreads, 0,
                                 s.stream>>>(s.x, s.n, s.n_el, s.ctl, s.geo, s.grid_mp, s.m_ind);
  else
    k_p2g_ind<<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el, s.ctl, s.geo,
                                                              s.grid_mp, s.m_ind);
  s.kernel_launches += 1;
  return 1;
}

int launch_p2g(DeviceSim& s, bool publish_diag) {
  int k = launch_p2g_gel(s) + launch_p2g_ind(s);
  if (publish_diag) {
    k_p2g_done<<<1, 1, 0, s.stream>>>(s.ctl);
    s.kernel_launches += 1;
    ++k;
  }
  return k;
}

int launch_grid_update(DeviceSim& s, int sms) {
  k_grid_update<<<window_blocks(sms), kThreads, 0, s.stream>>>(s.grid_mp, s.grid_v, s.ctl, s.geo);
  s.kernel_launches += 1;
  return 1;
}

int launch_g2p_gel_move(DeviceSim& s) {
  if (s.n_el <= 0) return 0;
  k_g2p_gel<true, true><<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(
      s.x, s.v, s.C, s.F, s.tag, s.n, s.n_el, s.ctl, s.geo, s.grid_v);
  s.kernel_launches += 1;
  return 1;
}

int launch_ind_move(DeviceSim& s) {
  if (s.n_ind <= 0) return 0;
  k_ind_move<true, true, true><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(
      s.x, s.v, s.n, s.n_el, s.ctl, s.geo);
  s.ind_v_uniform = true;
  s.kernel_launches += 1;
  return 1;
}

int launch_finalize_step(DeviceSim& s) {
  k_finalize<<<1, 1, 0, s.stream>>>(s.ctl, s.geo, kFinDiag | kFinAdvect | kFinWindow);
  s.kernel_launches += 1;
  return 1;
}

// Fused G2P + boundary + advect + finalize (the step path).
int launch_g2p_move(DeviceSim& s) {
  return launch_g2p_gel_move(s) + launch_ind_move(s) + launch_finalize_step(s);
}

int launch_phase_g2p(DeviceSim& s) {
  if (s.n_el > 0)
    k_g2p_gel<false, false><<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(
        s.x, s.v, s.C, s.F, s.tag, s.n, s.n_el, s.ctl, s.geo, s.grid_v);
  s.kernel_launches += 1;
  return 1;
}

int launch_phase_boundary(DeviceSim& s) {
  if (s.n_el > 0)
    k_gel_boundary<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.v, s.tag, s.n, s.n_el, s.ctl);
  if (s.n_ind > 0)
    k_ind_move<true, false, true><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(
        s.x, s.v, s.n, s.n_el, s.ctl, s.geo);
  if (s.n_ind > 0) s.ind_v_uniform = true;
  s.kernel_launches += 2;
  return 2;
}

int launch_phase_advect(DeviceSim& s) {
  if (s.n_el > 0)
    k_gel_advect<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el, s.ctl,
                                                                s.geo);
  if (s.n_ind > 0)
  {
    if (s.ind_v_uniform)
      k_ind_move<false, true, true><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(
          s.x, s.v, s.n, s.n_el, s.ctl, s.geo);
    else
      k_ind_move<false, true, false><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(
          s.x, s.v, s.n, s.n_el, s.ctl, s.geo);
  }
  k_finalize<<<1, 1, 0, s.stream>>>(s.ctl, s.geo, kFinAdvect);
  s.kernel_launches += 3;
  return 3;
}

int launch_reset(DeviceSim& s) {
  k_reset<<<1, 1, 0, s.stream>>>(s.ctl);
  s.kernel_launches += 1;
  return 1;
}

int launch_gather_box(DeviceSim& s, const int lo[3], const int hi[3], double* mass, double* mom,
                      double* vel) {
  k_gather_box<<<1024, kThreads, 0, s.stream>>>(s.grid_mp, s.grid_v, s.geo,
                                                make_int3(lo[0], lo[1], lo[2]),
                                                make_int3(hi[0], hi[1], hi[2]), mass, mom, vel);
  s.kernel_launches += 1;
  return 1;
}

}  // namespace tacchi_b200
