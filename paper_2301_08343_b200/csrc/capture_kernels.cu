// Fused capture path for sm_100a: extract_surface_depth -> crop_align ->
// surface_normals -> phong_render (sim::capture, scene_builder.cpp:80-89).
//
// The reference materialises a 713x713 full-surface map, then a 640x480 crop,
// then a normal map, then the image (four serial passes, ~50 ms). Here one
// kernel computes each crop pixel's depth on the fly from the 101x101 surface
// lattice (both bilinear stages restated exactly), stages a 34x10 depth tile
// (+1 halo for the [-1,0,1] normal stencil) in shared memory, and shades.
// All arithmetic uses the non-contracting _rn intrinsics in the reference's
// expression order, so the depth map is bit-identical to the CPU's for
// identical particle positions; the image differs only where pow() rounding
// lands on a .5 quantisation boundary.
#include <cmath>
#include <cstring>
#include <string>

#include "engine.cuh"
#include "tacchi_cuda.h"

namespace tacchi_b200 {

struct ShadeParams {
  double ka, kd, ks, shininess;
  double ambient[3];
  double view[3];         // normalised on host (phong.cpp:51)
  int n_lights;
  double lights[8][9];    // directions normalised on host (phong.cpp:53-54)
};

struct LinMap {  // extract_surface_depth's per-axis lattice coordinate tables
  int n;         // nx or ny
  double c;      // centre (cx or cy)
  double o;      // lattice origin x0 / y0
  double s;      // spacing sx / sy
  int len;       // full-map width / height
};

struct CropMap {  // crop_align geometry
  double c_src, c_out, scale, off;
  int src_len;
};

// depth_extract.cpp:30-47: lattice coordinate of full-map pixel `u`.
__device__ __forceinline__ void lattice_coord(const LinMap& m, int u, double r, int& i0,
                                              double& f) {
  const double xx = add_rn(m.c, mul_rn(sub_rn(static_cast<double>(u), mul_rn(0.5, static_cast<double>(m.len - 1))), r));
  double gi = div_rn(sub_rn(xx, m.o), m.s);
  const double hi = static_cast<double>(m.n) - 1.0;
  gi = gi < 0.0 ? 0.0 : (gi > hi ? hi : gi);
  i0 = min(static_cast<int>(gi), m.n - 2);
  f = sub_rn(gi, static_cast<double>(i0));
}

// depth_map.cpp:85-95: source coordinate of crop pixel `u`.
__device__ __forceinline__ void crop_coord(const CropMap& m, int u, int& x0, double& f) {
  double sx = add_rn(add_rn(m.c_src, mul_rn(m.scale, sub_rn(static_cast<double>(u), m.c_out))), m.off);
  const double hi = static_cast<double>(m.src_len - 1);
  sx = sx < 0.0 ? 0.0 : (sx > hi ? hi : sx);
  x0 = min(static_cast<int>(sx), m.src_len - 2);
  f = sub_rn(sx, static_cast<double>(x0));
}

__device__ __forceinline__ double bilerp(double f_outer, double f_inner, double d00, double d10,
                                         double d01, double d11) {
  // (1 - fo) * ((1 - fi) * d00 + fi * d10) + fo * ((1 - fi) * d01 + fi * d11)
  const double gi = sub_rn(1.0, f_inner), go = sub_rn(1.0, f_outer);
  const double a = add_rn(mul_rn(gi, d00), mul_rn(f_inner, d10));
  const double b = add_rn(mul_rn(gi, d01), mul_rn(f_inner, d11));
  return add_rn(mul_rn(go, a), mul_rn(f_outer, b));
}

// Full-map value at (row, col): depth_extract.cpp:40-45 with
// d00 = (i0, j0), d10 = (i0 + 1, j0), d01 = (i0, j0 + 1).
__device__ __forceinline__ double full_value(const double* __restrict__ dg, int ny, int i0,
                                             double fi, int j0, double fj) {
  const double d00 = dg[static_cast<size_t>(i0) * ny + j0];
  const double d10 = dg[static_cast<size_t>(i0 + 1) * ny + j0];
  const double d01 = dg[static_cast<size_t>(i0) * ny + j0 + 1];
  const double d11 = dg[static_cast<size_t>(i0 + 1) * ny + j0 + 1];
  return bilerp(fj, fi, d00, d10, d01, d11);
}

// phong.cpp:56-80 for one pixel with normal from gradients (gx, gy).
__device__ __forceinline__ void shade(const ShadeParams& P, double gx, double gy,
                                      const uint8_t* bg_px, uint8_t* out) {
  // n = (gx, gy, -1) / |.|   (phong.cpp:36-37)
  const double nrm = sqrt(add_rn(add_rn(mul_rn(gx, gx), mul_rn(gy, gy)), 1.0));
  const double n0 = div_rn(gx, nrm), n1 = div_rn(gy, nrm), n2 = div_rn(-1.0, nrm);
  double col[3];
#pragma unroll
  for (int c = 0; c < 3; ++c)
    col[c] = bg_px ? mul_rn(P.ka, div_rn(static_cast<double>(bg_px[c]), 255.0))
                   : mul_rn(P.ka, P.ambient[c]);
  for (int l = 0; l < P.n_lights; ++l) {
    const double* L = P.lights[l];
    const double ln = add_rn(add_rn(mul_rn(L[0], n0), mul_rn(L[1], n1)), mul_rn(L[2], n2));
    if (ln <= 0.0) continue;
    const double kdl = mul_rn(P.kd, ln);
#pragma unroll
    for (int c = 0; c < 3; ++c) col[c] = add_rn(col[c], mul_rn(kdl, L[3 + c]));
    const double t = mul_rn(2.0, ln);
    const double r0 = sub_rn(mul_rn(t, n0), L[0]);
    const double r1 = sub_rn(mul_rn(t, n1), L[1]);
    const double r2 = sub_rn(mul_rn(t, n2), L[2]);
    const double rv = add_rn(add_rn(mul_rn(r0, P.view[0]), mul_rn(r1, P.view[1])), mul_rn(r2, P.view[2]));
    if (rv > 0.0) {
      const double sp = mul_rn(P.ks, pow(rv, P.shininess));
#pragma unroll
      for (int c = 0; c < 3; ++c) col[c] = add_rn(col[c], mul_rn(sp, L[6 + c]));
    }
  }
#pragma unroll
  for (int c = 0; c < 3; ++c) {
    const double cc = col[c] < 0.0 ? 0.0 : (col[c] > 1.0 ? 1.0 : col[c]);
    out[c] = static_cast<uint8_t>(llround(mul_rn(cc, 255.0)));
  }
}

// Surface heights sampled on the reference lattice (depth_extract.cpp:18-20).
__global__ void k_surface_depth(const double* __restrict__ xz, const uint32_t* __restrict__ idx,
                                int count, double z0, double* __restrict__ dg) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s < count) dg[s] = sub_rn(z0, xz[idx[s]]);
}

constexpr int kTileW = 32, kTileH = 8;

// Fused crop depth + normals + Phong. One CTA per 32x8 output tile.
__global__ void __launch_bounds__(kTileW * kTileH) k_capture(
    const double* __restrict__ dg, int ny_lat, LinMap mx, LinMap my, double r_full, CropMap cx,
    CropMap cy, int ow, int oh, double r_out, ShadeParams P, const uint8_t* __restrict__ bg,
    double* __restrict__ depth_out, uint8_t* __restrict__ rgb_out) {
  __shared__ double tile[kTileH + 2][kTileW + 2];
  const int u0 = blockIdx.x * kTileW, v0 = blockIdx.y * kTileH;
  const int tid = threadIdx.y * kTileW + threadIdx.x;
  for (int e = tid; e < (kTileW + 2) * (kTileH + 2); e += kTileW * kTileH) {
    const int tu = e % (kTileW + 2), tv = e / (kTileW + 2);
    const int u = min(max(u0 + tu - 1, 0), ow - 1);
    const int v = min(max(v0 + tv - 1, 0), oh - 1);
    // crop_align: source pixel (x0, y0) and weights in the full map.
    int sx0, sy0;
    double fx, fy;
    crop_coord(cx, u, sx0, fx);
    crop_coord(cy, v, sy0, fy);
    // The four full-map samples; full(row, col) uses col -> lattice i, row -> j.
    int i0a, i0b, j0a, j0b;
    double fia, fib, fja, fjb;
    lattice_coord(mx, sx0, r_full, i0a, fia);
    lattice_coord(mx, sx0 + 1, r_full, i0b, fib);
    lattice_coord(my, sy0, r_full, j0a, fja);
    lattice_coord(my, sy0 + 1, r_full, j0b, fjb);
    const double d00 = full_value(dg, ny_lat, i0a, fia, j0a, fja);  // (y0, x0)
    const double d01 = full_value(dg, ny_lat, i0b, fib, j0a, fja);  // (y0, x0+1)
    const double d10 = full_value(dg, ny_lat, i0a, fia, j0b, fjb);  // (y0+1, x0)
    const double d11 = full_value(dg, ny_lat, i0b, fib, j0b, fjb);  // (y0+1, x0+1)
    // depth_map.cpp:96: (1-fy)*((1-fx)*d00 + fx*d01) + fy*((1-fx)*d10 + fx*d11)
    tile[tv][tu] = bilerp(fy, fx, d00, d01, d10, d11);
  }
  __syncthreads();
  const int u = u0 + threadIdx.x, v = v0 + threadIdx.y;
  if (u >= ow || v >= oh) return;
  const int tu = threadIdx.x + 1, tv = threadIdx.y + 1;
  const double inv_2r = div_rn(1.0, mul_rn(2.0, r_out));
  const double inv_r = div_rn(1.0, r_out);
  // phong.cpp:17-35 with H = -depth.
  double gx, gy;
  if (u == 0) gx = mul_rn(sub_rn(-tile[tv][tu + 1], -tile[tv][tu]), inv_r);
  else if (u == ow - 1) gx = mul_rn(sub_rn(-tile[tv][tu], -tile[tv][tu - 1]), inv_r);
  else gx = mul_rn(sub_rn(-tile[tv][tu + 1], -tile[tv][tu - 1]), inv_2r);
  if (v == 0) gy = mul_rn(sub_rn(-tile[tv + 1][tu], -tile[tv][tu]), inv_r);
  else if (v == oh - 1) gy = mul_rn(sub_rn(-tile[tv][tu], -tile[tv - 1][tu]), inv_r);
  else gy = mul_rn(sub_rn(-tile[tv + 1][tu], -tile[tv - 1][tu]), inv_2r);
  const size_t px = static_cast<size_t>(v) * ow + u;
  if (depth_out) depth_out[px] = tile[tv][tu];
  shade(P, gx, gy, bg ? bg + 3 * px : nullptr, rgb_out + 3 * px);
}

// render::extract_surface_depth at an arbitrary pixel grid (depth_extract.cpp:10-49).
__global__ void k_extract(const double* __restrict__ dg, int ny_lat, LinMap mx, LinMap my,
                          double r, int w, int h, double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= w || v >= h) return;
  int i0, j0;
  double fi, fj;
  lattice_coord(mx, u, r, i0, fi);
  lattice_coord(my, v, r, j0, fj);
  out[static_cast<size_t>(v) * w + u] = full_value(dg, ny_lat, i0, fi, j0, fj);
}

// render::crop_align on a device depth map (depth_map.cpp:84-98).
__global__ void k_crop(const double* __restrict__ src, int sw, CropMap cx, CropMap cy, int ow,
                       int oh, double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= ow || v >= oh) return;
  int x0, y0;
  double fx, fy;
  crop_coord(cx, u, x0, fx);
  crop_coord(cy, v, y0, fy);
  const double d00 = src[static_cast<size_t>(y0) * sw + x0], d01 = src[static_cast<size_t>(y0) * sw + x0 + 1];
  const double d10 = src[static_cast<size_t>(y0 + 1) * sw + x0];
  const double d11 = src[static_cast<size_t>(y0 + 1) * sw + x0 + 1];
  out[static_cast<size_t>(v) * ow + u] = bilerp(fy, fx, d00, d01, d10, d11);
}

__device__ __forceinline__ void gradients(const double* __restrict__ d, int w, int h, int u, int v,
                                          double r, double& gx, double& gy) {
  const double inv_2r = div_rn(1.0, mul_rn(2.0, r));
  const double inv_r = div_rn(1.0, r);
  auto H = [&](int row, int col) { return -d[static_cast<size_t>(row) * w + col]; };
  if (u == 0) gx = mul_rn(sub_rn(H(v, 1), H(v, 0)), inv_r);
  else if (u == w - 1) gx = mul_rn(sub_rn(H(v, u), H(v, u - 1)), inv_r);
  else gx = mul_rn(sub_rn(H(v, u + 1), H(v, u - 1)), inv_2r);
  if (v == 0) gy = mul_rn(sub_rn(H(1, u), H(0, u)), inv_r);
  else if (v == h - 1) gy = mul_rn(sub_rn(H(v, u), H(v - 1, u)), inv_r);
  else gy = mul_rn(sub_rn(H(v + 1, u), H(v - 1, u)), inv_2r);
}

// render::surface_normals (phong.cpp:10-41).
__global__ void k_normals(const double* __restrict__ d, int w, int h, double r,
                          double* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= w || v >= h) return;
  double gx, gy;
  gradients(d, w, h, u, v, r, gx, gy);
  const double nrm = sqrt(add_rn(add_rn(mul_rn(gx, gx), mul_rn(gy, gy)), 1.0));
  double* o = out + 3 * (static_cast<size_t>(v) * w + u);
  o[0] = div_rn(gx, nrm);
  o[1] = div_rn(gy, nrm);
  o[2] = div_rn(-1.0, nrm);
}

// render::phong_render on a device depth map (phong.cpp:43-84).
__global__ void k_phong(const double* __restrict__ d, int w, int h, double r, ShadeParams P,
                        const uint8_t* __restrict__ bg, uint8_t* __restrict__ out) {
  const int u = blockIdx.x * blockDim.x + threadIdx.x, v = blockIdx.y * blockDim.y + threadIdx.y;
  if (u >= w || v >= h) return;
  double gx, gy;
  gradients(d, w, h, u, v, r, gx, gy);
  const size_t px = static_cast<size_t>(v) * w + u;
  shade(P, gx, gy, bg ? bg + 3 * px : nullptr, out + 3 * px);
}

// ---------------------------------------------------------------------------
// Host-side launch helpers.
// ---------------------------------------------------------------------------

namespace {

void normalize_host(double* v) {  // Eigen normalize(): v / sqrt(squaredNorm)
  const double n2 = v[0] * v[0] + v[1] * v[1] + v[2] * v[2];
  if (n2 > 0.0) {
    const double n = std::sqrt(n2);
    v[0] /= n; v[1] /= n; v[2] /= n;
  }
}

ShadeParams make_shade(const tg_render& r) {
  ShadeParams P{};
  P.ka = r.ambient_k;
  P.kd = r.diffuse_k;
  P.ks = r.specular_k;
  P.shininess = r.shininess;
  for (int c = 0; c < 3; ++c) {
    P.ambient[c] = r.ambient_rgb[c];
    P.view[c] = r.view_dir[c];
  }
  normalize_host(P.view);  // phong.cpp:51
  P.n_lights = r.n_lights;
  for (int l = 0; l < r.n_lights; ++l) {
    for (int k = 0; k < 9; ++k) P.lights[l][k] = r.lights[l][k];
    normalize_host(P.lights[l]);  // phong.cpp:53-54
  }
  return P;
}

LinMap make_linmap(int n, double o, double s, int len) {
  LinMap m;
  m.n = n;
  m.o = o;
  m.s = s;
  m.c = o + 0.5 * (n - 1) * s;  // depth_extract.cpp:28-29
  m.len = len;
  return m;
}

CropMap make_cropmap(int src_len, int out_len, double scale, double off) {
  CropMap m;
  m.c_src = 0.5 * (src_len - 1);
  m.c_out = 0.5 * (out_len - 1);
  m.scale = scale;
  m.off = off;
  m.src_len = src_len;
  return m;
}

// depth_map.cpp:63,73-82
int check_crop(int sw, int sh, double off_x, double off_y, double scale, int ow, int oh,
               std::string& msg) {
  if (!(scale > 0.0)) {
    msg = "crop_align: scale must be > 0";
    return kErrConfig;
  }
  const double cx_src = 0.5 * (sw - 1), cy_src = 0.5 * (sh - 1);
  const double cx_out = 0.5 * (ow - 1), cy_out = 0.5 * (oh - 1);
  for (int corner = 0; corner < 4; ++corner) {
    const double u = (corner & 1) ? ow - 1 : 0;
    const double v = (corner & 2) ? oh - 1 : 0;
    const double sx = cx_src + scale * (u - cx_out) + off_x;
    const double sy = cy_src + scale * (v - cy_out) + off_y;
    if (sx < -1e-9 || sx > sw - 1 + 1e-9 || sy < -1e-9 || sy > sh - 1 + 1e-9) {
      msg = "crop window leaves the source depth map (source " + std::to_string(sw) + "x" +
            std::to_string(sh) + ")";
      return kErrCropOutOfBounds;
    }
  }
  return kOk;
}

int check_render(const tg_render& r, int w, int h, std::string& msg) {
  if (r.n_lights < 1 || r.n_lights > 8) {
    msg = "phong_render: at least one light source required (max 8)";
    return kErrConfig;
  }
  (void)w;
  (void)h;
  return kOk;
}

}  // namespace

void full_surface_size(const DeviceSim& s, double r, int* w, int* h) {
  // depth_extract.cpp:54-55
  *w = static_cast<int>(std::ceil((s.surf_nx - 1) * s.surf_geom[2] / r)) + 1;
  *h = static_cast<int>(std::ceil((s.surf_ny - 1) * s.surf_geom[3] / r)) + 1;
}

static int ensure_capture_buffers(DeviceSim& s, size_t pixels, bool want_bg) {
  if (pixels > s.cap_pixels) {
    cudaFree(s.cap_depth);
    cudaFree(s.cap_rgb);
    cudaFreeHost(s.h_depth_pinned);
    cudaFreeHost(s.h_rgb_pinned);
    s.cap_depth = nullptr;
    s.cap_rgb = nullptr;
    s.h_depth_pinned = nullptr;
    s.h_rgb_pinned = nullptr;
    if (cudaMalloc(&s.cap_depth, pixels * sizeof(double)) != cudaSuccess ||
        cudaMalloc(&s.cap_rgb, pixels * 3) != cudaSuccess ||
        cudaMallocHost(&s.h_depth_pinned, pixels * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&s.h_rgb_pinned, pixels * 3) != cudaSuccess)
      return TG_ERR_CUDA;
    s.cap_pixels = pixels;
  }
  if (want_bg && pixels > s.cap_bg_pixels) {
    cudaFree(s.cap_bg);
    if (cudaMalloc(&s.cap_bg, pixels * 3) != cudaSuccess) return TG_ERR_CUDA;
    s.cap_bg_pixels = pixels;
  }
  return TG_OK;
}

static void launch_surface_depth(DeviceSim& s) {
  const int count = s.surf_nx * s.surf_ny;
  k_surface_depth<<<(count + 255) / 256, 256, 0, s.stream>>>(s.x + 2 * s.n, s.surf_idx, count,
                                                            s.surf_geom[4], s.surf_depth);
  s.kernel_launches += 1;
}

// sim::capture. depth_host / rgb_host may be null (device-resident result).
// Enqueues sim::capture on the handle's stream: the fused kernel and, when
// requested, the D2H copies of depth / RGB into the handle's pinned buffers.
int capture_enqueue_to(DeviceSim& s, const tg_render& r, double* depth_pinned, uint8_t* rgb_pinned,
                       std::string& msg, cudaStream_t shade = nullptr,
                       cudaEvent_t surface_done = nullptr);

int capture_enqueue(DeviceSim& s, const tg_render& r, bool want_depth, bool want_rgb,
                    std::string& msg) {
  if (s.cap_pixels < static_cast<size_t>(r.width) * r.height || !s.h_depth_pinned) {
    // allocate (ensure_capture_buffers) before taking the pinned pointers
    const int rc = capture_enqueue_to(s, r, nullptr, nullptr, msg);
    if (rc) return rc;
    if (!want_depth && !want_rgb) return TG_OK;
    // the capture ran; only the read-back is left
    const size_t pixels = static_cast<size_t>(r.width) * r.height;
    if (want_depth)
      cudaMemcpyAsync(s.h_depth_pinned, s.cap_depth, pixels * sizeof(double),
                      cudaMemcpyDeviceToHost, s.stream);
    if (want_rgb)
      cudaMemcpyAsync(s.h_rgb_pinned, s.cap_rgb, pixels * 3, cudaMemcpyDeviceToHost, s.stream);
    return TG_OK;
  }
  return capture_enqueue_to(s, r, want_depth ? s.h_depth_pinned : nullptr,
                            want_rgb ? s.h_rgb_pinned : nullptr, msg);
}

// sim::capture on the handle's stream; the depth / RGB read-backs (if the
// destinations are given: pinned host buffers) are enqueued after it.
// With `shade` (and `surface_done`): only the surface gather runs on the
// handle's stream (it is all that reads the particles); the shading kernel
// and the read-backs run on `shade` after `surface_done`, beside whatever the
// handle's stream does next (the pipelined frames' next substeps).
int capture_enqueue_to(DeviceSim& s, const tg_render& r, double* depth_pinned, uint8_t* rgb_pinned,
                       std::string& msg, cudaStream_t shade, cudaEvent_t surface_done) {
  if (s.surf_nx < 2 || s.surf_ny < 2 || !s.surf_idx) {
    msg = "extract_surface_depth: state has no surface lattice";
    return kErrNoSurface;
  }
  if (!(r.pixel_to_meter > 0.0)) {
    msg = "extract_surface_depth: bad pixel grid";
    return kErrConfig;
  }
  int fw, fh;
  full_surface_size(s, r.pixel_to_meter, &fw, &fh);
  if (fw < 2 || fh < 2) {
    msg = "extract_surface_depth: bad pixel grid";
    return kErrConfig;
  }
  const int ow = r.width, oh = r.height;
  int rc = check_crop(fw, fh, r.crop_offset[0], r.crop_offset[1], r.crop_scale, ow, oh, msg);
  if (rc) return rc;
  rc = check_render(r, ow, oh, msg);
  if (rc) return rc;
  const size_t pixels = static_cast<size_t>(ow) * oh;
  rc = ensure_capture_buffers(s, pixels, r.background != nullptr);
  if (rc) {
    msg = "capture: device allocation failed";
    return rc;
  }
  if (r.background)
    cudaMemcpyAsync(s.cap_bg, r.background, pixels * 3, cudaMemcpyHostToDevice, s.stream);
  launch_surface_depth(s);
  cudaStream_t st = s.stream;
  if (shade && surface_done) {
    cudaEventRecord(surface_done, s.stream);
    cudaStreamWaitEvent(shade, surface_done, 0);
    st = shade;
  }
  const LinMap mx = make_linmap(s.surf_nx, s.surf_geom[0], s.surf_geom[2], fw);
  const LinMap my = make_linmap(s.surf_ny, s.surf_geom[1], s.surf_geom[3], fh);
  const CropMap cx = make_cropmap(fw, ow, r.crop_scale, r.crop_offset[0]);
  const CropMap cy = make_cropmap(fh, oh, r.crop_scale, r.crop_offset[1]);
  const double r_out = r.pixel_to_meter * r.crop_scale;  // depth_map.cpp:68
  const dim3 grid((ow + kTileW - 1) / kTileW, (oh + kTileH - 1) / kTileH);
  k_capture<<<grid, dim3(kTileW, kTileH), 0, st>>>(
      s.surf_depth, s.surf_ny, mx, my, r.pixel_to_meter, cx, cy, ow, oh, r_out, make_shade(r),
      r.background ? s.cap_bg : nullptr, s.cap_depth, s.cap_rgb);
  s.kernel_launches += 1;
  if (depth_pinned)
    cudaMemcpyAsync(depth_pinned, s.cap_depth, pixels * sizeof(double), cudaMemcpyDeviceToHost, st);
  if (rgb_pinned) cudaMemcpyAsync(rgb_pinned, s.cap_rgb, pixels * 3, cudaMemcpyDeviceToHost, st);
  s.cap_last_pixels = pixels;
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    msg = cudaGetErrorString(e);
    return TG_ERR_CUDA;
  }
  return TG_OK;
}

// After the stream is synchronised: copies the pinned results to caller
// buffers (skipped when the caller passes the pinned buffers themselves,
// see tg_capture_buffers).
void capture_collect(DeviceSim& s, double* depth_host, uint8_t* rgb_host) {
  const size_t pixels = s.cap_last_pixels;
  if (depth_host && depth_host != s.h_depth_pinned)
    std::memcpy(depth_host, s.h_depth_pinned, pixels * sizeof(double));
  if (rgb_host && rgb_host != s.h_rgb_pinned) std::memcpy(rgb_host, s.h_rgb_pinned, pixels * 3);
}

int capture(DeviceSim& s, const tg_render& r, double* depth_host, uint8_t* rgb_host,
            std::string& msg) {
  const int rc = capture_enqueue(s, r, depth_host != nullptr, rgb_host != nullptr, msg);
  if (rc) return rc;
  if (depth_host || rgb_host) {
    if (cudaStreamSynchronize(s.stream) != cudaSuccess) {
      msg = cudaGetErrorString(cudaGetLastError());
      return TG_ERR_CUDA;
    }
    capture_collect(s, depth_host, rgb_host);
  }
  return TG_OK;
}

// The handle's pinned capture buffers for r's output size (allocated here).
int capture_buffers(DeviceSim& s, const tg_render& r, double** depth, uint8_t** rgb,
                    std::string& msg) {
  if (r.width < 2 || r.height < 2) {
    msg = "capture: render image size too small";
    return kErrConfig;
  }
  if (ensure_capture_buffers(s, static_cast<size_t>(r.width) * r.height, false)) {
    msg = "capture: allocation failed";
    return TG_ERR_CUDA;
  }
  if (depth) *depth = s.h_depth_pinned;
  if (rgb) *rgb = s.h_rgb_pinned;
  return TG_OK;
}

// render::extract_surface_depth(state, w, h, r) into a host buffer.
int extract_depth(DeviceSim& s, int w, int h, double r, double* out, std::string& msg) {
  if (s.surf_nx < 2 || s.surf_ny < 2 || !s.surf_idx) {
    msg = "extract_surface_depth: state has no surface lattice";
    return kErrNoSurface;
  }
  if (w < 2 || h < 2 || !(r > 0.0)) {
    msg = "extract_surface_depth: bad pixel grid";
    return kErrConfig;
  }
  const size_t pixels = static_cast<size_t>(w) * h;
  double* d = nullptr;
  if (cudaMalloc(&d, pixels * sizeof(double)) != cudaSuccess) {
    msg = "extract_surface_depth: device allocation failed";
    return TG_ERR_CUDA;
  }
  launch_surface_depth(s);
  const LinMap mx = make_linmap(s.surf_nx, s.surf_geom[0], s.surf_geom[2], w);
  const LinMap my = make_linmap(s.surf_ny, s.surf_geom[1], s.surf_geom[3], h);
  k_extract<<<dim3((w + 31) / 32, (h + 7) / 8), dim3(32, 8), 0, s.stream>>>(s.surf_depth, s.surf_ny,
                                                                          mx, my, r, w, h, d);
  s.kernel_launches += 1;
  cudaMemcpyAsync(out, d, pixels * sizeof(double), cudaMemcpyDeviceToHost, s.stream);
  const cudaError_t e = cudaStreamSynchronize(s.stream);
  cudaFree(d);
  if (e != cudaSuccess) {
    msg = cudaGetErrorString(e);
    return TG_ERR_CUDA;
  }
  return TG_OK;
}

// Standalone render functions on host depth maps (render::crop_align,
// surface_normals, phong_render); mode 0 crop, 1 normals, 2 phong.
int render_standalone(int mode, const double* src, int sw, int sh, double r, double off_x,
                      double off_y, double scale, int ow, int oh, const tg_render* rp,
                      double* out_d, uint8_t* out_u8, std::string& msg) {
  int rc = kOk;
  if (mode == 0) rc = check_crop(sw, sh, off_x, off_y, scale, ow, oh, msg);
  if (mode == 1 && !(r > 0.0)) {
    msg = "surface_normals: pixel_to_meter <= 0";
    rc = kErrConfig;
  }
  if (mode == 2) {
    rc = check_render(*rp, sw, sh, msg);
    if (!rc && !(r > 0.0)) {
      msg = "surface_normals: pixel_to_meter <= 0";
      rc = kErrConfig;
    }
  }
  if (rc) return rc;
  const size_t in_px = static_cast<size_t>(sw) * sh;
  const size_t out_px = mode == 0 ? static_cast<size_t>(ow) * oh : in_px;
  double* d_src = nullptr;
  double* d_out = nullptr;
  uint8_t* d_u8 = nullptr;
  uint8_t* d_bg = nullptr;
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  bool ok = cudaMalloc(&d_src, in_px * sizeof(double)) == cudaSuccess;
  if (ok && mode == 0) ok = cudaMalloc(&d_out, out_px * sizeof(double)) == cudaSuccess;
  if (ok && mode == 1) ok = cudaMalloc(&d_out, out_px * 3 * sizeof(double)) == cudaSuccess;
  if (ok && mode == 2) ok = cudaMalloc(&d_u8, out_px * 3) == cudaSuccess;
  if (ok && mode == 2 && rp->background) ok = cudaMalloc(&d_bg, in_px * 3) == cudaSuccess;
  if (ok) {
    cudaMemcpyAsync(d_src, src, in_px * sizeof(double), cudaMemcpyHostToDevice, st);
    if (d_bg) cudaMemcpyAsync(d_bg, rp->background, in_px * 3, cudaMemcpyHostToDevice, st);
    const dim3 blk(32, 8);
    if (mode == 0) {
      k_crop<<<dim3((ow + 31) / 32, (oh + 7) / 8), blk, 0, st>>>(
          d_src, sw, make_cropmap(sw, ow, scale, off_x), make_cropmap(sh, oh, scale, off_y), ow, oh,
          d_out);
      cudaMemcpyAsync(out_d, d_out, out_px * sizeof(double), cudaMemcpyDeviceToHost, st);
    } else if (mode == 1) {
      k_normals<<<dim3((sw + 31) / 32, (sh + 7) / 8), blk, 0, st>>>(d_src, sw, sh, r, d_out);
      cudaMemcpyAsync(out_d, d_out, out_px * 3 * sizeof(double), cudaMemcpyDeviceToHost, st);
    } else {
      k_phong<<<dim3((sw + 31) / 32, (sh + 7) / 8), blk, 0, st>>>(d_src, sw, sh, r,
                                                                  make_shade(*rp), d_bg, d_u8);
      cudaMemcpyAsync(out_u8, d_u8, out_px * 3, cudaMemcpyDeviceToHost, st);
    }
    ok = cudaStreamSynchronize(st) == cudaSuccess;
  }
  if (!ok) msg = cudaGetErrorString(cudaGetLastError());
  cudaFree(d_src);
  cudaFree(d_out);
  cudaFree(d_u8);
  cudaFree(d_bg);
  cudaStreamDestroy(st);
  return ok ? static_cast<int>(kOk) : static_cast<int>(TG_ERR_CUDA);
}

}  // namespace tacchi_b200
