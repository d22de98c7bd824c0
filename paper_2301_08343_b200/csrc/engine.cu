// DeviceSim lifecycle, the substep launch plan (with CUDA-graph replay), state
// transfer, and the C-ABI entry points of include/tacchi_cuda.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "engine.cuh"
#include "tacchi_cuda.h"

namespace tacchi_b200 {

// mpm_kernels.cu
int launch_reset(DeviceSim& s, int mask);
int launch_window(DeviceSim& s);
int launch_clear(DeviceSim& s, int sms);
int launch_p2g(DeviceSim& s, bool publish_diag);
int launch_p2g_gel(DeviceSim& s);
int launch_p2g_ind(DeviceSim& s);
int launch_grid_update(DeviceSim& s, int sms, bool zero);
int launch_g2p2g_gel(DeviceSim& s, bool lookahead, bool with_indenter = false);
int launch_ind_move(DeviceSim& s, bool lookahead);
int launch_finalize_step(DeviceSim& s, bool walk_fix = false);
int launch_snapshot_ctl(DeviceSim& s, Ctl* out);
int launch_ind_walks_on(DeviceSim& s, cudaStream_t st);
int launch_chain_begin(DeviceSim& s);
int launch_ind_cols(DeviceSim& s, bool move);
int launch_ind_catchup(DeviceSim& s);
int launch_phase_g2p(DeviceSim& s);
int launch_phase_boundary(DeviceSim& s);
int launch_phase_advect(DeviceSim& s);
int launch_gather_box(DeviceSim& s, const int lo[3], const int hi[3], double* mass, double* mom,
                      double* vel);
void configure_gel_tiling(DeviceSim& s, int nx, int ny, int nz);
void permute_gel_lanes(DeviceSim& s, const double* x_in);
unsigned gel_block_count(const DeviceSim& s);
constexpr int kResetAll = 7;
// capture_kernels.cu
int capture(DeviceSim& s, const tg_render& r, double* depth_host, uint8_t* rgb_host,
            std::string& msg);
int capture_enqueue(DeviceSim& s, const tg_render& r, bool want_depth, bool want_rgb,
                    std::string& msg);
void capture_collect(DeviceSim& s, double* depth_host, uint8_t* rgb_host);
int capture_buffers(DeviceSim& s, const tg_render& r, double** depth, uint8_t** rgb,
                    std::string& msg);
int step_submit(DeviceSim& s, const double vind[3], int n_substeps);
int step_finish(DeviceSim& s, int n_substeps);
int extract_depth(DeviceSim& s, int w, int h, double r, double* out, std::string& msg);
void full_surface_size(const DeviceSim& s, double r, int* w, int* h);
int render_standalone(int mode, const double* src, int sw, int sh, double r, double off_x,
                      double off_y, double scale, int ow, int oh, const tg_render* rp,
                      double* out_d, uint8_t* out_u8, std::string& msg);

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

static const char* error_name(int code) {
  switch (code) {
    case kErrGridTooSmall: return "GridTooSmall";
    case kErrEmptyScene: return "EmptyScene";
    case kErrOutOfGrid: return "OutOfGrid";
    case kErrDegenerateF: return "DegenerateF";
    case kErrConfig: return "ConfigError";
    default: return "Error";
  }
}

#define CUDA_TRY(expr)                                                             \
  do {                                                                             \
    const cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                         \
      return fail(TG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

DeviceSim::~DeviceSim() {
  if (device >= 0) cudaSetDevice(device);
  if (stream) cudaStreamSynchronize(stream);
  for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
  cudaFree(x);
  cudaFree(v);
  cudaFree(C);
  cudaFree(F);
  cudaFree(tag);
  cudaFree(geo.cta_box);
  cudaFree(grid_slab);  // grid_mp, grid_v, grid_mi live in one allocation
  cudaFree(col_start);
  cudaFree(ind_moves);
  cudaFree(surf_idx);
  cudaFree(surf_depth);
  cudaFree(cap_depth);
  cudaFree(cap_rgb);
  cudaFree(cap_bg);
  cudaFree(ctl);
  cudaFreeHost(h_ctl);
  cudaFreeHost(h_vind);
  cudaFreeHost(h_depth_pinned);
  cudaFreeHost(h_rgb_pinned);
  if (walk_stream) cudaStreamSynchronize(walk_stream);
  if (walk_stream) cudaStreamDestroy(walk_stream);
  if (ev_fork) cudaEventDestroy(ev_fork);
  if (ev_join) cudaEventDestroy(ev_join);
  if (copy_stream) cudaStreamSynchronize(copy_stream);
  for (FrameSlot& f : frames) {
    cudaFreeHost(f.depth);
    cudaFreeHost(f.rgb);
    cudaFreeHost(f.ctl);
    cudaFree(f.d_snap);
    if (f.ev) cudaEventDestroy(f.ev);
    if (f.captured) cudaEventDestroy(f.captured);
  }
  if (copy_stream) cudaStreamDestroy(copy_stream);
  if (stream) cudaStreamDestroy(stream);
}

static int sm_count(int device) {
  static int cached[64] = {0};
  if (device < 0 || device >= 64) return 148;
  if (!cached[device]) {
    int v = 148;
    cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
    cached[device] = v;
  }
  return cached[device];
}

static int check_device(int device) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(TG_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  if (device < 0 || device >= count)
    return fail(TG_ERR_INVALID_ARGUMENT, "device index out of range");
  cudaDeviceProp prop;
  CUDA_TRY(cudaGetDeviceProperties(&prop, device));
  if (prop.major < 10)
    return fail(TG_ERR_CUDA, std::string("device ") + prop.name + " is not sm_100-class");
  CUDA_TRY(cudaSetDevice(device));
  return TG_OK;
}

// Host copy of zero_grid's base_index (engine.cpp:47-49).
static int host_base(double x, double origin, double inv_dx) {
  return static_cast<int>(std::floor((x - origin) * inv_dx - 0.5));
}

int upload(DeviceSim& s, const double* x, const double* v, const double* Cm, const double* Fm,
           bool init);
int configure_device(int device);  // mpm_kernels.cu

// Host <-> device copies ordered on the handle's (non-blocking) stream and
// completed before returning: every upload is ordered after the kernels
// already queued on the handle and before the ones that follow.
cudaError_t copy_sync(DeviceSim& s, void* dst, const void* src, size_t bytes,
                             cudaMemcpyKind kind) {
  const cudaError_t e = cudaMemcpyAsync(dst, src, bytes, kind, s.stream);
  if (e != cudaSuccess) return e;
  return cudaStreamSynchronize(s.stream);
}

// The grid arrays in one allocation (A.lo | A.hi | V.xy | V.z | M_I) over
// the node box [lo, lo + dim) of the logical grid, zeroed on the stream.
static bool alloc_grid(DeviceSim& s, const int lo[3], const int dim[3]) {
  const size_t n = static_cast<size_t>(dim[0]) * dim[1] * dim[2];
  const size_t b2 = n * sizeof(double2);
  // +2: the staging reads vz rows from an even node over an even count
  const size_t bz = ((n + 2) * sizeof(double) + 255) & ~size_t(255);
  const size_t b1 = n * sizeof(double);
  void* slab = nullptr;
  if (cudaMalloc(&slab, 3 * b2 + bz + 2 * b1) != cudaSuccess) return false;  // M_I x 2
  cudaFree(s.grid_slab);
  s.grid_slab = slab;
  s.grid_slab_bytes = 3 * b2 + bz + 2 * b1;
  s.geo.mi_stride = n;
  s.n_nodes = n;
  for (int a = 0; a < 3; ++a) {
    s.geo.ga_lo[a] = lo[a];
    s.geo.ga_dim[a] = dim[a];
  }
  char* p = static_cast<char*>(slab);
  s.grid_mp.lo = reinterpret_cast<double2*>(p);
  s.grid_mp.hi = reinterpret_cast<double2*>(p + b2);
  s.grid_v.xy = reinterpret_cast<double2*>(p + 2 * b2);
  s.grid_v.z = reinterpret_cast<double*>(p + 3 * b2);
  s.grid_mi = reinterpret_cast<double*>(p + 3 * b2 + bz);
  cudaMemsetAsync(slab, 0, s.grid_slab_bytes, s.stream);
  return true;
}

// Node margin around the boxes the step path scatters into when the
// allocation is (re)sized: room for the elastomer to deform and move before
// the next regrow.
constexpr int kAllocMargin = 4;
// The indenter's look-ahead walks touch nodes up to 3 outside the elastomer
// node box (its box widened by one node, plus the 3-node stencil).
constexpr int kWalkReach = 3;

// The allocation box that covers [lo, hi) with kAllocMargin (clamped to the
// logical grid, z start and length even where the grid allows: the velocity
// staging copies vz rows in 16-byte units).
static void alloc_box_for(const DeviceSim& s, const int lo[3], const int hi[3], int out_lo[3],
                          int out_dim[3]) {
  for (int a = 0; a < 3; ++a) {
    int l = std::max(lo[a] - kAllocMargin, 0);
    int h = std::min(hi[a] + kAllocMargin, s.geo.res[a]);
    if (a == 2) {
      // z rows padded to a multiple of kZPad nodes (128-byte aligned rows of
      // the 8-byte arrays), even start
      l &= ~1;
      const int pad = s.zpad;
      int d = ((h - l + pad - 1) / pad) * pad;
      if (l + d > s.geo.res[a]) l = std::max(s.geo.res[a] - d, 0) & ~1;
      h = std::min(l + d, s.geo.res[a]);
      if ((h - l) & 1) h = h < s.geo.res[a] ? h + 1 : h;
    }
    out_lo[a] = l;
    out_dim[a] = std::max(h - l, 1);
  }
  if (const char* e = std::getenv("TACCHI_DENSE_GRID"))
    if (std::atoi(e))
      for (int a = 0; a < 3; ++a) {
        out_lo[a] = 0;
        out_dim[a] = s.geo.res[a];
      }
}

static void drop_graphs(DeviceSim& s) {
  for (auto& kv : s.graphs) cudaGraphExecDestroy(kv.second);
  s.graphs.clear();
  s.graph_kernels.clear();
}

// Grows the node arrays so that they cover [lo, hi) (and what they covered
// before). The arrays come back zeroed: any look-ahead scatter is dropped.
// Kernel parameters (pointers, Geometry) change, so the cached graphs go.
static int ensure_alloc(DeviceSim& s, const int lo[3], const int hi[3]) {
  bool inside = true;
  for (int a = 0; a < 3; ++a)
    inside = inside && lo[a] >= s.geo.ga_lo[a] && hi[a] <= s.geo.ga_lo[a] + s.geo.ga_dim[a];
  if (inside && s.grid_slab) return TG_OK;
  int want_lo[3], want_hi[3];
  for (int a = 0; a < 3; ++a) {
    want_lo[a] = s.grid_slab ? std::min(lo[a], s.geo.ga_lo[a]) : lo[a];
    want_hi[a] = s.grid_slab ? std::max(hi[a], s.geo.ga_lo[a] + s.geo.ga_dim[a]) : hi[a];
  }
  int blo[3], bdim[3];
  alloc_box_for(s, want_lo, want_hi, blo, bdim);
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  if (!alloc_grid(s, blo, bdim)) return fail(TG_ERR_CUDA, "grid allocation failed");
  drop_graphs(s);
  s.grid_ready = false;
  s.grid_dirty = false;
  s.grid_ref = false;
  s.regrows += 1;
  return TG_OK;
}

int create(int device, const tg_params* P, const tg_particles* in, const tg_surface* surf,
           DeviceSim** out) {
  if (!P || !in || !out) return fail(TG_ERR_INVALID_ARGUMENT, "tg_create: null argument");
  if (in->n <= 0 || in->n_elastomer < 0 || in->n_elastomer > in->n)
    return fail(TG_ERR_EMPTY_SCENE, "init_scene: both elastomer and indenter particle sets must be non-empty");
  if (!in->x || !in->v || !in->mass || !in->volume0 || !in->tag)
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_create: x, v, mass, volume0 and tag are required");
  if (!(P->dt > 0.0)) return fail(TG_ERR_CONFIG, "dt must be > 0");
  if (P->res[0] < 4 || P->res[1] < 4 || P->res[2] < 4)
    return fail(TG_ERR_CONFIG, "grid resolution must be >= 4 per axis");
  if (!(P->dx > 0.0)) return fail(TG_ERR_CONFIG, "grid spacing must be > 0");
  if (!(P->youngs_modulus > 0.0)) return fail(TG_ERR_CONFIG, "youngs_modulus must be > 0");
  if (!(P->poisson_ratio >= 0.0 && P->poisson_ratio < 0.5))
    return fail(TG_ERR_CONFIG, "poisson_ratio must be in [0, 0.5)");
  if (!(P->density > 0.0)) return fail(TG_ERR_CONFIG, "density must be > 0");
  const int64_t n = in->n, n_el = in->n_elastomer, n_ind = n - n_el;
  for (int64_t p = 0; p < n; ++p) {
    const bool is_ind = in->tag[p] == kIndenter;
    if (is_ind != (p >= n_el))
      return fail(TG_ERR_CONFIG, "tg_create: elastomer particles must precede the indenter");
  }
  // init_scene assigns one mass / rest volume per material (scene.cpp:48-66).
  for (int64_t p = 0; p < n; ++p) {
    const int64_t ref = p < n_el ? 0 : n_el;
    if (in->mass[p] != in->mass[ref] || in->volume0[p] != in->volume0[ref])
      return fail(TG_ERR_CONFIG, "tg_create: mass / volume0 must be uniform per material");
  }
  int rc = check_device(device);
  if (rc) return rc;
  if (configure_device(device))
    return fail(TG_ERR_CUDA, "tg_create: could not set the kernels' shared-memory limits");

  auto* s = new DeviceSim();
  s->device = device;
  s->n = n;
  s->n_el = n_el;
  s->n_ind = n_ind;
  if (n_el > 0) { s->m_el = in->mass[0]; s->vol_el = in->volume0[0]; }
  if (n_ind > 0) { s->m_ind = in->mass[n_el]; s->vol_ind = in->volume0[n_el]; }
  Geometry& g = s->geo;
  for (int a = 0; a < 3; ++a) {
    g.res[a] = P->res[a];
    g.origin[a] = P->origin[a];
    g.gravity[a] = P->gravity[a];
    g.gdt[a] = P->gravity[a] * P->dt;  // engine.cpp:183
  }
  g.dx = P->dx;
  g.inv_dx = 1.0 / P->dx;
  g.dt = P->dt;
  // MaterialParams::mu / lambda (material.hpp:14-18)
  g.mu = P->youngs_modulus / (2.0 * (1.0 + P->poisson_ratio));
  g.lambda = P->youngs_modulus * P->poisson_ratio /
             ((1.0 + P->poisson_ratio) * (1.0 - 2.0 * P->poisson_ratio));
  g.with_gravity = (P->gravity[0] * P->gravity[0] + P->gravity[1] * P->gravity[1] +
                    P->gravity[2] * P->gravity[2]) > 0.0;
  g.stress_scale = -P->dt * 4.0 * g.inv_dx * g.inv_dx;
  if (const char* m = std::getenv("TACCHI_SCATTER")) g.scatter_mode = std::atoi(m);
  if (const char* f = std::getenv("TACCHI_FULL_INDENTER")) s->full_indenter = std::atoi(f) != 0;
  // launch-shape A/B switches (tools/README.md); defaults are the measured best
  s->zpad = 2;
  if (const char* e = std::getenv("TACCHI_AB_NO_WALKS")) s->ab_no_walks = std::atoi(e) != 0;
  if (const char* e = std::getenv("TACCHI_ZPAD")) s->zpad = std::max(2, std::atoi(e) & ~1);
  g.gu_bps = 5;  // one wave of resident blocks (1367 vs 1360 frames/s with 10)
  g.pdl_early = 1;
  g.gel_trigger = 1;
  if (const char* e = std::getenv("TACCHI_GEL_TRIGGER")) g.gel_trigger = std::atoi(e);
  g.fin_trigger = 1;
  g.det_skip0 = 1;
  g.det_fast4 = 1;
  if (const char* e = std::getenv("TACCHI_DET_FAST4")) g.det_fast4 = std::atoi(e);
  if (const char* e = std::getenv("TACCHI_DET_SKIP0")) g.det_skip0 = std::atoi(e);
  if (const char* e = std::getenv("TACCHI_FIN_TRIGGER")) g.fin_trigger = std::atoi(e);
  g.ind_first = 1;
  if (const char* e = std::getenv("TACCHI_GU_BPS")) g.gu_bps = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("TACCHI_PDL_EARLY")) g.pdl_early = std::atoi(e);
  if (const char* e = std::getenv("TACCHI_IND_FIRST")) g.ind_first = std::atoi(e);
  s->sms = sm_count(device);
  // Deterministic-mode fixed-point scales (powers of two): A resolves 2^-50
  // of one elastomer particle's mass (momentum: of its mass x 1 m/s), range
  // 2^12 of them per node; M_I (sums of B-spline weights <= 1) resolves 2^-52.
  {
    const double m_ref = s->m_el > 0 ? s->m_el : (s->m_ind > 0 ? s->m_ind : 1.0);
    int ex = 0;
    std::frexp(m_ref, &ex);  // m_ref in [2^(ex-1), 2^ex)
    g.fx_s = std::ldexp(1.0, 50 - ex);
    g.fx_inv = std::ldexp(1.0, ex - 50);
    g.fxi_s = std::ldexp(1.0, 52);
    g.fxi_inv = std::ldexp(1.0, -52);
    g.det = 0;
  }

  // Indenter particles are re-ordered by base cell so that P2G scatters from
  // neighbouring lanes hit neighbouring nodes; perm maps back.
  s->perm.resize(n);
  std::iota(s->perm.begin(), s->perm.end(), 0);
  std::vector<int64_t> col_starts;
  // Order: base cell (bx, by) of the initial position, then z. Under the press
  // (motion along z) the order stays sorted by (bx, by, bz) for the whole
  // episode, which keeps runs of equal base cell contiguous for the chunked
  // indenter scatter (k_p2g_ind_chunk).
  if (n_ind > 1) {
    std::vector<long long> key(n_ind);
    for (int64_t q = 0; q < n_ind; ++q) {
      const double* xp = in->x + 3 * (n_el + q);
      long long k = 0;
      for (int a = 0; a < 2; ++a) {
        const int b = std::min(std::max(host_base(xp[a], g.origin[a], g.inv_dx), -1), g.res[a]);
        k = k * (g.res[a] + 2) + (b + 1);
      }
      key[q] = k;
    }
    std::stable_sort(s->perm.begin() + n_el, s->perm.end(), [&](int64_t a, int64_t b) {
      const long long ka = key[a - n_el], kb = key[b - n_el];
      if (ka != kb) return ka < kb;
      return in->x[3 * a + 2] < in->x[3 * b + 2];
    });
    col_starts.push_back(n_el);
    for (int64_t q = n_el + 1; q < n; ++q)
      if (key[s->perm[q] - n_el] != key[s->perm[q - 1] - n_el]) col_starts.push_back(q);
    col_starts.push_back(n);
  } else if (n_ind == 1) {
    col_starts = {n_el, n};
  }
  // Lattice metadata (particle_set.hpp:16-17): the surface is the top layer
  // of an nx x ny x nz elastomer lattice; the CTA tiling follows it, and the
  // elastomer's storage order within each warp's slots is dealt for the
  // shared-memory banks (permute_gel_lanes, folded into perm).
  if (surf && surf->particle && surf->nx >= 2 && surf->ny >= 2) {
    const int64_t cols = static_cast<int64_t>(surf->nx) * surf->ny;
    if (n_el % cols == 0) {
      configure_gel_tiling(*s, surf->nx, surf->ny, static_cast<int>(n_el / cols));
      permute_gel_lanes(*s, in->x);
    }
  }
  // Stream priorities: the handle's stream (grid_update, elastomer kernel:
  // the substep's critical path) above the walk stream, whose kernel has the
  // whole substep to finish before the join (1362 vs 1358.5 frames/s;
  // TACCHI_WALK_PRIO=0 gives both the default priority). Graph replays run
  // every node at the launch stream's priority: instantiating with
  // cudaGraphInstantiateFlagUseNodePriority measured slower either way
  // (DESIGN 4.5).
  int prio_lo = 0, prio_hi = 0;
  cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi);
  const bool prio = !std::getenv("TACCHI_WALK_PRIO") || std::atoi(std::getenv("TACCHI_WALK_PRIO"));
  if (prio)
    cudaStreamCreateWithPriority(&s->stream, cudaStreamNonBlocking, prio_hi);
  else
    cudaStreamCreateWithFlags(&s->stream, cudaStreamNonBlocking);
  if (const char* e = std::getenv("TACCHI_WALKS")) s->fork_walks = std::string(e) != "fused";
  if (s->fork_walks &&
      (cudaStreamCreateWithPriority(&s->walk_stream, cudaStreamNonBlocking,
                                    prio ? prio_lo : 0) != cudaSuccess ||
       cudaEventCreateWithFlags(&s->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
       cudaEventCreateWithFlags(&s->ev_join, cudaEventDisableTiming) != cudaSuccess))
    s->fork_walks = false;
  // Node arrays over the elastomer's node box plus the walks' reach (the
  // step path touches nothing else); the whole window when there is no
  // elastomer. They grow on demand (ensure_alloc).
  int alo[3], ahi[3], adim[3];
  {
    const int64_t b = n_el > 0 ? 0 : n_el, e = n_el > 0 ? n_el : n;
    for (int a = 0; a < 3; ++a) {
      double lo = in->x[3 * b + a], hi = lo;
      for (int64_t p = b; p < e; ++p) {
        lo = std::min(lo, in->x[3 * p + a]);
        hi = std::max(hi, in->x[3 * p + a]);
      }
      alo[a] = host_base(lo, g.origin[a], g.inv_dx) - kWalkReach;
      ahi[a] = host_base(hi, g.origin[a], g.inv_dx) + 3 + kWalkReach;
    }
    alloc_box_for(*s, alo, ahi, alo, adim);
  }
  bool ok = cudaMalloc(&s->x, 3 * n * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->v, 3 * n * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->C, std::max<int64_t>(9 * n_el, 1) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->F, std::max<int64_t>(9 * n_el, 1) * sizeof(double)) == cudaSuccess &&
            cudaMalloc(&s->tag, std::max<int64_t>(n_el, 1)) == cudaSuccess &&
            alloc_grid(*s, alo, adim) &&
            cudaMalloc(&s->col_start, std::max<size_t>(col_starts.size(), 1) * sizeof(int64_t)) ==
                cudaSuccess &&
            cudaMalloc(&s->ind_moves, std::max<int64_t>(n_ind, 1)) == cudaSuccess &&
            cudaMalloc(&s->ctl, sizeof(Ctl)) == cudaSuccess &&
            cudaMallocHost(&s->h_ctl, sizeof(Ctl)) == cudaSuccess &&
            cudaMallocHost(&s->h_vind, 3 * sizeof(double)) == cudaSuccess;
  if (!ok) {
    delete s;
    return fail(TG_ERR_CUDA, "tg_create: device allocation failed");
  }
  cudaMemsetAsync(s->ind_moves, 0, std::max<int64_t>(n_ind, 1), s->stream);
  s->n_cols = col_starts.empty() ? 0 : static_cast<int>(col_starts.size()) - 1;
  if (s->n_cols > 0)
    copy_sync(*s, s->col_start, col_starts.data(), col_starts.size() * sizeof(int64_t),
              cudaMemcpyHostToDevice);
  std::memset(s->h_ctl, 0, sizeof(Ctl));
  s->h_ctl->err = kNoError;
  for (int a = 0; a < 3; ++a) s->h_ctl->vind[a] = in->indenter_velocity[a];
  // Is the indenter velocity uniform (it is for init_scene's output)?
  s->ind_v_uniform = true;
  for (int64_t p = n_el + 1; p < n && s->ind_v_uniform; ++p)
    for (int a = 0; a < 3; ++a)
      if (in->v[3 * p + a] != in->v[3 * n_el + a]) s->ind_v_uniform = false;
  for (int a = 0; a < 3; ++a) s->h_ctl->ind_v[a] = n_ind > 0 ? in->v[3 * n_el + a] : 0.0;
  s->h_ctl->diag_min_det_f = 1.0;
  cudaMemcpyAsync(s->ctl, s->h_ctl, sizeof(Ctl), cudaMemcpyHostToDevice, s->stream);
  launch_reset(*s, kResetAll);

  // Tags of the elastomer (Elastomer / ElastomerBottom).
  std::vector<uint8_t> tags(std::max<int64_t>(n_el, 1));
  for (int64_t p = 0; p < n_el; ++p) tags[p] = in->tag[s->perm[p]];
  copy_sync(*s, s->tag, tags.data(), n_el, cudaMemcpyHostToDevice);

  rc = upload(*s, in->x, in->v, in->C, in->F, true);
  if (rc) {
    delete s;
    return rc;
  }
  if (surf && surf->particle && surf->nx >= 2 && surf->ny >= 2) {
    s->surf_nx = surf->nx;
    s->surf_ny = surf->ny;
    s->surf_geom[0] = surf->x0;
    s->surf_geom[1] = surf->y0;
    s->surf_geom[2] = surf->sx;
    s->surf_geom[3] = surf->sy;
    s->surf_geom[4] = surf->z0;
    const size_t cnt = static_cast<size_t>(surf->nx) * surf->ny;
    std::vector<int64_t> inv(n);
    for (int64_t q = 0; q < n; ++q) inv[s->perm[q]] = q;
    std::vector<uint32_t> idx(cnt);
    for (size_t k = 0; k < cnt; ++k) {
      if (surf->particle[k] >= static_cast<uint64_t>(n)) {
        delete s;
        return fail(TG_ERR_NO_SURFACE, "surface lattice index out of range");
      }
      idx[k] = static_cast<uint32_t>(inv[surf->particle[k]]);
    }
    ok = cudaMalloc(&s->surf_idx, cnt * sizeof(uint32_t)) == cudaSuccess &&
         cudaMalloc(&s->surf_depth, cnt * sizeof(double)) == cudaSuccess;
    if (!ok) {
      delete s;
      return fail(TG_ERR_CUDA, "tg_create: device allocation failed");
    }
    copy_sync(*s, s->surf_idx, idx.data(), cnt * sizeof(uint32_t), cudaMemcpyHostToDevice);
  }
  // Per-CTA tile boxes carried from each P2G to the next G2P (mpm_kernels.cu).
  const size_t ctas = std::max<size_t>(gel_block_count(*s), 1);
  if (cudaMalloc(&s->geo.cta_box, ctas * 8 * sizeof(int)) != cudaSuccess) {
    delete s;
    return fail(TG_ERR_CUDA, "tg_create: device allocation failed");
  }
  cudaMemsetAsync(s->geo.cta_box, 0, ctas * 8 * sizeof(int), s->stream);
  const cudaError_t e = cudaStreamSynchronize(s->stream);
  if (e != cudaSuccess) {
    delete s;
    return fail(TG_ERR_CUDA, std::string("tg_create: ") + cudaGetErrorString(e));
  }
  *out = s;
  return TG_OK;
}

// Applies the open indenter chain's pending advects and closes the chain.
static void flush_indenter(DeviceSim& s) {
  if (!s.chain_open) return;
  if (s.n_cols > 0 && !s.full_indenter) launch_ind_catchup(s);
  s.chain_open = false;
  s.chain_len = 0;
}

// Reads back the control block and converts a latched device error into the
// reference's exception semantics. `end_substep` is the absolute substep index
// one past the last substep this call asked for: an error raised for a later
// substep (the next zero_grid's window check) is not this call's error; the
// window is just recomputed on the next call, which then raises it itself.
static int sync_and_check(DeviceSim& s, int end_substep) {
  CUDA_TRY(cudaMemcpyAsync(s.h_ctl, s.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s.stream));
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  CUDA_TRY(cudaGetLastError());
  const Ctl& c = *s.h_ctl;
  s.host_substep = c.substep;
  if (c.err == kNoError) return TG_OK;
  flush_indenter(s);  // the state at the throw includes the indenter's advects
  const int code = err_code_of(c.err);
  const int at = err_substep_of(c.err);
  // Clear the latch; the next call re-derives the window from the state.
  static const unsigned long long clear = kNoError;
  CUDA_TRY(cudaMemcpyAsync(&s.ctl->err, &clear, sizeof(clear), cudaMemcpyHostToDevice, s.stream));
  launch_reset(s, kResetAll);
  s.window_valid = false;
  s.grid_dirty = false;
  s.grid_ready = false;
  if (code == kErrRegrow) {
    // A scatter of substep `at` would have left the node arrays: every
    // substep before `at` is complete; grow the arrays over the boxes of
    // substep `at` (finalize wrote them) and let the caller run the rest.
    int lo[3], hi[3];
    const bool walks = s.n_cols > 0 && !s.full_indenter && s.ind_v_uniform && s.n_el > 0;
    for (int a = 0; a < 3; ++a) {
      lo[a] = walks ? c.box_lo[0][a] - kWalkReach : c.win_lo[a];
      hi[a] = walks ? c.box_hi[0][a] + kWalkReach : c.win_hi[a];
    }
    const int rc = ensure_alloc(s, lo, hi);
    if (rc) return rc;
    s.resume_substeps = std::max(end_substep - at, 0);
    return kResume;
  }
  // A look-ahead scatter may have started anywhere in the grid: reset the
  // accumulators wholesale (errors are rare; this keeps the invariant simple).
  CUDA_TRY(cudaMemsetAsync(s.grid_slab, 0, s.grid_slab_bytes, s.stream));
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  if (at >= end_substep) return TG_OK;
  const char* what = code == kErrOutOfGrid
                         ? "particles left the stencil-safe margin (check dt and scene size)"
                         : code == kErrDegenerateF ? "particle_to_grid: det(F) <= 0" : "device error";
  return fail(code, std::string(error_name(code)) + ": " + what);
}

// The substep plan of one mpm::step call (see mpm_kernels.cu): a standalone
// scatter for the first substep, then per substep grid_update (re-zeroing the
// accumulators), the fused G2P(+boundary+advect)+look-ahead-P2G kernel and
// finalize, with the indenter's look-ahead walks on the walk stream beside
// the first two (forked after the previous finalize, joined before this one).
// When the previous call already scattered this call's first substep
// (grid_ready), the standalone scatter is skipped; every substep, the last one
// included, scatters the next substep's particles, so consecutive step() calls
// chain without a standalone scatter.
// One substep of the step path.
static int record_substep(DeviceSim& s, int sms, bool cols) {
  if (cols && s.n_el > 0 && s.fork_walks && s.walk_stream) {
    // the walks of substep s need only the previous finalize (box, chain),
    // the indenter's own state and M_I buffer (s + 1) & 1: fork them beside
    // grid_update and the elastomer kernel, join before this finalize (which
    // completes them if the elastomer left their box)
    cudaEventRecord(s.ev_fork, s.stream);
    cudaStreamWaitEvent(s.walk_stream, s.ev_fork, 0);
    int k = launch_ind_walks_on(s, s.walk_stream);
    cudaEventRecord(s.ev_join, s.walk_stream);
    k += launch_grid_update(s, sms, true);
    k += launch_g2p2g_gel(s, true, false);
    cudaStreamWaitEvent(s.stream, s.ev_join, 0);
    k += launch_finalize_step(s, true);
    return k;
  }
  int k = launch_grid_update(s, sms, true);
  if (cols && s.n_el > 0) {
    // the indenter's column walks run as extra blocks of the elastomer kernel
    k += launch_g2p2g_gel(s, true, true);
    k += launch_finalize_step(s, true);
    return k;
  }
  k += launch_g2p2g_gel(s, true);
  k += cols ? launch_ind_cols(s, true) : launch_ind_move(s, true);
  k += launch_finalize_step(s);
  return k;
}

static int record_substeps(DeviceSim& s, int n_substeps) {
  int k = 0;
  const int sms = sm_count(s.device);
  const bool cols = s.n_cols > 0 && !s.full_indenter;
  if (!s.grid_ready) {
    if (s.grid_dirty) k += launch_clear(s, sms);
    k += launch_p2g_gel(s);
    k += (cols && s.ind_v_uniform) ? launch_ind_cols(s, false) : launch_p2g_ind(s);
  }
  for (int i = 0; i < n_substeps; ++i) k += record_substep(s, sms, cols);
  return k;
}

// Enqueues mpm::step's n_substeps (engine.cpp:288-297) on the handle's stream.
constexpr int kChainMax = 200;

int step_submit(DeviceSim& s, const double vind[3], int n_substeps) {
  CUDA_TRY(cudaSetDevice(s.device));
  s.pending_start = s.host_substep;
  if (n_substeps <= 0) return TG_OK;
  for (int a = 0; a < 3; ++a) s.h_vind[a] = vind[a];
  // the indenter chain continues only with the same velocity (bitwise) and
  // for at most kChainMax substeps (the per-particle move counters are 8-bit;
  // 200 = tg_step's chunk, so every 200 substeps of a long run pay one catch-up)
  if (s.chain_open && (std::memcmp(s.chain_vind, vind, sizeof(s.chain_vind)) != 0 ||
                       s.chain_len + n_substeps > kChainMax))
    flush_indenter(s);
  // zero_grid of the first substep (a failing window latches OutOfGrid for
  // this substep and every later kernel exits early); it reads positions.
  if (!s.window_valid) {
    flush_indenter(s);
    launch_window(s);
  }
  s.window_valid = true;
  if (!s.chain_open) {
    launch_chain_begin(s);
    s.chain_open = true;
    std::memcpy(s.chain_vind, vind, sizeof(s.chain_vind));
  }
  s.chain_len += n_substeps;
  if (s.use_graphs) {
    const int key = n_substeps * 32 + (s.grid_dirty ? 1 : 0) + (s.ind_v_uniform ? 2 : 0) +
                    (s.grid_ready ? 4 : 0);
    auto it = s.graphs.find(key);
    const bool replay = it != s.graphs.end();
    if (!replay) {
      cudaGraph_t graph;
      const int64_t before = s.kernel_launches;
      CUDA_TRY(cudaStreamBeginCapture(s.stream, cudaStreamCaptureModeThreadLocal));
      cudaMemcpyAsync(&s.ctl->vind[0], s.h_vind, 3 * sizeof(double), cudaMemcpyHostToDevice,
                      s.stream);
      const int k = record_substeps(s, n_substeps);
      CUDA_TRY(cudaStreamEndCapture(s.stream, &graph));
      cudaGraphExec_t exec;
      CUDA_TRY(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      s.kernel_launches = before;  // counted per replay below
      it = s.graphs.emplace(key, exec).first;
      s.graph_kernels[key] = k;
    }
    CUDA_TRY(cudaGraphLaunch(it->second, s.stream));
    s.kernel_launches += s.graph_kernels[key];
  } else {
    CUDA_TRY(cudaMemcpyAsync(&s.ctl->vind[0], s.h_vind, 3 * sizeof(double),
                             cudaMemcpyHostToDevice, s.stream));
    record_substeps(s, n_substeps);
  }
  s.grid_dirty = false;
  s.ind_v_uniform = true;
  s.grid_ready = true;
  s.grid_ref = false;  // the grid now holds the next substep's look-ahead scatter
  return TG_OK;
}

int step_finish(DeviceSim& s, int n_substeps) {
  CUDA_TRY(cudaSetDevice(s.device));
  return sync_and_check(s, s.pending_start + std::max(n_substeps, 0));
}

int phase(DeviceSim& s, int ph, const double vind[3]);

int step(DeviceSim& s, const double vind[3], int n_substeps) {
  if (s.keep_grid && n_substeps > 0) {
    // The fused plan leaves a look-ahead scatter in the grid; with keep_grid
    // the last substep runs the six phases (engine.cpp:288-297) so that the
    // grid afterwards holds that substep's P2G and grid_update, as the
    // reference's does.
    for (int left = n_substeps - 1; left > 0;) {  // chunks as tg_step's
      const int c = left > 200 ? 200 : left;
      const int rc = step_submit(s, vind, c);
      if (rc) return rc;
      const int e = step_finish(s, c);
      if (e == kResume) {  // node arrays grown mid-chunk: run the rest of it
        left -= c - s.resume_substeps;
        continue;
      }
      if (e) return e;
      left -= c;
    }
    for (int ph = TG_PHASE_ZERO_GRID; ph <= TG_PHASE_ADVECT; ++ph)
      if (const int e = phase(s, ph, vind)) return e;
    return TG_OK;
  }
  for (int left = n_substeps;;) {
    const int rc = step_submit(s, vind, left);
    if (rc) return rc;
    const int e = step_finish(s, left);
    if (e != kResume) return e;
    left = s.resume_substeps;  // node arrays grown mid-call: run the rest
    if (left <= 0) return TG_OK;
  }
}

int check_device_public(int device) { return check_device(device); }
void flush_indenter_public(DeviceSim& s) { flush_indenter(s); }
void drop_graphs_public(DeviceSim& s) { drop_graphs(s); }

// Per-kernel device times of the substep plan (CUDA events between the
// launches, no graph), averaged over `reps` substeps: one mpm::step call of
// `reps` substeps launched kernel by kernel. Order of out_ms:
// [p2g_elastomer (standalone, first substep only), p2g_indenter (standalone),
//  grid_update, g2p2g_elastomer (G2P+boundary+advect+look-ahead P2G),
//  indenter_move_p2g, finalize]. Used by bench.py for the roofline.
int time_phases(DeviceSim& s, const double vind[3], int reps, double* out_ms) {
  CUDA_TRY(cudaSetDevice(s.device));
  const int sms = sm_count(s.device);
  constexpr int kGroups = 6;
  cudaEvent_t ev[kGroups + 1];
  for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
  for (int g = 0; g < kGroups; ++g) out_ms[g] = 0.0;
  for (int a = 0; a < 3; ++a) s.h_vind[a] = vind[a];
  const int start = s.host_substep;
  flush_indenter(s);
  if (!s.window_valid) launch_window(s);
  s.window_valid = true;
  CUDA_TRY(cudaMemcpyAsync(&s.ctl->vind[0], s.h_vind, 3 * sizeof(double), cudaMemcpyHostToDevice,
                           s.stream));
  if (s.grid_ready) {  // discard the previous call's look-ahead scatter
    s.grid_ready = false;
    s.grid_dirty = true;
  }
  if (s.grid_dirty) launch_clear(s, sms);
  const bool cols = s.n_cols > 0 && !s.full_indenter;
  launch_chain_begin(s);
  float ms = 0.f;
  cudaEventRecord(ev[0], s.stream);
  launch_p2g_gel(s);
  cudaEventRecord(ev[1], s.stream);
  if (cols && s.ind_v_uniform) launch_ind_cols(s, false);
  else launch_p2g_ind(s);
  cudaEventRecord(ev[2], s.stream);
  CUDA_TRY(cudaEventSynchronize(ev[2]));
  cudaEventElapsedTime(&ms, ev[0], ev[1]);
  out_ms[0] = ms;
  cudaEventElapsedTime(&ms, ev[1], ev[2]);
  out_ms[1] = ms;
  for (int r = 0; r < reps; ++r) {
    cudaEventRecord(ev[2], s.stream);
    launch_grid_update(s, sms, true);
    cudaEventRecord(ev[3], s.stream);
    launch_g2p2g_gel(s, true);
    cudaEventRecord(ev[4], s.stream);
    if (cols) launch_ind_cols(s, true);
    else launch_ind_move(s, true);
    cudaEventRecord(ev[5], s.stream);
    launch_finalize_step(s);
    cudaEventRecord(ev[6], s.stream);
    CUDA_TRY(cudaEventSynchronize(ev[6]));
    for (int g = 2; g < kGroups; ++g) {
      cudaEventElapsedTime(&ms, ev[g], ev[g + 1]);
      out_ms[g] += ms / reps;
    }
  }
  if (cols) launch_ind_catchup(s);
  for (auto& e : ev) cudaEventDestroy(e);
  s.grid_ready = true;  // the last substep scattered the next one, as in step()
  s.grid_ref = false;
  const int rc = sync_and_check(s, start + reps);
  // grown mid-run: the timings cover a partial run; the state is consistent
  return rc == kResume ? TG_OK : rc;
}

int phase(DeviceSim& s, int ph, const double vind[3]) {
  CUDA_TRY(cudaSetDevice(s.device));
  flush_indenter(s);  // the phases read and move every particle
  if (s.grid_ready) {  // phases drive zero_grid / P2G themselves
    s.grid_ready = false;
    s.grid_dirty = true;
  }
  const int start = s.host_substep;
  const int sms = sm_count(s.device);
  // The phase path touches the whole active window (every indenter particle
  // scatters): grow the node arrays over it and the box zero_grid clears.
  auto cover_window = [&]() -> int {
    CUDA_TRY(cudaMemcpyAsync(s.h_ctl, s.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s.stream));
    CUDA_TRY(cudaStreamSynchronize(s.stream));
    const Ctl& c = *s.h_ctl;
    if (c.err != kNoError) return TG_OK;  // reported by sync_and_check below
    int lo[3], hi[3];
    for (int a = 0; a < 3; ++a) {
      const bool clr = c.clr_hi[a] > c.clr_lo[a];
      lo[a] = clr ? std::min(c.win_lo[a], c.clr_lo[a]) : c.win_lo[a];
      hi[a] = clr ? std::max(c.win_hi[a], c.clr_hi[a]) : c.win_hi[a];
      if (hi[a] <= lo[a]) return TG_OK;  // no window yet
    }
    return ensure_alloc(s, lo, hi);
  };
  switch (ph) {
    case TG_PHASE_ZERO_GRID: {
      launch_window(s);
      if (const int rc = cover_window()) return rc;
      launch_clear(s, sms);
      break;
    }
    case TG_PHASE_PARTICLE_TO_GRID:
      if (const int rc = cover_window()) return rc;
      launch_p2g(s, true);
      break;
    case TG_PHASE_GRID_UPDATE: launch_grid_update(s, sms, false); break;
    case TG_PHASE_GRID_TO_PARTICLE: launch_phase_g2p(s); break;
    case TG_PHASE_APPLY_BOUNDARY:
      for (int a = 0; a < 3; ++a) s.h_vind[a] = vind[a];
      CUDA_TRY(cudaMemcpyAsync(&s.ctl->vind[0], s.h_vind, 3 * sizeof(double),
                               cudaMemcpyHostToDevice, s.stream));
      launch_phase_boundary(s);
      break;
    case TG_PHASE_ADVECT: launch_phase_advect(s); break;
    default: return fail(TG_ERR_INVALID_ARGUMENT, "tg_phase: bad phase id");
  }
  s.window_valid = false;  // phases drive zero_grid explicitly
  s.grid_ref = true;       // the phases keep the grid exactly as the reference's
  const int rc = sync_and_check(s, start + 1);
  if (rc == kResume)  // a scatter outside the node arrays (P2G without zero_grid)
    return fail(TG_ERR_INVALID_ARGUMENT,
                "particle_to_grid: particles outside the grid window; call zero_grid first");
  return rc;
}

static void to_component_major(const double* src, int64_t n, int ncomp, const std::vector<int64_t>& perm,
                               int64_t begin, int64_t end, std::vector<double>& dst) {
  const int64_t cnt = end - begin;
  dst.resize(static_cast<size_t>(ncomp) * cnt);
  for (int64_t q = begin; q < end; ++q) {
    const int64_t r = perm[q];
    for (int c = 0; c < ncomp; ++c) dst[static_cast<size_t>(c) * cnt + (q - begin)] = src[ncomp * r + c];
  }
  (void)n;
}

int upload(DeviceSim& s, const double* x, const double* v, const double* Cm, const double* Fm,
           bool init) {
  CUDA_TRY(cudaSetDevice(s.device));
  flush_indenter(s);
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  std::vector<double> buf;
  auto put3 = [&](const double* src, double* dst) -> int {
    to_component_major(src, s.n, 3, s.perm, 0, s.n, buf);
    const cudaError_t e = copy_sync(s, dst, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice);
    return e == cudaSuccess ? 0 : fail(TG_ERR_CUDA, cudaGetErrorString(e));
  };
  auto put9 = [&](const double* src, double* dst, bool identity) -> int {
    if (s.n_el == 0) return 0;
    if (src) {
      to_component_major(src, s.n, 9, s.perm, 0, s.n_el, buf);
    } else {
      buf.assign(static_cast<size_t>(9) * s.n_el, 0.0);
      if (identity)
        for (int d = 0; d < 3; ++d)
          std::fill(buf.begin() + static_cast<size_t>(4 * d) * s.n_el,
                    buf.begin() + static_cast<size_t>(4 * d + 1) * s.n_el, 1.0);
    }
    const cudaError_t e = copy_sync(s, dst, buf.data(), buf.size() * sizeof(double), cudaMemcpyHostToDevice);
    return e == cudaSuccess ? 0 : fail(TG_ERR_CUDA, cudaGetErrorString(e));
  };
  int rc = 0;
  if (x && (rc = put3(x, s.x))) return rc;
  if (v && (rc = put3(v, s.v))) return rc;
  if (v && s.n_ind > 0 && !init) {
    bool uniform = true;
    for (int64_t p = s.n_el + 1; p < s.n && uniform; ++p)
      for (int a = 0; a < 3; ++a)
        if (v[3 * p + a] != v[3 * s.n_el + a]) uniform = false;
    s.ind_v_uniform = uniform;
    if (uniform) CUDA_TRY(copy_sync(s, &s.ctl->ind_v[0], v + 3 * s.n_el, 3 * sizeof(double),
                                    cudaMemcpyHostToDevice));
  }
  if ((Cm || init) && (rc = put9(Cm, s.C, false))) return rc;
  if ((Fm || init) && (rc = put9(Fm, s.F, true))) return rc;
  s.window_valid = false;
  if (s.grid_ready) {  // the look-ahead scatter used the old state
    s.grid_ready = false;
    s.grid_dirty = true;
  }
  return TG_OK;
}

int download(DeviceSim& s, double* x, double* v, double* Cm, double* Fm) {
  CUDA_TRY(cudaSetDevice(s.device));
  flush_indenter(s);
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  std::vector<double> buf;
  auto get3 = [&](const double* src, double* dst) -> int {
    buf.resize(3 * s.n);
    const cudaError_t e = copy_sync(s, buf.data(), src, buf.size() * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(TG_ERR_CUDA, cudaGetErrorString(e));
    for (int64_t q = 0; q < s.n; ++q)
      for (int c = 0; c < 3; ++c) dst[3 * s.perm[q] + c] = buf[static_cast<size_t>(c) * s.n + q];
    return 0;
  };
  auto get9 = [&](const double* src, double* dst, bool identity) -> int {
    if (s.n_el > 0) {
      buf.resize(9 * s.n_el);
      const cudaError_t e = copy_sync(s, buf.data(), src, buf.size() * sizeof(double), cudaMemcpyDeviceToHost);
      if (e != cudaSuccess) return fail(TG_ERR_CUDA, cudaGetErrorString(e));
      for (int64_t q = 0; q < s.n_el; ++q)  // perm: the lane order within warps
        for (int c = 0; c < 9; ++c) dst[9 * s.perm[q] + c] = buf[static_cast<size_t>(c) * s.n_el + q];
    }
    // Indenter particles keep C = 0 and F = I (engine.cpp:218; scene.cpp:67-68).
    for (int64_t q = s.n_el; q < s.n; ++q)
      for (int c = 0; c < 9; ++c) dst[9 * q + c] = (identity && (c % 4 == 0)) ? 1.0 : 0.0;
    return 0;
  };
  int rc = 0;
  if (x && (rc = get3(s.x, x))) return rc;
  if (v && (rc = get3(s.v, v))) return rc;
  if (v && s.ind_v_uniform && s.n_ind > 0) {
    double u[3];
    CUDA_TRY(copy_sync(s, u, &s.ctl->ind_v[0], sizeof u, cudaMemcpyDeviceToHost));
    for (int64_t q = s.n_el; q < s.n; ++q)
      for (int a = 0; a < 3; ++a) v[3 * s.perm[q] + a] = u[a];
  }
  if (Cm && (rc = get9(s.C, Cm, false))) return rc;
  if (Fm && (rc = get9(s.F, Fm, true))) return rc;
  return TG_OK;
}

// ---------------------------------------------------------------------------
// Pipelined control steps: frame k's read-back overlaps frame k+1's substeps.
// ---------------------------------------------------------------------------
int capture_enqueue_to(DeviceSim& s, const tg_render& r, double* depth_pinned, uint8_t* rgb_pinned,
                       std::string& msg, cudaStream_t shade = nullptr,
                       cudaEvent_t surface_done = nullptr);

static int frame_buffers(DeviceSim& s, FrameSlot& f, size_t pixels) {
  if (!s.copy_stream && cudaStreamCreateWithFlags(&s.copy_stream, cudaStreamNonBlocking) != cudaSuccess)
    return fail(TG_ERR_CUDA, "pipelined capture: stream creation failed");
  if ((!f.ev && cudaEventCreateWithFlags(&f.ev, cudaEventDisableTiming) != cudaSuccess) ||
      (!f.captured && cudaEventCreateWithFlags(&f.captured, cudaEventDisableTiming) != cudaSuccess))
    return fail(TG_ERR_CUDA, "pipelined capture: event creation failed");
  if ((!f.ctl && cudaMallocHost(&f.ctl, sizeof(Ctl)) != cudaSuccess) ||
      (!f.d_snap && cudaMalloc(&f.d_snap, sizeof(Ctl)) != cudaSuccess))
    return fail(TG_ERR_CUDA, "pipelined capture: allocation failed");
  if (pixels > f.pixels) {
    cudaFreeHost(f.depth);
    cudaFreeHost(f.rgb);
    f.depth = nullptr;
    f.rgb = nullptr;
    if (cudaMallocHost(&f.depth, pixels * sizeof(double)) != cudaSuccess ||
        cudaMallocHost(&f.rgb, pixels * 3) != cudaSuccess)
      return fail(TG_ERR_CUDA, "pipelined capture: pinned allocation failed");
    f.pixels = pixels;
  }
  return TG_OK;
}

// mpm::step + sim::capture of one frame, synchronously, into the slot (the
// keep_grid path, a frame that follows a grown allocation).
static int frame_run_sync(DeviceSim& s, FrameSlot& f) {
  // pending read-backs of other frames must drain the capture buffers first
  if (s.copy_stream) CUDA_TRY(cudaStreamSynchronize(s.copy_stream));
  int rc = step(s, f.v, f.n);
  if (rc) return rc;
  std::string msg;
  rc = capture_enqueue_to(s, f.r, f.depth, f.rgb, msg);
  if (rc) return fail(rc, msg);
  CUDA_TRY(cudaStreamSynchronize(s.stream));
  return TG_OK;
}

int frame_submit(DeviceSim& s, const double v[3], int n, const tg_render& r, bool read_back,
                 int64_t* ticket) {
  CUDA_TRY(cudaSetDevice(s.device));
  if (n < 0 || n > 200) return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_submit: n outside [0, 200]");
  FrameSlot& f = s.frames[s.frames_submitted % 2];
  if (f.live)
    return fail(TG_ERR_INVALID_ARGUMENT,
                "tg_step_capture_submit: two frames in flight; wait for the oldest first");
  int rc = frame_buffers(s, f, static_cast<size_t>(std::max(r.width, 0)) * std::max(r.height, 0));
  if (rc) return rc;
  for (int a = 0; a < 3; ++a) f.v[a] = v[a];
  f.n = n;
  f.r = r;
  f.replay = false;
  f.status = 0;
  f.msg.clear();
  if (s.keep_grid) {  // the last substep runs the (synchronous) phase path
    rc = frame_run_sync(s, f);
    if (rc) return rc;
    CUDA_TRY(cudaMemcpyAsync(f.ctl, s.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, s.stream));
    CUDA_TRY(cudaEventRecord(f.ev, s.stream));
  } else {
    // handle stream: the substeps, a device snapshot of the control block
    // and (once the previous frame's shading has released the capture
    // buffers) the surface gather; copy stream: the shading kernel and the
    // read-backs, while the handle stream already runs the next frame
    const int start = s.host_substep;
    rc = step_submit(s, v, n);
    if (rc) return rc;
    launch_snapshot_ctl(s, f.d_snap);
    const FrameSlot& prev = s.frames[(s.frames_submitted + 1) % 2];
    if (prev.used) CUDA_TRY(cudaStreamWaitEvent(s.stream, prev.ev, 0));
    std::string msg;
    rc = capture_enqueue_to(s, r, read_back ? f.depth : nullptr, read_back ? f.rgb : nullptr, msg,
                            s.copy_stream, f.captured);
    if (rc) return fail(rc, msg);
    CUDA_TRY(cudaMemcpyAsync(f.ctl, f.d_snap, sizeof(Ctl), cudaMemcpyDeviceToHost, s.copy_stream));
    CUDA_TRY(cudaEventRecord(f.ev, s.copy_stream));
    f.end_substep = start + n;
    s.host_substep = start + n;  // the host's view until the frame is waited for
  }
  f.used = true;
  f.live = true;
  f.read_back = read_back;
  *ticket = s.frames_submitted++;
  return TG_OK;
}

int frame_wait(DeviceSim& s, int64_t ticket, double** depth, uint8_t** rgb) {
  CUDA_TRY(cudaSetDevice(s.device));
  if (ticket != s.frames_collected)
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_wait: frames are waited for in order");
  FrameSlot& f = s.frames[ticket % 2];
  if (!f.live) return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_wait: no such frame");
  f.live = false;
  s.frames_collected++;
  CUDA_TRY(cudaEventSynchronize(f.ev));
  int rc = TG_OK;
  if (f.status) {
    rc = fail(f.status, f.msg);  // an earlier frame failed; this one ran as a no-op
  } else if (f.replay) {
    rc = frame_run_sync(s, f);
  } else if (f.ctl->err != kNoError) {
    // the frame (or a later substep) latched an error: drain what follows it
    // (no-ops under the latch) and clean up as tg_step does
    CUDA_TRY(cudaStreamSynchronize(s.stream));
    CUDA_TRY(cudaStreamSynchronize(s.copy_stream));
    rc = sync_and_check(s, f.end_substep);
    FrameSlot& next = s.frames[(ticket + 1) % 2];
    if (rc == kResume) {  // node arrays grown: finish this frame, replay the next
      rc = step(s, f.v, s.resume_substeps);
      std::string msg;
      if (!rc) rc = capture_enqueue_to(s, f.r, f.depth, f.rgb, msg);
      if (!rc && cudaStreamSynchronize(s.stream) != cudaSuccess) rc = fail(TG_ERR_CUDA, "capture failed");
      if (rc && !msg.empty()) rc = fail(rc, msg);
      if (next.live) next.replay = true;
    } else if (rc && next.live) {
      next.status = rc;
      next.msg = std::string("an earlier pipelined frame failed: ") + g_last_error;
    }
  }
  // (on success the host's substep count was already advanced at submit: a
  // later frame may be in flight, so it is not reset from this snapshot)
  if (rc) return rc;
  if (depth) *depth = f.read_back ? f.depth : nullptr;
  if (rgb) *rgb = f.read_back ? f.rgb : nullptr;
  return TG_OK;
}

}  // namespace tacchi_b200

// ===========================================================================
// C-ABI
// ===========================================================================

using tacchi_b200::DeviceSim;
using tacchi_b200::fail;
using tacchi_b200::g_last_error;

struct tg_sim : DeviceSim {};

static DeviceSim* H(tg_handle h) { return static_cast<DeviceSim*>(reinterpret_cast<void*>(h)); }

// Pipelined frames own the handle until they are waited for.
static int in_flight(tg_handle h, const char* who) {
  const DeviceSim& s = *H(h);
  if (s.frames_submitted != s.frames_collected)
    return fail(TG_ERR_INVALID_ARGUMENT,
                std::string(who) + ": pipelined frames are in flight; tg_step_capture_wait first");
  return TG_OK;
}

extern "C" {

const char* tg_last_error(void) { return g_last_error.c_str(); }
const char* tg_version(void) { return "tacchi_b200 0.1 (sm_100a)"; }

int tg_create(int device, const tg_params* params, const tg_particles* particles,
              const tg_surface* surface, tg_handle* out) {
  DeviceSim* s = nullptr;
  const int rc = tacchi_b200::create(device, params, particles, surface, &s);
  if (rc) return rc;
  *out = reinterpret_cast<tg_handle>(s);
  return TG_OK;
}

void tg_destroy(tg_handle h) { delete H(h); }

int tg_step(tg_handle h, const double v[3], int n) {
  if (!h || !v) return fail(TG_ERR_INVALID_ARGUMENT, "tg_step: null argument");
  if (const int rc = in_flight(h, "tg_step")) return rc;
  if (H(h)->keep_grid) return tacchi_b200::step(*H(h), v, n);
  // The per-call indenter move counters are 8-bit: long calls run in chunks
  // (identical results; one extra host sync per 200 substeps).
  while (n > 0) {
    const int chunk = n > 200 ? 200 : n;
    const int rc = tacchi_b200::step(*H(h), v, chunk);
    if (rc) return rc;
    n -= chunk;
  }
  return TG_OK;
}

int tg_phase(tg_handle h, int phase, const double v[3]) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_phase: null handle");
  if (const int rc = in_flight(h, "tg_phase")) return rc;
  const double zero[3] = {0, 0, 0};
  return tacchi_b200::phase(*H(h), phase, v ? v : zero);
}

int64_t tg_num_particles(tg_handle h) { return h ? H(h)->n : 0; }
int64_t tg_num_elastomer(tg_handle h) { return h ? H(h)->n_el : 0; }

int tg_download(tg_handle h, double* x, double* v, double* C, double* F) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_download: null handle");
  if (const int rc = in_flight(h, "tg_download")) return rc;
  return tacchi_b200::download(*H(h), x, v, C, F);
}

int tg_upload(tg_handle h, const double* x, const double* v, const double* C, const double* F) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_upload: null handle");
  if (const int rc = in_flight(h, "tg_upload")) return rc;
  return tacchi_b200::upload(*H(h), x, v, C, F, false);
}

int tg_diag(tg_handle h, double* min_det_f, double* max_speed, int64_t* step_count,
            double indenter_velocity[3]) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_diag: null handle");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  if (cudaMemcpyAsync(s.h_ctl, s.ctl, sizeof(tacchi_b200::Ctl), cudaMemcpyDeviceToHost, s.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(s.stream) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_diag: readback failed");
  if (min_det_f) *min_det_f = s.h_ctl->diag_min_det_f;
  if (max_speed) *max_speed = s.h_ctl->diag_max_speed;
  if (step_count) *step_count = s.h_ctl->step_count;
  if (indenter_velocity)
    for (int a = 0; a < 3; ++a) indenter_velocity[a] = s.h_ctl->vind[a];
  return TG_OK;
}

int tg_grid_window(tg_handle h, int lo[3], int hi[3]) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_grid_window: null handle");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  cudaMemcpyAsync(s.h_ctl, s.ctl, sizeof(tacchi_b200::Ctl), cudaMemcpyDeviceToHost, s.stream);
  if (cudaStreamSynchronize(s.stream) != cudaSuccess) return fail(TG_ERR_CUDA, "readback failed");
  for (int a = 0; a < 3; ++a) {
    lo[a] = s.h_ctl->ref_lo[a];
    hi[a] = s.h_ctl->ref_hi[a];
  }
  return TG_OK;
}

int tg_download_grid(tg_handle h, const int lo[3], const int hi[3], double* mass, double* mom,
                     double* vel) {
  if (!h || !lo || !hi) return fail(TG_ERR_INVALID_ARGUMENT, "tg_download_grid: null argument");
  DeviceSim& s = *H(h);
  for (int a = 0; a < 3; ++a)
    if (lo[a] < 0 || hi[a] > s.geo.res[a] || hi[a] <= lo[a])
      return fail(TG_ERR_INVALID_ARGUMENT, "tg_download_grid: box outside the grid");
  if (!s.grid_ref)
    return fail(TG_ERR_INVALID_ARGUMENT,
                "tg_download_grid: the last tg_step ran the fused substep plan, whose grid holds "
                "the next substep's look-ahead scatter; call tg_set_keep_grid(h, 1) before "
                "stepping to keep the reference's post-step grid");
  cudaSetDevice(s.device);
  const size_t cnt = static_cast<size_t>(hi[0] - lo[0]) * (hi[1] - lo[1]) * (hi[2] - lo[2]);
  double* d = nullptr;
  if (cudaMalloc(&d, cnt * 7 * sizeof(double)) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_download_grid: allocation failed");
  tacchi_b200::launch_gather_box(s, lo, hi, d, d + cnt, d + 4 * cnt);
  std::vector<double> buf(cnt * 7);
  cudaMemcpyAsync(buf.data(), d, cnt * 7 * sizeof(double), cudaMemcpyDeviceToHost, s.stream);
  const cudaError_t e = cudaStreamSynchronize(s.stream);
  cudaFree(d);
  if (e != cudaSuccess) return fail(TG_ERR_CUDA, cudaGetErrorString(e));
  if (mass) std::memcpy(mass, buf.data(), cnt * sizeof(double));
  if (mom) std::memcpy(mom, buf.data() + cnt, 3 * cnt * sizeof(double));
  if (vel) std::memcpy(vel, buf.data() + 4 * cnt, 3 * cnt * sizeof(double));
  return TG_OK;
}

int tg_capture(tg_handle h, const tg_render* r, double* depth_out, uint8_t* rgb_out) {
  if (!h || !r) return fail(TG_ERR_INVALID_ARGUMENT, "tg_capture: null argument");
  if (const int rc = in_flight(h, "tg_capture")) return rc;
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  std::string msg;
  const int rc = tacchi_b200::capture(s, *r, depth_out, rgb_out, msg);
  return rc ? fail(rc, msg) : TG_OK;
}

int tg_capture_buffers(tg_handle h, const tg_render* r, double** depth, uint8_t** rgb) {
  if (!h || !r) return fail(TG_ERR_INVALID_ARGUMENT, "tg_capture_buffers: null argument");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  std::string msg;
  const int rc = tacchi_b200::capture_buffers(s, *r, depth, rgb, msg);
  return rc ? fail(rc, msg) : TG_OK;
}

// One control step of the co-simulation loop (session.cpp:86 + 42): the
// substeps and the capture are submitted together, with one host sync.
int tg_step_capture(tg_handle h, const double v[3], int n, const tg_render* r, double* depth_out,
                    uint8_t* rgb_out) {
  if (!h || !v || !r) return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture: null argument");
  if (const int rc = in_flight(h, "tg_step_capture")) return rc;
  DeviceSim& s = *H(h);
  if (s.keep_grid) {  // the step ends on the phase path; capture afterwards
    const int rc = tacchi_b200::step(s, v, n);
    if (rc) return rc;
    std::string msg;
    const int crc = tacchi_b200::capture(s, *r, depth_out, rgb_out, msg);
    return crc ? fail(crc, msg) : TG_OK;
  }
  while (n > 200) {  // long calls: chunks as tg_step
    const int rc = tacchi_b200::step(s, v, 200);
    if (rc) return rc;
    n -= 200;
  }
  int rc = tacchi_b200::step_submit(s, v, n);
  if (rc) return rc;
  std::string msg;
  const int crc = tacchi_b200::capture_enqueue(s, *r, depth_out != nullptr, rgb_out != nullptr, msg);
  rc = tacchi_b200::step_finish(s, n);  // syncs the stream; the step's error wins
  if (rc == tacchi_b200::kResume) {  // node arrays grown mid-call: finish, capture again
    rc = tacchi_b200::step(s, v, s.resume_substeps);
    if (rc) return rc;
    const int c2 = tacchi_b200::capture(s, *r, depth_out, rgb_out, msg);
    return c2 ? fail(c2, msg) : TG_OK;
  }
  if (rc) return rc;
  if (crc) return fail(crc, msg);
  tacchi_b200::capture_collect(s, depth_out, rgb_out);
  return TG_OK;
}

int tg_extract_depth(tg_handle h, int w, int hgt, double r, double* out, int* out_w, int* out_h) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_extract_depth: null handle");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  if (w <= 0 || hgt <= 0) {
    if (s.surf_nx < 2 || s.surf_ny < 2)
      return fail(TG_ERR_NO_SURFACE, "extract_surface_depth: state has no surface lattice");
    tacchi_b200::full_surface_size(s, r, &w, &hgt);
  }
  if (out_w) *out_w = w;
  if (out_h) *out_h = hgt;
  if (!out) return TG_OK;
  std::string msg;
  const int rc = tacchi_b200::extract_depth(s, w, hgt, r, out, msg);
  return rc ? fail(rc, msg) : TG_OK;
}

int tg_crop_align(int device, const double* src, int sw, int sh, double off_x, double off_y,
                  double scale, int ow, int oh, double* out) {
  int rc = tacchi_b200::check_device_public(device);
  if (rc) return rc;
  std::string msg;
  rc = tacchi_b200::render_standalone(0, src, sw, sh, 0.0, off_x, off_y, scale, ow, oh, nullptr,
                                      out, nullptr, msg);
  return rc ? fail(rc, msg) : TG_OK;
}

int tg_surface_normals(int device, const double* depth, int w, int hgt, double r, double* out) {
  int rc = tacchi_b200::check_device_public(device);
  if (rc) return rc;
  std::string msg;
  rc = tacchi_b200::render_standalone(1, depth, w, hgt, r, 0, 0, 1, w, hgt, nullptr, out, nullptr,
                                      msg);
  return rc ? fail(rc, msg) : TG_OK;
}

int tg_phong_render(int device, const double* depth, int w, int hgt, double r,
                    const tg_render* render, uint8_t* out) {
  if (!render) return fail(TG_ERR_INVALID_ARGUMENT, "tg_phong_render: null render params");
  int rc = tacchi_b200::check_device_public(device);
  if (rc) return rc;
  std::string msg;
  rc = tacchi_b200::render_standalone(2, depth, w, hgt, r, 0, 0, 1, w, hgt, render, nullptr, out,
                                      msg);
  return rc ? fail(rc, msg) : TG_OK;
}

// Submits every handle's work before waiting on any of them; a handle whose
// submission fails is still accounted for, the others are finished normally.
// Returns the first failing handle's code and message; per-handle codes go to
// `status` when given.
static int many(tg_handle* hs, int n_handles, const double* velocities, int n_substeps,
                const tg_render* renders, int n_renders, double** depth_outs,
                uint8_t** rgb_outs, int* status, const char* who) {
  if (!hs || !velocities || n_handles < 0)
    return fail(TG_ERR_INVALID_ARGUMENT, std::string(who) + ": null argument");
  if (n_substeps < 0 || n_substeps > 200)
    return fail(TG_ERR_INVALID_ARGUMENT, std::string(who) + ": n_substeps outside [0, 200]");
  for (int i = 0; i < n_handles; ++i) {
    if (!hs[i]) return fail(TG_ERR_INVALID_ARGUMENT, std::string(who) + ": null handle");
    if (const int rc = in_flight(hs[i], who)) return rc;
  }
  std::vector<int> rc(n_handles, TG_OK), crc(n_handles, TG_OK);
  std::vector<std::string> msg(n_handles);
  std::vector<char> submitted(n_handles, 0), stepped(n_handles, 0);
  for (int i = 0; i < n_handles; ++i) {
    DeviceSim& s = *H(hs[i]);
    // keep_grid handles step to completion here (their last substep runs
    // the phase path), the others are only submitted
    stepped[i] = s.keep_grid;
    rc[i] = s.keep_grid ? tacchi_b200::step(s, velocities + 3 * i, n_substeps)
                        : tacchi_b200::step_submit(s, velocities + 3 * i, n_substeps);
    if (rc[i]) {
      msg[i] = g_last_error;
      continue;
    }
    submitted[i] = 1;
    if (renders) {
      const tg_render& r = renders[n_renders == 1 ? 0 : i];
      crc[i] = tacchi_b200::capture_enqueue(s, r, depth_outs && depth_outs[i],
                                            rgb_outs && rgb_outs[i], msg[i]);
    }
  }
  int first = -1;
  for (int i = 0; i < n_handles; ++i) {
    if (submitted[i]) {
      DeviceSim& s = *H(hs[i]);
      if (stepped[i])
        rc[i] = cudaStreamSynchronize(s.stream) == cudaSuccess
                    ? TG_OK
                    : fail(TG_ERR_CUDA, "capture failed on the device");
      else
        rc[i] = tacchi_b200::step_finish(s, n_substeps);  // the step's error wins
      if (rc[i] == tacchi_b200::kResume) {  // node arrays grown mid-call
        rc[i] = tacchi_b200::step(s, velocities + 3 * i, s.resume_substeps);
        if (!rc[i] && renders && !crc[i]) {
          const tg_render& r = renders[n_renders == 1 ? 0 : i];
          crc[i] = tacchi_b200::capture(s, r, depth_outs ? depth_outs[i] : nullptr,
                                        rgb_outs ? rgb_outs[i] : nullptr, msg[i]);
          if (!crc[i]) stepped[i] = 2;  // outputs already delivered
        }
      }
      if (rc[i]) {
        msg[i] = g_last_error;
      } else if (crc[i]) {
        rc[i] = crc[i];
      } else if (renders && stepped[i] != 2) {
        tacchi_b200::capture_collect(s, depth_outs ? depth_outs[i] : nullptr,
                                     rgb_outs ? rgb_outs[i] : nullptr);
      }
    }
    if (status) status[i] = rc[i];
    if (rc[i] && first < 0) first = i;
  }
  return first < 0 ? TG_OK : fail(rc[first], msg[first]);
}

int tg_step_many(tg_handle* hs, int n_handles, const double* velocities, int n_substeps) {
  return many(hs, n_handles, velocities, n_substeps, nullptr, 0, nullptr, nullptr, nullptr,
              "tg_step_many");
}

int tg_step_capture_many(tg_handle* hs, int n_handles, const double* velocities, int n_substeps,
                         const tg_render* renders, int n_renders, double** depth_outs,
                         uint8_t** rgb_outs, int* status) {
  if (!renders || (n_renders != 1 && n_renders != n_handles))
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_many: renders must hold 1 or n entries");
  return many(hs, n_handles, velocities, n_substeps, renders, n_renders, depth_outs, rgb_outs,
              status, "tg_step_capture_many");
}

int tg_sync(tg_handle h) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_sync: null handle");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  const cudaError_t e = cudaStreamSynchronize(s.stream);
  return e == cudaSuccess ? TG_OK : fail(TG_ERR_CUDA, cudaGetErrorString(e));
}

int tg_time_phases(tg_handle h, const double v[3], int reps, double* out_ms) {
  if (!h || !v || !out_ms || reps <= 0)
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_time_phases: bad argument");
  return tacchi_b200::time_phases(*H(h), v, reps, out_ms);
}

void* tg_stream(tg_handle h) { return h ? static_cast<void*>(H(h)->stream) : nullptr; }
int64_t tg_kernel_launches(tg_handle h) { return h ? H(h)->kernel_launches : 0; }
int tg_stats(tg_handle h, int64_t out[7]) {
  if (!h || !out) return fail(TG_ERR_INVALID_ARGUMENT, "tg_stats: null argument");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  if (cudaMemcpyAsync(s.h_ctl, s.ctl, sizeof(tacchi_b200::Ctl), cudaMemcpyDeviceToHost, s.stream) !=
          cudaSuccess ||
      cudaStreamSynchronize(s.stream) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_stats: readback failed");
  out[0] = s.kernel_launches;
  out[1] = s.regrows;
  out[2] = static_cast<int64_t>(s.grid_slab_bytes);
  out[3] = s.h_ctl->walk_fixups;
  out[4] = static_cast<int64_t>(s.n_nodes);
  out[5] = static_cast<int64_t>(s.graphs.size());
  out[6] = static_cast<int64_t>(s.h_ctl->ind_walked);
  return TG_OK;
}

int tg_step_capture_submit(tg_handle h, const double v[3], int n, const tg_render* r,
                           int read_back, int64_t* ticket) {
  if (!h || !v || !r || !ticket)
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_submit: null argument");
  return tacchi_b200::frame_submit(*H(h), v, n, *r, read_back != 0, ticket);
}

int tg_step_capture_wait(tg_handle h, int64_t ticket, double** depth, uint8_t** rgb) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_step_capture_wait: null handle");
  return tacchi_b200::frame_wait(*H(h), ticket, depth, rgb);
}

int tg_set_deterministic(tg_handle h, int enabled) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_set_deterministic: null handle");
  DeviceSim& s = *H(h);
  const int want = enabled != 0;
  if (s.geo.det == want) return TG_OK;
  cudaSetDevice(s.device);
  // the accumulators change format: drop any pending scatter and the graphs
  // (Geometry is captured by value)
  tacchi_b200::flush_indenter_public(s);
  if (cudaStreamSynchronize(s.stream) != cudaSuccess ||
      cudaMemsetAsync(s.grid_slab, 0, s.grid_slab_bytes, s.stream) != cudaSuccess ||
      cudaStreamSynchronize(s.stream) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_set_deterministic: device error");
  tacchi_b200::drop_graphs_public(s);
  s.geo.det = want;
  s.grid_ready = false;
  s.grid_dirty = false;
  s.grid_ref = false;
  s.window_valid = false;
  return TG_OK;
}

int tg_set_keep_grid(tg_handle h, int enabled) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_set_keep_grid: null handle");
  H(h)->keep_grid = enabled != 0;
  return TG_OK;
}

int tg_download_constants(tg_handle h, double* mass, double* volume0, uint8_t* tag) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_download_constants: null handle");
  DeviceSim& s = *H(h);
  cudaSetDevice(s.device);
  std::vector<uint8_t> el_tag(static_cast<size_t>(std::max<int64_t>(s.n_el, 1)));
  if (tag && s.n_el > 0) {
    const cudaError_t e = tacchi_b200::copy_sync(s, el_tag.data(), s.tag, s.n_el, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return fail(TG_ERR_CUDA, cudaGetErrorString(e));
  }
  for (int64_t q = 0; q < s.n; ++q) {
    const int64_t r = s.perm[q];  // reference index
    const bool el = q < s.n_el;
    if (mass) mass[r] = el ? s.m_el : s.m_ind;
    if (volume0) volume0[r] = el ? s.vol_el : s.vol_ind;
    if (tag) tag[r] = el ? el_tag[q] : tacchi_b200::kIndenter;
  }
  return TG_OK;
}

int tg_set_graphs(tg_handle h, int enabled) {
  if (!h) return fail(TG_ERR_INVALID_ARGUMENT, "tg_set_graphs: null handle");
  H(h)->use_graphs = enabled != 0;
  return TG_OK;
}

}  // extern "C"
