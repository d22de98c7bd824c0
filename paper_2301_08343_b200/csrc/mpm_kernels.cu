// MLS-MPM substep kernels for sm_100a.
//
// Step path (mpm::step, engine.cpp:288-297), per substep s (CUDA graph, each
// kernel launched with programmatic stream serialization):
//   k_grid_update_boxes  grid_update (engine.cpp:180-205) over the elastomer
//                        and indenter node boxes; reads Grid::mass/momentum
//                        (A, M_I), writes Grid::velocity (V) and re-zeroes A /
//                        M_I, so the next scatter needs no zero_grid clear.
//   k_g2p2g_gel          grid_to_particle + apply_boundary + advect for the
//                        elastomer (engine.cpp:207-279) from a TMA-staged
//                        velocity tile and, fused in the same CTA,
//                        particle_to_grid of substep s+1 (engine.cpp:107-178:
//                        det F, Newton polar, corotated stress, APIC) through
//                        a shared-memory node tile: 27 barrier-separated
//                        conflict-free accumulation phases, then one TMA bulk
//                        reduction per tile row (the particles' storage order
//                        within each CTA's slots is dealt for the banks,
//                        permute_gel_lanes).
//   k_ind_cols           (on the handle's walk stream, forked after the
//                        previous finalize and joined before this one; with
//                        TACCHI_WALKS=fused, extra blocks of k_g2p2g_gel) the
//                        rigid indenter's apply_boundary + advect + s+1
//                        scatter (ind_cols_block: warp per z-sorted column,
//                        run-length accumulation of B-spline weight sums, one
//                        RED.F64 per touched node into M_I buffer (s+1) & 1;
//                        the indenter's momentum is M_I * v, v uniform).
//   k_finalize           advect's in_range check / step_count / max_speed and
//                        the next zero_grid window (engine.cpp:53-68, 279-285).
// grid_update triggers the elastomer kernel's launch right after its own
// griddepcontrol.wait, and the elastomer kernel reads its particle state and
// staging box (written by its previous launch, complete by then) before its
// own wait.
// The first substep of a call without a pending look-ahead starts with a
// standalone scatter (k_p2g_gel_tile, k_ind_cols<false>); every substep
// scatters the next one, so consecutive calls chain; k_ind_catchup applies
// the advects of indenter particles the column walks did not visit once the
// chain of same-velocity calls ends. Errors
// are latched in Ctl::err_code with the substep they belong to; every kernel
// of a later or equal substep exits early, reproducing the reference's
// "state at the throwing phase".
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <vector>
#include <string>
#include <mutex>

#include "engine.cuh"
#include "tacchi_cuda.h"

namespace tacchi_b200 {

namespace {

// Programmatic dependent launch: the step-path kernels are launched with
// programmatic stream serialization so each is dispatched while its
// predecessor drains; this waits until the predecessor's writes are visible
// (a no-op for ordinary launches).
#ifdef TACCHI_TRACE
// Per-CTA stage timestamps of the elastomer kernel (diagnostic builds only,
// tools/trace_gel.py): [0] globaltimer at entry, [1] smid, [2..13] clock64 at
// the stage marks, [14] globaltimer at exit, [15] block kind.
__device__ unsigned long long g_trace[16384 * 16];
__device__ __forceinline__ unsigned long long trace_gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define TRACE_MARK(i)                                                                   \
  do {                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x < 16384) g_trace[blockIdx.x * 16 + 2 + (i)] = clock64(); \
  } while (0)
#define TRACE_BEGIN(kind)                                                               \
  do {                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x < 16384) {                                      \
      unsigned sm;                                                                     \
      asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));                                  \
      g_trace[blockIdx.x * 16 + 0] = trace_gtime();                                    \
      g_trace[blockIdx.x * 16 + 1] = sm;                                               \
      g_trace[blockIdx.x * 16 + 15] = (kind);                                          \
      g_trace[blockIdx.x * 16 + 2] = clock64();                                        \
    }                                                                                  \
  } while (0)
#define TRACE_END()                                                                     \
  do {                                                                                 \
    if (threadIdx.x == 0 && blockIdx.x < 16384) g_trace[blockIdx.x * 16 + 14] = trace_gtime(); \
  } while (0)
#else
#define TRACE_MARK(i)
#define TRACE_BEGIN(kind)
#define TRACE_END()
#endif

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ void raise(Ctl* ctl, int code, int substep) {
  atomicMin(&ctl->err, err_key(substep, code));
}

// True when an error latched for substep <= s (the work of substep s must not run).
__device__ __forceinline__ bool stale(const Ctl* ctl, int s) {
  return (*reinterpret_cast<volatile const unsigned long long*>(&ctl->err) >> 8) <=
         static_cast<unsigned long long>(s);
}

// Block-uniform version (one read, broadcast through shared memory) for
// kernels that use __syncthreads after the check.
__device__ __forceinline__ bool stale_block(const Ctl* ctl, int s) {
  __shared__ int flag;
  if (threadIdx.x == 0) flag = stale(ctl, s) ? 1 : 0;
  __syncthreads();
  const bool r = flag != 0;
  __syncthreads();
  return r;
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

// Block reduction of advect's quantities (engine.cpp:273-282): max |v|^2 and
// the bbox of x. Warp shuffles, one shared-memory pass, then 7 atomics per
// block. Every thread of the block must call it.
__device__ void reduce_motion(unsigned long long* max_v2, unsigned long long* lo_keys,
                              unsigned long long* hi_keys, bool active, double v2, double x0,
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
  __syncthreads();
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
      if (max_v2) atomicMax(max_v2, static_cast<unsigned long long>(__double_as_longlong(r[0])));
      atomicMin(&lo_keys[0], order_key(r[1]));
      atomicMin(&lo_keys[1], order_key(r[2]));
      atomicMin(&lo_keys[2], order_key(r[3]));
      atomicMax(&hi_keys[0], order_key(r[4]));
      atomicMax(&hi_keys[1], order_key(r[5]));
      atomicMax(&hi_keys[2], order_key(r[6]));
    }
  }
}

// 16-byte store with an L2 evict_last policy (grid data reused by the next
// kernel; the particle streams around it are evict-first).
__device__ __forceinline__ void st_keep(double2* p, double a, double b) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(a), "d"(b),
               "l"(pol)
               : "memory");
}

__device__ __forceinline__ void st_keep1(double* p, double a) {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(a), "l"(pol) : "memory");
}

__device__ __forceinline__ size_t node_index(const Geometry& g, int i, int j, int k) {
  return (static_cast<size_t>(i - g.ga_lo[0]) * g.ga_dim[1] + (j - g.ga_lo[1])) * g.ga_dim[2] +
         (k - g.ga_lo[2]);
}

// The M_I buffer of substep s (double-buffered by parity, Geometry::mi_stride).
__device__ __forceinline__ double* mi_at(const Geometry& g, double* mi, int s) {
  return mi + static_cast<size_t>(s & 1) * g.mi_stride;
}

// The node box [lo, hi) lies inside the node arrays' allocation box.
__device__ __forceinline__ bool box_in_alloc(const Geometry& g, int l0, int l1, int l2, int h0,
                                             int h1, int h2) {
  return l0 >= g.ga_lo[0] && l1 >= g.ga_lo[1] && l2 >= g.ga_lo[2] &&
         h0 <= g.ga_lo[0] + g.ga_dim[0] && h1 <= g.ga_lo[1] + g.ga_dim[1] &&
         h2 <= g.ga_lo[2] + g.ga_dim[2];
}
// A particle's 27 stencil nodes [base, base + 3) are allocated.
__device__ __forceinline__ bool stencil_in_alloc(const Geometry& g, const int* b) {
  return box_in_alloc(g, b[0], b[1], b[2], b[0] + 3, b[1] + 3, b[2] + 3);
}

__device__ __forceinline__ void red_add(double* p, double v) { atomicAdd(p, v); }

// Deterministic mode: v as 64-bit fixed point (v * scale rounded to nearest);
// |v * scale| must stay below 2^62 (the sums of a node then cannot wrap).
__device__ __forceinline__ long long to_fixed(double v, double scale, Ctl* ctl) {
  const double t = v * scale;
  if (!(fabs(t) < 4.611686018427388e18)) {
    if (ctl) atomicMin(&ctl->err, err_key(ctl->substep, kErrFixedRange));
    return 0;
  }
  return __double2ll_rn(t);
}
// llrint(v * scale) without F2I: two round-to-integer additions of
// 1.5 * 2^52 (exact for |v * scale| < 2^62; `bad` is set outside that range),
// returned as the int64's bit pattern in a double register. (A one-addition
// path for |v * scale| < 2^51 behind a per-value branch measured slower:
// 60.6 vs 59.5 us on the deterministic config-2a elastomer kernel.)
__device__ __forceinline__ double fixed_bits(double v, double scale, bool& bad) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  constexpr long long kMagicBits = 0x4338000000000000LL;
  const double y = v * scale;  // exact (power-of-two scale)
  bad |= !(fabs(y) < 4.611686018427388e18);
  const double h = __dadd_rn(__fma_rn(y, 0x1p-32, kMagic), -kMagic);  // round(y / 2^32)
  const double r = __fma_rn(-h, 0x1p32, y);                           // y - h 2^32, exact
  const long long hi = __double_as_longlong(__dadd_rn(h, kMagic)) - kMagicBits;
  const long long lo = __double_as_longlong(__dadd_rn(r, kMagic)) - kMagicBits;  // round(r)
  return __longlong_as_double((hi << 32) + lo);
}

// fixed_bits of a node's four sums: where every |v * scale| < 2^51 (node
// sums of a few particle masses, ~2^48, and every momentum; tested on the
// exponent bits, no fp64 compare) one round-to-integer addition each gives
// llrint (round half to even, as the two-addition path), else fixed_bits.
__device__ __forceinline__ void fixed_bits4(double2& lo, double2& hi, double scale, bool& bad) {
  constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
  constexpr long long kMagicBits = 0x4338000000000000LL;
  constexpr unsigned kExp51 = (1023u + 51u) << 20;  // |y| < 2^51 <=> biased exponent < 1074
  const double y[4] = {lo.x * scale, lo.y * scale, hi.x * scale, hi.y * scale};
  bool small = true;
#pragma unroll
  for (int i = 0; i < 4; ++i)
    small &= (static_cast<unsigned>(__double2hiint(y[i])) & 0x7ff00000u) < kExp51;
  double r[4];
  if (small) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      r[i] = __longlong_as_double(__double_as_longlong(__dadd_rn(y[i], kMagic)) - kMagicBits);
  } else {
#pragma unroll
    for (int i = 0; i < 4; ++i) r[i] = fixed_bits(y[i], 1.0, bad);
  }
  lo = make_double2(r[0], r[1]);
  hi = make_double2(r[2], r[3]);
}

__device__ __forceinline__ double from_fixed(double bits, double inv) {
  return static_cast<double>(__double_as_longlong(bits)) * inv;
}
// One scalar added to a node accumulator: RED.F64, or in deterministic mode
// the exact integer RED.64 of its fixed-point value.
__device__ __forceinline__ void acc_add(double* p, double v, bool det, double scale, Ctl* ctl) {
  if (det)
    atomicAdd(reinterpret_cast<unsigned long long*>(p),
              static_cast<unsigned long long>(to_fixed(v, scale, ctl)));
  else
    atomicAdd(p, v);
}
// Accumulation mode of a code path: kDet < 0 reads Geometry::det at run
// time; 0 / 1 fix it at compile time (the elastomer kernel is instantiated
// per mode so the fast path carries no fixed-point code).
template <int kDet>
__device__ __forceinline__ bool det_on(const Geometry& g) {
  return kDet < 0 ? g.det != 0 : kDet != 0;
}

// M_I (indenter weight sums).
template <int kDet = -1>
__device__ __forceinline__ void mi_add(const Geometry& g, double* p, double v, Ctl* ctl) {
  acc_add(p, v, det_on<kDet>(g), g.fxi_s, ctl);
}

__device__ __forceinline__ bool stencil_in_grid(const Geometry& g, const Stencil& st) {
  return st.base[0] >= 0 && st.base[1] >= 0 && st.base[2] >= 0 && st.base[0] + 2 < g.res[0] &&
         st.base[1] + 2 < g.res[1] && st.base[2] + 2 < g.res[2];
}

// advect: x += dt * v with the reference's rounding (no FMA, engine.cpp:276).
__device__ __forceinline__ double advance(double x, double dt, double v) {
  return add_rn(x, mul_rn(dt, v));
}

}  // namespace

// ---------------------------------------------------------------------------
// Elastomer particle -> CTA mapping. With lattice metadata, a CTA owns a
// (ti x tj x nz) block of lattice columns (particle (i,j,k) at
// (i*ny + j)*nz + k, particle_set.hpp:16-17), which keeps its scatter
// footprint compact; otherwise 256 consecutive particles.
// ---------------------------------------------------------------------------
struct GelMap {
  int lat[3];
  int tile[3];
  int tiles[3];
};

// The rigid indenter's look-ahead column walks, run by extra blocks of the
// elastomer kernel (blocks [ind_lo, ind_lo + walk blocks)) instead of a kernel
// of their own.
struct IndArgs {
  const int64_t* col_start;
  uint8_t* moves;
  double* mi;
  int n_cols;
  int gel_ctas;  // 0: no indenter blocks
  int gel_lo;    // first elastomer block (the indenter blocks come first: they are
                 // short, and the elastomer CTAs then end the kernel in full waves)
  int ind_lo;    // first indenter block
};

namespace {

__device__ __forceinline__ int64_t gel_particle(const GelMap& M, int64_t n_el, int cta) {
  if (M.lat[0] > 0) {
    const int t = threadIdx.x;
    const int per_col = M.tile[2];
    const int kk = t % per_col;
    const int jj = (t / per_col) % M.tile[1];
    const int ii = t / (per_col * M.tile[1]);
    if (ii >= M.tile[0]) return -1;
    const int bj = cta % M.tiles[1];
    const int bi = cta / M.tiles[1];
    const int i = bi * M.tile[0] + ii, j = bj * M.tile[1] + jj;
    if (i >= M.lat[0] || j >= M.lat[1] || kk >= M.lat[2]) return -1;
    return (static_cast<int64_t>(i) * M.lat[1] + j) * M.lat[2] + kk;
  }
  const int64_t p = static_cast<int64_t>(cta) * blockDim.x + threadIdx.x;
  return p < n_el ? p : -1;
}

// ---------------------------------------------------------------------------
// Shared-memory node tile for the elastomer scatter.
// ---------------------------------------------------------------------------
#ifndef TACCHI_TILE_CAP
#define TACCHI_TILE_CAP 2816
#endif
#ifndef TACCHI_F_EARLY
#define TACCHI_F_EARLY 7  // F components loaded before the staging wait (DESIGN 4.5)
#endif
#ifndef TACCHI_GEL_THREADS
#define TACCHI_GEL_THREADS 256
#endif
constexpr int kTileCap = TACCHI_TILE_CAP;  // nodes; 2816 -> 32 B x 2816 + 4 B x 2816 = 101 KB
constexpr int kGelThreads = TACCHI_GEL_THREADS;
constexpr int kGelMinBlocks = (2 * 256) / TACCHI_GEL_THREADS;

// Node tile in the grid's split layout (NodeBuf: two 16-byte halves per node
// in two arrays), so that a z-row of the CTA's node box is one contiguous run
// per half in both shared and global memory (node (i,j,k) at
// (i*res1 + j)*res2 + k, k fastest): rows move with bulk-async (TMA) copies /
// reductions, and 16-byte lanes of one half fall in distinct bank slots for
// nodes up to 8 apart.
struct P2GTile {
  double2 nlo[kTileCap];  // {m, px} / {vx, vy}
  double2 nhi[kTileCap];  // {py, pz} / vz rows (as doubles, pitch zp, offset zoff)
  int owner[kTileCap];
  int lo[3], hi[3], dim[3];
  int blo[3], bhi[3];  // block_motion_box's node box reduction
  int cur_s, cur_stale;  // the substep and its stale flag (thread 0, after the wait)
  int ok;
  int pitch;     // node row pitch (>= dim[2], tile_pitch)
  int rd;        // rows per x-slab (dim[1] + kRowPad)
  int zp, zoff;  // staged vz: node (row r, column c) at ((double*)nhi)[r * zp + zoff + c]
  unsigned long long bar;  // mbarrier of the staging copies
};

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}

// Generic-proxy shared-memory writes -> visible to the async (bulk) proxy.
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Row pitches of the tile: 16-byte node slots, pitch = 5 mod 8 nodes, and
// x-slabs of dim[1] + kRowPad rows; with the elastomer's storage order dealt
// by the residue of the node offsets (permute_gel_lanes) these spread a
// quarter-warp's 128-bit accesses over the bank slots best (a bank model of
// config 2a's CTAs: 1.12x the ideal wavefronts vs 1.30x with pitch = 1 mod 8
// and unpadded slabs). The staged vz rows (8-byte elements, 16-byte aligned
// starts) use an even pitch = 6 mod 16.
#ifndef TACCHI_PITCH_RES
#define TACCHI_PITCH_RES 5
#endif
#ifndef TACCHI_ZPITCH_RES
#define TACCHI_ZPITCH_RES 6
#endif
#ifndef TACCHI_ROW_PAD
#define TACCHI_ROW_PAD 2
#endif
__host__ __device__ __forceinline__ int tile_pitch(int d2) { return d2 + ((TACCHI_PITCH_RES - d2) & 7); }
__host__ __device__ __forceinline__ int tile_zpitch(int zcnt) {
  return zcnt + ((TACCHI_ZPITCH_RES - zcnt) & 15);
}
// Rows of one x-slab of the tile (the j extent padded by kRowPad rows).
constexpr int kRowPad = TACCHI_ROW_PAD;

// The CTA's P2G node box as every thread holds it (block_motion_box computes
// it from T.blo / T.bhi in each thread, so the tile zeroing needs no barrier
// to publish it; thread 0 also stores it in T for the flush).
struct TileBox {
  int lo[3], hi[3], dim[3];
  int pitch, rd, ok;
};

__device__ __forceinline__ TileBox tile_box_of(const int* blo, const int* bhi) {
  TileBox b;
  const bool any = blo[0] != INT_MAX;
  for (int a = 0; a < 3; ++a) {
    b.lo[a] = blo[a];
    b.hi[a] = bhi[a];
    b.dim[a] = any ? bhi[a] - blo[a] + 3 : 0;
  }
  b.pitch = tile_pitch(b.dim[2]);
  b.rd = b.dim[1] + kRowPad;
  const int rows = b.dim[0] * b.rd;
  b.ok = any && rows * b.pitch <= kTileCap && rows * tile_zpitch(b.dim[2] + 2) <= 2 * kTileCap;
  return b;
}

// Adds the CTA's node box into the global grid: one bulk-async reduction
// (UBLKRED.ADD.F64, element-wise atomic in L2) per z-row and half, issued by
// the first 2*dim0*dim1 threads. Call after a __syncthreads that follows the
// last tile write (and a fence_proxy_async by every writer).
template <int kDet>
__device__ __forceinline__ void tile_bulk_reduce(const P2GTile& T, const Geometry& g,
                                                 NodeBuf grid) {
  const int rows = T.dim[0] * T.dim[1];
  const int d2 = T.dim[2];
  bool issued = false;
  for (int t = threadIdx.x; t < 2 * rows; t += blockDim.x) {
    const int r = t >> 1, half = t & 1;
    const int i = r / T.dim[1], j = r - i * T.dim[1];
    double2* dst = (half ? grid.hi : grid.lo) + node_index(g, T.lo[0] + i, T.lo[1] + j, T.lo[2]);
    const double2* src = (half ? T.nhi : T.nlo) + (i * T.rd + j) * T.pitch;
    if (det_on<kDet>(g))  // fixed-point node sums: exact integer adds
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.u64 [%0], [%1], %2;" ::"l"(dst),
          "r"(smem_addr(src)), "r"(static_cast<unsigned>(d2 * sizeof(double2)))
          : "memory");
    else
      asm volatile(
          "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f64 [%0], [%1], %2;" ::"l"(dst),
          "r"(smem_addr(src)), "r"(static_cast<unsigned>(d2 * sizeof(double2)))
          : "memory");
    issued = true;
  }
  if (issued) {
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // the tile must stay intact until the bulk engine has read it
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

// Staging of grid rows [lo, lo + dim) of `src` (both halves) into T as
// bulk-async copies completing on T.bar (tile_bulk_wait), in two parts:
// tile_bulk_stage_init (thread 0: pitches, mbarrier, expected bytes) and,
// after a barrier, tile_bulk_stage_copies (every thread, one copy per row and
// half). T.dim / T.lo / T.ok are set.
// vz rows are 8-byte elements: each row is copied from the even node at or
// below its start (16-byte aligned; res2 is even, so every row of the box
// has the same parity zoff) over an even count, into rows of pitch zp.
__device__ __forceinline__ void tile_bulk_stage_init(P2GTile& T) {
  const int rows = T.dim[0] * T.dim[1];
  const int d2 = T.dim[2];
  const unsigned bar = smem_addr(&T.bar);
  const int zoff = T.lo[2] & 1;
  const int zcnt = (zoff + d2 + 1) & ~1;
  T.zp = tile_zpitch(zcnt);
  T.zoff = zoff;
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
               "r"(static_cast<unsigned>(rows * (d2 * sizeof(double2) + zcnt * sizeof(double))))
               : "memory");
}

__device__ __forceinline__ void tile_bulk_stage_copies(P2GTile& T, const Geometry& g, VelBuf src) {
  const int rows = T.dim[0] * T.dim[1];
  const int d2 = T.dim[2];
  const unsigned bar = smem_addr(&T.bar);
  unsigned long long pol;  // V is dead once the CTAs around it have staged it
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  const int zoff = T.zoff, zp = T.zp;
  const int zcnt = (zoff + d2 + 1) & ~1;
  double* zs = reinterpret_cast<double*>(T.nhi);
  for (int t = threadIdx.x; t < 2 * rows; t += blockDim.x) {
    const int r = t >> 1, half = t & 1;
    const int i = r / T.dim[1], j = r - i * T.dim[1];
    const int sr = i * T.rd + j;  // the row in the tile
    const size_t nd = node_index(g, T.lo[0] + i, T.lo[1] + j, T.lo[2]);
    const void* sp = half ? static_cast<const void*>(src.z + (nd - zoff))
                          : static_cast<const void*>(src.xy + nd);
    void* dp = half ? static_cast<void*>(zs + sr * zp) : static_cast<void*>(T.nlo + sr * T.pitch);
    const unsigned bytes = half ? zcnt * sizeof(double) : d2 * sizeof(double2);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], "
        "[%1], %2, [%3], %4;" ::"r"(smem_addr(dp)),
        "l"(sp), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
  }
}

__device__ __forceinline__ void tile_bulk_wait(P2GTile& T) {
  const unsigned bar = smem_addr(&T.bar);
  asm volatile(
      "{\n"
      ".reg .pred done;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 done, [%0], 0;\n"
      "@!done bra WAIT_%=;\n"
      "}\n" ::"r"(bar)
      : "memory");
}

// One particle's P2G payload (engine.cpp:128-145): stencil, m v and the
// APIC + stress affine matrix.
struct P2GPayload {
  Stencil st;
  double mv[3];
  double aff[9];
};

template <int kDet>
__device__ __forceinline__ void scatter_direct(const Geometry& g, NodeBuf grid, double m,
                                               const P2GPayload& q, Ctl* ctl) {
  const bool det = det_on<kDet>(g);
  const double fs = g.fx_s;
  const double dx = g.dx;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double wa = q.st.w[0][a];
    const double dxa = (a - q.st.fx[0]) * dx;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double wab = wa * q.st.w[1][b];
      const double dxb = (b - q.st.fx[1]) * dx;
      const double m0 = q.mv[0] + q.aff[0] * dxa + q.aff[1] * dxb;
      const double m1 = q.mv[1] + q.aff[3] * dxa + q.aff[4] * dxb;
      const double m2 = q.mv[2] + q.aff[6] * dxa + q.aff[7] * dxb;
      const size_t row = node_index(g, q.st.base[0] + a, q.st.base[1] + b, q.st.base[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = wab * q.st.w[2][c];
        const double dxc = (c - q.st.fx[2]) * dx;
        double* lo = reinterpret_cast<double*>(grid.lo + row + c);
        double* hi = reinterpret_cast<double*>(grid.hi + row + c);
        acc_add(lo + 0, w * m, det, fs, ctl);
        acc_add(lo + 1, w * (m0 + q.aff[2] * dxc), det, fs, ctl);
        acc_add(hi + 0, w * (m1 + q.aff[5] * dxc), det, fs, ctl);
        acc_add(hi + 1, w * (m2 + q.aff[8] * dxc), det, fs, ctl);
      }
    }
  }
}

// Walks the flat indices e = first, first + stride, ... of a (d0, d1, d2) box
// (k fastest) keeping (i, j, k) up to date with carries instead of a div/mod
// per step.
struct BoxIter {
  int e, i, j, k;
  int di, dj, dk, stride;
  __device__ __forceinline__ BoxIter(int first, int step, int d1, int d2) {
    e = first;
    stride = step;
    k = first % d2;
    const int r = first / d2;
    j = r % d1;
    i = r / d1;
    dk = step % d2;
    const int rs = step / d2;
    dj = rs % d1;
    di = rs / d1;
  }
  __device__ __forceinline__ void next(int d1, int d2) {
    e += stride;
    k += dk;
    j += dj;
    i += di;
    if (k >= d2) {
      k -= d2;
      ++j;
    }
    if (j >= d1) {
      j -= d1;
      ++i;
    }
  }
};

// The CTA's node box [min base, max base + 3) per axis; T.ok when it fits
// the tile. All threads of the block must call it (3 barriers).
__device__ void tile_box(P2GTile& T, bool active, const int* base) {
  const int tid = threadIdx.x;
  __syncthreads();  // previous users of T.lo / T.hi are done
  if (tid == 0) {
    T.lo[0] = T.lo[1] = T.lo[2] = INT_MAX;
    T.hi[0] = T.hi[1] = T.hi[2] = INT_MIN;
  }
  __syncthreads();
  if (active) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(&T.lo[a], base[a]);
      atomicMax(&T.hi[a], base[a]);
    }
  }
  __syncthreads();
  if (tid == 0) {
    const bool any = T.lo[0] != INT_MAX;
    for (int a = 0; a < 3; ++a) T.dim[a] = any ? T.hi[a] - T.lo[a] + 3 : 0;
    T.pitch = tile_pitch(T.dim[2]);
    T.rd = T.dim[1] + kRowPad;
    const int rows = T.dim[0] * T.rd;
    T.ok = any && rows * T.pitch <= kTileCap && rows * tile_zpitch(T.dim[2] + 2) <= 2 * kTileCap;
  }
  __syncthreads();
}

// The look-ahead kernel's block reductions: advect's max |v|^2 and bbox of x
// (engine.cpp:273-282) into the substep-s slots of the control block, the
// min det F of substep s + 1 (engine.cpp:119,135), and the CTA's P2G node box
// into T (as tile_box). Warps reduce with shuffles; the node box goes into
// T.blo / T.bhi with shared int atomics (set to the empty box at the
// kernel's entry); after the first barrier warp w reduces quantity w over the
// eight warps and issues its one RED into the control block (one per CTA and
// quantity: per-warp REDs on these eight words measured 83 vs 66 us), and
// thread 0 derives the tile box. All threads of the block must call it; the
// first barrier also retires every earlier reader of T (the G2P gathers).
__device__ void block_motion_box(P2GTile& T, Ctl* ctl, int s, bool moved, double v2, double x0,
                                 double x1, double x2, bool go, double J, const int* base,
                                 TileBox& box) {
  static_assert(kGelThreads / 32 == 8, "one warp per reduced quantity");
  __shared__ double redd[8][8];
  double r[8];
  r[0] = moved ? v2 : 0.0;
  r[1] = moved ? x0 : INFINITY;
  r[2] = moved ? x1 : INFINITY;
  r[3] = moved ? x2 : INFINITY;
  r[4] = moved ? x0 : -INFINITY;
  r[5] = moved ? x1 : -INFINITY;
  r[6] = moved ? x2 : -INFINITY;
  r[7] = go ? J : 1.0;
  r[0] = warp_max(r[0]);
#pragma unroll
  for (int a = 1; a < 4; ++a) r[a] = warp_min(r[a]);
#pragma unroll
  for (int a = 4; a < 7; ++a) r[a] = warp_max(r[a]);
  r[7] = warp_min(r[7]);
  int bi[6];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    bi[a] = __reduce_min_sync(0xffffffffu, go ? base[a] : INT_MAX);
    bi[3 + a] = __reduce_max_sync(0xffffffffu, go ? base[a] : INT_MIN);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int a = 0; a < 8; ++a) redd[a][warp] = r[a];
    if (bi[0] != INT_MAX) {
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        atomicMin(&T.blo[a], bi[a]);
        atomicMax(&T.bhi[a], bi[3 + a]);
      }
    }
  }
  __syncthreads();
  {
    // quantity `warp`: 0 max v^2, 1-3 min x, 4-6 max x, 7 min det F
    const int q = warp;
    const double ident = q == 0 ? 0.0 : (q < 4 ? INFINITY : (q < 7 ? -INFINITY : 1.0));
    double v = lane < 8 ? redd[q][lane] : ident;
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      const double w = __shfl_xor_sync(0xffffffffu, v, o);
      v = (q == 0 || (q >= 4 && q < 7)) ? fmax(v, w) : fmin(v, w);
    }
    if (lane == 0) {
      if (q == 0) {
        if (v > 0.0)
          atomicMax(&ctl->max_v2[s & 1], static_cast<unsigned long long>(__double_as_longlong(v)));
      } else if (q < 4) {
        if (v < INFINITY) atomicMin(&ctl->bb_lo[s & 1][q - 1], order_key(v));
      } else if (q < 7) {
        if (v > -INFINITY) atomicMax(&ctl->bb_hi[s & 1][q - 4], order_key(v));
      } else if (v < 1.0) {
        atomicMin(&ctl->min_detf[(s + 1) & 1], order_key(v));
      }
    }
  }
  // every thread derives the box (T.blo / T.bhi are final after the barrier);
  // thread 0 stores it for the flush, which follows later barriers
  box = tile_box_of(T.blo, T.bhi);
  if (threadIdx.x == 0) {
    for (int a = 0; a < 3; ++a) {
      T.lo[a] = box.lo[a];
      T.hi[a] = box.hi[a];
      T.dim[a] = box.dim[a];
    }
    T.pitch = box.pitch;
    T.rd = box.rd;
    T.ok = box.ok;
  }
}

// CTA-cooperative scatter. All threads of the block must call it.
// Phase (a,b,c) adds each particle's contribution to node base + (a,b,c);
// two particles of the CTA collide in a phase only if they share a base cell,
// which an elastomer lattice coarser than the grid (0.2 mm vs 0.129 mm) never
// does; the rare duplicates (detected through the owner table) and CTAs whose
// footprint exceeds the tile fall back to direct REDs.
// s_scatter: the substep whose P2G this is (a scatter that would leave the
// node arrays' allocation latches kErrRegrow for it instead of writing).
template <int kDet>
__device__ void p2g_tile_scatter(P2GTile& T, bool active, const P2GPayload& q, double m,
                                 const Geometry& g, NodeBuf grid, int cta, const TileBox* given,
                                 Ctl* ctl, int s_scatter, bool owners_reset) {
  const int tid = threadIdx.x;
  if (g.scatter_mode == 1 || g.scatter_mode == 3) {  // A/B switches without a tile
    if (tid == 0 && g.cta_box) g.cta_box[8 * cta + 6] = 0;  // next G2P: no staged box
    if (g.scatter_mode == 1 && active) {  // per-particle REDs (3: no scatter)
      if (stencil_in_alloc(g, q.st.base)) scatter_direct<kDet>(g, grid, m, q, ctl);
      else raise(ctl, kErrRegrow, s_scatter);
    }
    return;
  }
  TileBox B;
  if (given) {
    B = *given;
  } else {
    tile_box(T, active, q.st.base);
    for (int a = 0; a < 3; ++a) {
      B.lo[a] = T.lo[a];
      B.hi[a] = T.hi[a];
      B.dim[a] = T.dim[a];
    }
    B.pitch = T.pitch;
    B.rd = T.dim[1] + kRowPad;
    B.ok = T.ok;
  }
  // every node this CTA can touch, [min base, max base + 3), must be
  // allocated (block-uniform: every thread holds the same box)
  if (B.lo[0] != INT_MAX &&
      !box_in_alloc(g, B.lo[0], B.lo[1], B.lo[2], B.hi[0] + 3, B.hi[1] + 3, B.hi[2] + 3)) {
    if (tid == 0) {
      raise(ctl, kErrRegrow, s_scatter);
      if (g.cta_box) g.cta_box[8 * cta + 6] = 0;
    }
    return;
  }
  if (tid == 0 && g.cta_box) {  // the next G2P of these particles stages this box
    int* b = g.cta_box + 8 * cta;
    for (int a = 0; a < 3; ++a) {
      b[a] = B.lo[a];
      b[3 + a] = B.dim[a];
    }
    b[6] = B.ok;
  }
  const int d1 = B.rd, d2 = B.pitch;  // x-slab rows, row pitch
  const int vol = B.dim[0] * d1 * d2;
  const bool use_tile = B.ok != 0;
  // Deterministic mode: a duplicate's contributions reach the grid as
  // separately rounded fixed-point REDs, the owner's inside the tile sum, so
  // the owner of a shared base cell must not depend on timing: the highest
  // thread takes it (atomicMax). With the owner table reset at kernel entry
  // (owners_reset) the claims go in before the zeroing barrier and are read
  // after it; otherwise they need a barrier of their own.
  const bool det = det_on<kDet>(g);
  const bool pre = det && owners_reset;
  int base_idx = 0;
  if (active && use_tile) {
    base_idx = ((q.st.base[0] - B.lo[0]) * d1 + (q.st.base[1] - B.lo[1])) * d2 +
               (q.st.base[2] - B.lo[2]);
    if (pre) atomicMax(&T.owner[base_idx], tid);
  }
  if (use_tile) {
    const double2 z2 = make_double2(0.0, 0.0);
    for (int e = tid; e < vol; e += blockDim.x) {
      T.nlo[e] = z2;
      T.nhi[e] = z2;
      if (!pre) T.owner[e] = -1;
    }
  }
  __syncthreads();
  bool tiled = false;
  TRACE_MARK(5);
  if (active && use_tile) {
    if (pre)
      tiled = T.owner[base_idx] == tid;
    else if (det)
      atomicMax(&T.owner[base_idx], tid);
    else  // fast mode: first come
      tiled = atomicCAS(&T.owner[base_idx], -1, tid) == -1;
  }
  if (det && !pre && use_tile) {  // block-uniform
    __syncthreads();
    if (active) tiled = T.owner[base_idx] == tid;
  }
  if (active && !tiled) scatter_direct<kDet>(g, grid, m, q, ctl);
  if (!use_tile) return;  // block-uniform
  const double dx = g.dx;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double dxa = (a - q.st.fx[0]) * dx;
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      const double dxb = (b - q.st.fx[1]) * dx;
      const double wab = q.st.w[0][a] * q.st.w[1][b];
      const double m0 = q.mv[0] + q.aff[0] * dxa + q.aff[1] * dxb;
      const double m1 = q.mv[1] + q.aff[3] * dxa + q.aff[4] * dxb;
      const double m2 = q.mv[2] + q.aff[6] * dxa + q.aff[7] * dxb;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        // phase (0,0,0) follows the zeroing barrier directly (the owner CAS
        // touches only the owner table)
        if (a | b | c) __syncthreads();
        if (tiled && g.scatter_mode != 2) {
          const double dxc = (c - q.st.fx[2]) * dx;
          const double w = wab * q.st.w[2][c];
          const int e = base_idx + (a * d1 + b) * d2 + c;
          double2 lo2 = T.nlo[e], hi2 = T.nhi[e];
          lo2.x += w * m;
          lo2.y += w * (m0 + q.aff[2] * dxc);
          hi2.x += w * (m1 + q.aff[5] * dxc);
          hi2.y += w * (m2 + q.aff[8] * dxc);
          T.nlo[e] = lo2;
          T.nhi[e] = hi2;
        }
      }
    }
  }
  TRACE_MARK(6);
  if (det_on<kDet>(g)) {
    // deterministic mode: the tile's node sums (a fixed phase order within
    // the CTA) become 64-bit fixed point in place and reach the grid with
    // integer bulk reductions, exact in any order across CTAs (a whole-block
    // conversion pass; per-warp convert-and-issue measured slower, 84 vs
    // 76 us on config 2a)
    __syncthreads();
    const double fs = g.fx_s;
    bool bad = false;
    for (int e = tid; e < vol; e += blockDim.x) {
      const double2 a = T.nlo[e], b = T.nhi[e];
      // untouched nodes (slab / pitch padding, empty corners) are +0: bits 0
      if (g.det_skip0 && (__double_as_longlong(a.x) | __double_as_longlong(a.y) |
                          __double_as_longlong(b.x) | __double_as_longlong(b.y)) == 0)
        continue;
      double2 lo2 = a, hi2 = b;
      if (g.det_fast4) {
        fixed_bits4(lo2, hi2, fs, bad);
      } else {
        lo2 = make_double2(fixed_bits(a.x, fs, bad), fixed_bits(a.y, fs, bad));
        hi2 = make_double2(fixed_bits(b.x, fs, bad), fixed_bits(b.y, fs, bad));
      }
      T.nlo[e] = lo2;
      T.nhi[e] = hi2;
    }
    if (bad) raise(ctl, kErrFixedRange, s_scatter);
  }
  fence_proxy_async();
  __syncthreads();
  tile_bulk_reduce<kDet>(T, g, grid);
  TRACE_MARK(7);
}

// det F check + polar + stress + affine (engine.cpp:130-139). Returns false
// (and latches DegenerateF for substep s) when det F <= 0.
__device__ __forceinline__ bool make_payload(const Geometry& g, Ctl* ctl, int s, double m,
                                             double vol0, const double* F, const double* Cm,
                                             const double* v, double x0, double x1, double x2,
                                             P2GPayload& q, double& J) {
  J = det3(F);
  if (!(J > 0.0)) {
    raise(ctl, kErrDegenerateF, s);
    return false;
  }
  make_stencil(x0, x1, x2, g.origin, g.inv_dx, q.st);
  double R[9], S[9];
  polar_rotation(F, R);
  corotated_stress(F, R, J, g.mu, g.lambda, S);
  const double ks = g.stress_scale * vol0;
#pragma unroll
  for (int i = 0; i < 9; ++i) q.aff[i] = m * Cm[i] + ks * S[i];
  q.mv[0] = m * v[0];
  q.mv[1] = m * v[1];
  q.mv[2] = m * v[2];
  return true;
}

// StepDiagnostics::min_det_f of substep s, seeded with 1.0 (engine.cpp:119,135).
__device__ __forceinline__ void reduce_min_detf(Ctl* ctl, int s, bool active, double J) {
  const double w = warp_min(active ? J : 1.0);
  if ((threadIdx.x & 31) == 0 && w < 1.0) atomicMin(&ctl->min_detf[s & 1], order_key(w));
}

}  // namespace

// ---------------------------------------------------------------------------
// Window / bbox / finalize
// ---------------------------------------------------------------------------

enum : int { kResetMotion = 1, kResetIndBox = 2, kResetDetF = 4 };

__global__ void k_reset(Ctl* ctl, int mask) {
  for (int slot = 0; slot < 2; ++slot) {
    for (int a = 0; a < 3; ++a) {
      if (mask & kResetMotion) {
        ctl->bb_lo[slot][a] = order_key(INFINITY);
        ctl->bb_hi[slot][a] = order_key(-INFINITY);
      }
      if (mask & kResetIndBox) {
        ctl->ind_lo[slot][a] = order_key(INFINITY);
        ctl->ind_hi[slot][a] = order_key(-INFINITY);
      }
    }
    if (mask & kResetMotion) ctl->max_v2[slot] = 0ull;
  }
  if (mask & kResetDetF) ctl->min_detf[0] = ctl->min_detf[1] = order_key(1.0);
}

// particle_bbox (engine.cpp:31-45) over [begin, end): elastomer part into
// bb_*, indenter part into ind_* (then advanced analytically by finalize),
// slot (substep + next) & 1: next = 1 for the positions before this substep's
// P2G (they are "after the advect of substep - 1"), 0 after an advect.
__global__ void k_bbox(const double* __restrict__ x, int64_t n, int64_t begin, int64_t end,
                       Ctl* ctl, int indenter, int next) {
  const int64_t p = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < end;
  const int sl = (ctl->substep + next) & 1;
  reduce_motion(nullptr, indenter ? ctl->ind_lo[sl] : ctl->bb_lo[sl],
                indenter ? ctl->ind_hi[sl] : ctl->bb_hi[sl],
                active, 0.0, active ? x[p] : 0.0, active ? x[n + p] : 0.0,
                active ? x[2 * n + p] : 0.0);
}

// kFinWalkFix: the step path's indenter look-ahead walks (run beside the
// elastomer kernel) used the previous elastomer box widened by one node;
// finalize checks the new box against it and, if the elastomer moved out of
// it, scatters the indenter particles the walks missed (k_finalize's extra
// warps) so M_I is exact wherever the elastomer reads the grid.
enum : int { kFinAdvect = 1, kFinWindow = 2, kFinDiag = 4, kFinIndShift = 8, kFinWalkFix = 16 };

// Node boxes handed from finalize's first warp to the walk fix-up.
struct FinFix {
  int need;               // the new elastomer box is not inside the widened old one
  int old_ok;             // the walks ran (the old box was non-empty)
  int wlo[3], whi[3];     // old elastomer box widened by one node (what the walks used)
  int elo[3], ehi[3];     // new (exact) elastomer box of the substep being scattered
  int s;                  // the substep whose advect this finalize completes
};

// grid.cpp:29-36: in_range divides by dx.
__device__ bool in_range(const Geometry& g, const double* x) {
  for (int a = 0; a < 3; ++a) {
    const double xn = div_rn(sub_rn(x[a], g.origin[a]), g.dx);
    const int b = static_cast<int>(floor(sub_rn(xn, 0.5)));
    if (b < 0 || b + 2 >= g.res[a]) return false;
  }
  return true;
}

// One warp; lanes 0-2 own one axis each (the per-axis work is independent:
// bbox shift, in_range, window, material boxes, clear box), lane 0 the
// scalar diagnostics. Each lane reads only its fields, once, and writes its
// results once, so no read waits on an aliasing store; cross-axis decisions
// (in_range of all axes, the previous window's emptiness) are warp votes.
__device__ __forceinline__ int base_of(const Geometry& g, int a, double x) {
  return static_cast<int>(floor(sub_rn(mul_rn(sub_rn(x, g.origin[a]), g.inv_dx), 0.5)));
}

__device__ void finalize_warp(Ctl* ctl, const Geometry& g, int mode, FinFix& fx) {
  const int lane = threadIdx.x;
  const bool ax = lane < 3;
  const int a = ax ? lane : 0;
  // Every input is loaded in one round trip (both parity slots of the
  // slotted reductions; the substep picks one afterwards): finalize sits on
  // the substep's critical path, between the elastomer kernel and the next
  // grid_update.
  const int s = ctl->substep;
  const unsigned long long errk = *reinterpret_cast<volatile const unsigned long long*>(&ctl->err);
  unsigned long long kbl[2], kbh[2], kil[2], kih[2], ki0l[2], ki0h[2];
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    kbl[q] = ctl->bb_lo[q][a];
    kbh[q] = ctl->bb_hi[q][a];
    kil[q] = ctl->ind_lo[q][a];
    kih[q] = ctl->ind_hi[q][a];
    ki0l[q] = ctl->ind_lo[q][0];
    ki0h[q] = ctl->ind_hi[q][0];
  }
  const double va = ctl->vind[a];
  const double u0 = ctl->vind[0], u1 = ctl->vind[1], u2 = ctl->vind[2];
  const int pl = ctl->prev_lo[a], ph = ctl->prev_hi[a];
  const int olo = ctl->box_lo[0][a], ohi = ctl->box_hi[0][a];
  const unsigned long long kdf[2] = {ctl->min_detf[0], ctl->min_detf[1]};
  const unsigned long long kv2[2] = {ctl->max_v2[0], ctl->max_v2[1]};
  const long long steps = ctl->step_count;
  const int wl_old = ctl->win_lo[a], wh_old = ctl->win_hi[a];
  const long long fixups = ctl->walk_fixups;
  if ((errk >> 8) <= static_cast<unsigned long long>(s)) return;  // stale(ctl, s)
  // after an advect the reductions of substep s are in slot s & 1; a window
  // of the current positions (before P2G(s)) reads slot (s + 1) & 1
  const int cur = (mode & kFinAdvect) ? (s & 1) : ((s + 1) & 1);
  // the indenter box is advanced from the previous slot when shifting
  const int isl = (mode & kFinIndShift) ? (cur ^ 1) : cur;
  // per-axis inputs
  const bool ind_any = order_val(ki0l[isl]) <= order_val(ki0h[isl]);
  double bl = order_val(kbl[cur]), bh = order_val(kbh[cur]);
  double il = order_val(kil[isl]), ih = order_val(kih[isl]);
  const bool shift = (mode & kFinIndShift) && ind_any;
  if (shift) {
    // The indenter moved rigidly with vind: fl(x + fl(dt v)) is monotone in
    // x, so its bbox moves by exactly the same rounded step as its particles.
    const double d = mul_rn(g.dt, va);
    il = add_rn(il, d);
    ih = add_rn(ih, d);
  }
  const double lo = fmin(bl, il), hi = fmax(bh, ih);
  int err = 0;  // warp-uniform
  // (olo, ohi: the elastomer box the look-ahead walks of this substep used,
  // read above before it is replaced below)
  if (mode & kFinAdvect) {
    // engine.cpp:279-285 (grid.cpp:29-36 per axis: xn = (x - o) / dx)
    bool ok = true;
    if (ax) {
      const int b0 = static_cast<int>(floor(sub_rn(div_rn(sub_rn(lo, g.origin[a]), g.dx), 0.5)));
      const int b1 = static_cast<int>(floor(sub_rn(div_rn(sub_rn(hi, g.origin[a]), g.dx), 0.5)));
      ok = b0 >= 0 && b0 + 2 < g.res[a] && b1 >= 0 && b1 + 2 < g.res[a];
    }
    if (__any_sync(0xffffffffu, !ok)) err = 1;
  }
  int wlo = 0, whi = 0;
  if (!err && (mode & kFinWindow)) {
    // engine.cpp:60-85 — window [base(lo), base(hi) + 3); clear prev ∪ new.
    bool ok = true;
    if (ax) {
      const int b0 = base_of(g, a, lo), b1 = base_of(g, a, hi);
      ok = !(b0 < 0 || b1 + 2 >= g.res[a]);
      wlo = b0;
      whi = b1 + 3;
    }
    if (__any_sync(0xffffffffu, !ok)) err = 2;
  }
  const bool prev_empty = __any_sync(0xffffffffu, ax && ph - pl <= 0);
  if (lane == 0) {
    if (mode & kFinDiag) {  // particle_to_grid's min_det_f (engine.cpp:119,177)
      ctl->diag_min_det_f = order_val(kdf[s & 1]);
      ctl->min_detf[s & 1] = order_key(1.0);
    }
    if (mode & kFinAdvect) {
      double v2 = __longlong_as_double(static_cast<long long>(kv2[cur]));
      if (shift) v2 = fmax(v2, u0 * u0 + u1 * u1 + u2 * u2);
      ctl->diag_max_speed = sqrt(v2);
      ctl->step_count = steps + 1;
      ctl->substep = s + 1;
    }
    if (err) raise(ctl, kErrOutOfGrid, err == 1 ? s : ((mode & kFinAdvect) ? s + 1 : s));
  }
  if (ax && shift) {
    ctl->ind_lo[cur][a] = order_key(il);
    ctl->ind_hi[cur][a] = order_key(ih);
  }
  if (err) return;
  if (ax && (mode & kFinWindow)) {
    // The two materials' own node boxes: grid_update only needs their union
    // (the stretch of the combined window between the gel and the indenter
    // holds no mass). An empty set gives an empty box.
    const double l[2] = {bl, il}, h[2] = {bh, ih};
    for (int m = 0; m < 2; ++m) {
      const bool any = l[m] <= h[m];
      ctl->box_lo[m][a] = any ? base_of(g, a, l[m]) : 0;
      ctl->box_hi[m][a] = any ? base_of(g, a, h[m]) + 3 : 0;
    }
    if (mode & kFinWalkFix) {
      const bool any = bl <= bh;
      fx.wlo[a] = olo - 1;
      fx.whi[a] = ohi + 1;
      fx.elo[a] = any ? base_of(g, a, bl) : 0;
      fx.ehi[a] = any ? base_of(g, a, bh) + 3 : 0;
    }
    ctl->clr_lo[a] = prev_empty ? wlo : min(wlo, pl);
    ctl->clr_hi[a] = prev_empty ? whi : max(whi, ph);
    // the reference's Grid::active window: after a step it is the window of
    // the last substep's zero_grid (the one ending here), else the new one
    const bool after_step = (mode & kFinAdvect) != 0;
    ctl->ref_lo[a] = after_step ? wl_old : wlo;
    ctl->ref_hi[a] = after_step ? wh_old : whi;
    ctl->win_lo[a] = ctl->prev_lo[a] = wlo;
    ctl->win_hi[a] = ctl->prev_hi[a] = whi;
  }
  if ((mode & kFinAdvect) && ax) {  // the next advect reduces into the other slot
    ctl->bb_lo[cur ^ 1][a] = order_key(INFINITY);
    ctl->bb_hi[cur ^ 1][a] = order_key(-INFINITY);
  }
  if ((mode & kFinAdvect) && lane == 0) ctl->max_v2[cur ^ 1] = 0ull;
  if ((mode & kFinWalkFix) && (mode & kFinWindow)) {
    // The walks covered the new box iff it lies inside the widened old one.
    const bool old_ok = __all_sync(0xffffffffu, !ax || ohi > olo);
    const bool new_any = __all_sync(0xffffffffu, !ax || bl <= bh);
    const bool inside = __all_sync(0xffffffffu, !ax || (fx.elo[a] >= fx.wlo[a] && fx.ehi[a] <= fx.whi[a]));
    if (lane == 0) {
      fx.old_ok = old_ok;
      fx.need = new_any && !(old_ok && inside);
      fx.s = s;
      if (fx.need) ctl->walk_fixups = fixups + 1;
    }
  }
}

// zero_grid's clear of Grid::mass / momentum / velocity over Ctl::clr
// (engine.cpp:72-83).
__global__ void k_clear(NodeBuf grid, double* __restrict__ mi, VelBuf vel, Ctl* ctl, Geometry g) {
  if (stale(ctl, ctl->substep)) return;
  // both M_I buffers: the phase path's grid_update leaves its M_I in place,
  // and the next substep's look-ahead scatter goes into the other one
  // (the host grows the allocation over the window before the phase path
  // runs; clamped so a stale box can never index outside it)
  const int lx = max(ctl->clr_lo[0], g.ga_lo[0]), ly = max(ctl->clr_lo[1], g.ga_lo[1]),
            lz = max(ctl->clr_lo[2], g.ga_lo[2]);
  const int ny = max(min(ctl->clr_hi[1], g.ga_lo[1] + g.ga_dim[1]) - ly, 0);
  const int nz = max(min(ctl->clr_hi[2], g.ga_lo[2] + g.ga_dim[2]) - lz, 0);
  const int64_t total =
      static_cast<int64_t>(max(min(ctl->clr_hi[0], g.ga_lo[0] + g.ga_dim[0]) - lx, 0)) * ny * nz;
  const double2 z = make_double2(0, 0);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = static_cast<int>(t % nz);
    const int64_t r = t / nz;
    const int j = static_cast<int>(r % ny);
    const int i = static_cast<int>(r / ny);
    const size_t nd = node_index(g, lx + i, ly + j, lz + k);
    grid.lo[nd] = z;
    grid.hi[nd] = z;
    mi[nd] = 0.0;
    mi[g.mi_stride + nd] = 0.0;
    vel.xy[nd] = z;
    vel.z[nd] = 0.0;
  }
}

// ---------------------------------------------------------------------------
// particle_to_grid
// ---------------------------------------------------------------------------

// Standalone elastomer scatter (first substep of a call / phase API).
__global__ void __launch_bounds__(kGelThreads, kGelMinBlocks) k_p2g_gel_tile(
    const double* __restrict__ x, const double* __restrict__ v, const double* __restrict__ Cm,
    const double* __restrict__ Fm, int64_t n, int64_t n_el, GelMap M, Ctl* ctl, Geometry g,
    NodeBuf grid, double m, double vol0) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2GTile& T = *reinterpret_cast<P2GTile*>(smem_raw);
  const int s = ctl->substep;
  if (stale_block(ctl, s)) return;
  const int64_t p = gel_particle(M, n_el, blockIdx.x);
  bool active = p >= 0;
  P2GPayload q;
  double J = 1.0;
  if (active) {
    double F[9], C9[9], vv[3];
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      F[i] = Fm[i * n_el + p];
      C9[i] = Cm[i * n_el + p];
    }
    vv[0] = v[p];
    vv[1] = v[n + p];
    vv[2] = v[2 * n + p];
    active = make_payload(g, ctl, s, m, vol0, F, C9, vv, x[p], x[n + p], x[2 * n + p], q, J);
    if (active && !stencil_in_grid(g, q.st)) active = false;  // zero_grid already raised
  }
  reduce_min_detf(ctl, s, active, J);
  p2g_tile_scatter<-1>(T, active, q, m, g, grid, blockIdx.x, nullptr, ctl, s, false);
}

// Indenter scatter with a non-uniform velocity (only possible before the
// first apply_boundary after tg_create / tg_upload): direct REDs of w m and
// w m v into A.
__global__ void __launch_bounds__(256) k_p2g_ind_direct(const double* __restrict__ x,
                                                        const double* __restrict__ v, int64_t n,
                                                        int64_t n_el, Ctl* ctl, Geometry g,
                                                        NodeBuf grid, double m) {
  if (stale(ctl, ctl->substep)) return;
  const int64_t p = n_el + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  P2GPayload q;
  make_stencil(x[p], x[n + p], x[2 * n + p], g.origin, g.inv_dx, q.st);
  if (!stencil_in_grid(g, q.st)) return;
  if (!stencil_in_alloc(g, q.st.base)) {
    raise(ctl, kErrRegrow, ctl->substep);
    return;
  }
  q.mv[0] = m * v[p];
  q.mv[1] = m * v[n + p];
  q.mv[2] = m * v[2 * n + p];
#pragma unroll
  for (int i = 0; i < 9; ++i) q.aff[i] = 0.0;
  scatter_direct<-1>(g, grid, m, q, ctl);
}

// Rigid indenter: optional apply_boundary + advect (kMove) and the scatter of
// the (next) substep (kScatter). Every node receives (sum_p w_p) m (1, v)
// (C = 0, uniform v, engine.cpp:130,144), so only the weight sums M_I are
// scattered. Particles are sorted by (bx, by, z) at creation (engine.cu), so
// consecutive particles share a base cell in runs of ~particles-per-cell.
//   1. each thread moves kIndK consecutive particles (32-byte vector
//      loads/stores) and sums their 27 stencil weights in registers (an
//      in-chunk base change, rare, is flushed with direct REDs);
//   2. the per-thread partial sums go to shared memory with the base key;
//      threads with equal keys form contiguous runs;
//   3. (run, component) tasks sum a run's partials and issue one RED.F64 per
//      node (~1.5 per particle instead of 108).
constexpr int kIndThreads = 256;
constexpr int kIndK = 4;

struct IndSmem {
  double w[27][kIndThreads + 1];  // +1: (run, component) tasks read down columns
  long long key[kIndThreads];
  int run_start[kIndThreads + 1];
  int nruns;
  int warp_heads[kIndThreads / 32];
};

__device__ __forceinline__ long long base_key(const Geometry& g, const int* b) {
  return static_cast<long long>(node_index(g, b[0], b[1], b[2]));
}

template <bool kMove, bool kScatter>
__global__ void __launch_bounds__(kIndThreads) k_ind_move_p2g(double* __restrict__ x, int64_t n,
                                                              int64_t n_el, Ctl* ctl, Geometry g,
                                                              double* __restrict__ mi) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  IndSmem& S = *reinterpret_cast<IndSmem*>(smem_raw);
  const int s = ctl->substep;
  if (stale(ctl, s)) return;  // stable: nothing raises for substep s while this runs
  const int tid = threadIdx.x;
  const int64_t gt = static_cast<int64_t>(blockIdx.x) * kIndThreads + tid;
  const int s_scatter = kMove ? s + 1 : s;
  mi = mi_at(g, mi, s_scatter);
  if (gt == 0) {
    // apply_boundary: every indenter velocity becomes the command
    // (engine.cpp:260-261); M_I's velocity for grid_update of s_scatter
    for (int a = 0; a < 3; ++a) {
      if (kMove) ctl->ind_v[a] = ctl->vind[a];
      if (kScatter) ctl->ind_vp[s_scatter & 1][a] = kMove ? ctl->vind[a] : ctl->ind_v[a];
    }
  }
  // Coalesced move: the warp's 32 * kIndK consecutive particles, lane l
  // touching elements l + 32 i; then a register transpose (shuffles) gives
  // lane l the kIndK consecutive elements kIndK*l .. kIndK*l + kIndK - 1.
  const int lane = tid & 31;
  const int64_t wbase = n_el + (static_cast<int64_t>(blockIdx.x) * kIndThreads + (tid & ~31)) * kIndK;
  double cx[kIndK], cy[kIndK], cz[kIndK];
#pragma unroll
  for (int i = 0; i < kIndK; ++i) {
    const int64_t p = wbase + lane + 32 * i;
    const bool ok = p < n;
    cx[i] = ok ? x[p] : 0.0;
    cy[i] = ok ? x[n + p] : 0.0;
    cz[i] = ok ? x[2 * n + p] : 0.0;
  }
  if (kMove) {
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = mul_rn(g.dt, ctl->vind[a]);
#pragma unroll
    for (int i = 0; i < kIndK; ++i) {
      const int64_t p = wbase + lane + 32 * i;
      if (p < n) {
        cx[i] = add_rn(cx[i], d[0]);
        cy[i] = add_rn(cy[i], d[1]);
        cz[i] = add_rn(cz[i], d[2]);
        x[p] = cx[i];
        x[n + p] = cy[i];
        x[2 * n + p] = cz[i];
      }
    }
  }
  if (!kScatter) return;
  double px[kIndK], py[kIndK], pz[kIndK];
  const int reg = (kIndK * lane) >> 5;  // register slot holding this lane's elements
#pragma unroll
  for (int j = 0; j < kIndK; ++j) {
    const int src = (kIndK * lane + j) & 31;
    px[j] = py[j] = pz[j] = 0.0;
#pragma unroll
    for (int r = 0; r < kIndK; ++r) {
      const double vx = __shfl_sync(0xffffffffu, cx[r], src);
      const double vy = __shfl_sync(0xffffffffu, cy[r], src);
      const double vz = __shfl_sync(0xffffffffu, cz[r], src);
      if (r == reg) {
        px[j] = vx;
        py[j] = vy;
        pz[j] = vz;
      }
    }
  }
  const int64_t p0 = wbase + kIndK * lane;
  const int cnt = p0 >= n ? 0 : (n - p0 < kIndK ? static_cast<int>(n - p0) : kIndK);
  double acc[27];
#pragma unroll
  for (int i = 0; i < 27; ++i) acc[i] = 0.0;
  int cb[3] = {0, 0, 0};
  bool have = false;
#pragma unroll
  for (int j = 0; j < kIndK; ++j) {
    if (j >= cnt) break;
    Stencil st;
    make_stencil(px[j], py[j], pz[j], g.origin, g.inv_dx, st);
    if (!stencil_in_grid(g, st)) continue;  // finalize raises OutOfGrid
    if (!stencil_in_alloc(g, st.base)) {    // the host grows the allocation
      raise(ctl, kErrRegrow, s_scatter);
      continue;
    }
    if (have && (st.base[0] != cb[0] || st.base[1] != cb[1] || st.base[2] != cb[2])) {
      // rare: the chunk crosses a base cell; flush the first part directly
#pragma unroll
      for (int i = 0; i < 27; ++i) {
        if (acc[i] != 0.0)
          mi_add(g, mi + node_index(g, cb[0] + i / 9, cb[1] + (i / 3) % 3, cb[2] + i % 3), acc[i],
                 ctl);
        acc[i] = 0.0;
      }
    }
    cb[0] = st.base[0];
    cb[1] = st.base[1];
    cb[2] = st.base[2];
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
  // 2. partials + keys to shared memory; runs of equal keys.
  const long long key = have ? base_key(g, cb) : -1 - static_cast<long long>(tid);
  S.key[tid] = key;
#pragma unroll
  for (int i = 0; i < 27; ++i) S.w[i][tid] = acc[i];
  __syncthreads();
  const bool head = have && (tid == 0 || S.key[tid - 1] != key);
  const unsigned bal = __ballot_sync(0xffffffffu, head);
  const int warp = tid >> 5;
  if (lane == 0) S.warp_heads[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += S.warp_heads[w];
  const int rank = before + __popc(bal & ((1u << lane) - 1));
  if (head) S.run_start[rank] = tid;
  if (tid == kIndThreads - 1) {
    int total = 0;
    for (int w = 0; w < kIndThreads / 32; ++w) total += S.warp_heads[w];
    S.nruns = total;
  }
  __syncthreads();
  // 3. (run, component) tasks. A run ends at the next head or at the first
  // thread whose key differs (empty chunks carry unique negative keys).
  const int nruns = S.nruns;
  for (int task = tid; task < nruns * 27; task += kIndThreads) {
    const int r = task / 27, c = task % 27;
    const int t0 = S.run_start[r];
    const long long k0 = S.key[t0];
    double sum = 0.0;
    for (int t = t0; t < kIndThreads && S.key[t] == k0; ++t) sum += S.w[c][t];
    if (sum != 0.0) {
      const int64_t node = k0;  // node index of the base cell
      const int a = c / 9, b = (c / 3) % 3, cc = c % 3;
      mi_add(g, mi + node + (static_cast<int64_t>(a) * g.ga_dim[1] + b) * g.ga_dim[2] + cc, sum,
             ctl);
    }
  }
}

// ---------------------------------------------------------------------------
// Rigid-indenter scatter restricted to where it matters (step path).
//
// Grid velocities are only ever read by elastomer particles (the indenter
// skips G2P, engine.cpp:218), at nodes of their own stencils, i.e. inside the
// elastomer's node box. An indenter particle whose stencil misses that box
// changes nothing the simulation reads, so the step path scatters only the
// particles whose stencil meets it; M_I is then exact on every node that has
// elastomer mass. Within each column of the (bx, by, z)-sorted cloud z is
// ascending and stays so under the rigid translation (fl(z + d) is monotone),
// so base_z is non-decreasing: a warp walks its column upward and stops at the
// first particle above the box. Particles are still advected every substep in
// exact arithmetic: the ones visited here are moved in place, the others
// accumulate pending moves that k_ind_catchup applies (the same sequence of
// rounded adds) when the chain of same-velocity step calls ends (engine.cu
// flush_indenter: a velocity change, any access to the particle state, an
// error, or 255 substeps).
// ---------------------------------------------------------------------------
__global__ void k_chain_begin(Ctl* ctl) { ctl->chain_start = ctl->substep; }

constexpr int kColWarps = 8;  // the walk blocks inside the elastomer kernel (TACCHI_WALKS=fused)
#ifndef TACCHI_WALK_WARPS
#define TACCHI_WALK_WARPS 4
#endif
// Warps (columns) per block of the walk kernel of its own: small blocks
// retire as soon as their columns are done instead of holding shared memory
// and registers for their longest column.
constexpr int kWalkWarps = TACCHI_WALK_WARPS;

template <int W>
struct ColSmemT {
  double w[W][27][33];
  long long key[W][32];
  int run_start[W][33];
  int run_end[W][33];
};
using ColSmem = ColSmemT<kColWarps>;

// One block's column walks (blk = block index among the indenter blocks).
// box_mode: 0 = Ctl::box[0] (the elastomer box of the substep being
// scattered: standalone scatter), 1 = from Ctl::bb (the elastomer bbox after
// this substep's advect), 2 = Ctl::box[0] of this substep widened by one node
// on every side (look-ahead scatter running alongside the elastomer kernel:
// the elastomer moves less than one cell per substep, which k_finalize checks).
// An indenter particle with stencil st is scattered by a walk over the
// elastomer node box [glo, ghi) iff its stencil is in the grid and its 27
// nodes meet the box (base_z is non-decreasing along a column, so the walk's
// stop at the first particle with base_z >= ghi_z drops none of these).
__device__ __forceinline__ bool walk_contrib(const Geometry& g, const Stencil& st, const int* glo,
                                             const int* ghi) {
  bool c = stencil_in_grid(g, st);
#pragma unroll
  for (int a = 0; a < 3; ++a) c = c && st.base[a] + 2 >= glo[a] && st.base[a] <= ghi[a] - 1;
  return c;
}

template <bool kMove, int kDet = -1, int W = kColWarps>
__device__ __forceinline__ void ind_cols_block(ColSmemT<W>& S, int blk, double* __restrict__ x,
                                               int64_t n, int64_t n_el,
                                               const int64_t* __restrict__ col_start, int n_cols,
                                               uint8_t* __restrict__ moves, Ctl* ctl,
                                               const Geometry& g, double* __restrict__ mi,
                                               int box_mode, int s) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s_scatter = kMove ? s + 1 : s;
  mi = mi_at(g, mi, s_scatter);
  if (blk == 0 && threadIdx.x == 0 && !stale(ctl, s)) {
    for (int a = 0; a < 3; ++a) {
      if (kMove) ctl->ind_v[a] = ctl->vind[a];  // apply_boundary (engine.cpp:260-261)
      ctl->ind_vp[s_scatter & 1][a] = kMove ? ctl->vind[a] : ctl->ind_v[a];
    }
  }
  const int c = blk * W + warp;
  if (c >= n_cols) return;  // warp-uniform; only __syncwarp below
  // Every input of the walk is loaded up front (one round trip for the
  // column bounds, the box, the chain start and the velocity instead of a
  // chain of dependent reads), then the column's first chunk.
  const int64_t a0 = col_start[c], a1 = col_start[c + 1];
  int blo0[3], bhi0[3];
  for (int a = 0; a < 3; ++a) {
    blo0[a] = ctl->box_lo[0][a];
    bhi0[a] = ctl->box_hi[0][a];
  }
  const int chain_start = ctl->chain_start;
  double vind[3];
  for (int a = 0; a < 3; ++a) vind[a] = ctl->vind[a];
  double nx = 0, ny = 0, nz = 0;
  int ndone = 0;
  if (a0 + lane < a1) {
    const int64_t p = a0 + lane;
    nx = __ldcs(x + p);
    ny = __ldcs(x + n + p);
    nz = __ldcs(x + 2 * n + p);
    ndone = moves[p - n_el];
  }
  // (k_ind_cols checks staleness here, after issuing its loads)
  if (stale(ctl, s)) return;
  // Elastomer node box of the substep being scattered.
  int glo[3], ghi[3];
  for (int a = 0; a < 3; ++a) {
    if (box_mode == 1) {
      const double l = order_val(ctl->bb_lo[s & 1][a]), h = order_val(ctl->bb_hi[s & 1][a]);
      if (!(l <= h)) return;  // no elastomer: nothing reads the grid
      glo[a] = static_cast<int>(floor(sub_rn(mul_rn(sub_rn(l, g.origin[a]), g.inv_dx), 0.5)));
      ghi[a] = static_cast<int>(floor(sub_rn(mul_rn(sub_rn(h, g.origin[a]), g.inv_dx), 0.5))) + 3;
    } else {
      const int widen = box_mode == 2 ? 1 : 0;
      glo[a] = blo0[a];
      ghi[a] = bhi0[a];
      if (ghi[a] <= glo[a]) return;
      glo[a] -= widen;
      ghi[a] += widen;
    }
  }
  const int target = s - chain_start + (kMove ? 1 : 0);  // chain advects after this kernel
  double d[3] = {0, 0, 0};
  for (int a = 0; a < 3; ++a) d[a] = mul_rn(g.dt, vind[a]);
  // the next chunk's loads are issued one chunk ahead (most columns take two
  // or three chunks; each was a dependent DRAM round trip)
  unsigned walked = 0;
  for (int64_t b0 = a0; b0 < a1; b0 += 32) {
    const int64_t p = b0 + lane;
    const bool valid = p < a1;
    double px = nx, py = ny, pz = nz;
    const int done = ndone;
    if (b0 + 32 + lane < a1) {
      const int64_t q = b0 + 32 + lane;
      nx = __ldcs(x + q);
      ny = __ldcs(x + n + q);
      nz = __ldcs(x + 2 * n + q);
      ndone = moves[q - n_el];
    }
    Stencil st;
    bool beyond = false, contrib = false, moved = false;
    if (valid) {
      moved = done < target;
      if (moved) {
        for (int k = done; k < target; ++k) {
          px = add_rn(px, d[0]);
          py = add_rn(py, d[1]);
          pz = add_rn(pz, d[2]);
        }
        __stcs(x + p, px);
        __stcs(x + n + p, py);
        __stcs(x + 2 * n + p, pz);
        moves[p - n_el] = static_cast<uint8_t>(target);
      }
      make_stencil(px, py, pz, g.origin, g.inv_dx, st);
      beyond = st.base[2] > ghi[2] - 1;  // this and every later particle of the column miss
      contrib = walk_contrib(g, st, glo, ghi);
      if (contrib && !stencil_in_alloc(g, st.base)) {  // the host grows the allocation
        raise(ctl, kErrRegrow, kMove ? s + 1 : s);
        contrib = false;
      }
    }
    walked += __popc(__ballot_sync(0xffffffffu, moved));
    const unsigned bey = __ballot_sync(0xffffffffu, beyond);
    const int first_beyond = bey ? __ffs(bey) - 1 : 32;
    if (lane > first_beyond) contrib = false;
    if (!__any_sync(0xffffffffu, contrib)) {  // nothing to scatter in this chunk
      if (bey) break;
      continue;
    }
    const long long key = contrib ? static_cast<long long>(node_index(g, st.base[0], st.base[1], st.base[2]))
                                  : -1 - static_cast<long long>(lane);
#pragma unroll
    for (int a = 0; a < 3; ++a)
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const double wab = contrib ? st.w[0][a] * st.w[1][b] : 0.0;
#pragma unroll
        for (int cc = 0; cc < 3; ++cc) S.w[warp][9 * a + 3 * b + cc][lane] = wab * (contrib ? st.w[2][cc] : 0.0);
      }
    S.key[warp][lane] = key;
    __syncwarp();
    // runs of equal keys (contributing lanes only): heads and tails ranked
    // by ballot, so the sums below walk [start, end) without key compares
    const bool head = contrib && (lane == 0 || S.key[warp][lane - 1] != key);
    const bool tail = contrib && (lane == 31 || S.key[warp][lane + 1] != key);
    const unsigned hb = __ballot_sync(0xffffffffu, head);
    const unsigned tb = __ballot_sync(0xffffffffu, tail);
    if (head) S.run_start[warp][__popc(hb & ((1u << lane) - 1))] = lane;
    if (tail) S.run_end[warp][__popc(tb & ((1u << lane) - 1))] = lane + 1;
    __syncwarp();
    const int nruns = __popc(hb);
    for (int task = lane; task < nruns * 27; task += 32) {
      const int r = task / 27, comp = task % 27;
      const int t0 = S.run_start[warp][r], t1 = S.run_end[warp][r];
      const long long k0 = S.key[warp][t0];
      double sum = 0.0;
      for (int t = t0; t < t1; ++t) sum += S.w[warp][comp][t];
      if (sum != 0.0)
        mi_add<kDet>(g, mi + k0 + (static_cast<int64_t>(comp / 9) * g.ga_dim[1] + (comp / 3) % 3) * g.ga_dim[2] +
                    comp % 3,
               sum, ctl);
    }
    __syncwarp();
    if (bey) break;  // the rest of the column is above the elastomer box
  }
  // tg_stats' walked count: one RED per column (per chunk, they queued on
  // one control-block word)
  if (lane == 0 && walked) atomicAdd(&ctl->ind_walked, static_cast<unsigned long long>(walked));
}

template <bool kMove>
__global__ void __launch_bounds__(kWalkWarps * 32) k_ind_cols(
    double* __restrict__ x, int64_t n, int64_t n_el, const int64_t* __restrict__ col_start,
    int n_cols, uint8_t* __restrict__ moves, Ctl* ctl, Geometry g, double* __restrict__ mi,
    int box_mode) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  ColSmemT<kWalkWarps>& S = *reinterpret_cast<ColSmemT<kWalkWarps>*>(smem_raw);
  pdl_wait();
  // staleness is checked inside, once the walk's loads are in flight
  ind_cols_block<kMove, -1, kWalkWarps>(S, blockIdx.x, x, n, n_el, col_start, n_cols, moves, ctl,
                                        g, mi, box_mode, ctl->substep);
}

// Applies the pending advects of the indenter particles the column walks did
// not visit, so every particle has moved exactly (completed substeps of the
// chain) times, then resets the move counters.
__global__ void k_ind_catchup(double* __restrict__ x, int64_t n, int64_t n_el,
                              uint8_t* __restrict__ moves, Ctl* ctl, Geometry g) {
  pdl_wait();
  const int64_t p = n_el + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int total = ctl->substep - ctl->chain_start;  // advects completed in the chain
  const int done = moves[p - n_el];
  if (done < total) {
    double d[3];
    for (int a = 0; a < 3; ++a) d[a] = mul_rn(g.dt, ctl->vind[a]);
    double px = __ldcs(x + p), py = __ldcs(x + n + p), pz = __ldcs(x + 2 * n + p);
    for (int k = done; k < total; ++k) {
      px = add_rn(px, d[0]);
      py = add_rn(py, d[1]);
      pz = add_rn(pz, d[2]);
    }
    __stcs(x + p, px);
    __stcs(x + n + p, py);
    __stcs(x + 2 * n + p, pz);
  }
  if (done) moves[p - n_el] = 0;
}

// Fix-up of the look-ahead walks (rare: the elastomer moved out of the box
// the walks used, i.e. more than a cell in one substep): every warp of
// finalize's block walks whole columns and scatters the particles whose
// stencil meets the new box but not the widened old one (the walks scattered
// exactly the latter), at their positions after this substep's advect
// (pending advects applied on the fly, as the walks do).
__device__ void ind_walk_fixup(const FinFix& fx, const double* __restrict__ x, int64_t n,
                               int64_t n_el, const int64_t* __restrict__ col_start, int n_cols,
                               const uint8_t* __restrict__ moves, Ctl* ctl,
                               const Geometry& g, double* __restrict__ mi) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int target = fx.s - ctl->chain_start + 1;
  mi = mi_at(g, mi, fx.s + 1);
  double d[3];
  for (int a = 0; a < 3; ++a) d[a] = mul_rn(g.dt, ctl->vind[a]);
  for (int c = warp; c < n_cols; c += nw) {
    const int64_t a1 = col_start[c + 1];
    for (int64_t p = col_start[c] + lane; p < a1; p += 32) {
      double px = x[p], py = x[n + p], pz = x[2 * n + p];
      for (int k = moves[p - n_el]; k < target; ++k) {
        px = add_rn(px, d[0]);
        py = add_rn(py, d[1]);
        pz = add_rn(pz, d[2]);
      }
      Stencil st;
      make_stencil(px, py, pz, g.origin, g.inv_dx, st);
      if (!walk_contrib(g, st, fx.elo, fx.ehi)) continue;
      if (fx.old_ok && walk_contrib(g, st, fx.wlo, fx.whi)) continue;  // the walk had it
      if (!stencil_in_alloc(g, st.base)) {
        raise(ctl, kErrRegrow, fx.s + 1);
        continue;
      }
#pragma unroll
      for (int i = 0; i < 27; ++i) {
        const int ia = i / 9, ib = (i / 3) % 3, ic = i % 3;
        mi_add(g, mi + node_index(g, st.base[0] + ia, st.base[1] + ib, st.base[2] + ic),
               st.w[0][ia] * st.w[1][ib] * st.w[2][ic], ctl);
      }
    }
  }
}

// Walk fix-up arguments (the step path's column data).
struct FixArgs {
  const double* x;
  int64_t n, n_el;
  const int64_t* col_start;
  int n_cols;
  const uint8_t* moves;
  double* mi;
};

// advect's in_range / step_count / max_speed and the next zero_grid window
// (finalize_warp, warp 0); with kFinWalkFix the other warps of the block
// stand by for the walk fix-up.
__global__ void __launch_bounds__(256) k_finalize(Ctl* ctl, Geometry g, int mode, FixArgs fa) {
  // every kernel that follows finalize in a step plan (grid_update,
  // k_ind_catchup) reads nothing before its own wait: let it launch while
  // this block runs -- by default before finalize's own wait, so the next
  // grid_update's blocks fill the SMs the elastomer kernel's tail frees and
  // are resident when finalize completes
  if (g.fin_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  pdl_wait();
  if (!g.fin_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  __shared__ FinFix fx;
  if (threadIdx.x == 0) fx.need = 0;
  if (blockDim.x > 32) __syncthreads();
  if (threadIdx.x < 32) finalize_warp(ctl, g, mode, fx);
  if (blockDim.x == 32) return;
  __syncthreads();
  if (fx.need)
    ind_walk_fixup(fx, fa.x, fa.n, fa.n_el, fa.col_start, fa.n_cols, fa.moves, ctl, g, fa.mi);
}

// ---------------------------------------------------------------------------
// grid_update (engine.cpp:180-205)
// ---------------------------------------------------------------------------
// grid_update of one node (engine.cpp:186-203) from its accumulators: the
// elastomer's A = {m, p} plus the indenter's weight sum wi (mass m_ind wi,
// momentum m_ind wi u). Massless nodes get v = 0.
__device__ __forceinline__ double4 node_velocity(const Geometry& g, double4 q, double wi,
                                                 double m_ind, double u0, double u1, double u2,
                                                 int i, int j, int k) {
  double4 o = make_double4(0, 0, 0, 0);
  double mass = q.x, p0 = q.y, p1 = q.z, p2 = q.w;
  if (wi != 0.0) {  // explicit roundings: tg_download_grid forms the same sums
    const double M = __dmul_rn(wi, m_ind);
    mass = __dadd_rn(mass, M);
    p0 = __dadd_rn(p0, __dmul_rn(M, u0));
    p1 = __dadd_rn(p1, __dmul_rn(M, u1));
    p2 = __dadd_rn(p2, __dmul_rn(M, u2));
  }
  if (mass > 0.0) {
    // p / mass, correctly rounded (Markstein: y = RN(1/mass), q = RN(p y),
    // q + (p - mass q) y rounded once is RN(p / mass) for normal operands):
    // one reciprocal shared by the three components.
    const double y = __drcp_rn(mass);
    double q0 = p0 * y, q1 = p1 * y, q2 = p2 * y;
    q0 = fma(fma(-q0, mass, p0), y, q0);
    q1 = fma(fma(-q1, mass, p1), y, q1);
    q2 = fma(fma(-q2, mass, p2), y, q2);
    o.x = q0;
    o.y = q1;
    o.z = q2;
    if (g.with_gravity) {
      o.x = o.x + g.gdt[0];
      o.y = o.y + g.gdt[1];
      o.z = o.z + g.gdt[2];
    }
    if (i == 0 || i == g.res[0] - 1) o.x = 0.0;
    if (j == 0 || j == g.res[1] - 1) o.y = 0.0;
    if (k == 0 || k == g.res[2] - 1) o.z = 0.0;
    o.w = 1.0;  // has mass (not part of Grid::velocity)
  }
  return o;
}

// Node update of the grid_update kernels; kZero also re-zeroes A / M_I.
// with_mi: the node may hold indenter weight (inside the indenter box).
template <bool kZero>
__device__ __forceinline__ void update_node(NodeBuf mp, double* __restrict__ mi,
                                            VelBuf vel, const Geometry& g,
                                            double m_ind, double u0, double u1, double u2, int i,
                                            int j, int k, bool with_mi) {
  const size_t nd = node_index(g, i, j, k);
  const double2 qa = mp.lo[nd], qb = mp.hi[nd];
  // the accumulators' bits (fixed point in deterministic mode)
  const bool filled = __double_as_longlong(qa.x) | __double_as_longlong(qa.y) |
                      __double_as_longlong(qb.x) | __double_as_longlong(qb.y);
  double4 q = make_double4(qa.x, qa.y, qb.x, qb.y);
  double wi = with_mi ? mi[nd] : 0.0;
  if (g.det) {
    q = make_double4(from_fixed(qa.x, g.fx_inv), from_fixed(qa.y, g.fx_inv),
                     from_fixed(qb.x, g.fx_inv), from_fixed(qb.y, g.fx_inv));
    wi = from_fixed(wi, g.fxi_inv);
  }
  double4 o = node_velocity(g, q, wi, m_ind, u0, u1, u2, i, j, k);
  const bool massive = o.w != 0.0;
  o.w = 0.0;
  // Step path: nodes without mass keep their (finite) stale velocity; every
  // G2P read of such a node carries B-spline weight exactly 0 (the particle's
  // own scatter would have given it mass otherwise).
  if (!kZero || massive) {  // read back by the next G2P staging: keep in L2
    st_keep(vel.xy + nd, o.x, o.y);
    st_keep1(vel.z + nd, o.z);
  }
  if (kZero) {
    if (filled) {  // next scatter target
      st_keep(mp.lo + nd, 0.0, 0.0);
      st_keep(mp.hi + nd, 0.0, 0.0);
    }
    if (wi != 0.0) mi[nd] = 0.0;
  }
}

// Phase API: the full active window, as the reference (Grid::velocity is 0
// on every massless window node).
__global__ void k_grid_update_window(NodeBuf mp, double* __restrict__ mi, VelBuf vel,
                                     Ctl* ctl, Geometry g,
                                     double m_ind) {
  if (stale(ctl, ctl->substep)) return;
  mi = mi_at(g, mi, ctl->substep);
  const int lx = max(ctl->win_lo[0], g.ga_lo[0]), ly = max(ctl->win_lo[1], g.ga_lo[1]),
            lz = max(ctl->win_lo[2], g.ga_lo[2]);
  const int ny = max(min(ctl->win_hi[1], g.ga_lo[1] + g.ga_dim[1]) - ly, 0);
  const int nz = max(min(ctl->win_hi[2], g.ga_lo[2] + g.ga_dim[2]) - lz, 0);
  const int vol = max(min(ctl->win_hi[0], g.ga_lo[0] + g.ga_dim[0]) - lx, 0) * ny * nz;
  const double u0 = ctl->ind_v[0], u1 = ctl->ind_v[1], u2 = ctl->ind_v[2];
  for (BoxIter it(blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x, ny, nz); it.e < vol;
       it.next(ny, nz))
    update_node<false>(mp, mi, vel, g, m_ind, u0, u1, u2, lx + it.i, ly + it.j, lz + it.k, true);
}

// Step path: only the union of the elastomer and indenter node boxes (every
// node a scatter can have touched), re-zeroing the accumulators. M_I is read
// only inside the indenter box.
__global__ void __launch_bounds__(256, 5) k_grid_update_boxes(NodeBuf mp, double* __restrict__ mi, VelBuf vel,
                                    Ctl* ctl, Geometry g,
                                    double m_ind) {
  pdl_wait();
  // The elastomer kernel that follows reads its particle state (written two
  // kernels back, complete now) before its own wait: let it launch early.
  if (g.pdl_early) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int s = ctl->substep;
  if (stale(ctl, s)) return;
  mi = mi_at(g, mi, s);
  int lo[2][3], dm[2][3], vol[2];
  for (int m = 0; m < 2; ++m) {  // each box clamped to the allocation (no mass outside)
    vol[m] = 1;
    for (int a = 0; a < 3; ++a) {
      lo[m][a] = max(ctl->box_lo[m][a], g.ga_lo[a]);
      dm[m][a] = max(min(ctl->box_hi[m][a], g.ga_lo[a] + g.ga_dim[a]) - lo[m][a], 0);
      vol[m] *= dm[m][a];
    }
  }
  // the indenter velocity its M_I scatter was made with (the walks of the
  // previous substep may already be writing the other slot)
  const double u0 = ctl->ind_vp[s & 1][0], u1 = ctl->ind_vp[s & 1][1], u2 = ctl->ind_vp[s & 1][2];
  const int first = blockIdx.x * blockDim.x + threadIdx.x, step = gridDim.x * blockDim.x;
  auto in_box = [&](int m, int i, int j, int k) {
    return vol[m] > 0 && i >= lo[m][0] && i < lo[m][0] + dm[m][0] && j >= lo[m][1] &&
           j < lo[m][1] + dm[m][1] && k >= lo[m][2] && k < lo[m][2] + dm[m][2];
  };
  if (vol[0] > 0)
    for (BoxIter it(first, step, dm[0][1], dm[0][2]); it.e < vol[0]; it.next(dm[0][1], dm[0][2])) {
      const int i = lo[0][0] + it.i, j = lo[0][1] + it.j, k = lo[0][2] + it.k;
      update_node<true>(mp, mi, vel, g, m_ind, u0, u1, u2, i, j, k, in_box(1, i, j, k));
    }
  if (vol[1] > 0)
    for (BoxIter it(first, step, dm[1][1], dm[1][2]); it.e < vol[1]; it.next(dm[1][1], dm[1][2])) {
      const int i = lo[1][0] + it.i, j = lo[1][1] + it.j, k = lo[1][2] + it.k;
      if (in_box(0, i, j, k)) continue;  // already handled in the elastomer box
      update_node<true>(mp, mi, vel, g, m_ind, u0, u1, u2, i, j, k, true);
    }
}

// ---------------------------------------------------------------------------
// grid_to_particle (+ apply_boundary + advect) [+ next particle_to_grid]
// ---------------------------------------------------------------------------

namespace {
// engine.cpp:217-249 for one particle: v and C from the node velocities.
// kGuard: nodes outside the allocation read as 0 (phase path, where positions
// may have been uploaded after zero_grid); in the step path every stencil
// lies in the box its own P2G scattered to, so no check is compiled in.
template <bool kGuard>
__device__ __forceinline__ void g2p_gather(const Geometry& g, VelBuf vel,
                                           double px0, double px1, double px2, double* vv,
                                           double* Cn) {
  Stencil st;
  make_stencil(px0, px1, px2, g.origin, g.inv_dx, st);
  const bool inside = !kGuard || stencil_in_alloc(g, st.base);
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
      const size_t row = node_index(g, st.base[0] + a, st.base[1] + b, st.base[2]);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = wab * st.w[2][c];
        const double dc = c - st.fx[2];
        // nodes outside the allocation hold no mass: velocity 0 (as the
        // reference's cleared grid)
        const bool in = inside || box_in_alloc(g, st.base[0] + a, st.base[1] + b, st.base[2] + c,
                                               st.base[0] + a + 1, st.base[1] + b + 1,
                                               st.base[2] + c + 1);
        const double2 qa = in ? __ldg(vel.xy + row + c) : make_double2(0.0, 0.0);
        const double2 qb = make_double2(in ? __ldg(vel.z + row + c) : 0.0, 0.0);
        const double wv0 = w * qa.x, wv1 = w * qa.y, wv2 = w * qb.x;
        v0 += wv0; v1 += wv1; vz += wv2;
        b00 += wv0 * da; b01 += wv0 * db; b02 += wv0 * dc;
        b10 += wv1 * da; b11 += wv1 * db; b12 += wv1 * dc;
        b20 += wv2 * da; b21 += wv2 * db; b22 += wv2 * dc;
      }
    }
  }
  vv[0] = v0;
  vv[1] = v1;
  vv[2] = vz;
  const double k = 4.0 * g.inv_dx;
  Cn[0] = k * b00; Cn[1] = k * b01; Cn[2] = k * b02;
  Cn[3] = k * b10; Cn[4] = k * b11; Cn[5] = k * b12;
  Cn[6] = k * b20; Cn[7] = k * b21; Cn[8] = k * b22;
}
}  // namespace

// G2P gather from the CTA's node box staged in shared memory (vx, vy, vz in
// T.nlo[.].x/y, T.nhi[.].x), same arithmetic as g2p_gather.
__device__ __forceinline__ void g2p_gather_smem(const Geometry& g, const P2GTile& T,
                                                const Stencil& st, double* vv, double* Cn) {
  const int d1 = T.rd, d2 = T.pitch, zp = T.zp;
  const int r0 = (st.base[0] - T.lo[0]) * d1 + (st.base[1] - T.lo[1]);
  const int c0 = st.base[2] - T.lo[2];
  const double* zs = reinterpret_cast<const double*>(T.nhi);
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
      const int r = r0 + a * d1 + b;
      const int row = r * d2 + c0, zrow = r * zp + T.zoff + c0;
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        const double w = wab * st.w[2][c];
        const double dc = c - st.fx[2];
        const double2 vxy = T.nlo[row + c];
        const double vzz = zs[zrow + c];
        const double wv0 = w * vxy.x, wv1 = w * vxy.y, wv2 = w * vzz;
        v0 += wv0; v1 += wv1; vz += wv2;
        b00 += wv0 * da; b01 += wv0 * db; b02 += wv0 * dc;
        b10 += wv1 * da; b11 += wv1 * db; b12 += wv1 * dc;
        b20 += wv2 * da; b21 += wv2 * db; b22 += wv2 * dc;
      }
    }
  }
  vv[0] = v0;
  vv[1] = v1;
  vv[2] = vz;
  const double k = 4.0 * g.inv_dx;
  Cn[0] = k * b00; Cn[1] = k * b01; Cn[2] = k * b02;
  Cn[3] = k * b10; Cn[4] = k * b11; Cn[5] = k * b12;
  Cn[6] = k * b20; Cn[7] = k * b21; Cn[8] = k * b22;
}

template <bool kBoundary, bool kAdvect, bool kLookahead, int kDet = -1>
__global__ void __launch_bounds__(kGelThreads, kGelMinBlocks) k_g2p2g_gel(
    double* __restrict__ x, double* __restrict__ v, double* __restrict__ Cm,
    double* __restrict__ Fm, const uint8_t* __restrict__ tag, int64_t n, int64_t n_el, GelMap M,
    Ctl* ctl, Geometry g, VelBuf vel, NodeBuf grid, double m,
    double vol0, IndArgs ia) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  P2GTile& T = *reinterpret_cast<P2GTile*>(smem_raw);
  const bool with_ind = kLookahead && ia.gel_ctas > 0;
  const int cta = with_ind ? static_cast<int>(blockIdx.x) - ia.gel_lo : static_cast<int>(blockIdx.x);
  const bool gel_block = !with_ind || (cta >= 0 && cta < ia.gel_ctas);
  TRACE_BEGIN(gel_block ? 1 : 2);
  const int64_t p = gel_block ? gel_particle(M, n_el, cta) : -1;
  const bool active = p >= 0;
  double px0 = 0, px1 = 0, px2 = 0, v2 = 0;
  bool bottom = false;
  if (active) {
    // particle state streams through once per substep: evict-first loads and
    // stores (ld/st .cs) keep L2 for the grid arrays the next kernels reuse.
    // x, F and cta_box were last written by the previous launch of this
    // kernel, which is complete once the kernel before this one passed its
    // own griddepcontrol.wait (the only way this grid can have been
    // launched), so they are read before this grid's wait, overlapping the
    // tail of grid_update. F is loaded once the stencil is computed (loaded
    // into registers this early it is spilled; an L2 prefetch of it here
    // measured 0.6 % slower than none, round 2).
    px0 = __ldcs(x + p);
    px1 = __ldcs(x + n + p);
    px2 = __ldcs(x + 2 * n + p);
    if (kBoundary) bottom = __ldg(tag + p) == kElastomerBottom;
  }
  int ctl_s = 0;
  bool ctl_stale = false;
  if (kLookahead && gel_block && threadIdx.x == 0) {
    // The control block as the previous finalize left it, read beside the
    // tile box (one round trip instead of two): finalize(s - 1) is complete
    // once grid_update passed its own wait (the only way this grid can have
    // been launched), grid_update raises nothing, and the walks beside it
    // raise only for s + 1, so neither the substep nor its stale flag can
    // change before this grid's wait.
    ctl_s = ctl->substep;
    ctl_stale = stale(ctl, ctl_s);
    // The G2P footprint is the tile box of the P2G that scattered these
    // particles at these positions (the previous kernel of this CTA).
    const int* b = g.cta_box + 8 * cta;
    for (int a = 0; a < 3; ++a) {
      T.lo[a] = b[a];
      T.dim[a] = b[3 + a];
    }
    // vz row staging needs even allocation rows (even start and length in z)
    T.ok = b[6] && (g.ga_dim[2] & 1) == 0 && (g.ga_lo[2] & 1) == 0;
    T.pitch = tile_pitch(T.dim[2]);
    T.rd = T.dim[1] + kRowPad;
    if (T.ok && g.scatter_mode != 5) tile_bulk_stage_init(T);
    for (int a = 0; a < 3; ++a) {  // the empty box for block_motion_box
      T.blo[a] = INT_MAX;
      T.bhi[a] = INT_MIN;
    }
  }
  if (kLookahead && kDet == 1 && gel_block) {
    // the deterministic scatter's owner table (p2g_tile_scatter owners_reset),
    // shared memory only: before the wait, published by the start barrier
    for (int e = threadIdx.x; e < kTileCap; e += blockDim.x) T.owner[e] = -1;
  }
  pdl_wait();
  // Let finalize (which waits for this whole grid) be launched once every CTA
  // of it has started: it is then resident when the last CTA retires
  // instead of being launched after it (TACCHI_GEL_TRIGGER=0: off)
  if (kLookahead && g.gel_trigger) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (kLookahead && gel_block && threadIdx.x == 0) {
    // the substep and its stale flag, shared at the barrier below
    T.cur_s = ctl_s;
    T.cur_stale = ctl_stale ? 1 : 0;
  }
  TRACE_MARK(1);
  if (!gel_block) {
    // indenter blocks: the s+1 column walks (they touch only indenter x and
    // M_I; the elastomer box comes from the previous finalize, widened)
    const int s = ctl->substep;
    if (stale(ctl, s)) return;
    ind_cols_block<true, kDet>(*reinterpret_cast<ColSmem*>(smem_raw), blockIdx.x - ia.ind_lo, x, n,
                         n_el, ia.col_start, ia.n_cols, ia.moves, ctl, g, ia.mi, 2, s);
    TRACE_END();
    return;
  }
  double F[9], vv[3], Cn[9];  // defined for active particles only
  bool staged = false;
  Stencil st_old;
  int s;
  if (kLookahead) {
    // Stage the grid velocities of the CTA's G2P footprint (coalesced rows
    // along z) in the shared tile before the gathers. One barrier publishes
    // thread 0's tile box, mbarrier and control-block read.
    __syncthreads();
    s = T.cur_s;
    if (T.cur_stale) return;  // block-uniform; no copy issued yet
    staged = T.ok != 0;
    if (staged && g.scatter_mode != 5) tile_bulk_stage_copies(T, g, vel);
  } else {
    s = ctl->substep;
    if (stale_block(ctl, s)) return;
  }
  const bool staging = kLookahead && staged && g.scatter_mode != 5;
  // the stencil needs x: its loads complete while the staging copies fly
  if (active) make_stencil(px0, px1, px2, g.origin, g.inv_dx, st_old);
  // F is loaded while the staging copies complete: loaded at entry it was
  // spilled (the spill store waited for the load), loaded after the gather
  // its latency was exposed (DESIGN 4.5)
  double F0[9];
  if (active) {
#pragma unroll
    for (int i = 0; i < TACCHI_F_EARLY; ++i) F0[i] = __ldcs(Fm + i * n_el + p);
  }
  if (staging) tile_bulk_wait(T);
  TRACE_MARK(2);
  if (active) {
#pragma unroll
    for (int i = TACCHI_F_EARLY; i < 9; ++i) F0[i] = __ldcs(Fm + i * n_el + p);
  }
  if (active) {
    if (g.scatter_mode == 5) {  // A/B timing: no velocity staging / gather
      vv[0] = vv[1] = vv[2] = 0.0;
      for (int i = 0; i < 9; ++i) Cn[i] = 0.0;
    } else if (staged) g2p_gather_smem(g, T, st_old, vv, Cn);
    else g2p_gather<!kLookahead>(g, vel, px0, px1, px2, vv, Cn);
    TRACE_MARK(8);
    double G[9];
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) G[3 * i + j] = (i == j ? 1.0 : 0.0) + g.dt * Cn[3 * i + j];
    matmul3(G, F0, F);  // F <- (I + dt C) F  (engine.cpp:250)
#pragma unroll
    for (int i = 0; i < 9; ++i) {
      if (g.scatter_mode != 6) __stcs(Cm + i * n_el + p, Cn[i]);  // 6: A/B timing, no C / v
      __stcs(Fm + i * n_el + p, F[i]);
    }
    if (bottom) vv[0] = vv[1] = vv[2] = 0.0;
    if (g.scatter_mode != 6) {
      __stcs(v + p, vv[0]);
      __stcs(v + n + p, vv[1]);
      __stcs(v + 2 * n + p, vv[2]);
    }
    if (kAdvect) {
      px0 = advance(px0, g.dt, vv[0]);
      px1 = advance(px1, g.dt, vv[1]);
      px2 = advance(px2, g.dt, vv[2]);
      __stcs(x + p, px0);
      __stcs(x + n + p, px1);
      __stcs(x + 2 * n + p, px2);
      v2 = vv[0] * vv[0] + vv[1] * vv[1] + vv[2] * vv[2];
    }
  }
  TRACE_MARK(9);
  if (kAdvect && !kLookahead)
    reduce_motion(&ctl->max_v2[s & 1], ctl->bb_lo[s & 1], ctl->bb_hi[s & 1], active, v2, px0, px1,
                  px2);
  TRACE_MARK(3);
  if (kLookahead) {
    static_assert(!kLookahead || kAdvect, "the look-ahead scatter follows an advect");
    // particle_to_grid of substep s + 1 with the state just written.
    P2GPayload q;
    double J = 1.0;
    bool go = active;
    if (go && g.scatter_mode == 4) {
      make_stencil(px0, px1, px2, g.origin, g.inv_dx, q.st);
      q.mv[0] = q.mv[1] = q.mv[2] = 0.0;
      for (int i = 0; i < 9; ++i) q.aff[i] = 0.0;
    } else if (go) {
      go = make_payload(g, ctl, s + 1, m, vol0, F, Cn, vv, px0, px1, px2, q, J);
      if (go && !stencil_in_grid(g, q.st)) go = false;  // finalize raises OutOfGrid
    }
    TRACE_MARK(4);
    // advect's motion reductions, min det F of s + 1 and the tile box together
    TileBox box;
    block_motion_box(T, ctl, s, active, v2, px0, px1, px2, go, J, q.st.base, box);
    p2g_tile_scatter<kDet>(T, go, q, m, g, grid, cta, &box, ctl, s + 1, kDet == 1);
  }
  TRACE_END();
}

// A copy of the control block (the pipelined frames' snapshot, taken in
// stream order right after the frame's capture).
__global__ void k_snapshot_ctl(const Ctl* __restrict__ ctl, Ctl* __restrict__ out) {
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(ctl);
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(out);
  for (int i = threadIdx.x; i < static_cast<int>(sizeof(Ctl) / 8); i += blockDim.x) dst[i] = src[i];
}

int launch_snapshot_ctl(DeviceSim& s, Ctl* out) {
  k_snapshot_ctl<<<1, 64, 0, s.stream>>>(s.ctl, out);
  s.kernel_launches += 1;
  return 1;
}

// Phase-API pieces (engine.cpp:254-286).
__global__ void k_gel_boundary(double* __restrict__ v, const uint8_t* __restrict__ tag, int64_t n,
                               int64_t n_el, Ctl* ctl) {
  if (stale(ctl, ctl->substep)) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p < n_el && tag[p] == kElastomerBottom) {
    v[p] = 0.0;
    v[n + p] = 0.0;
    v[2 * n + p] = 0.0;
  }
}

__global__ void k_gel_advect(double* __restrict__ x, const double* __restrict__ v, int64_t n,
                             int64_t n_el, Ctl* ctl, Geometry g) {
  if (stale_block(ctl, ctl->substep)) return;
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n_el;
  double px0 = 0, px1 = 0, px2 = 0, v2 = 0;
  if (active) {
    const double v0 = v[p], v1 = v[n + p], vz = v[2 * n + p];
    px0 = advance(x[p], g.dt, v0);
    px1 = advance(x[n + p], g.dt, v1);
    px2 = advance(x[2 * n + p], g.dt, vz);
    x[p] = px0;
    x[n + p] = px1;
    x[2 * n + p] = px2;
    v2 = v0 * v0 + v1 * v1 + vz * vz;
  }
  const int sl = ctl->substep & 1;
  reduce_motion(&ctl->max_v2[sl], ctl->bb_lo[sl], ctl->bb_hi[sl], active, v2, px0, px1, px2);
}

// Indenter advect in phase mode with its current (possibly non-uniform)
// velocity; the indenter bbox is recomputed afterwards by k_bbox.
template <bool kUniform>
__global__ void k_ind_advect(double* __restrict__ x, const double* __restrict__ v, int64_t n,
                             int64_t n_el, Ctl* ctl, Geometry g) {
  if (stale(ctl, ctl->substep)) return;
  const int64_t p = n_el + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool active = p < n;
  double v2 = 0;
  if (active) {
    const double v0 = kUniform ? ctl->ind_v[0] : v[p];
    const double v1 = kUniform ? ctl->ind_v[1] : v[n + p];
    const double vz = kUniform ? ctl->ind_v[2] : v[2 * n + p];
    x[p] = advance(x[p], g.dt, v0);
    x[n + p] = advance(x[n + p], g.dt, v1);
    x[2 * n + p] = advance(x[2 * n + p], g.dt, vz);
    v2 = v0 * v0 + v1 * v1 + vz * vz;
  }
  const double m = warp_max(active ? v2 : 0.0);
  if ((threadIdx.x & 31) == 0 && m > 0.0)
    atomicMax(&ctl->max_v2[ctl->substep & 1],
              static_cast<unsigned long long>(__double_as_longlong(m)));
}

__global__ void k_ind_boundary(Ctl* ctl) {
  if (stale(ctl, ctl->substep)) return;
  for (int a = 0; a < 3; ++a) ctl->ind_v[a] = ctl->vind[a];
}

// End of particle_to_grid in phase mode: publish min_det_f (engine.cpp:177).
__global__ void k_p2g_done(Ctl* ctl) {
  const int s = ctl->substep;
  if (stale(ctl, s)) return;
  ctl->mi_last = s;  // the M_I buffer tg_download_grid reads
  ctl->diag_min_det_f = order_val(ctl->min_detf[s & 1]);
  ctl->min_detf[s & 1] = order_key(1.0);
}

// Copies a node box [lo, hi) into dense staging buffers (tg_download_grid):
// Grid::mass / momentum as the reference holds them (elastomer + indenter).
__global__ void k_gather_box(NodeBuf mp, const double* __restrict__ mi, VelBuf vel,
                             const Ctl* ctl, Geometry g,
                             double m_ind, int3 lo, int3 hi, double* __restrict__ mass,
                             double* __restrict__ mom, double* __restrict__ velo) {
  const int ny = hi.y - lo.y, nz = hi.z - lo.z;
  const int64_t total = static_cast<int64_t>(hi.x - lo.x) * ny * nz;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int k = lo.z + static_cast<int>(t % nz);
    const int64_t r = t / nz;
    const int j = lo.y + static_cast<int>(r % ny);
    const int i = lo.x + static_cast<int>(r / ny);
    // Grid nodes outside the reference's active window are zero there
    // (zero_grid cleared them when the window moved, engine.cpp:72-83)
    const bool in_win = i >= ctl->ref_lo[0] && i < ctl->ref_hi[0] && j >= ctl->ref_lo[1] &&
                        j < ctl->ref_hi[1] && k >= ctl->ref_lo[2] && k < ctl->ref_hi[2];
    const bool alloc = i >= g.ga_lo[0] && i < g.ga_lo[0] + g.ga_dim[0] && j >= g.ga_lo[1] &&
                       j < g.ga_lo[1] + g.ga_dim[1] && k >= g.ga_lo[2] &&
                       k < g.ga_lo[2] + g.ga_dim[2];
    if (!in_win || !alloc) {
      mass[t] = 0.0;
      for (int c = 0; c < 3; ++c) mom[3 * t + c] = velo[3 * t + c] = 0.0;
      continue;
    }
    const size_t nd = node_index(g, i, j, k);
    const double2 qa = mp.lo[nd], qb = mp.hi[nd];
    double4 q = make_double4(qa.x, qa.y, qb.x, qb.y);
    double wi = mi[static_cast<size_t>(ctl->mi_last & 1) * g.mi_stride + nd];
    if (g.det) {
      q = make_double4(from_fixed(qa.x, g.fx_inv), from_fixed(qa.y, g.fx_inv),
                       from_fixed(qb.x, g.fx_inv), from_fixed(qb.y, g.fx_inv));
      wi = from_fixed(wi, g.fxi_inv);
    }
    const double M = __dmul_rn(wi, m_ind);
    const double2 ua = vel.xy[nd];
    const double4 u = make_double4(ua.x, ua.y, vel.z[nd], 0.0);
    // the node sums exactly as grid_update forms them (node_velocity)
    const bool ind = wi != 0.0;
    mass[t] = ind ? __dadd_rn(q.x, M) : q.x;
    mom[3 * t] = ind ? __dadd_rn(q.y, __dmul_rn(M, ctl->ind_v[0])) : q.y;
    mom[3 * t + 1] = ind ? __dadd_rn(q.z, __dmul_rn(M, ctl->ind_v[1])) : q.z;
    mom[3 * t + 2] = ind ? __dadd_rn(q.w, __dmul_rn(M, ctl->ind_v[2])) : q.w;
    velo[3 * t] = u.x;
    velo[3 * t + 1] = u.y;
    velo[3 * t + 2] = u.z;
  }
}

// ---------------------------------------------------------------------------
// Launch helpers (host).
// ---------------------------------------------------------------------------

namespace {
// cudaLaunchKernelEx with programmatic stream serialization (see pdl_wait).
template <typename... KArgs, typename... Args>
void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

constexpr int kThreads = 256;
constexpr size_t kTileSmem = sizeof(P2GTile);
static_assert(sizeof(ColSmem) <= sizeof(P2GTile), "indenter blocks reuse the tile's shared memory");
static_assert(kGelThreads == kColWarps * 32, "indenter blocks of the elastomer kernel: 8 warps");
constexpr size_t kIndSmem = sizeof(IndSmem);

inline unsigned blocks_for(int64_t n) {
  const int64_t b = (n + kThreads - 1) / kThreads;
  return static_cast<unsigned>(b > 0 ? b : 1);
}
inline unsigned window_blocks(int sms) { return static_cast<unsigned>(sms * 8); }

GelMap gel_map(const DeviceSim& s) {
  GelMap M;
  for (int a = 0; a < 3; ++a) {
    M.lat[a] = s.lat[a];
    M.tile[a] = s.tile[a];
    M.tiles[a] = s.tiles[a];
  }
  return M;
}

unsigned gel_blocks(const DeviceSim& s);
}  // namespace
unsigned gel_block_count(const DeviceSim& s) { return gel_blocks(s); }
namespace {
unsigned gel_blocks(const DeviceSim& s) {
  if (s.lat[0] > 0) return static_cast<unsigned>(s.tiles[0] * s.tiles[1]);
  return static_cast<unsigned>((s.n_el + kGelThreads - 1) / kGelThreads);
}

// Dynamic shared-memory opt-ins are per device (per primary context): set
// once for every device a handle is created on (configure_device, called by
// tg_create after the device is selected), never lazily during a graph
// capture. A mutex guards the per-device flags (handles on different devices
// may be created from different threads).
std::mutex g_cfg_mutex;
bool g_cfg_done[64] = {};
}  // namespace

int configure_device(int device) {
  std::lock_guard<std::mutex> lock(g_cfg_mutex);
  if (device < 0 || device >= 64) return 1;
  if (g_cfg_done[device]) return 0;
  int cur = -1;
  cudaGetDevice(&cur);
  cudaSetDevice(device);
  const int tile = static_cast<int>(kTileSmem);
  cudaError_t e = cudaSuccess;
  auto set = [&](const void* f, int bytes) {
    const cudaError_t r = cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (r != cudaSuccess && e == cudaSuccess) e = r;
  };
  set(reinterpret_cast<const void*>(k_p2g_gel_tile), tile);
  set(reinterpret_cast<const void*>(k_g2p2g_gel<true, true, true, 0>), tile);
  set(reinterpret_cast<const void*>(k_g2p2g_gel<true, true, true, 1>), tile);
  set(reinterpret_cast<const void*>(k_ind_move_p2g<false, true>), static_cast<int>(kIndSmem));
  set(reinterpret_cast<const void*>(k_ind_move_p2g<true, true>), static_cast<int>(kIndSmem));
  set(reinterpret_cast<const void*>(k_ind_cols<true>), static_cast<int>(sizeof(ColSmemT<kWalkWarps>)));
  set(reinterpret_cast<const void*>(k_ind_cols<false>), static_cast<int>(sizeof(ColSmemT<kWalkWarps>)));
  if (cur >= 0 && cur != device) cudaSetDevice(cur);
  if (e != cudaSuccess) return 2;
  g_cfg_done[device] = true;
  return 0;
}
namespace {
}  // namespace

// Chooses the lattice-block CTA tiling of the elastomer (engine.cuh).
void configure_gel_tiling(DeviceSim& s, int nx, int ny, int nz) {
  if (nx <= 0 || ny <= 0 || nz <= 0 || static_cast<int64_t>(nx) * ny * nz != s.n_el ||
      nz > kGelThreads) {
    s.lat[0] = s.lat[1] = s.lat[2] = 0;
    return;
  }
  s.lat[0] = nx;
  s.lat[1] = ny;
  s.lat[2] = nz;
  const int cols = kGelThreads / nz > 0 ? kGelThreads / nz : 1;
  int ti = 1;
  while ((ti + 1) * (ti + 1) <= cols) ++ti;
  const int tj = cols / ti > 0 ? cols / ti : 1;
  s.tile[0] = ti;
  s.tile[1] = tj;
  s.tile[2] = nz;
  s.tiles[0] = (nx + ti - 1) / ti;
  s.tiles[1] = (ny + tj - 1) / tj;
  s.tiles[2] = 1;
}

// Lane order of the lattice-block CTAs: within each warp, the particles of
// the warp's 32 lattice slots are stored in an order dealt by the residue
// mod 8 of their tile node offsets, so a quarter-warp's 128-bit tile
// accesses spread over the shared-memory banks. A 128-bit shared access is
// served a quarter-warp (8 lanes) at a time; in lattice order a quarter-warp
// holds 8 consecutive particles of a column whose z bases, 1.55 cells
// apart, span more than the 8 bank slots, so its tile accesses took ~2x the
// ideal wavefronts (ncu). Slots are sorted by the residue at the initial
// positions (tile box and pitch as the kernel derives them) and dealt round
// robin to the quarter-warps; the result permutes the elastomer part of
// DeviceSim::perm within each warp's slots, so the warp's particles, and the
// memory sectors it touches, stay the same. Any order is correct: the node
// sums of the tile do not depend on it (the phases fix the order per node).
void permute_gel_lanes(DeviceSim& s, const double* x_in) {
  if (s.lat[0] <= 0 || !x_in) return;
  int mode = 2;  // 0: lattice order, 1: dealt within each warp, 2: across the CTA
  if (const char* e = std::getenv("TACCHI_GEL_LANES")) mode = std::atoi(e);
  if (mode <= 0) return;
  const int ctas = s.tiles[0] * s.tiles[1];
  const Geometry& g = s.geo;
  auto base_of_x = [&](double x, int a) {
    return static_cast<int>(std::floor((x - g.origin[a]) * g.inv_dx - 0.5));
  };
  const std::vector<int64_t> perm0(s.perm.begin(), s.perm.begin() + s.n_el);
  for (int cta = 0; cta < ctas; ++cta) {
    int b[kGelThreads][3];
    int64_t slot[kGelThreads];  // lattice (storage) index of thread t's slot, -1: none
    int lo[3] = {INT_MAX, INT_MAX, INT_MAX}, hi[3] = {INT_MIN, INT_MIN, INT_MIN};
    for (int t = 0; t < kGelThreads; ++t) {
      const int per_col = s.tile[2];
      const int kk = t % per_col, jj = (t / per_col) % s.tile[1], ii = t / (per_col * s.tile[1]);
      const int bj = cta % s.tiles[1], bi = cta / s.tiles[1];
      const int i = bi * s.tile[0] + ii, j = bj * s.tile[1] + jj;
      const bool act = ii < s.tile[0] && i < s.lat[0] && j < s.lat[1] && kk < s.lat[2];
      slot[t] = act ? (static_cast<int64_t>(i) * s.lat[1] + j) * s.lat[2] + kk : -1;
      if (!act) continue;
      const int64_t r = perm0[slot[t]];
      for (int a = 0; a < 3; ++a) {
        b[t][a] = base_of_x(x_in[3 * r + a], a);
        lo[a] = std::min(lo[a], b[t][a]);
        hi[a] = std::max(hi[a], b[t][a]);
      }
    }
    const int d1 = hi[1] - lo[1] + 3 + kRowPad, pitch = tile_pitch(hi[2] - lo[2] + 3);
    auto residue = [&](int t) {
      const long e = (static_cast<long>(b[t][0] - lo[0]) * d1 + (b[t][1] - lo[1])) * pitch +
                     (b[t][2] - lo[2]);
      return static_cast<int>(e & 7);
    };
    if (mode == 2) {
      // across the CTA: the slots stay where they are (each warp reads the
      // same memory), the particles are dealt to the 32 quarter-warps in
      // residue order, one per quarter in turn, skipping full quarters
      std::vector<int> order;
      std::vector<int> quarter_slots[kGelThreads / 8];
      for (int t = 0; t < kGelThreads; ++t)
        if (slot[t] >= 0) {
          order.push_back(t);
          quarter_slots[t / 8].push_back(t);
        }
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return residue(x) < residue(y); });
      std::vector<size_t> fill(kGelThreads / 8, 0);
      std::vector<int> src(kGelThreads, -1);  // thread -> the thread slot whose particle it takes
      int q = 0;
      for (int t : order) {
        while (fill[q] >= quarter_slots[q].size()) q = (q + 1) % (kGelThreads / 8);
        src[quarter_slots[q][fill[q]++]] = t;
        q = (q + 1) % (kGelThreads / 8);
      }
      // Keep the lattice order where it already spreads the banks (a gel
      // spacing below one cell, config 2b: 8 consecutive z particles span
      // fewer than 8 nodes): the bank cost of an order is the sum over
      // quarter-warps of the largest number of distinct tile nodes sharing a
      // 16-byte slot (the same for every tile phase: the phases shift all
      // lanes' nodes by one offset).
      auto cost = [&](auto&& who) {
        long c = 0;
        for (int q4 = 0; q4 < kGelThreads / 8; ++q4) {
          long node[8];
          int cnt = 0;
          for (int l = 0; l < 8; ++l) {
            const int t = who(8 * q4 + l);
            if (t < 0) continue;
            node[cnt++] = (static_cast<long>(b[t][0] - lo[0]) * d1 + (b[t][1] - lo[1])) * pitch +
                          (b[t][2] - lo[2]);
          }
          int worst = 0;
          for (int r = 0; r < 8; ++r) {
            int m = 0;
            for (int i = 0; i < cnt; ++i) {
              if ((node[i] & 7) != r) continue;
              bool dup = false;
              for (int k = 0; k < i; ++k) dup = dup || node[k] == node[i];
              m += dup ? 0 : 1;
            }
            worst = std::max(worst, m);
          }
          c += worst;
        }
        return c;
      };
      const long c_lat = cost([&](int t) { return slot[t] >= 0 ? t : -1; });
      const long c_deal = cost([&](int t) { return src[t]; });
      if (10 * c_deal < 9 * c_lat)
        for (int t = 0; t < kGelThreads; ++t)
          if (src[t] >= 0) s.perm[slot[t]] = perm0[slot[src[t]]];
      continue;
    }
    for (int w = 0; w < kGelThreads / 32; ++w) {
      std::vector<int> used;
      for (int l = 0; l < 32; ++l)
        if (slot[32 * w + l] >= 0) used.push_back(32 * w + l);
      if (used.size() < 2) continue;
      std::vector<int> order = used;
      std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return residue(x) < residue(y); });
      // the k-th particle in residue order goes to quarter k % 4; the warp's
      // occupied slots (in lane order) are refilled quarter by quarter
      std::vector<int> dealt;
      for (int q4 = 0; q4 < 4; ++q4)
        for (size_t k = q4; k < order.size(); k += 4) dealt.push_back(order[k]);
      // lanes of the warp with a slot, in order: lane u gets the particle of
      // slot dealt[u'] (u' its rank among the occupied lanes)
      for (size_t u = 0; u < used.size(); ++u) s.perm[slot[used[u]]] = perm0[slot[dealt[u]]];
    }
  }
}

int launch_reset(DeviceSim& s, int mask) {
  k_reset<<<1, 1, 0, s.stream>>>(s.ctl, mask);
  s.kernel_launches += 1;
  return 1;
}

// zero_grid's window from the current positions (both bboxes recomputed).
int launch_window(DeviceSim& s) {
  int k = launch_reset(s, kResetMotion | kResetIndBox | kResetDetF);
  if (s.n_el > 0) {
    k_bbox<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.x, s.n, 0, s.n_el, s.ctl, 0, 1);
    ++k;
  }
  if (s.n_ind > 0) {
    k_bbox<<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.n, s.n_el, s.n, s.ctl, 1, 1);
    ++k;
  }
  k_finalize<<<1, 32, 0, s.stream>>>(s.ctl, s.geo, kFinWindow, FixArgs{});
  s.kernel_launches += k;  // reset counted in launch_reset
  return k + 1;
}

int launch_clear(DeviceSim& s, int sms) {
  k_clear<<<window_blocks(sms), kThreads, 0, s.stream>>>(s.grid_mp, s.grid_mi, s.grid_v, s.ctl,
                                                        s.geo);
  s.kernel_launches += 1;
  s.grid_dirty = false;
  return 1;
}

int launch_p2g_gel(DeviceSim& s) {
  if (s.n_el <= 0) return 0;
  k_p2g_gel_tile<<<gel_blocks(s), kGelThreads, kTileSmem, s.stream>>>(
      s.x, s.v, s.C, s.F, s.n, s.n_el, gel_map(s), s.ctl, s.geo, s.grid_mp, s.m_el, s.vol_el);
  s.kernel_launches += 1;
  return 1;
}

inline unsigned ind_blocks(const DeviceSim& s) {
  const int64_t seg = static_cast<int64_t>(kIndThreads) * kIndK;
  return static_cast<unsigned>((s.n_ind + seg - 1) / seg);
}

int launch_p2g_ind(DeviceSim& s) {
  if (s.n_ind <= 0) return 0;
  if (s.ind_v_uniform)
    k_ind_move_p2g<false, true><<<ind_blocks(s), kIndThreads, kIndSmem, s.stream>>>(
        s.x, s.n, s.n_el, s.ctl, s.geo, s.grid_mi);
  else
    k_p2g_ind_direct<<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el, s.ctl,
                                                                     s.geo, s.grid_mp, s.m_ind);
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
  s.grid_dirty = true;
  return k;
}

int launch_grid_update(DeviceSim& s, int sms, bool zero) {
  if (zero)
    launch_pdl(k_grid_update_boxes, dim3(static_cast<unsigned>(sms * s.geo.gu_bps)), dim3(kThreads), 0, s.stream,
               s.grid_mp, s.grid_mi, s.grid_v, s.ctl, s.geo, s.m_ind);
  else
    k_grid_update_window<<<window_blocks(sms), kThreads, 0, s.stream>>>(
        s.grid_mp, s.grid_mi, s.grid_v, s.ctl, s.geo, s.m_ind);
  s.kernel_launches += 1;
  return 1;
}

// G2P + boundary + advect for the elastomer, with the look-ahead scatter.
int launch_g2p2g_gel(DeviceSim& s, bool lookahead, bool with_indenter) {
  if (s.n_el <= 0) return 0;
  IndArgs ia{};
  unsigned extra = 0;
  if (with_indenter) {  // the indenter's look-ahead column walks ride along
    // (TACCHI_AB_NO_WALKS: A/B timing only, the indenter then scatters nothing)
    extra = s.ab_no_walks ? 0u : static_cast<unsigned>((s.n_cols + kColWarps - 1) / kColWarps);
    const int gel = static_cast<int>(gel_blocks(s));
    const bool ind_first = s.geo.ind_first != 0;
    ia = IndArgs{s.col_start, s.ind_moves, s.grid_mi, s.n_cols, gel,
                 ind_first ? static_cast<int>(extra) : 0, ind_first ? 0 : gel};
    s.ind_v_uniform = true;
  }
  if (lookahead)
    launch_pdl(s.geo.det ? k_g2p2g_gel<true, true, true, 1> : k_g2p2g_gel<true, true, true, 0>,
               dim3(gel_blocks(s) + extra), dim3(kGelThreads), kTileSmem, s.stream, s.x, s.v, s.C,
               s.F, s.tag, s.n, s.n_el, gel_map(s), s.ctl, s.geo, s.grid_v, s.grid_mp, s.m_el,
               s.vol_el, ia);
  else
    k_g2p2g_gel<true, true, false><<<gel_blocks(s), kGelThreads, 0, s.stream>>>(
        s.x, s.v, s.C, s.F, s.tag, s.n, s.n_el, gel_map(s), s.ctl, s.geo, s.grid_v, s.grid_mp,
        s.m_el, s.vol_el, IndArgs{});
  s.kernel_launches += 1;
  return 1;
}

int launch_ind_move(DeviceSim& s, bool lookahead) {
  if (s.n_ind <= 0) return 0;
  if (lookahead)
    k_ind_move_p2g<true, true><<<ind_blocks(s), kIndThreads, kIndSmem, s.stream>>>(
        s.x, s.n, s.n_el, s.ctl, s.geo, s.grid_mi);
  else
    k_ind_move_p2g<true, false><<<ind_blocks(s), kIndThreads, 0, s.stream>>>(
        s.x, s.n, s.n_el, s.ctl, s.geo, s.grid_mi);
  s.ind_v_uniform = true;
  s.kernel_launches += 1;
  return 1;
}

constexpr size_t kColSmem = sizeof(ColSmemT<kWalkWarps>);  // the walk kernel of its own

int launch_chain_begin(DeviceSim& s) {
  k_chain_begin<<<1, 1, 0, s.stream>>>(s.ctl);
  s.kernel_launches += 1;
  return 1;
}

// Indenter scatter of the step path: standalone (first substep of a call,
// positions as they are) or fused with this substep's advect (look-ahead).
int launch_ind_cols(DeviceSim& s, bool move) {
  if (s.n_ind <= 0 || s.n_cols <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>((s.n_cols + kWalkWarps - 1) / kWalkWarps);
  if (move)
    launch_pdl(k_ind_cols<true>, dim3(blocks), dim3(kWalkWarps * 32), kColSmem, s.stream, s.x,
               s.n, s.n_el, static_cast<const int64_t*>(s.col_start), s.n_cols, s.ind_moves,
               s.ctl, s.geo, s.grid_mi, 1);
  else
    k_ind_cols<false><<<blocks, kWalkWarps * 32, kColSmem, s.stream>>>(
        s.x, s.n, s.n_el, s.col_start, s.n_cols, s.ind_moves, s.ctl, s.geo, s.grid_mi, 0);
  s.ind_v_uniform = true;
  s.kernel_launches += 1;
  return 1;
}

// The look-ahead walks as a kernel of their own on `st` (the forked walk
// stream of the substep plan): the previous finalize's elastomer box widened
// by one node, completed by this substep's finalize if the elastomer leaves it.
int launch_ind_walks_on(DeviceSim& s, cudaStream_t st) {
  if (s.n_ind <= 0 || s.n_cols <= 0) return 0;
  const unsigned blocks = static_cast<unsigned>((s.n_cols + kWalkWarps - 1) / kWalkWarps);
  k_ind_cols<true><<<blocks, kWalkWarps * 32, kColSmem, st>>>(
      s.x, s.n, s.n_el, s.col_start, s.n_cols, s.ind_moves, s.ctl, s.geo, s.grid_mi, 2);
  s.ind_v_uniform = true;
  s.kernel_launches += 1;
  return 1;
}

int launch_ind_catchup(DeviceSim& s) {
  if (s.n_ind <= 0) return 0;
  launch_pdl(k_ind_catchup, dim3(blocks_for(s.n_ind)), dim3(kThreads), 0, s.stream, s.x, s.n,
             s.n_el, s.ind_moves, s.ctl, s.geo);
  s.kernel_launches += 1;
  return 1;
}

int launch_finalize_step(DeviceSim& s, bool walk_fix) {
  const int mode = kFinDiag | kFinAdvect | kFinWindow | (s.n_ind > 0 ? kFinIndShift : 0) |
                   (walk_fix ? kFinWalkFix : 0);
  const FixArgs fa{s.x, s.n, s.n_el, s.col_start, s.n_cols, s.ind_moves, s.grid_mi};
  launch_pdl(k_finalize, dim3(1), dim3(walk_fix ? 256 : 32), 0, s.stream, s.ctl, s.geo, mode, fa);
  s.kernel_launches += 1;
  return 1;
}

int launch_phase_g2p(DeviceSim& s) {
  if (s.n_el <= 0) return 0;
  k_g2p2g_gel<false, false, false><<<gel_blocks(s), kGelThreads, 0, s.stream>>>(
      s.x, s.v, s.C, s.F, s.tag, s.n, s.n_el, gel_map(s), s.ctl, s.geo, s.grid_v, s.grid_mp,
      s.m_el, s.vol_el, IndArgs{});
  s.kernel_launches += 1;
  return 1;
}

int launch_phase_boundary(DeviceSim& s) {
  int k = 0;
  if (s.n_el > 0) {
    k_gel_boundary<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.v, s.tag, s.n, s.n_el, s.ctl);
    ++k;
  }
  if (s.n_ind > 0) {
    k_ind_boundary<<<1, 1, 0, s.stream>>>(s.ctl);
    s.ind_v_uniform = true;
    ++k;
  }
  s.kernel_launches += k;
  return k;
}

// advect (engine.cpp:268-286) in phase mode: move, recompute the indenter box,
// then finalize's in_range check.
int launch_phase_advect(DeviceSim& s) {
  int k = 0;
  if (s.n_el > 0) {
    k_gel_advect<<<blocks_for(s.n_el), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el, s.ctl,
                                                                s.geo);
    ++k;
  }
  if (s.n_ind > 0) {
    if (s.ind_v_uniform)
      k_ind_advect<true><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el,
                                                                        s.ctl, s.geo);
    else
      k_ind_advect<false><<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.v, s.n, s.n_el,
                                                                         s.ctl, s.geo);
    k_reset<<<1, 1, 0, s.stream>>>(s.ctl, kResetIndBox);
    k_bbox<<<blocks_for(s.n_ind), kThreads, 0, s.stream>>>(s.x, s.n, s.n_el, s.n, s.ctl, 1, 0);
    k += 3;
  }
  k_finalize<<<1, 32, 0, s.stream>>>(s.ctl, s.geo, kFinAdvect, FixArgs{});
  ++k;
  s.kernel_launches += k;
  return k;
}

int launch_gather_box(DeviceSim& s, const int lo[3], const int hi[3], double* mass, double* mom,
                      double* vel) {
  k_gather_box<<<1024, kThreads, 0, s.stream>>>(s.grid_mp, s.grid_mi, s.grid_v, s.ctl, s.geo,
                                                s.m_ind, make_int3(lo[0], lo[1], lo[2]),
                                                make_int3(hi[0], hi[1], hi[2]), mass, mom, vel);
  s.kernel_launches += 1;
  return 1;
}

}  // namespace tacchi_b200

// ---------------------------------------------------------------------------
// Instrumentation: the material functions the P2G kernels call, on a batch of
// deformation gradients (tg_polar; known-answer tests of material.cpp:18-89,
// including the SVD fallback the Newton iteration reaches only for
// pathological F).
// ---------------------------------------------------------------------------
namespace tacchi_b200 {
__global__ void k_polar(const double* __restrict__ F, int64_t n, int mode, double mu, double lambda,
                        double* __restrict__ R, double* __restrict__ S) {
  const int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (p >= n) return;
  double f[9], r[9];
  for (int i = 0; i < 9; ++i) f[i] = F[9 * p + i];
  if (mode == 1) polar_rotation_svd(f, r);
  else polar_rotation(f, r);
  for (int i = 0; i < 9; ++i) R[9 * p + i] = r[i];
  if (S) {
    double st[9];
    corotated_stress(f, r, det3(f), mu, lambda, st);
    for (int i = 0; i < 9; ++i) S[9 * p + i] = st[i];
  }
}
int check_device_public(int device);
int fail(int code, const std::string& msg);
}  // namespace tacchi_b200

extern "C" int tg_polar(int device, const double* F, int64_t n, int mode, double youngs_modulus,
                        double poisson_ratio, double* R, double* S) {
  using namespace tacchi_b200;
  if (!F || !R || n < 0 || (mode != 0 && mode != 1))
    return fail(TG_ERR_INVALID_ARGUMENT, "tg_polar: bad argument");
  int rc = check_device_public(device);
  if (rc) return rc;
  if (n == 0) return TG_OK;
  const double mu = youngs_modulus / (2.0 * (1.0 + poisson_ratio));  // material.hpp:14-18
  const double lambda =
      youngs_modulus * poisson_ratio / ((1.0 + poisson_ratio) * (1.0 - 2.0 * poisson_ratio));
  double *dF = nullptr, *dR = nullptr, *dS = nullptr;
  const size_t bytes = static_cast<size_t>(n) * 9 * sizeof(double);
  cudaError_t e = cudaMalloc(&dF, bytes);
  if (e == cudaSuccess) e = cudaMalloc(&dR, bytes);
  if (e == cudaSuccess && S) e = cudaMalloc(&dS, bytes);
  if (e == cudaSuccess) e = cudaMemcpy(dF, F, bytes, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    k_polar<<<static_cast<unsigned>((n + 127) / 128), 128>>>(dF, n, mode, mu, lambda, dR, dS);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpy(R, dR, bytes, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess && S) e = cudaMemcpy(S, dS, bytes, cudaMemcpyDeviceToHost);
  cudaFree(dF);
  cudaFree(dR);
  cudaFree(dS);
  return e == cudaSuccess ? TG_OK : fail(TG_ERR_CUDA, std::string("tg_polar: ") + cudaGetErrorString(e));
}

#ifdef TACCHI_TRACE
// Diagnostic builds only: copies the elastomer kernel's per-CTA stage marks.
extern "C" int tg_debug_trace(unsigned long long* out, int n_ctas) {
  if (n_ctas > 16384) n_ctas = 16384;
  return cudaMemcpyFromSymbol(out, tacchi_b200::g_trace, sizeof(unsigned long long) * 16 * n_ctas) ==
                 cudaSuccess
             ? n_ctas
             : -1;
}
#endif
