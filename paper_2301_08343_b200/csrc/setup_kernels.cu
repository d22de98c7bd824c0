// Episode setup on the device: the indenter cloud's
// rejection sampling (geo::generate_shape_cloud, shapes.cpp:231-249) and
// its placement (place_for_press, scene_builder.cpp:48-61) for sm_100a,
// bit-identical to the host restatement (host_setup.cpp) and so to the
// reference.
//
//   k_mt_stream   std::mt19937_64's output stream: one CTA keeps the 312-word
//                 state in shared memory and twists it in two parallel halves
//                 (words 0-155 read only old words; 156-311 read the new
//                 0-155), then tempers all 312 at once.
//   k_candidates  candidate i takes words 3i, 3i+1, 3i+2 as the 53-bit
//                 uniforms of x, y, z (lo + span u, mm), tests the shape, and
//                 counts accepted candidates per block.
//   k_compact     writes the accepted points (m) in stream order at the
//                 blocks' exclusive offsets (block scan of the counts).
//   k_place       place_indenter's rotation about z / translation to the
//                 press position, with the bbox of the rotated cloud reduced
//                 exactly (min / max of order keys).
// Every arithmetic operation is spelled with a round-to-nearest intrinsic (no
// FMA contraction), as the host code is compiled with -ffp-contract=off.
// The subsample (particle_set.cpp:60-90) is a sequential partial
// Fisher-Yates over the same kind of stream: its index draw stays on the
// host (1e5 swaps), the gather of the chosen points runs here.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <random>
#include <string>
#include <vector>

#include "host_config.hpp"
#include "mpm_device.cuh"
#include "setup_shapes.h"
#include "tacchi_cuda.h"

namespace tacchi_b200 {

int fail(int code, const std::string& msg);
namespace host {
bool shape_table(const std::string& name, ShapeTable& t);
}

namespace {

constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kMtA = 0xB5026F5AA96619E9ull;
constexpr unsigned long long kUpper = 0xFFFFFFFF80000000ull, kLower = 0x7FFFFFFFull;

__device__ __forceinline__ unsigned long long mt_temper(unsigned long long y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  y ^= y >> 43;
  return y;
}

// `blocks` twists of the state (kept in `state` between launches), each
// producing 312 tempered words at out[312 b + k].
__global__ void __launch_bounds__(kMtN) k_mt_stream(unsigned long long* __restrict__ state,
                                                    unsigned long long* __restrict__ out,
                                                    int blocks) {
  __shared__ unsigned long long mt[kMtN];
  const int k = threadIdx.x;
  mt[k] = state[k];
  __syncthreads();
  for (int b = 0; b < blocks; ++b) {
    // words 0..155: mt[k+1] and mt[k+156] are still the old ones
    unsigned long long v = 0;
    if (k < kMtM) {
      const unsigned long long y = (mt[k] & kUpper) | (mt[k + 1] & kLower);
      v = mt[k + kMtM] ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
    }
    __syncthreads();
    if (k < kMtM) mt[k] = v;
    __syncthreads();
    // words 156..311: mt[k-156] is new, mt[k+1] old (mt[0] new for k = 311)
    if (k >= kMtM) {
      const unsigned long long y = (mt[k] & kUpper) | (mt[(k + 1) % kMtN] & kLower);
      v = mt[k - kMtM] ^ (y >> 1) ^ ((y & 1ull) ? kMtA : 0ull);
    }
    __syncthreads();
    if (k >= kMtM) mt[k] = v;
    __syncthreads();
    out[static_cast<size_t>(b) * kMtN + k] = mt_temper(mt[k]);
  }
  state[k] = mt[k];
}

__device__ __forceinline__ double m_(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double a_(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double s_(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double d_(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double sq(double v) { return m_(v, v); }
__device__ __forceinline__ double r2(double x, double y) { return a_(m_(x, x), m_(y, y)); }
__device__ __forceinline__ bool disk(double x, double y, double r) { return r2(x, y) <= m_(r, r); }
__device__ __forceinline__ bool rect(double x, double y, double hx, double hy) {
  return fabs(x) <= hx && fabs(y) <= hy;
}

// The shape predicates of shapes.cpp:79-206 (host_setup.cpp make_shape).
__device__ bool inside(const ShapeTable& t, double x, double y, double z) {
  constexpr double kPi = 3.14159265358979323846;
  switch (t.id) {
    case kShSphere: return a_(r2(x, y), sq(s_(z, 3.0))) <= 9.0;
    case kShSphere2: return a_(r2(x, y), sq(s_(z, 2.0))) <= 4.0;
    case kShCone: return r2(x, y) <= m_(z, z) && z <= 3.5;
    case kShCylinder: return disk(x, y, 3.0);
    case kShCylinderShell: {
      const double q = r2(x, y);
      return q <= 9.0 && q >= sq(2.1);
    }
    case kShCylinderSide: return a_(sq(x), sq(s_(z, 2.0))) <= 4.0;
    case kShCurvedSurface: return z >= d_(r2(x, y), 24.0);
    case kShFlatSlab: return true;
    case kShDotIn: return disk(x, y, 3.5) && !(disk(x, y, 0.7) && z < 0.9);
    case kShDots: {
      if (z >= 1.0) return rect(x, y, 3.5, 3.5);
      const double gx = m_(round(d_(x, 2.2)), 2.2);
      const double gy = m_(round(d_(y, 2.2)), 2.2);
      return fabs(gx) <= 2.3 && fabs(gy) <= 2.3 && disk(s_(x, gx), s_(y, gy), 0.55);
    }
    case kShHexagon:
    case kShTriangle:
      for (int k = 0; k < t.n_planes; ++k)
        if (a_(m_(x, t.ca[k]), m_(y, t.sa[k])) > t.apothem) return false;
      return true;
    case kShPrism: return fabs(x) <= z && z <= 3.0;
    case kShLine: return rect(x, y, 0.6, 4.0);
    case kShParallelLines: {
      if (z >= 1.5) return rect(x, y, 3.4, 4.0);
      const double gx = m_(round(d_(x, 2.4)), 2.4);
      return fabs(gx) <= 2.5 && fabs(s_(x, gx)) <= 0.45 && fabs(y) <= 4.0;
    }
    case kShCrossLines:
      if (z >= 1.5) return rect(x, y, 4.0, 4.0);
      return (fabs(x) <= 0.45 || fabs(y) <= 0.45) && rect(x, y, 4.0, 4.0);
    case kShMoon: return disk(x, y, 3.0) && !disk(s_(x, 1.4), y, 2.4);
    case kShPacman: return disk(x, y, 3.0) && fabs(atan2(y, x)) > d_(kPi, 6.0);
    case kShTorus: {
      const double rho = __dsqrt_rn(r2(x, y));
      return a_(sq(s_(rho, 2.3)), sq(s_(z, 0.9))) <= sq(0.9);
    }
    case kShWave1:
      return z >= m_(0.5, a_(1.0, sin(d_(m_(m_(2.0, kPi), x), 2.7))));
    case kShRandom: {
      double h = 0.0;
      for (int i = 0; i < 28; ++i)
        h = a_(h, m_(t.amp[i],
                     exp(m_(-a_(sq(s_(x, t.bx[i])), sq(s_(y, t.by[i]))), t.inv_s2[i]))));
      return z >= fmin(h, 1.4);
    }
    default: return false;
  }
}

__device__ __forceinline__ double u53(unsigned long long w) {
  return static_cast<double>(w >> 11) * 0x1.0p-53;
}

constexpr int kCandThreads = 256;

// Candidate i of this chunk: flags its acceptance and counts per block.
__global__ void __launch_bounds__(kCandThreads) k_candidates(
    const unsigned long long* __restrict__ words, int64_t n_cand, ShapeTable t,
    uint8_t* __restrict__ flag, int* __restrict__ block_count) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kCandThreads + threadIdx.x;
  bool ok = false;
  if (i < n_cand) {
    const double x = a_(t.lo[0], m_(t.span[0], u53(words[3 * i])));
    const double y = a_(t.lo[1], m_(t.span[1], u53(words[3 * i + 1])));
    const double z = a_(t.lo[2], m_(t.span[2], u53(words[3 * i + 2])));
    ok = inside(t, x, y, z);
    flag[i] = ok;
  }
  const int c = __syncthreads_count(ok);
  if (threadIdx.x == 0) block_count[blockIdx.x] = c;
}

// Accepted candidates of block b go to out[offset[b] + rank], rank = the
// number of accepted candidates before them in the block; only the first
// `limit` accepted points of the stream are written (metres).
__global__ void __launch_bounds__(kCandThreads) k_compact(
    const unsigned long long* __restrict__ words, int64_t n_cand, ShapeTable t,
    const uint8_t* __restrict__ flag, const int64_t* __restrict__ offset, int64_t limit,
    double* __restrict__ out) {
  __shared__ int warp_tot[kCandThreads / 32];
  const int64_t i = static_cast<int64_t>(blockIdx.x) * kCandThreads + threadIdx.x;
  const bool ok = i < n_cand && flag[i];
  const unsigned bal = __ballot_sync(0xffffffffu, ok);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) warp_tot[warp] = __popc(bal);
  __syncthreads();
  int before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  const int64_t dst = offset[blockIdx.x] + before + __popc(bal & ((1u << lane) - 1));
  if (!ok || dst >= limit) return;
  const double x = a_(t.lo[0], m_(t.span[0], u53(words[3 * i])));
  const double y = a_(t.lo[1], m_(t.span[1], u53(words[3 * i + 1])));
  const double z = a_(t.lo[2], m_(t.span[2], u53(words[3 * i + 2])));
  out[3 * dst] = m_(x, 1e-3);
  out[3 * dst + 1] = m_(y, 1e-3);
  out[3 * dst + 2] = m_(z, 1e-3);
}

// subsample's gather: out[k] = in[idx[k]] (idx ascending, particle_set.cpp:84-89).
__global__ void k_gather_points(const double* __restrict__ in, const uint32_t* __restrict__ idx,
                                int64_t n, double* __restrict__ out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= n) return;
  const int64_t s = idx[k];
  out[3 * k] = in[3 * s];
  out[3 * k + 1] = in[3 * s + 1];
  out[3 * k + 2] = in[3 * s + 2];
}

// place_indenter (particle_set.cpp:92-102): x' = c x - s y + tx,
// y' = s x + c y + ty, z' = z + tz; optionally the bbox of the result
// (order keys, exact min / max) into box[6].
__global__ void k_place(const double* __restrict__ in, int64_t n, double c, double s, double tx,
                        double ty, double tz, double* __restrict__ out,
                        unsigned long long* __restrict__ box) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  double v[3] = {INFINITY, INFINITY, INFINITY}, w[3] = {-INFINITY, -INFINITY, -INFINITY};
  if (k < n) {
    const double px = in[3 * k], py = in[3 * k + 1], pz = in[3 * k + 2];
    const double x = a_(s_(m_(c, px), m_(s, py)), tx);
    const double y = a_(a_(m_(s, px), m_(c, py)), ty);
    const double z = a_(pz, tz);
    out[3 * k] = x;
    out[3 * k + 1] = y;
    out[3 * k + 2] = z;
    v[0] = w[0] = x;
    v[1] = w[1] = y;
    v[2] = w[2] = z;
  }
  if (!box) return;
  for (int a = 0; a < 3; ++a)
    for (int o = 16; o > 0; o >>= 1) {
      v[a] = fmin(v[a], __shfl_xor_sync(0xffffffffu, v[a], o));
      w[a] = fmax(w[a], __shfl_xor_sync(0xffffffffu, w[a], o));
    }
  if ((threadIdx.x & 31) == 0 && v[0] <= w[0])
    for (int a = 0; a < 3; ++a) {
      atomicMin(&box[a], order_key(v[a]));
      atomicMax(&box[3 + a], order_key(w[a]));
    }
}

// std::mt19937_64(seed)'s initial state (the seeding recurrence).
void mt_seed(uint64_t seed, unsigned long long* st) {
  st[0] = seed;
  for (int i = 1; i < kMtN; ++i)
    st[i] = 6364136223846793005ull * (st[i - 1] ^ (st[i - 1] >> 62)) + static_cast<uint64_t>(i);
}

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() { cudaFree(p); }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
  bool alloc(size_t bytes) { return cudaMalloc(&p, bytes) == cudaSuccess; }
};

#define SETUP_TRY(expr)                                                                      \
  do {                                                                                       \
    const cudaError_t _e = (expr);                                                           \
    if (_e != cudaSuccess) return fail(TG_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

}  // namespace

// generate_shape_cloud on `device` into `d_out` (device, n x 3 m): rejection
// sampling over chunks of the mt19937_64 stream until n points are accepted.
int device_shape_cloud(int device, const std::string& shape, int64_t n, uint64_t seed,
                       double* d_out) {
  ShapeTable t;
  if (!host::shape_table(shape, t)) return fail(TG_ERR_CONFIG, "unknown shape: " + shape);
  if (n <= 0) return TG_OK;
  SETUP_TRY(cudaSetDevice(device));
  constexpr int64_t kChunk = int64_t(1) << 21;  // candidates per chunk
  constexpr int kTwists = static_cast<int>((3 * kChunk + kMtN - 1) / kMtN);
  // a chunk's candidates: its words plus up to two carried, in triples
  const int64_t max_cand = (static_cast<int64_t>(kTwists) * kMtN + 2) / 3;
  const int blocks = static_cast<int>((max_cand + kCandThreads - 1) / kCandThreads);
  DevBuf state, words, flag, counts, offsets;
  if (!state.alloc(kMtN * 8) || !words.alloc(static_cast<size_t>(kTwists) * kMtN * 8) ||
      !flag.alloc(static_cast<size_t>(max_cand)) || !counts.alloc(blocks * sizeof(int)) ||
      !offsets.alloc(blocks * sizeof(int64_t)))
    return fail(TG_ERR_CUDA, "shape cloud: device allocation failed");
  unsigned long long st[kMtN];
  mt_seed(seed, st);
  SETUP_TRY(cudaMemcpy(state.p, st, sizeof st, cudaMemcpyHostToDevice));
  // The stream is consumed three words per candidate; a chunk's twists
  // produce whole 312-word blocks, so a remainder carries to the next chunk.
  std::vector<int> cnt(blocks);
  std::vector<int64_t> off(blocks);
  int64_t accepted = 0;
  std::vector<unsigned long long> carry;  // words generated but not yet consumed
  DevBuf carry_dev;
  if (!carry_dev.alloc(3 * 8)) return fail(TG_ERR_CUDA, "shape cloud: device allocation failed");
  const size_t words_per_chunk = static_cast<size_t>(kTwists) * kMtN;
  DevBuf stream;  // carry (< 3 words) + this chunk's words
  if (!stream.alloc((words_per_chunk + 3) * 8))
    return fail(TG_ERR_CUDA, "shape cloud: device allocation failed");
  for (int guard = 0; accepted < n; ++guard) {
    if (guard > 4096) return fail(TG_ERR_CONFIG, "shape cloud: acceptance too low for " + shape);
    k_mt_stream<<<1, kMtN>>>(state.as<unsigned long long>(), words.as<unsigned long long>(), kTwists);
    const size_t nc = carry.size();
    if (nc) SETUP_TRY(cudaMemcpy(stream.p, carry.data(), nc * 8, cudaMemcpyHostToDevice));
    SETUP_TRY(cudaMemcpy(stream.as<unsigned long long>() + nc, words.p, words_per_chunk * 8,
                         cudaMemcpyDeviceToDevice));
    const size_t avail = nc + words_per_chunk;
    const int64_t n_cand = static_cast<int64_t>(avail / 3);
    const int nb = static_cast<int>((n_cand + kCandThreads - 1) / kCandThreads);
    k_candidates<<<nb, kCandThreads>>>(stream.as<unsigned long long>(), n_cand, t,
                                       flag.as<uint8_t>(), counts.as<int>());
    SETUP_TRY(cudaGetLastError());
    SETUP_TRY(cudaMemcpy(cnt.data(), counts.p, nb * sizeof(int), cudaMemcpyDeviceToHost));
    int64_t run = accepted;
    for (int b = 0; b < nb; ++b) {
      off[b] = run;
      run += cnt[b];
    }
    SETUP_TRY(cudaMemcpy(offsets.p, off.data(), nb * sizeof(int64_t), cudaMemcpyHostToDevice));
    k_compact<<<nb, kCandThreads>>>(stream.as<unsigned long long>(), n_cand, t, flag.as<uint8_t>(),
                                    offsets.as<int64_t>(), n, d_out);
    SETUP_TRY(cudaGetLastError());
    accepted = run;
    const size_t used = static_cast<size_t>(n_cand) * 3;
    carry.resize(avail - used);
    if (!carry.empty())
      SETUP_TRY(cudaMemcpy(carry.data(), stream.as<unsigned long long>() + used,
                           carry.size() * 8, cudaMemcpyDeviceToHost));
  }
  SETUP_TRY(cudaDeviceSynchronize());
  return TG_OK;
}

// indenter_cloud_for (scene_builder.cpp:33-46) for a generated shape on the
// device: the rejection-sampled source cloud, subsampled to target_points
// (the partial Fisher-Yates index draw is the host's: sequential, 1e5 steps;
// the gather runs here). Result: `n` points (m) in device memory.
int device_indenter_cloud(int device, const std::string& shape, uint64_t source_points,
                          uint64_t target_points, uint64_t seed, double** d_cloud, int64_t* n_out) {
  const int64_t ns = static_cast<int64_t>(source_points);
  double* src = nullptr;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaMalloc(&src, static_cast<size_t>(std::max<int64_t>(ns, 1)) * 3 * 8) != cudaSuccess)
    return fail(TG_ERR_CUDA, "indenter: device allocation failed");
  int rc = device_shape_cloud(device, shape, ns, seed, src);
  if (rc) {
    cudaFree(src);
    return rc;
  }
  const uint64_t target = std::max<uint64_t>(target_points, 1);
  if (target >= source_points) {
    *d_cloud = src;
    *n_out = ns;
    return TG_OK;
  }
  std::vector<uint32_t> idx(static_cast<size_t>(ns));
  for (int64_t i = 0; i < ns; ++i) idx[i] = static_cast<uint32_t>(i);
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < target; ++i) {  // draw_below (particle_set.cpp:48-56)
    const uint64_t bound = source_points - i;
    const uint64_t limit = UINT64_MAX - UINT64_MAX % bound;
    uint64_t x;
    do {
      x = rng();
    } while (x >= limit);
    std::swap(idx[i], idx[i + x % bound]);
  }
  idx.resize(target);
  std::sort(idx.begin(), idx.end());
  const int64_t n = static_cast<int64_t>(target);
  DevBuf d_idx;
  double* sub = nullptr;
  if (!d_idx.alloc(idx.size() * 4) || cudaMalloc(&sub, static_cast<size_t>(n) * 3 * 8) != cudaSuccess) {
    cudaFree(src);
    return fail(TG_ERR_CUDA, "indenter: device allocation failed");
  }
  cudaMemcpy(d_idx.p, idx.data(), idx.size() * 4, cudaMemcpyHostToDevice);
  k_gather_points<<<static_cast<unsigned>((n + 255) / 256), 256>>>(src, d_idx.as<uint32_t>(), n, sub);
  const cudaError_t e = cudaDeviceSynchronize();
  cudaFree(src);
  if (e != cudaSuccess) {
    cudaFree(sub);
    return fail(TG_ERR_CUDA, std::string("indenter: ") + cudaGetErrorString(e));
  }
  *d_cloud = sub;
  *n_out = n;
  return TG_OK;
}

// place_for_press (scene_builder.cpp:48-61) of a device cloud: rotate about
// z, reduce the bbox, translate so the cloud's xy-centre sits at
// (centre + off_x, centre + off_y) and its lowest point at top_plus_gap;
// the placed points come back to `out` (host).
int device_place_for_press(const double* d_cloud, int64_t n, double z_rotation, double centre,
                           double top_plus_gap, double off_x, double off_y,
                           std::vector<host::V3>& out) {
  DevBuf rot, placed, box;
  if (!rot.alloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * 3 * 8) ||
      !placed.alloc(static_cast<size_t>(std::max<int64_t>(n, 1)) * 3 * 8) || !box.alloc(6 * 8))
    return fail(TG_ERR_CUDA, "indenter: device allocation failed");
  unsigned long long init[6];
  for (int a = 0; a < 3; ++a) {
    init[a] = ~0ull;  // above order_key(+inf)
    init[3 + a] = 0ull;
  }
  SETUP_TRY(cudaMemcpy(box.p, init, sizeof init, cudaMemcpyHostToDevice));
  const unsigned nb = static_cast<unsigned>((n + 255) / 256);
  k_place<<<nb, 256>>>(d_cloud, n, std::cos(z_rotation), std::sin(z_rotation), 0.0, 0.0, 0.0,
                       rot.as<double>(), box.as<unsigned long long>());
  unsigned long long bk[6];
  SETUP_TRY(cudaMemcpy(bk, box.p, sizeof bk, cudaMemcpyDeviceToHost));
  double lo[3], hi[3];
  for (int a = 0; a < 3; ++a) {
    lo[a] = order_val(bk[a]);
    hi[a] = order_val(bk[3 + a]);
  }
  const double tx = centre + off_x - 0.5 * (lo[0] + hi[0]);
  const double ty = centre + off_y - 0.5 * (lo[1] + hi[1]);
  const double tz = top_plus_gap - lo[2];
  k_place<<<nb, 256>>>(rot.as<double>(), n, std::cos(0.0), std::sin(0.0), tx, ty, tz,
                       placed.as<double>(), nullptr);
  std::vector<double> h(static_cast<size_t>(n) * 3);
  SETUP_TRY(cudaMemcpy(h.data(), placed.p, h.size() * 8, cudaMemcpyDeviceToHost));
  out.resize(static_cast<size_t>(n));
  for (int64_t k = 0; k < n; ++k) out[k] = {h[3 * k], h[3 * k + 1], h[3 * k + 2]};
  return TG_OK;
}

}  // namespace tacchi_b200

namespace tacchi_b200 {
void device_free(void* p) { cudaFree(p); }
}  // namespace tacchi_b200

extern "C" int tg_generate_cloud_device(int device, const char* shape, int64_t n, uint64_t seed,
                                        double* out) {
  using namespace tacchi_b200;
  if (!shape || !out || n < 0) return fail(TG_ERR_INVALID_ARGUMENT, "tg_generate_cloud_device: bad argument");
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(TG_ERR_CUDA, "no CUDA device available (the B200 path has no CPU fallback)");
  double* d = nullptr;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaMalloc(&d, static_cast<size_t>(std::max<int64_t>(n, 1)) * 3 * 8) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_generate_cloud_device: device allocation failed");
  int rc = device_shape_cloud(device, shape, n, seed, d);
  if (!rc && cudaMemcpy(out, d, static_cast<size_t>(n) * 3 * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    rc = fail(TG_ERR_CUDA, "tg_generate_cloud_device: copy failed");
  cudaFree(d);
  return rc;
}
