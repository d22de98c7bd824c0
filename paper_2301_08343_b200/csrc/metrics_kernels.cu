// Image metrics on the GPU: metrics::ssim / psnr / mae
// (/root/reference/proj/src/metrics/image_metrics.cpp:57-112) for a batch of
// image pairs in one launch, for `compare` over thousands of frames.
//
// Layout: `count` pairs of height x width x 3 uint8 images, interleaved RGB
// (Image8::data), pair-major. One CTA column (blockIdx.y) per pair:
//   - SSIM: one thread per 8x8 window (top-left (x, y), x + 8 <= w,
//     y + 8 <= h), grey = (r + g + b) / 3.0 (image_metrics.cpp:25-30); the
//     five window sums are taken directly instead of through summed-area
//     tables, so SSIM agrees with the reference to rounding (~1e-11).
//   - squared / absolute channel differences are integers: accumulated
//     exactly in 64-bit integers, so PSNR and MAE equal the reference's.
// Per-CTA partials are reduced in a fixed order by a second kernel, so the
// results are run-to-run deterministic.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <string>
#include <vector>

#include "tacchi_cuda.h"

namespace tacchi_b200 {
int fail(int code, const std::string& msg);

namespace {

constexpr int kWin = 8;
constexpr double kC1 = (0.01 * 255.0) * (0.01 * 255.0);
constexpr double kC2 = (0.03 * 255.0) * (0.03 * 255.0);
constexpr int kThreads = 256;

struct Partial {
  double ssim;
  unsigned long long se, ae;
};

__device__ __forceinline__ double grey(const uint8_t* p) {
  return (static_cast<double>(p[0]) + p[1] + p[2]) / 3.0;
}

// Grid: x = CTAs over max(windows, pixels*3) of one pair, y = pair.
__global__ void __launch_bounds__(kThreads) k_metrics(const uint8_t* __restrict__ a,
                                                      const uint8_t* __restrict__ b, int w,
                                                      int h, Partial* __restrict__ partials) {
  const int pair = blockIdx.y;
  const size_t img = static_cast<size_t>(w) * h * 3;
  const uint8_t* A = a + pair * img;
  const uint8_t* B = b + pair * img;
  const int wx = w - kWin + 1, wy = h - kWin + 1;
  const int64_t windows = static_cast<int64_t>(wx) * wy;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * kThreads;

  double ssim = 0.0;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x; t < windows;
       t += stride) {
    const int x0 = static_cast<int>(t % wx), y0 = static_cast<int>(t / wx);
    double sa = 0, sb = 0, saa = 0, sbb = 0, sab = 0;
    for (int dy = 0; dy < kWin; ++dy) {
      const uint8_t* ra = A + (static_cast<size_t>(y0 + dy) * w + x0) * 3;
      const uint8_t* rb = B + (static_cast<size_t>(y0 + dy) * w + x0) * 3;
#pragma unroll
      for (int dx = 0; dx < kWin; ++dx) {
        const double ga = grey(ra + 3 * dx), gb = grey(rb + 3 * dx);
        sa += ga;
        sb += gb;
        saa += ga * ga;
        sbb += gb * gb;
        sab += ga * gb;
      }
    }
    const double n = kWin * kWin;
    const double mu_a = sa / n, mu_b = sb / n;
    const double var_a = saa / n - mu_a * mu_a;
    const double var_b = sbb / n - mu_b * mu_b;
    const double cov = sab / n - mu_a * mu_b;
    const double num = (2.0 * mu_a * mu_b + kC1) * (2.0 * cov + kC2);
    const double den = (mu_a * mu_a + mu_b * mu_b + kC1) * (var_a + var_b + kC2);
    ssim += num / den;
  }
  unsigned long long se = 0, ae = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * kThreads + threadIdx.x;
       i < static_cast<int64_t>(img); i += stride) {
    const int d = static_cast<int>(A[i]) - static_cast<int>(B[i]);
    se += static_cast<unsigned long long>(d * d);
    ae += static_cast<unsigned long long>(d < 0 ? -d : d);
  }
  // CTA reduction in a fixed order
  __shared__ double s_ssim[kThreads / 32];
  __shared__ unsigned long long s_se[kThreads / 32], s_ae[kThreads / 32];
  for (int o = 16; o > 0; o >>= 1) {
    ssim += __shfl_down_sync(0xffffffffu, ssim, o);
    se += __shfl_down_sync(0xffffffffu, se, o);
    ae += __shfl_down_sync(0xffffffffu, ae, o);
  }
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (lane == 0) {
    s_ssim[warp] = ssim;
    s_se[warp] = se;
    s_ae[warp] = ae;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    Partial p{0.0, 0ull, 0ull};
    for (int k = 0; k < kThreads / 32; ++k) {
      p.ssim += s_ssim[k];
      p.se += s_se[k];
      p.ae += s_ae[k];
    }
    partials[static_cast<size_t>(pair) * gridDim.x + blockIdx.x] = p;
  }
}

// One thread per pair: fixed-order sum of its CTA partials -> ssim, psnr, mae.
__global__ void k_metrics_finish(const Partial* __restrict__ partials, int ctas, int count,
                                 int w, int h, double* __restrict__ out) {
  const int pair = blockIdx.x * blockDim.x + threadIdx.x;
  if (pair >= count) return;
  double ssim = 0.0;
  unsigned long long se = 0, ae = 0;
  for (int k = 0; k < ctas; ++k) {
    const Partial& p = partials[static_cast<size_t>(pair) * ctas + k];
    ssim += p.ssim;
    se += p.se;
    ae += p.ae;
  }
  const double windows = static_cast<double>(w - kWin + 1) * (h - kWin + 1);
  const double n = static_cast<double>(w) * h * 3;
  const double mse = static_cast<double>(se) / n;
  out[3 * pair + 0] = ssim / windows;
  // the mse (exact: an integer sum over n); tg_image_metrics turns it into
  // PSNR on the host with the host's log10, the reference's own call
  // (image_metrics.cpp:99) — the device log10 differs in the last ulp
  out[3 * pair + 1] = mse;
  out[3 * pair + 2] = static_cast<double>(ae) / n / 255.0 * 100.0;
}

}  // namespace

// Batched metrics on device buffers (stream-ordered): per pair {ssim, mse,
// mae %}; the caller forms PSNR from the mse on the host (psnr_from_mse).
int image_metrics_device(const uint8_t* d_a, const uint8_t* d_b, int w, int h, int count,
                         double* d_out, cudaStream_t stream) {
  int sms = 148;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  // ~4 CTAs per SM over the whole batch, at least one per pair
  const int ctas = std::max(1, std::min(64, (4 * sms + count - 1) / count));
  Partial* partials = nullptr;
  if (cudaMallocAsync(&partials, sizeof(Partial) * ctas * count, stream) != cudaSuccess)
    return fail(TG_ERR_CUDA, "image_metrics: allocation failed");
  k_metrics<<<dim3(ctas, count), kThreads, 0, stream>>>(d_a, d_b, w, h, partials);
  k_metrics_finish<<<(count + 127) / 128, 128, 0, stream>>>(partials, ctas, count, w, h, d_out);
  cudaFreeAsync(partials, stream);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(TG_ERR_CUDA, std::string("image_metrics: ") + cudaGetErrorString(e));
  return TG_OK;
}

}  // namespace tacchi_b200

extern "C" int tg_image_metrics(int device, const uint8_t* a, const uint8_t* b, int w, int h,
                                int count, double* out) {
  using tacchi_b200::fail;
  if (!a || !b || !out || count < 0) return fail(TG_ERR_INVALID_ARGUMENT, "tg_image_metrics: null");
  if (count == 0) return TG_OK;
  if (w <= 0 || h <= 0) return fail(TG_ERR_SHAPE_MISMATCH, "empty image");
  if (w < 8 || h < 8) return fail(TG_ERR_SHAPE_MISMATCH, "image smaller than the SSIM window");
  if (cudaSetDevice(device) != cudaSuccess) return fail(TG_ERR_CUDA, "tg_image_metrics: no device");
  cudaStream_t s;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess)
    return fail(TG_ERR_CUDA, "tg_image_metrics: stream");
  const size_t bytes = static_cast<size_t>(w) * h * 3 * count;
  uint8_t *da = nullptr, *db = nullptr;
  double* dout = nullptr;
  int rc = TG_OK;
  if (cudaMallocAsync(&da, bytes, s) != cudaSuccess || cudaMallocAsync(&db, bytes, s) != cudaSuccess ||
      cudaMallocAsync(&dout, sizeof(double) * 3 * count, s) != cudaSuccess) {
    rc = fail(TG_ERR_CUDA, "tg_image_metrics: allocation failed");
  } else {
    cudaMemcpyAsync(da, a, bytes, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(db, b, bytes, cudaMemcpyHostToDevice, s);
    rc = tacchi_b200::image_metrics_device(da, db, w, h, count, dout, s);
    if (rc == TG_OK) cudaMemcpyAsync(out, dout, sizeof(double) * 3 * count, cudaMemcpyDeviceToHost, s);
  }
  if (da) cudaFreeAsync(da, s);
  if (db) cudaFreeAsync(db, s);
  if (dout) cudaFreeAsync(dout, s);
  const cudaError_t e = cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
  if (rc == TG_OK && e != cudaSuccess)
    rc = fail(TG_ERR_CUDA, std::string("tg_image_metrics: ") + cudaGetErrorString(e));
  if (rc == TG_OK)  // PSNR from the exact mse with the reference's expression
    for (int p = 0; p < count; ++p) {
      const double mse = out[3 * p + 1];
      out[3 * p + 1] = mse == 0.0 ? std::numeric_limits<double>::infinity()
                                  : 10.0 * std::log10(255.0 * 255.0 / mse);
    }
  return rc;
}
