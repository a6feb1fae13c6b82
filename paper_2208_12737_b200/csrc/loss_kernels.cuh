// loss_kernels.cuh -- fused image-similarity loss + pixel gradient
// (SURVEY 8(f) row 1), restating metrics.py of the reference:
//   neg_zncc: a_hat = (a - mu_a)/sigma_a (population sigma, metrics.py:26-31),
//             raw = mean(a_hat * b_hat), value = -clip(raw, -1, 1)
//             (metrics.py:41-53), grad = -(b_hat - raw a_hat)/(N sigma_a)
//             (metrics.py:78-84);
//   l2:       value = ||a - b||, grad = (a - b)/value (0 when value == 0)
//             (metrics.py:56-59,85-90).
// One CTA per image: a fixed-order block reduction of the five moments in
// f64, then a second sweep writes the fp32 pixel gradient that drr_backward
// consumes.  sigma == 0 (constant image) is reported through `status`
// (metrics.py:29-30 MetricUndefinedError) instead of a host round trip.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace drr {

constexpr int kLossThreads = 512;

__device__ __forceinline__ void block_sum5(double v[5], double* sm) {
  // fixed-order: xor butterfly in the warp, then warps in index order
#pragma unroll
  for (int k = 0; k < 5; ++k)
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) sm[warp * 5 + k] = v[k];
  __syncthreads();
  if (threadIdx.x < 5) {
    double s = 0.0;
    for (int w = 0; w < kLossThreads / 32; ++w) s += sm[w * 5 + threadIdx.x];
    sm[kLossThreads / 32 * 5 + threadIdx.x] = s;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 5; ++k) v[k] = sm[kLossThreads / 32 * 5 + k];
}

// kind 0 = neg_zncc, 1 = l2.  fixed may be shared by all images (fixed_stride 0).
template <typename IT>
__global__ void __launch_bounds__(kLossThreads)
    k_image_loss(const IT* __restrict__ img, const IT* __restrict__ fixed,
                 int64_t fixed_stride, int64_t npix, int kind,
                 double* __restrict__ value, float* __restrict__ grad,
                 int* __restrict__ status) {
  __shared__ double sm[(kLossThreads / 32 + 1) * 5];
  const int b = blockIdx.x;
  const IT* a = img + static_cast<int64_t>(b) * npix;
  const IT* f = fixed + static_cast<int64_t>(b) * fixed_stride;
  float* g = grad ? grad + static_cast<int64_t>(b) * npix : nullptr;
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  for (int64_t i = threadIdx.x; i < npix; i += kLossThreads) {
    const double x = static_cast<double>(a[i]), y = static_cast<double>(f[i]);
    if (kind == 0) {
      v[0] += x; v[1] += x * x; v[2] += y; v[3] += y * y; v[4] += x * y;
    } else {
      const double dd = x - y;
      v[0] += dd * dd;
    }
  }
  block_sum5(v, sm);
  const double N = static_cast<double>(npix);
  if (kind == 0) {
    const double ma = v[0] / N, mb = v[2] / N;
    const double va = fmax(v[1] / N - ma * ma, 0.0), vb = fmax(v[3] / N - mb * mb, 0.0);
    const double sa = sqrt(va), sb = sqrt(vb);
    const bool undefined = !(sa > 0.0) || !(sb > 0.0);
    const double raw = undefined ? 0.0 : (v[4] / N - ma * mb) / (sa * sb);
    if (threadIdx.x == 0) {
      value[b] = undefined ? NAN : -fmin(1.0, fmax(-1.0, raw));
      if (status) status[b] = undefined ? 1 : 0;
    }
    if (g) {
      const double inv_sa = undefined ? 0.0 : 1.0 / sa, inv_sb = undefined ? 0.0 : 1.0 / sb;
      const double scale = undefined ? 0.0 : -1.0 / (N * sa);
      for (int64_t i = threadIdx.x; i < npix; i += kLossThreads) {
        const double ah = (static_cast<double>(a[i]) - ma) * inv_sa;
        const double bh = (static_cast<double>(f[i]) - mb) * inv_sb;
        g[i] = static_cast<float>(scale * (bh - raw * ah));
      }
    }
  } else {
    const double norm = sqrt(v[0]);
    if (threadIdx.x == 0) {
      value[b] = norm;
      if (status) status[b] = 0;
    }
    if (g) {
      const double inv = norm > 0.0 ? 1.0 / norm : 0.0;
      for (int64_t i = threadIdx.x; i < npix; i += kLossThreads)
        g[i] = static_cast<float>((static_cast<double>(a[i]) - static_cast<double>(f[i])) * inv);
    }
  }
}

}  // namespace drr
