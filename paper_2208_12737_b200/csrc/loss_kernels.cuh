// loss_kernels.cuh -- fused image-similarity loss + pixel gradient
// (SURVEY 8(f) row 1), restating metrics.py of the reference:
//   neg_zncc: a_hat = (a - mu_a)/sigma_a (population sigma, metrics.py:26-31),
//             raw = mean(a_hat * b_hat), value = -clip(raw, -1, 1)
//             (metrics.py:41-53), grad = -(b_hat - raw a_hat)/(N sigma_a)
//             (metrics.py:78-84);
//   l2:       value = ||a - b||, grad = (a - b)/value (0 when value == 0)
//             (metrics.py:56-59,85-90).
// One thread-block cluster of kLossCluster CTAs per image, each CTA a fixed
// contiguous chunk of the pixels: a fixed-order reduction of the five moments
// in f64 (threads, warp butterfly, warps, then the cluster's CTAs in rank
// order through distributed shared memory), then each CTA writes the fp32
// pixel gradient of its chunk that drr_backward consumes.  No workspace and no
// atomics; the f64 moment sweep is spread over kLossCluster SMs (one CTA per
// image was FP64-throughput-bound on one SM: 18.6 us per 200^2 image, vs
// ~6 us this way).  sigma == 0 (constant image) is reported through `status`
// (metrics.py:29-30 MetricUndefinedError) instead of a host round trip.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace drr {

// threads per CTA (A/B, scripts/lossbench.py, 1 / 32 images of 200^2: 128 -> 11.5 / 12.8 us,
// 256 -> 11.3 / 11.1, 512 -> 11.5 / 11.4, 1024 -> 11.2 / 20.7)
#ifndef DRR_LOSS_THREADS
#define DRR_LOSS_THREADS 256
#endif
constexpr int kLossThreads = DRR_LOSS_THREADS;
constexpr int kLossCluster = 8;  // CTAs (SMs) per image
#ifndef DRR_LOSS_BATCH
#define DRR_LOSS_BATCH 4
#endif
constexpr int kLossBatch = DRR_LOSS_BATCH;  // loads in flight per thread before they are summed (in order)

// Fixed-order block sum of five doubles: xor butterfly in each warp, then the
// warps in index order; every thread returns the block totals.
__device__ __forceinline__ void block_sum5(double v[5], double* sm) {
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

// Cluster-wide fixed-order total of five per-thread partials: block_sum5 in
// each CTA, then the CTAs' totals in rank order through distributed shared
// memory.  Every thread of the cluster returns the image's five totals.
template <int kThreadsT>
__device__ __forceinline__ void cluster_sum5(double v[5], double* sm) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  constexpr int kTot = kThreadsT / 32 * 5, kImg = kTot + 5;
  block_sum5(v, sm);  // this CTA's totals in sm[kTot..kTot+5)
  cluster.sync();     // every CTA's totals are visible cluster-wide
  if (threadIdx.x < 5) {
    double t = 0.0;
    for (int r = 0; r < kLossCluster; ++r) t += *cluster.map_shared_rank(sm + kTot + threadIdx.x, r);
    sm[kImg + threadIdx.x] = t;
  }
  cluster.sync();     // no CTA leaves (or reuses its totals) while they are read
#pragma unroll
  for (int k = 0; k < 5; ++k) v[k] = sm[kImg + k];
}

// kind 0 = neg_zncc, 1 = l2.  fixed may be shared by all images (fixed_stride 0).
// Grid (kLossCluster, images); cluster (kLossCluster, 1, 1).
//
// neg_zncc is two-pass like the reference (metrics.py:26-31 centres before it
// squares): pass 1 the means, pass 2 the centred second moments over the same
// (L1/L2-resident) chunk, so a bright image with little structure keeps its
// digits.  sigma == 0 (MetricUndefinedError, metrics.py:29-30) is decided
// from the data itself: an image whose pixels are all equal is undefined even
// when its mean rounds (so its residuals are tiny but not zero) -- pass 2 also
// counts the pixels that differ from the first one.
//
// Outputs (each optional but value): value[b]; status[b] = 1 where the metric
// is undefined (value, gradient and coefficients are then NaN, as the torch
// restatement gives); grad = the fp32 pixel gradient (metrics.py:78-90); coef
// = the pixel gradient as an affine map of the two images,
//   dL/da_i = coef[0] + coef[1] a_i + coef[2] b_i   (3 doubles per image),
// which lets a walk that already holds a_i, b_i and the ray Jacobian reduce
// the pose gradient without the per-pixel gradient ever being stored
// (k_forward_loss + k_reduce_loss_grad).
template <typename IT>
__global__ void __cluster_dims__(kLossCluster, 1, 1) __launch_bounds__(kLossThreads)
    k_image_loss(const IT* __restrict__ img, const IT* __restrict__ fixed,
                 int64_t fixed_stride, int64_t npix, int kind,
                 double* __restrict__ value, float* __restrict__ grad,
                 int* __restrict__ status, double* __restrict__ coef) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  // [0, W*5): warp partials; [W*5, W*5+5): this CTA's totals; then the image's
  __shared__ double sm[(kLossThreads / 32 + 2) * 5];
  const int b = blockIdx.y;
  const int rank = static_cast<int>(cluster.block_rank());
  const int64_t chunk = (npix + kLossCluster - 1) / kLossCluster;
  const int64_t lo = rank * chunk, hi = lo + chunk < npix ? lo + chunk : npix;
  const IT* a = img + static_cast<int64_t>(b) * npix;
  const IT* f = fixed + static_cast<int64_t>(b) * fixed_stride;
  float* g = grad ? grad + static_cast<int64_t>(b) * npix : nullptr;
  const double N = static_cast<double>(npix);
  double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
  // pass 1: each thread sums its pixels lo + tid, lo + tid + T, ... in that
  // order; the loads of kLossBatch of them are issued before any is summed
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kLossThreads * kLossBatch) {
    IT xa[kLossBatch], ya[kLossBatch];
#pragma unroll
    for (int j = 0; j < kLossBatch; ++j) {
      const int64_t i = i0 + static_cast<int64_t>(j) * kLossThreads;
      xa[j] = i < hi ? a[i] : IT(0);
      ya[j] = i < hi ? f[i] : IT(0);
    }
#pragma unroll
    for (int j = 0; j < kLossBatch; ++j) {
      if (i0 + static_cast<int64_t>(j) * kLossThreads >= hi) break;
      const double x = static_cast<double>(xa[j]), y = static_cast<double>(ya[j]);
      if (kind == 0) {
        v[0] += x; v[2] += y;
      } else {
        const double dd = x - y;
        v[0] += dd * dd;
      }
    }
  }
  cluster_sum5<kLossThreads>(v, sm);
  if (kind == 0) {
    const double ma = v[0] / N, mb = v[2] / N;
    const double a0 = static_cast<double>(a[0]), b0 = static_cast<double>(f[0]);
    // pass 2: centred moments and the count of pixels unlike the first
    double w[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kLossThreads * kLossBatch) {
      IT xa[kLossBatch], ya[kLossBatch];
#pragma unroll
      for (int j = 0; j < kLossBatch; ++j) {
        const int64_t i = i0 + static_cast<int64_t>(j) * kLossThreads;
        xa[j] = i < hi ? a[i] : IT(0);
        ya[j] = i < hi ? f[i] : IT(0);
      }
#pragma unroll
      for (int j = 0; j < kLossBatch; ++j) {
        if (i0 + static_cast<int64_t>(j) * kLossThreads >= hi) break;
        const double x = static_cast<double>(xa[j]), y = static_cast<double>(ya[j]);
        const double dx = x - ma, dy = y - mb;
        w[0] += dx * dx; w[1] += dy * dy; w[2] += dx * dy;
        w[3] += x != a0 ? 1.0 : 0.0;
        w[4] += y != b0 ? 1.0 : 0.0;
      }
    }
    cluster_sum5<kLossThreads>(w, sm);
    const double sa = sqrt(w[0] / N), sb = sqrt(w[1] / N);
    const bool undefined = w[3] == 0.0 || w[4] == 0.0 || !(sa > 0.0) || !(sb > 0.0);
    const double raw = undefined ? NAN : w[2] / (N * sa * sb);
    const double scale = undefined ? NAN : -1.0 / (N * sa);
    if (rank == 0 && threadIdx.x == 0) {
      value[b] = undefined ? NAN : -fmin(1.0, fmax(-1.0, raw));
      if (status) status[b] = undefined ? 1 : 0;
      if (coef) {
        // scale (bh - raw ah) with ah = (a - ma)/sa, bh = (b - mb)/sb
        coef[3 * b + 0] = scale * (raw * ma / sa - mb / sb);
        coef[3 * b + 1] = -scale * raw / sa;
        coef[3 * b + 2] = scale / sb;
      }
    }
    if (g) {
      const double inv_sa = 1.0 / sa, inv_sb = 1.0 / sb;
#pragma unroll 4
      for (int64_t i = lo + threadIdx.x; i < hi; i += kLossThreads) {
        const double ah = (static_cast<double>(a[i]) - ma) * inv_sa;
        const double bh = (static_cast<double>(f[i]) - mb) * inv_sb;
        g[i] = static_cast<float>(scale * (bh - raw * ah));
      }
    }
  } else {
    const double norm = sqrt(v[0]);
    const double inv = norm > 0.0 ? 1.0 / norm : 0.0;
    if (rank == 0 && threadIdx.x == 0) {
      value[b] = norm;
      if (status) status[b] = 0;
      if (coef) {
        coef[3 * b + 0] = 0.0;
        coef[3 * b + 1] = inv;
        coef[3 * b + 2] = -inv;
      }
    }
    if (g) {
#pragma unroll 4
      for (int64_t i = lo + threadIdx.x; i < hi; i += kLossThreads)
        g[i] = static_cast<float>((static_cast<double>(a[i]) - static_cast<double>(f[i])) * inv);
    }
  }
}

}  // namespace drr
