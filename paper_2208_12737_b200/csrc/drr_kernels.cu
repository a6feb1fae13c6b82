// drr_kernels.cu -- sm_100a kernels and the extern "C" ABI of include/drr_b200.h.
//
// Every kernel generates its pixel rays in-kernel from the pose frame
// (geometry.py:152-175) and walks them with siddon_lean.cuh (the reference's
// _native.pyx:140-282 semantics, bit-identical crossing parameters).  No dense
// contraction anywhere, so no tensor cores.  CTAs cover pixel tiles whose warps
// are 8 x 4 quads, so neighbouring rays gather neighbouring voxels.
//   k_forward        image of a B x H x W batch
//   k_forward_jac    image + each ray's endpoint Jacobian dE/ds, dE/dp (one
//                    walk per ray for the whole fwd+bwd step)
//   k_backward_jac   contraction of the stored Jacobians with the pixel
//                    gradient, per-CTA partials of the 12 frame gradients
//   k_backward       the same gradient by re-walking the rays (Jacobian-budget
//                    fallback)
//   k_reduce_frames  fixed-order second pass over the CTA partials (no atomics
//                    anywhere, so gradients are bit-reproducible: SPEC.md:289)
//   k_raysum / k_raysum_grad  explicit-ray forms for the kernel-protocol
//                    backend (the reference's _kernels plugin boundary)
//   k_count          used voxel-steps per ray (roofline denominator)
// loss_kernels.cuh / pose_kernels.cuh hold the loss, pose-frame and
// registration-update kernels of the batched loss_and_gradient chain.
#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdarg.h>
#include <string.h>

#include "../../include/drr_b200.h"
#include "siddon_walk.cuh"
#include "siddon_lean.cuh"
#include "loss_kernels.cuh"
#include "pose_kernels.cuh"
#include "volume_pack.cuh"

namespace drr {

// Launch bounds (A/B on C2, 32 poses; scripts/gpu_ab.sh, gpu_ab_fast.sh): the
// forward at 6 CTAs/SM with a 4-deep gather pipeline, k_forward_jac and the
// re-walk k_backward at 6 with a 3-deep one (their derived-axis loops fit 80
// registers once the walk's end state is parked in shared memory and the
// pixel and direction are re-derived after it; k_backward 2.34 -> 2.17 ms
// going from 5 to 6); ptxas spills only outside the walk's fast path.
#ifndef DRR_BWD_MINB
#define DRR_BWD_MINB 6
#endif
#ifndef DRR_FJ_MINB
#define DRR_FJ_MINB 6
#endif
#ifndef DRR_FWD_MINB
#define DRR_FWD_MINB 6
#endif
#ifndef DRR_SPLIT_MINB
#define DRR_SPLIT_MINB 6
#endif
// the gradient walks with rays split over K > 1 lanes (a 4-deep gather
// pipeline, DRR_LEAN_PIPE_GRAD_SPLIT): A/B one C2 pose, fwd+jac 0.119 -> 0.107 ms
#ifndef DRR_SPLIT_MINB_GRAD
#define DRR_SPLIT_MINB_GRAD 5
#endif
constexpr int kThreads = 128;  // 4 warps per CTA
constexpr int kFrameGrads = 12;

// CTA pixel tile for K threads per ray (SURVEY 7 H2 ray splitting):
//   K = 1: each warp a kQuadW x (32 / kQuadW) quad of adjacent pixels
//          (neighbouring rays share L1/L2 lines of the CT), the CTA 2 x 2
//          quads (4 x 1 when kQuadW = 32);
//   K > 1: 128 / K rays as an 8 x (16 / K) tile; the K chunks of a ray are K
//          consecutive lanes of one warp, combined with xor shuffles.
#ifndef DRR_QUAD_W
#define DRR_QUAD_W 8
#endif
constexpr int kQuadW = DRR_QUAD_W, kQuadH = 32 / kQuadW;
constexpr int kCtaQuadsW = kQuadW == 32 ? 1 : 2, kCtaQuadsH = 4 / kCtaQuadsW;
template <int K>
struct Tile {
  static constexpr int W = K == 1 ? kQuadW * kCtaQuadsW : 8;
  static constexpr int H = K == 1 ? kQuadH * kCtaQuadsH : 16 / K;
};

struct DetDev {
  int H, W;
  int split;       // requested threads per ray (0 = auto)
  int pose_group;  // poses interleaved tile by tile in the CTA order (>= 1)
  double pitch_x, pitch_y;
  double half_h, half_w;  // (H-1)/2.0, (W-1)/2.0   (geometry.py:155-156)
};

// Which (tile, pose) a CTA of a pose launch renders.  The grid is (tiles x,
// tiles y, poses); the CTA's linear launch index is re-read with the poses of
// a group of det.pose_group fastest, then the tiles, then the groups.  With
// a group spanning the batch, the CTAs resident at any moment cover one band
// of detector tiles for every pose rather than the whole detector of a few
// poses: nearby poses cross the same part of the CT, whose lines then stay in
// L2.  Only the work assignment changes; every ray and every partial lands
// where it did.
struct CtaPos {
  int tx, ty, b;
};
// (the indices are read with volatile moves, so a kernel can recompute its
// pixel after the walk instead of holding it in registers across the loop)
__device__ __forceinline__ unsigned sreg_ctaid(int a) {
  unsigned v;
  if (a == 0) asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(v));
  else if (a == 1) asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(v));
  else asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(v));
  return v;
}
__device__ __forceinline__ CtaPos cta_pos(const DetDev& det) {
  const unsigned lin = sreg_ctaid(0) + gridDim.x * (sreg_ctaid(1) + gridDim.y * sreg_ctaid(2));
  const unsigned tiles = gridDim.x * gridDim.y, B = gridDim.z;
  const unsigned G = static_cast<unsigned>(det.pose_group);
  const unsigned gi = lin / (G * tiles);
  const unsigned gl = min(G, B - gi * G);  // the last group may be smaller
  const unsigned rem = lin - gi * G * tiles;
  const unsigned tile = rem / gl;
  return CtaPos{static_cast<int>(tile % gridDim.x), static_cast<int>(tile / gridDim.x),
                static_cast<int>(gi * G + rem % gl)};
}

template <int K>
__device__ __forceinline__ void tile_ray(const DetDev& det, int& h, int& w, int& chunk) {
  const CtaPos c = cta_pos(det);
  const int t = threadIdx.x;
  if (K == 1) {
    const int warp = t >> 5, lane = t & 31;
    w = c.tx * Tile<K>::W + (warp % kCtaQuadsW) * kQuadW + (lane % kQuadW);
    h = c.ty * Tile<K>::H + (warp / kCtaQuadsW) * kQuadH + (lane / kQuadW);
    chunk = 0;
  } else {
    const int ray = t / K;
    chunk = t % K;
    w = c.tx * Tile<K>::W + (ray & 7);
    h = c.ty * Tile<K>::H + (ray >> 3);
  }
}

// Fixed-order sum over the K lanes of a ray (all 32 lanes must call it).
template <int K, typename T>
__device__ __forceinline__ T chunk_sum(T x) {
#pragma unroll
  for (int off = K / 2; off > 0; off >>= 1) x += __shfl_xor_sync(0xffffffffu, x, off);
  return x;
}


// Pixel position (c + a_h e1) + a_w e2 in numpy's evaluation order
// (geometry.py:171-174); the TU is built --fmad=false, so this rounds
// exactly like numpy.
__device__ __forceinline__ void pixel_ray(const double* __restrict__ f,
                                          const DetDev& det, int h, int w,
                                          double* s, double* p, double& ah,
                                          double& aw) {
  ah = (static_cast<double>(h) - det.half_h) * det.pitch_y;
  aw = (static_cast<double>(w) - det.half_w) * det.pitch_x;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    s[a] = __ldg(f + a);
    p[a] = (__ldg(f + 3 + a) + ah * __ldg(f + 6 + a)) + aw * __ldg(f + 9 + a);
  }
}

// The direction p - s of pixel (h, w), re-read from the frames after a walk
// (volatile loads, so the compiler cannot keep the pre-walk values alive
// across the walk loop instead: registers there are what bound occupancy).
// Same operations as pixel_ray + ray_setup, so bit-identical.
__device__ __forceinline__ void reload_ray_d(const double* __restrict__ f, const DetDev& det,
                                             int h, int w, double* d, double& ah, double& aw) {
  ah = (static_cast<double>(h) - det.half_h) * det.pitch_y;
  aw = (static_cast<double>(w) - det.half_w) * det.pitch_x;
  double v[12];
#pragma unroll
  for (int i = 0; i < 12; ++i)
    asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(v[i]) : "l"(f + i));
#pragma unroll
  for (int a = 0; a < 3; ++a) d[a] = ((v[3 + a] + ah * v[6 + a]) + aw * v[9 + a]) - v[a];
}

__device__ __forceinline__ double ray_length(const double* d) {
  return sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
}

__device__ __forceinline__ double ray_length(const Ray& r) {
  return sqrt(r.d[0] * r.d[0] + r.d[1] * r.d[1] + r.d[2] * r.d[2]);
}

template <typename OT>
__device__ __forceinline__ void store_out(OT* p, double v) {
  *p = static_cast<OT>(v);
}

// The walk (siddon_lean.cuh) in its sum / count / gradient mode; chunked walks
// (K > 1) are described by the Ray itself (ray_setup).
template <typename VT, int kMode, bool kChunked>
__device__ __forceinline__ void walk_sums(const VT* __restrict__ vol, const GridDev& g,
                                          double* tab, const Ray& r, LeanSums& o) {
  lean_walk<VT, kMode, kChunked>(vol, g, tab, tab + plane_table_span(g), r, o);
}

// ---------------------------------------------------------------- forward
template <typename VT, typename OT, int K>
__global__ void __launch_bounds__(kThreads, K == 1 ? DRR_FWD_MINB : DRR_SPLIT_MINB)
    k_forward(const VT* __restrict__ vol, const GridDev g,
              const double* __restrict__ frames, const DetDev det,
              OT* __restrict__ img) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);  // s of this CTA's pose
  __syncthreads();
  int h, w, chunk;
  tile_ray<K>(det, h, w, chunk);
  const bool valid = h < det.H && w < det.W;
  if (K == 1 && !valid) return;
  const int b = cta_pos(det).b;
  double acc = 0.0, L = 0.0;
  if (valid) {
    double s[3], p[3], ah, aw;
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    Ray r;
    ray_setup(g, s, p, r, K, chunk);
    L = ray_length(r);
    if (r.hit) {
      LeanSums o;
      walk_sums<VT, kLeanSum, (K > 1)>(vol, g, tab, r, o);
      acc = o.acc;
    }
  }
  acc = chunk_sum<K>(acc);
  if (valid && chunk == 0)
    store_out(img + (static_cast<size_t>(b) * det.H + h) * det.W + w, L * acc);
}

template <typename VT, int K>
__global__ void __launch_bounds__(kThreads)
    k_count(const VT* __restrict__ vol, const GridDev g,
            const double* __restrict__ frames, const DetDev det,
            int* __restrict__ steps) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);  // s of this CTA's pose
  __syncthreads();
  int h, w, chunk;
  tile_ray<K>(det, h, w, chunk);
  const bool valid = h < det.H && w < det.W;
  if (K == 1 && !valid) return;
  const int b = cta_pos(det).b;
  int n = 0;
  if (valid) {
    double s[3], p[3], ah, aw;
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    Ray r;
    ray_setup(g, s, p, r, K, chunk);
    if (r.hit) {
      LeanSums o;
      walk_sums<VT, kLeanCount, (K > 1)>(vol, g, tab, r, o);
      n = o.steps;
    }
  }
  n = chunk_sum<K>(n);
  if (valid && chunk == 0) steps[(static_cast<size_t>(b) * det.H + h) * det.W + w] = n;
}

// Endpoint gradients from summed walk totals (acc, G, H): the same algebra as
// endpoint_grads, for chunked walks whose partial sums were combined.
// Correctly rounded x / y -- the Markstein form (the walk's) when y is in the
// normal range, else IEEE '/': the same bits either way, fewer instructions.
__device__ __forceinline__ double cr_div(double x, double y, double rcp) {
  return fabs(y) > 1e-20 ? div_rn(x, y, rcp) : x / y;
}

__device__ __forceinline__ void sums_to_endpoint_grads(const double* d, double acc,
                                                       const double* G, const double* Hh,
                                                       double L, double* dEds, double* dEdp) {
  const double rL = __drcp_rn(L);
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    double gs = 0.0, gp = 0.0;
    if (d[a] != 0.0) {
      const double rd = __drcp_rn(d[a]);
      gs = cr_div(L * (Hh[a] - G[a]), d[a], rd);
      gp = cr_div(-L * Hh[a], d[a], rd);
    }
    const double lt = cr_div(d[a], L, rL) * acc;
    dEds[a] = gs - lt;
    dEdp[a] = gp + lt;
  }
}
__device__ __forceinline__ void sums_to_endpoint_grads(const Ray& r, double acc,
                                                       const double* G, const double* Hh,
                                                       double L, double* dEds, double* dEdp) {
  sums_to_endpoint_grads(r.d, acc, G, Hh, L, dEds, dEdp);
}

// --------------------------------------------------------------- backward
template <typename VT, typename GT, typename OT, int K>
__global__ void __launch_bounds__(kThreads, K == 1 ? DRR_BWD_MINB : DRR_SPLIT_MINB_GRAD)
    k_backward(const VT* __restrict__ vol, const GridDev g,
               const double* __restrict__ frames, const DetDev det,
               const GT* __restrict__ grad_img, OT* __restrict__ img,
               double* __restrict__ partials) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);  // s of this CTA's pose
  __syncthreads();
  int h, w, chunk;
  tile_ray<K>(det, h, w, chunk);
  const int b = cta_pos(det).b;
  const bool valid = h < det.H && w < det.W;
  double acc12[kFrameGrads];
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) acc12[k] = 0.0;
  // this chunk's partial walk sums: acc, G[3], H[3]
  double part[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double s[3], p[3], ah = 0.0, aw = 0.0;
  Ray r;
  r.hit = false;
  if (valid) {
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    ray_setup(g, s, p, r, K, chunk);
    if (r.hit) {
      LeanSums o;
      walk_sums<VT, kLeanGrad, (K > 1)>(vol, g, tab, r, o);
      part[0] = o.acc;
      part[1] = o.G0; part[2] = o.G1; part[3] = o.G2;
      part[4] = o.H0; part[5] = o.H1; part[6] = o.H2;
    }
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) part[k] = chunk_sum<K>(part[k]);
  // the pixel and its ray again (volatile reads, as in k_forward_jac): nothing
  // of them is held across the walk; d and L are chunk-invariant
  tile_ray<K>(det, h, w, chunk);
  const int bp = cta_pos(det).b;
  if (h < det.H && w < det.W && chunk == 0) {
    const size_t pix = (static_cast<size_t>(bp) * det.H + h) * det.W + w;
    const double gpx = static_cast<double>(grad_img[pix]);
    double d[3];
    reload_ray_d(frames + 12 * bp, det, h, w, d, ah, aw);
    const double L = ray_length(d);
    const double e = L * part[0];
    if (part[0] != 0.0 || part[1] != 0.0 || part[2] != 0.0 || part[3] != 0.0 ||
        part[4] != 0.0 || part[5] != 0.0 || part[6] != 0.0) {
      double dEds[3], dEdp[3];
      sums_to_endpoint_grads(d, part[0], part + 1, part + 4, L, dEds, dEdp);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc12[a] = gpx * dEds[a];
        acc12[3 + a] = gpx * dEdp[a];
        acc12[6 + a] = gpx * ah * dEdp[a];
        acc12[9 + a] = gpx * aw * dEdp[a];
      }
    }
    if (img != nullptr) store_out(img + pix, e);
  }
  // Fixed-order CTA reduction: xor-butterfly inside each warp, then warps in
  // index order.
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) {
    double v = acc12[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    acc12[k] = v;
  }
  __shared__ double warp_part[kThreads / 32][kFrameGrads];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) warp_part[warp][k] = acc12[k];
  }
  __syncthreads();
  if (threadIdx.x < kFrameGrads) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kThreads / 32; ++q) v += warp_part[q][threadIdx.x];
    const int blocks_per_pose = gridDim.x * gridDim.y;
    const CtaPos c = cta_pos(det);
    const int blk = c.ty * gridDim.x + c.tx;
    partials[(static_cast<size_t>(b) * blocks_per_pose + blk) * kFrameGrads +
             threadIdx.x] = v;
  }
}

// ------------------------------------------------- forward + ray Jacobian
// One walk per ray yields the image AND the ray's endpoint derivatives
// dE/ds, dE/dp (the reverse-mode form of siddon_raysum_grad's tangents,
// _native.pyx:196-282): the reference's render_with_gradient also walks each
// ray once for energies and tangents together (gradients.py:45-58).  The
// pixel gradient is unknown until the loss has been evaluated, so the 6
// derivatives are stored (SoA, jac[c * npix_total + pix], f64) and
// k_backward_jac contracts them with it -- no second walk of the CT.
template <typename VT, typename OT, int K>
__global__ void __launch_bounds__(kThreads, K == 1 ? DRR_FJ_MINB : DRR_SPLIT_MINB_GRAD)
    k_forward_jac(const VT* __restrict__ vol, const GridDev g,
                  const double* __restrict__ frames, const DetDev det,
                  OT* __restrict__ img, double* __restrict__ jac, size_t npix_total) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);  // s of this CTA's pose
  __syncthreads();
  int h, w, chunk;
  tile_ray<K>(det, h, w, chunk);
  const bool valid = h < det.H && w < det.W;
  if (K == 1 && !valid) return;
  const int b = cta_pos(det).b;
  double part[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  double s[3], p[3], ah = 0.0, aw = 0.0;
  Ray r;
  r.hit = false;
  if (valid) {
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    ray_setup(g, s, p, r, K, chunk);
    if (r.hit) {
      LeanSums o;
      walk_sums<VT, kLeanGrad, (K > 1)>(vol, g, tab, r, o);
      part[0] = o.acc;
      part[1] = o.G0; part[2] = o.G1; part[3] = o.G2;
      part[4] = o.H0; part[5] = o.H1; part[6] = o.H2;
    }
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) part[k] = chunk_sum<K>(part[k]);
  // the pixel again (volatile index reads): nothing of it is held across the walk
  tile_ray<K>(det, h, w, chunk);
  const int bp = cta_pos(det).b;
  if (h < det.H && w < det.W && chunk == 0) {
    const size_t pix = (static_cast<size_t>(bp) * det.H + h) * det.W + w;
    double d[3], ah, aw;
    reload_ray_d(frames + 12 * bp, det, h, w, d, ah, aw);
    const double L = ray_length(d);
    double dEds[3] = {0.0, 0.0, 0.0}, dEdp[3] = {0.0, 0.0, 0.0};
    if (part[0] != 0.0 || part[1] != 0.0 || part[2] != 0.0 || part[3] != 0.0 ||
        part[4] != 0.0 || part[5] != 0.0 || part[6] != 0.0)
      sums_to_endpoint_grads(d, part[0], part + 1, part + 4, L, dEds, dEdp);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      jac[a * npix_total + pix] = dEds[a];
      jac[(3 + a) * npix_total + pix] = dEdp[a];
    }
    store_out(img + pix, L * part[0]);
  }
}

// ------------------------------------------ forward + fused loss gradient
// One walk per ray for a whole neg-ZNCC / L2 loss-and-gradient step
// (gradients.py:61-69 with metrics.py:71-91), with no per-ray Jacobian stored.
// Both losses have a pixel gradient that is affine in the two images,
// dL/da_i = c0 + c1 a_i + c2 b_i (k_image_loss's coefficients), so
//   dL/dframe = c0 sum_i J_i + c1 sum_i a_i J_i + c2 sum_i b_i J_i
// with J_i the ray's 12-vector (dE/ds, dE/dp, a_h dE/dp, a_w dE/dp).  The
// walk knows a_i (its own image value, as stored), b_i (the fixed image) and
// J_i, so each CTA reduces the three 12-vectors over its pixels in a fixed
// order and writes 36 doubles; k_reduce_loss_grad combines the CTAs
// (fixed order) with the coefficients once the loss kernel has run.  That
// removes the 48 B/pixel Jacobian store and its re-read (k_backward_jac) from
// the step, and any batch size takes the one-walk path.
constexpr int kLossSums = 3 * kFrameGrads;
template <typename VT, typename OT, int K>
__global__ void __launch_bounds__(kThreads, K == 1 ? DRR_FJ_MINB : DRR_SPLIT_MINB_GRAD)
    k_forward_loss(const VT* __restrict__ vol, const GridDev g,
                   const double* __restrict__ frames, const DetDev det,
                   OT* __restrict__ img, const OT* __restrict__ fixed, int64_t fixed_stride,
                   double* __restrict__ partials) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);  // s of this CTA's pose
  __syncthreads();
  int h, w, chunk;
  tile_ray<K>(det, h, w, chunk);
  const bool valid = h < det.H && w < det.W;
  const int b = cta_pos(det).b;
  double part[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  if (valid) {
    double s[3], p[3], ah, aw;
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    Ray r;
    ray_setup(g, s, p, r, K, chunk);
    if (r.hit) {
      LeanSums o;
      walk_sums<VT, kLeanGrad, (K > 1)>(vol, g, tab, r, o);
      part[0] = o.acc;
      part[1] = o.G0; part[2] = o.G1; part[3] = o.G2;
      part[4] = o.H0; part[5] = o.H1; part[6] = o.H2;
    }
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) part[k] = chunk_sum<K>(part[k]);
  // the pixel again (volatile index reads): nothing of it is held across the walk
  tile_ray<K>(det, h, w, chunk);
  const int bp = cta_pos(det).b;
  double J[kFrameGrads], av = 0.0, bv = 0.0;
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) J[k] = 0.0;
  if (h < det.H && w < det.W && chunk == 0) {
    const size_t pix = (static_cast<size_t>(bp) * det.H + h) * det.W + w;
    double d[3], ah, aw;
    reload_ray_d(frames + 12 * bp, det, h, w, d, ah, aw);
    const double L = ray_length(d);
    const OT e = static_cast<OT>(L * part[0]);
    img[pix] = e;
    av = static_cast<double>(e);  // the value the loss kernel reads
    bv = static_cast<double>(fixed[static_cast<size_t>(bp) * fixed_stride +
                                   static_cast<size_t>(h) * det.W + w]);
    if (part[0] != 0.0 || part[1] != 0.0 || part[2] != 0.0 || part[3] != 0.0 ||
        part[4] != 0.0 || part[5] != 0.0 || part[6] != 0.0) {
      double dEds[3], dEdp[3];
      sums_to_endpoint_grads(d, part[0], part + 1, part + 4, L, dEds, dEdp);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        J[a] = dEds[a];
        J[3 + a] = dEdp[a];
        J[6 + a] = ah * dEdp[a];
        J[9 + a] = aw * dEdp[a];
      }
    }
  }
  // Fixed-order CTA sums of w * J for w = 1, a, b: an xor butterfly in each
  // warp (all 36 chains independent), then the 4 warp rows in index order
  // after one CTA barrier -- one 36-sum row per CTA, so the reduction kernel
  // stays short for a single split pose.  A/B: the barrier costs ~0.6% at 256
  // poses against warps writing their own rows (warp rows made the C3
  // reduction 4x longer: +6 us per registration step), and a last-warp
  // counter instead (correct under release/acquire) is invisible to
  // compute-sanitizer's racecheck.
  __shared__ double warp_part[kThreads / 32][kLossSums];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int wsel = 0; wsel < 3; ++wsel) {
    const double wt = wsel == 0 ? 1.0 : (wsel == 1 ? av : bv);
    double v[kFrameGrads];
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) v[k] = wsel == 0 ? J[k] : wt * J[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1)
#pragma unroll
      for (int k = 0; k < kFrameGrads; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
    if (lane == 0)
#pragma unroll
      for (int k = 0; k < kFrameGrads; ++k) warp_part[warp][wsel * kFrameGrads + k] = v[k];
  }
  __syncthreads();
  if (threadIdx.x < kLossSums) {
    double sacc = 0.0;
#pragma unroll
    for (int q = 0; q < kThreads / 32; ++q) sacc += warp_part[q][threadIdx.x];
    const int blocks_per_pose = gridDim.x * gridDim.y;
    const CtaPos c = cta_pos(det);
    const int blk = c.ty * gridDim.x + c.tx;
    partials[(static_cast<size_t>(c.b) * blocks_per_pose + blk) * kLossSums + threadIdx.x] = sacc;
  }
}

// ------------------------------------------------------------ occupied box
// Per axis the min / max voxel index of any voxel that is not exactly zero
// (NaN counts as occupied), by integer atomics: order-free, so deterministic.
// out: lo[3] (init n), hi[3] (init -1, stored as max index; the host adds 1).
template <typename VT>
__global__ void __launch_bounds__(256)
    k_volume_bounds(const VT* __restrict__ vol, const GridDev g, int* __restrict__ out) {
  int lo[3] = {g.n[0], g.n[1], g.n[2]}, hi[3] = {-1, -1, -1};
  const int64_t n = g.total;
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const VT v = vol[f];
    if (!(v == VT(0))) {
      const int i = static_cast<int>(f % g.n[0]);
      const int j = static_cast<int>((f / g.n[0]) % g.n[1]);
      const int k = static_cast<int>(f / (static_cast<int64_t>(g.n[0]) * g.n[1]));
      lo[0] = min(lo[0], i); hi[0] = max(hi[0], i);
      lo[1] = min(lo[1], j); hi[1] = max(hi[1], j);
      lo[2] = min(lo[2], k); hi[2] = max(hi[2], k);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], off));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], off));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      atomicMin(out + a, lo[a]);
      atomicMax(out + 3 + a, hi[a]);
    }
  }
}

__global__ void k_bounds_init(const GridDev g, int* out) {
  if (threadIdx.x < 3) {
    out[threadIdx.x] = g.n[threadIdx.x];
    out[3 + threadIdx.x] = -1;
  }
}

__global__ void k_bounds_finish(int* out) {
  // [lo, max] -> [lo, max + 1); an empty volume -> [0, 0) on every axis
  if (threadIdx.x == 0) {
    const bool empty = out[3] < 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      out[a] = empty ? 0 : out[a];
      out[3 + a] = empty ? 0 : out[3 + a] + 1;
    }
  }
}

// The occupied hull: for each of the kHullDirs directions n_q, the min / max
// of n_q . (i, j, k) over the voxels that are not exactly zero (NaN counts),
// by integer atomics (order-free, deterministic).  out: lo[16], hi[16]
// (the first kHullDirs of each used).
template <typename VT>
__global__ void __launch_bounds__(256)
    k_volume_hull(const VT* __restrict__ vol, const GridDev g, int* __restrict__ out) {
  int lo[kHullDirs], hi[kHullDirs];
#pragma unroll
  for (int q = 0; q < kHullDirs; ++q) {
    lo[q] = INT_MAX;
    hi[q] = INT_MIN;
  }
  const int64_t n = g.total;
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (!(vol[f] == VT(0))) {
      const int c[3] = {static_cast<int>(f % g.n[0]), static_cast<int>((f / g.n[0]) % g.n[1]),
                        static_cast<int>(f / (static_cast<int64_t>(g.n[0]) * g.n[1]))};
#pragma unroll
      for (int q = 0; q < kHullDirs; ++q) {
        const int v = hull_dir(q, 0) * c[0] + hull_dir(q, 1) * c[1] + hull_dir(q, 2) * c[2];
        lo[q] = min(lo[q], v);
        hi[q] = max(hi[q], v);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < kHullDirs; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      lo[q] = min(lo[q], __shfl_xor_sync(0xffffffffu, lo[q], off));
      hi[q] = max(hi[q], __shfl_xor_sync(0xffffffffu, hi[q], off));
    }
  }
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int q = 0; q < kHullDirs; ++q) {
      atomicMin(out + q, lo[q]);
      atomicMax(out + 16 + q, hi[q]);
    }
  }
}

__global__ void k_hull_init(int* out) {
  if (threadIdx.x < 16) {
    out[threadIdx.x] = INT_MAX;
    out[16 + threadIdx.x] = INT_MIN;
  }
}

// ------------------------------------------------------ discrete signature
// Per pose, a 64-bit signature of every ray's traversal structure (SigVisitor:
// labels, used set, voxels, exit selector; a missed ray hashes as a miss),
// combined over the pixels by addition mod 2^64 of mix(pixel, ray hash) --
// order-free, so the atomics give the same bits every run.  Replaces
// gradients.py:124-142 discrete_signature for detect_fd_boundaries
// (gradients.py:145-167).  One thread per ray, the v4 visitor walk.
// kPerRay: each ray's own hash to sig[(b H + h) W + w] instead (per-ray
// boundary attribution of finite differences, fd.ray_fd_report); the pose
// signature is their wrapping sum.
template <typename VT, bool kPerRay>
__global__ void __launch_bounds__(kThreads)
    k_signature(const VT* __restrict__ vol, const GridDev g, const double* __restrict__ frames,
                const DetDev det, unsigned long long* __restrict__ sig) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, frames + 12 * cta_pos(det).b, tab);
  __syncthreads();
  int h, w, chunk;
  tile_ray<1>(det, h, w, chunk);
  const int b = cta_pos(det).b;
  uint64_t v = 0;
  if (h < det.H && w < det.W) {
    double s[3], p[3], ah, aw;
    pixel_ray(frames + 12 * b, det, h, w, s, p, ah, aw);
    Ray r;
    ray_setup(g, s, p, r);
    SigVisitor vis;
    if (r.hit) {
      vis.h = sig_mix(vis.h, static_cast<uint64_t>(r.lab_min));
      walk_select<VT, false>(vol, g, tab, r, vis);
    } else {
      vis.h = sig_mix(vis.h, 0xDEADull);  // miss
    }
    v = sig_mix(static_cast<uint64_t>(h) * det.W + w, vis.h);
    if constexpr (kPerRay) sig[(static_cast<size_t>(b) * det.H + h) * det.W + w] = v;
  }
  if constexpr (!kPerRay) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    if ((threadIdx.x & 31) == 0) atomicAdd(sig + b, static_cast<unsigned long long>(v));
  }
}

// One CTA per pose: the CTA partials of the three 12-vectors in a fixed order,
// combined with the loss kernel's coefficients into dL/dframe, then chained
// to the pose: dL/deta (drr_pose_grad's map).  Either output may be NULL.
// kReduceRows x 36 threads: thread (row r, sum k) adds tiles r, r + 8, ... of
// sum k (consecutive threads read consecutive doubles: coalesced), then the 8
// row totals are added in row order.  A single pose split over K lanes per ray
// has ~1250 small tiles; this keeps its reduction off the latency path.
constexpr int kReduceRows = 8;
constexpr int kReduceLossThreads = kReduceRows * kLossSums;  // 288
// With `reg.on`, the same kernel is also one registration iteration
// (registration.py:89-125): thread 0 applies register_update_one with this
// pose's dL/dframe and writes the frame of the updated pose for the next walk,
// so a whole iteration is three launches (walk, loss, this).
struct RegStep {
  int on;
  int iter;
  RegConfig cfg;
  double* eta;
  double* vel;
  const double* value;
  const int* status;
  int* state;
  int* n_rec;
  double* trace_eta;
  double* trace_loss;
  double* frames;  // next frames (the walk of the next iteration reads them)
  double iso0, iso1, iso2;
};

__global__ void __launch_bounds__(kReduceLossThreads)
    k_reduce_loss_grad(const double* __restrict__ partials, int blocks_per_pose,
                       const double* __restrict__ coef, const double* __restrict__ eta,
                       double* __restrict__ grad_frames, double* __restrict__ grad_eta,
                       RegStep reg) {
  const int b = blockIdx.x;
  const int k = threadIdx.x % kLossSums, r = threadIdx.x / kLossSums;
  __shared__ double sm[kReduceRows][kLossSums];
  __shared__ double gf[kFrameGrads];
  const double* base = partials + static_cast<size_t>(b) * blocks_per_pose * kLossSums + k;
  double v0 = 0.0, v1 = 0.0;  // tiles r + 16 i and r + 8 + 16 i: two independent chains
  int j = r;
  for (; j + kReduceRows < blocks_per_pose; j += 2 * kReduceRows) {
    v0 += base[static_cast<size_t>(j) * kLossSums];
    v1 += base[static_cast<size_t>(j + kReduceRows) * kLossSums];
  }
  if (j < blocks_per_pose) v0 += base[static_cast<size_t>(j) * kLossSums];
  sm[r][k] = v0 + v1;
  __syncthreads();
  if (threadIdx.x < kLossSums) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kReduceRows; ++q) t += sm[q][threadIdx.x];
    sm[0][threadIdx.x] = t;  // row 0 is read again only after the barrier below
  }
  __syncthreads();
  if (threadIdx.x < kFrameGrads) {
    const int c = threadIdx.x;
    const double c0 = coef[3 * b], c1 = coef[3 * b + 1], c2 = coef[3 * b + 2];
    const double gk = (c0 * sm[0][c] + c1 * sm[0][kFrameGrads + c]) + c2 * sm[0][2 * kFrameGrads + c];
    gf[c] = gk;
    if (grad_frames) grad_frames[b * kFrameGrads + c] = gk;
  }
  __syncthreads();
  if (threadIdx.x == 0 && grad_eta) {
    double ge[7];
    pose_grad(eta + 7 * b, gf, ge);
#pragma unroll
    for (int q = 0; q < 7; ++q) grad_eta[7 * b + q] = ge[q];
  }
  if (threadIdx.x == 0 && reg.on) {
    if (register_update_one(b, reg.eta, reg.vel, gf, reg.value[b], reg.status[b], reg.cfg,
                            reg.iter, reg.state, reg.n_rec, reg.trace_eta, reg.trace_loss))
      pose_frame_one(reg.eta + 7 * b, reg.iso0, reg.iso1, reg.iso2, reg.frames + 12 * b);
  }
}

// Contraction of the stored ray Jacobians with the upstream pixel gradient,
// reduced per CTA in the same fixed order as k_backward (16 x 8 tiles, warp
// butterflies, warps in index order), then k_reduce_frames.
template <typename GT>
__global__ void __launch_bounds__(kThreads)
    k_backward_jac(const double* __restrict__ jac, size_t npix_total, const DetDev det,
                   const GT* __restrict__ grad_img, double* __restrict__ partials) {
  int h, w, chunk;
  tile_ray<1>(det, h, w, chunk);
  const int b = cta_pos(det).b;
  double acc12[kFrameGrads];
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) acc12[k] = 0.0;
  if (h < det.H && w < det.W) {
    const size_t pix = (static_cast<size_t>(b) * det.H + h) * det.W + w;
    double js[3], jp[3];
    bool any = false;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      js[a] = __ldg(jac + a * npix_total + pix);
      jp[a] = __ldg(jac + (3 + a) * npix_total + pix);
      any = any || js[a] != 0.0 || jp[a] != 0.0;
    }
    if (any) {  // a missed ray contributes exactly nothing (as in k_backward)
      const double gpx = static_cast<double>(grad_img[pix]);
      const double ah = (static_cast<double>(h) - det.half_h) * det.pitch_y;
      const double aw = (static_cast<double>(w) - det.half_w) * det.pitch_x;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        acc12[a] = gpx * js[a];
        acc12[3 + a] = gpx * jp[a];
        acc12[6 + a] = gpx * ah * jp[a];
        acc12[9 + a] = gpx * aw * jp[a];
      }
    }
  }
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) {
    double v = acc12[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    acc12[k] = v;
  }
  __shared__ double warp_part[kThreads / 32][kFrameGrads];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) warp_part[warp][k] = acc12[k];
  }
  __syncthreads();
  if (threadIdx.x < kFrameGrads) {
    double v = 0.0;
#pragma unroll
    for (int q = 0; q < kThreads / 32; ++q) v += warp_part[q][threadIdx.x];
    const int blocks_per_pose = gridDim.x * gridDim.y;
    const CtaPos c = cta_pos(det);
    const int blk = c.ty * gridDim.x + c.tx;
    partials[(static_cast<size_t>(b) * blocks_per_pose + blk) * kFrameGrads +
             threadIdx.x] = v;
  }
}

// ------------------------------------------- loss + Jacobian contraction
// The stored-Jacobian step's tail in ONE kernel per image (one 8-CTA
// thread-block cluster, as k_image_loss): the two-pass neg-ZNCC / L2 moments
// give the value and the pixel gradient's affine coefficients (c0, c1, c2)
// on every thread; a third pass over the CTA's pixels contracts
// g_i = c0 + c1 a_i + c2 b_i (float64, never stored) with the ray's stored
// endpoint derivatives into the 12 frame sums, reduced in a fixed order
// (warp butterflies, warps, then the cluster's CTAs in rank order through
// distributed shared memory); rank 0 writes dL/dframe and, given eta,
// chains it to dL/deta.  Replaces k_image_loss + k_backward_jac +
// k_reduce_frames + k_pose_grad (four launches, and the fp32 pixel-gradient
// round trip) for gradients.py:61-69 with the losses of metrics.py:71-91.
// Launch-time choice (drr_loss_grad_jac): the TMA-staged contraction when the
// batch fills the GPU at least twice over (C2's 256 poses: 0.162 vs 0.197 ms),
// else the register-staged one (32 poses: 0.033 vs 0.038 ms) --
// scripts/gpu_lgj_tma.sh; both give the same bits.
#ifndef DRR_LGJ_TMA
#define DRR_LGJ_TMA 1
#endif
#ifndef DRR_LGJ_STAGES
#define DRR_LGJ_STAGES 3
#endif
constexpr int kLgjStages = DRR_LGJ_STAGES;  // Jacobian tiles in flight per CTA (TMA path)
template <typename IT, bool kTma>
__global__ void __cluster_dims__(kLossCluster, 1, 1) __launch_bounds__(kLossThreads)
    k_loss_grad_jac(const double* __restrict__ jac, size_t npix_total, const IT* __restrict__ img,
                    const IT* __restrict__ fixed, int64_t fixed_stride, const DetDev det,
                    int kind, double* __restrict__ value, int* __restrict__ status,
                    double* __restrict__ grad_frames, const double* __restrict__ eta,
                    double* __restrict__ grad_eta) {
  namespace cg = cooperative_groups;
  cg::cluster_group cluster = cg::this_cluster();
  __shared__ double sm[(kLossThreads / 32 + 2) * 5];
  __shared__ double wrow[kLossThreads / 32][kFrameGrads];
  __shared__ double ctot[kFrameGrads];
  const int b = blockIdx.y;
  const int rank = static_cast<int>(cluster.block_rank());
  const int64_t npix = static_cast<int64_t>(det.H) * det.W;
  const int64_t chunk = (npix + kLossCluster - 1) / kLossCluster;
  const int64_t lo = rank * chunk, hi = lo + chunk < npix ? lo + chunk : npix;
  const IT* a = img + static_cast<int64_t>(b) * npix;
  const IT* f = fixed + static_cast<int64_t>(b) * fixed_stride;
  const double N = static_cast<double>(npix);
  double c0 = 0.0, c1 = 0.0, c2 = 0.0;
  {
    double v[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    for (int64_t i = lo + threadIdx.x; i < hi; i += kLossThreads) {
      const double x = static_cast<double>(a[i]), y = static_cast<double>(f[i]);
      if (kind == 0) {
        v[0] += x; v[2] += y;
      } else {
        const double dd = x - y;
        v[0] += dd * dd;
      }
    }
    cluster_sum5<kLossThreads>(v, sm);
    if (kind == 0) {
      const double ma = v[0] / N, mb = v[2] / N;
      const double a0 = static_cast<double>(a[0]), b0 = static_cast<double>(f[0]);
      double w[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
      for (int64_t i = lo + threadIdx.x; i < hi; i += kLossThreads) {
        const double x = static_cast<double>(a[i]), y = static_cast<double>(f[i]);
        const double dx = x - ma, dy = y - mb;
        w[0] += dx * dx; w[1] += dy * dy; w[2] += dx * dy;
        w[3] += x != a0 ? 1.0 : 0.0;
        w[4] += y != b0 ? 1.0 : 0.0;
      }
      cluster_sum5<kLossThreads>(w, sm);
      const double sa = sqrt(w[0] / N), sb = sqrt(w[1] / N);
      const bool undefined = w[3] == 0.0 || w[4] == 0.0 || !(sa > 0.0) || !(sb > 0.0);
      const double raw = undefined ? NAN : w[2] / (N * sa * sb);
      const double scale = undefined ? NAN : -1.0 / (N * sa);
      c0 = scale * (raw * ma / sa - mb / sb);
      c1 = -scale * raw / sa;
      c2 = scale / sb;
      if (rank == 0 && threadIdx.x == 0) {
        value[b] = undefined ? NAN : -fmin(1.0, fmax(-1.0, raw));
        if (status) status[b] = undefined ? 1 : 0;
      }
    } else {
      const double norm = sqrt(v[0]);
      const double inv = norm > 0.0 ? 1.0 / norm : 0.0;
      c1 = inv;
      c2 = -inv;
      if (rank == 0 && threadIdx.x == 0) {
        value[b] = norm;
        if (status) status[b] = 0;
      }
    }
  }
  // contraction of this CTA's pixels (a missed ray's zero Jacobian adds nothing)
  double acc[kFrameGrads];
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) acc[k] = 0.0;
  const size_t pbase = static_cast<size_t>(b) * npix;
  // one pixel's contribution, in the same order whichever way its six
  // Jacobian entries arrived (thread t takes pixels lo + t, lo + t + T, ...)
  auto contract = [&](int64_t i, double xa, double yb, const double* js, const double* jp) {
    const double g = (c0 + c1 * xa) + c2 * yb;
    const int h = static_cast<int>(i / det.W), w = static_cast<int>(i % det.W);
    const double ah = (static_cast<double>(h) - det.half_h) * det.pitch_y;
    const double aw = (static_cast<double>(w) - det.half_w) * det.pitch_x;
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      acc[q] += g * js[q];
      acc[3 + q] += g * jp[q];
      acc[6 + q] += g * ah * jp[q];
      acc[9 + q] += g * aw * jp[q];
    }
  };
  if constexpr (kTma) {
  // The Jacobian streams through shared memory: per tile of kLossThreads
  // pixels, one thread issues six TMA bulk copies (one contiguous run per
  // component, cp.async.bulk ... mbarrier::complete_tx) kLgjStages tiles
  // ahead, so the loads in flight cost no registers (the register-staged
  // form held 128 registers: 2 CTAs per SM, ~44% of HBM).  Tiles whose run
  // is not 16-byte aligned / sized load directly.
  {
    __shared__ __align__(16) double stage[kLgjStages][6][kLossThreads];
    __shared__ __align__(8) unsigned long long bars[kLgjStages];
    const int64_t n = hi - lo;
    const int ntiles = static_cast<int>((n + kLossThreads - 1) / kLossThreads);
    // bulk copies need 16-byte aligned global runs: the Jacobian's base (any
    // pointer a C-ABI caller passes) and every run's first element
    const bool aligned = (reinterpret_cast<uintptr_t>(jac) & 15) == 0 &&
                         ((npix_total | (pbase + static_cast<size_t>(lo))) & 1) == 0;
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
    const uint32_t stage0 = static_cast<uint32_t>(__cvta_generic_to_shared(&stage[0][0][0]));
    auto tile_count = [&](int j) {
      const int64_t c = n - static_cast<int64_t>(j) * kLossThreads;
      return c < kLossThreads ? c : static_cast<int64_t>(kLossThreads);
    };
    auto tile_tma = [&](int j) { return aligned && (tile_count(j) & 1) == 0; };
    auto issue = [&](int j) {  // one thread
      if (j >= ntiles || !tile_tma(j)) return;
      const int k = j % kLgjStages;
      const uint32_t bytes = static_cast<uint32_t>(tile_count(j) * sizeof(double));
      const uint32_t bar = bar0 + 8u * k;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                   "r"(6u * bytes) : "memory");
      const size_t p0 = pbase + static_cast<size_t>(lo) + static_cast<size_t>(j) * kLossThreads;
#pragma unroll
      for (int q = 0; q < 6; ++q)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            ::"r"(stage0 + static_cast<uint32_t>(((k * 6 + q) * kLossThreads) * sizeof(double))),
            "l"(jac + q * npix_total + p0), "r"(bytes), "r"(bar) : "memory");
    };
    if (threadIdx.x == 0) {
      for (int k = 0; k < kLgjStages; ++k)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8u * k) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0)
      for (int j = 0; j < kLgjStages; ++j) issue(j);
    for (int j = 0; j < ntiles; ++j) {
      const int k = j % kLgjStages;
      const int64_t i = lo + static_cast<int64_t>(j) * kLossThreads + threadIdx.x;
      double js[3], jp[3];
      // the two image values (L2-resident after the moment passes) are
      // requested before waiting for the tile
      const double xa = i < hi ? static_cast<double>(a[i]) : 0.0;
      const double yb = i < hi ? static_cast<double>(f[i]) : 0.0;
      if (tile_tma(j)) {
        const uint32_t phase = static_cast<uint32_t>((j / kLgjStages) & 1);
        // bounded wait: a tile that never lands (a bad address or byte
        // count) traps after 2 s of wall time -- a launch error for the
        // caller instead of a kernel that never retires
        asm volatile(
            "{\n .reg .pred p;\n .reg .u64 t0, t1;\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @p bra DONE_%=;\n"
            " mov.u64 t0, %%globaltimer;\n"
            " WAIT_%=:\n"
            " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
            " @p bra DONE_%=;\n"
            " mov.u64 t1, %%globaltimer;\n"
            " sub.u64 t1, t1, t0;\n"
            " setp.gt.u64 p, t1, 2000000000;\n"
            " @p trap;\n"
            " bra WAIT_%=;\n"
            " DONE_%=:\n}\n" ::"r"(bar0 + 8u * k), "r"(phase) : "memory");
        if (i < hi) {
#pragma unroll
          for (int q = 0; q < 3; ++q) {
            js[q] = stage[k][q][threadIdx.x];
            jp[q] = stage[k][3 + q][threadIdx.x];
          }
        }
      } else if (i < hi) {
        const size_t pix = pbase + static_cast<size_t>(i);
#pragma unroll
        for (int q = 0; q < 3; ++q) {
          js[q] = __ldg(jac + q * npix_total + pix);
          jp[q] = __ldg(jac + (3 + q) * npix_total + pix);
        }
      }
      if (i < hi) contract(i, xa, yb, js, jp);
      __syncthreads();  // every thread is done with buffer k
      if (threadIdx.x == 0) issue(j + kLgjStages);
    }
  }
  } else {
  // kLossBatch pixels' loads in flight before any is accumulated (in order)
  for (int64_t i0 = lo + threadIdx.x; i0 < hi; i0 += kLossThreads * kLossBatch) {
    double js[kLossBatch][3], jp[kLossBatch][3], xa[kLossBatch], yb[kLossBatch];
#pragma unroll
    for (int u = 0; u < kLossBatch; ++u) {
      const int64_t i = i0 + static_cast<int64_t>(u) * kLossThreads;
      const bool in = i < hi;
      const size_t pix = pbase + (in ? i : lo);
#pragma unroll
      for (int q = 0; q < 3; ++q) {
        js[u][q] = in ? __ldg(jac + q * npix_total + pix) : 0.0;
        jp[u][q] = in ? __ldg(jac + (3 + q) * npix_total + pix) : 0.0;
      }
      xa[u] = in ? static_cast<double>(a[i]) : 0.0;
      yb[u] = in ? static_cast<double>(f[i]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kLossBatch; ++u) {
      const int64_t i = i0 + static_cast<int64_t>(u) * kLossThreads;
      if (i >= hi) break;
      contract(i, xa[u], yb[u], js[u], jp[u]);
    }
  }
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1)
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) acc[k] += __shfl_xor_sync(0xffffffffu, acc[k], off);
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) wrow[warp][k] = acc[k];
  __syncthreads();
  if (threadIdx.x < kFrameGrads) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < kLossThreads / 32; ++q) t += wrow[q][threadIdx.x];
    ctot[threadIdx.x] = t;
  }
  cluster.sync();  // every CTA's 12 totals are visible cluster-wide
  if (rank == 0) {
    __shared__ double gf[kFrameGrads];
    if (threadIdx.x < kFrameGrads) {
      double t = 0.0;
      for (int r = 0; r < kLossCluster; ++r) t += *cluster.map_shared_rank(ctot + threadIdx.x, r);
      gf[threadIdx.x] = t;
      if (grad_frames) grad_frames[b * kFrameGrads + threadIdx.x] = t;
    }
    __syncthreads();
    if (threadIdx.x == 0 && grad_eta != nullptr) {
      double ge[7];
      pose_grad(eta + 7 * b, gf, ge);
#pragma unroll
      for (int q = 0; q < 7; ++q) grad_eta[7 * b + q] = ge[q];
    }
  }
  cluster.sync();  // no CTA leaves while rank 0 reads its totals
}

// One CTA per pose: each thread sums a fixed strided subset of the CTA
// partials, then a fixed shared-memory tree.
constexpr int kReduceThreads = 128;
__global__ void __launch_bounds__(kReduceThreads)
    k_reduce_frames(const double* __restrict__ partials, int blocks_per_pose,
                    double* __restrict__ grad_frames) {
  const int b = blockIdx.x;
  __shared__ double sm[kReduceThreads][kFrameGrads + 1];
  double v[kFrameGrads];
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) v[k] = 0.0;
  const double* base = partials + static_cast<size_t>(b) * blocks_per_pose * kFrameGrads;
  for (int j = threadIdx.x; j < blocks_per_pose; j += kReduceThreads) {
#pragma unroll
    for (int k = 0; k < kFrameGrads; ++k) v[k] += base[j * kFrameGrads + k];
  }
#pragma unroll
  for (int k = 0; k < kFrameGrads; ++k) sm[threadIdx.x][k] = v[k];
  __syncthreads();
  for (int stride = kReduceThreads / 2; stride > 0; stride >>= 1) {
    if (threadIdx.x < stride) {
#pragma unroll
      for (int k = 0; k < kFrameGrads; ++k)
        sm[threadIdx.x][k] += sm[threadIdx.x + stride][k];
    }
    __syncthreads();
  }
  if (threadIdx.x < kFrameGrads)
    grad_frames[b * kFrameGrads + threadIdx.x] = sm[0][threadIdx.x];
}

// ----------------------------------------------------------- explicit rays
constexpr int kRayThreads = 128;

template <typename VT>
__global__ void __launch_bounds__(kRayThreads)
    k_raysum(const VT* __restrict__ vol, const GridDev g,
             const double* __restrict__ src, const double* __restrict__ pix,
             int64_t n_rays, double* __restrict__ out) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, src, tab);
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_rays) return;
  double s[3] = {__ldg(src), __ldg(src + 1), __ldg(src + 2)};
  double p[3] = {__ldg(pix + 3 * i), __ldg(pix + 3 * i + 1), __ldg(pix + 3 * i + 2)};
  Ray r;
  ray_setup(g, s, p, r);
  double e = 0.0;
  if (r.hit) {
    LeanSums o;
    walk_sums<VT, kLeanSum, false>(vol, g, tab, r, o);
    e = ray_length(r) * o.acc;
  }
  out[i] = e;
}

// With n_tan > 0 (drr_raysum_tangents) the epilogue contracts the endpoint
// derivatives with the caller's tangents instead of storing them:
// d_energy[i, t] = dE/ds . d_source[:, t] + dE/dp . d_pixels[i, :, t]
// (the reference's siddon_raysum_grad contract, _native.pyx:196-282), in a
// fixed order per (ray, tangent).
template <typename VT>
__global__ void __launch_bounds__(kRayThreads)
    k_raysum_grad(const VT* __restrict__ vol, const GridDev g,
                  const double* __restrict__ src,
                  const double* __restrict__ pix, int64_t n_rays,
                  double* __restrict__ out, double* __restrict__ dEds,
                  double* __restrict__ dEdp, int n_tan = 0,
                  const double* __restrict__ dsrc = nullptr,
                  const double* __restrict__ dpix = nullptr,
                  double* __restrict__ denergy = nullptr) {
  extern __shared__ __align__(16) double tab[];
  build_plane_table(g, src, tab);
  __syncthreads();
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_rays) return;
  double s[3] = {__ldg(src), __ldg(src + 1), __ldg(src + 2)};
  double p[3] = {__ldg(pix + 3 * i), __ldg(pix + 3 * i + 1), __ldg(pix + 3 * i + 2)};
  Ray r;
  ray_setup(g, s, p, r);
  double e = 0.0, gs[3] = {0.0, 0.0, 0.0}, gp[3] = {0.0, 0.0, 0.0};
  if (r.hit) {
    LeanSums o;
    walk_sums<VT, kLeanGrad, false>(vol, g, tab, r, o);
    const double L = ray_length(r);
    e = L * o.acc;
    const double G[3] = {o.G0, o.G1, o.G2}, Hh[3] = {o.H0, o.H1, o.H2};
    sums_to_endpoint_grads(r, o.acc, G, Hh, L, gs, gp);
  }
  out[i] = e;
  if (n_tan > 0) {
    const double* dp = dpix + 3 * i * n_tan;
    for (int t = 0; t < n_tan; ++t) {
      double v = gs[0] * __ldg(dsrc + t);
      v = v + gs[1] * __ldg(dsrc + n_tan + t);
      v = v + gs[2] * __ldg(dsrc + 2 * n_tan + t);
      v = v + gp[0] * __ldg(dp + t);
      v = v + gp[1] * __ldg(dp + n_tan + t);
      v = v + gp[2] * __ldg(dp + 2 * n_tan + t);
      denergy[i * n_tan + t] = v;
    }
    return;
  }
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dEds[3 * i + a] = gs[a];
    dEdp[3 * i + a] = gp[a];
  }
}

}  // namespace drr

// =================================================================== C ABI
#ifndef DRR_KERNELS_ONLY  // (scripts/sass_harness.cu compiles single kernels for SASS study)
namespace {

thread_local char g_err[512] = "";

int fail(int code, const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

int check_launch(const char* what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess)
    return fail(DRR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return DRR_OK;
}

// Dynamic shared memory: the per-CTA plane table plus the walk's per-thread
// ray records (every walk kernel has 128 threads).  Only what the walk mode
// uses is allocated -- shared memory comes out of the same 228 KB per SM as
// the L1 cache that serves the CT gathers.  >48 KB needs opt-in.
size_t table_bytes(const drr::GridDev& g, bool grad_walk) {
  const size_t per_thread = drr::lean_rec_doubles(grad_walk);
  return (static_cast<size_t>(drr::plane_table_span(g)) + per_thread * 128) * sizeof(double);
}

template <typename Kernel>
void ensure_smem(Kernel kernel, size_t bytes) {
  if (bytes > 48 * 1024)
    cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(bytes));
}

int make_grid(const drr_grid* in, drr::GridDev& g) {
  if (in == nullptr) return fail(DRR_ERR_INVALID_ARGUMENT, "grid is NULL");
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) {
    if (in->dims[a] < 1)
      return fail(DRR_ERR_INVALID_ARGUMENT, "dims must be >= 1, got %lld on axis %d",
                  (long long)in->dims[a], a);
    if (!(in->spacing[a] > 0.0) || !isfinite(in->spacing[a]))
      return fail(DRR_ERR_INVALID_ARGUMENT, "spacing must be positive, got %g on axis %d",
                  in->spacing[a], a);
    if (!isfinite(in->origin[a]))
      return fail(DRR_ERR_INVALID_ARGUMENT, "origin must be finite");
    total *= in->dims[a];
  }
  if (total >= (int64_t(1) << 31))
    return fail(DRR_ERR_INVALID_ARGUMENT, "volume has %lld voxels; limit is 2^31-1",
                (long long)total);
  for (int a = 0; a < 3; ++a) {
    g.n[a] = static_cast<int>(in->dims[a]);
    g.sp[a] = in->spacing[a];
    g.o[a] = in->origin[a];
    // Same expression as _native.pyx:34 (host double arithmetic is IEEE;
    // built without FMA contraction).
    volatile double prod = static_cast<double>(in->dims[a]) * in->spacing[a];
    g.hi[a] = in->origin[a] + prod;
  }
  g.stride[0] = 1;
  g.stride[1] = g.n[0];
  g.stride[2] = g.n[0] * g.n[1];
  g.total = static_cast<int>(total);
  // the occupied box (drr_volume_bounds); all-zero occ_hi = the whole volume
  const bool whole = in->occ_hi[0] == 0 && in->occ_hi[1] == 0 && in->occ_hi[2] == 0 &&
                     in->occ_lo[0] == 0 && in->occ_lo[1] == 0 && in->occ_lo[2] == 0;
  for (int a = 0; a < 3; ++a) {
    const int64_t lo = whole ? 0 : in->occ_lo[a], hi = whole ? in->dims[a] : in->occ_hi[a];
    if (lo < 0 || hi < lo || hi > in->dims[a])
      return fail(DRR_ERR_INVALID_ARGUMENT, "occupied box [%lld, %lld) outside [0, %lld] on axis %d",
                  (long long)lo, (long long)hi, (long long)in->dims[a], a);
    // the plane table's rounding of P(k) = o + k*sp (whole volume: o and hi)
    volatile double plo = static_cast<double>(lo) * in->spacing[a];
    volatile double phi = static_cast<double>(hi) * in->spacing[a];
    g.tlo[a] = in->origin[a] + plo;
    g.thi[a] = in->origin[a] + phi;
    g.isp[a] = static_cast<float>(1.0 / in->spacing[a]);
    g.ispd[a] = 1.0 / in->spacing[a];
  }
  // the occupied hull (drr_volume_hull): n . (i, j, k) ranges of the non-zero
  // voxels -> the supports of their boxes [i, i+1] x ..., widened by 1/16 voxel
  g.hull = in->hull_valid == drr::kHullDirs && !whole;
  for (int q = 0; q < drr::kHullDirs; ++q) {
    int pos = 0, neg = 0, l1 = 0;
    for (int a = 0; a < 3; ++a) {
      const int c = drr::hull_dir(q, a);
      pos += c > 0 ? c : 0;
      neg += c < 0 ? c : 0;
      l1 += c > 0 ? c : -c;
    }
    g.hlo[q] = static_cast<float>(in->hull_lo[q] + neg) - 0.0625f * l1;
    g.hhi[q] = static_cast<float>(in->hull_hi[q] + pos) + 0.0625f * l1;
  }
  if (table_bytes(g, true) > 227 * 1024)
    return fail(DRR_ERR_INVALID_ARGUMENT, "plane table of %zu bytes exceeds shared memory",
                table_bytes(g, true));
  return DRR_OK;
}

int make_det(const drr_detector* in, drr::DetDev& d) {
  if (in == nullptr) return fail(DRR_ERR_INVALID_ARGUMENT, "detector is NULL");
  if (in->height < 1 || in->width < 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "detector must be at least 1x1, got %dx%d",
                in->height, in->width);
  if (!(in->pitch_x > 0.0) || !(in->pitch_y > 0.0) || !isfinite(in->pitch_x) ||
      !isfinite(in->pitch_y))
    return fail(DRR_ERR_INVALID_ARGUMENT, "pixel pitch must be positive");
  if (in->ray_split != 0 && in->ray_split != 1 && in->ray_split != 2 && in->ray_split != 4 &&
      in->ray_split != 8)
    return fail(DRR_ERR_INVALID_ARGUMENT, "ray_split must be 0, 1, 2, 4 or 8, got %d",
                in->ray_split);
  d.H = in->height;
  d.W = in->width;
  d.split = in->ray_split;
  d.pose_group = 1;
  d.pitch_x = in->pitch_x;
  d.pitch_y = in->pitch_y;
  d.half_h = static_cast<double>(in->height - 1) / 2.0;
  d.half_w = static_cast<double>(in->width - 1) / 2.0;
  return DRR_OK;
}

// Streaming multiprocessors of the current device (cudaDevAttrMultiProcessorCount,
// cached per device): the auto ray split and the pose-group size below are
// sized in waves of resident CTAs, so a MIG slice or another SKU gets its own.
int device_sms() {
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}
constexpr int kResidentCtasPerSm = 6;  // the walk kernels' launch bounds (DRR_*_MINB)

// Threads per ray: explicit, or auto = the smallest K in {1, 2, 4, 8} with
// B*H*W*K >= 0.6 waves of resident threads (SMs x 6 CTAs x 128; 148 SMs on
// a B200).  A/B (scripts/kbench_split.py, one pose, fwd+jac+contraction /
// forward ms for K = 1 / 2 / 4 / 8), with occupied-box trimming
// (profiles/r02/rec1_kbench_split.json): C2 200^2 0.168 / 0.116 / 0.119 /
// 0.130 and 0.129 / 0.082 / 0.085 / 0.097 (K = 2 chosen); C1 100^2 forward
// 0.045 / 0.033 / 0.027 / 0.025 (K = 8).  (Untrimmed, r01: C2 0.218 / 0.150 /
// 0.147 / 0.161 -- the shorter trimmed rays favour fewer, longer chunks.)
int ray_split(const drr::DetDev& d, int n_poses) {
  if (d.split > 0) return d.split;
  const double rays = static_cast<double>(n_poses) * d.H * d.W;
  const double wave = static_cast<double>(device_sms()) * kResidentCtasPerSm * drr::kThreads;
  int k = 1;
  while (k < 8 && rays * k < 0.6 * wave) k *= 2;
  return k;
}

// Poses interleaved tile by tile in the CTA order (DetDev::pose_group):
// groups of ~18 waves of resident CTAs (16384 CTAs on a 148-SM B200, scaled by
// the SM count: G = 16384 x SMs / 148 / tiles per pose).  Interleaving pays when a
// tile's CT footprint is large next to the pose spread (nearby poses share
// it), and costs when tiles are many and small (each pose then brings its own
// lines).  A/B (scripts/gpu_ab_fast.sh, gpu_ab_configs.sh; fwd+jac ms or
// DRR/s for G = 1 / 2 / 4 / 8 / 16 / whole batch):
//   C2 (32 poses, 325 tiles):    2.40 / 2.35 / 2.30 / 2.25 / 2.24 / 2.24 ms
//   C4 (1024 poses, 512 tiles):  11473 / 11599 / 11760 / 11846 / 11895 / 12010
//   C5 (16 poses, 8192 tiles):   492 / 494 / 493 / 483 / 477 / 477
// DRR_POSE_GROUP > 0 fixes G (A/B builds).
#ifndef DRR_POSE_GROUP
#define DRR_POSE_GROUP 0
#endif
int pose_group(int n_poses, unsigned tiles) {
  const long group_ctas = 16384L * device_sms() / 148;
  long G = DRR_POSE_GROUP > 0 ? DRR_POSE_GROUP : group_ctas / (tiles > 0 ? tiles : 1);
  return static_cast<int>(G < 1 ? 1 : (G > n_poses ? n_poses : G));
}

// The launch grid of a pose kernel; also sets d.pose_group for it.
dim3 pose_grid(drr::DetDev& d, int n_poses, int K) {
  int tw, th;
  switch (K) {
    case 1: tw = drr::Tile<1>::W; th = drr::Tile<1>::H; break;
    case 2: tw = drr::Tile<2>::W; th = drr::Tile<2>::H; break;
    case 4: tw = drr::Tile<4>::W; th = drr::Tile<4>::H; break;
    default: tw = drr::Tile<8>::W; th = drr::Tile<8>::H; break;
  }
  const dim3 grd((d.W + tw - 1) / tw, (d.H + th - 1) / th, n_poses);
  d.pose_group = pose_group(n_poses, grd.x * grd.y);
  return grd;
}

// Dispatch a runtime K in {1, 2, 4, 8} to a template instantiation.
#define DRR_DISPATCH_K(K, ...)                      \
  switch (K) {                                       \
    case 1: { constexpr int kK = 1; __VA_ARGS__ } break; \
    case 2: { constexpr int kK = 2; __VA_ARGS__ } break; \
    case 4: { constexpr int kK = 4; __VA_ARGS__ } break; \
    default: { constexpr int kK = 8; __VA_ARGS__ } break; \
  }

template <typename VT, typename GT>
void launch_backward(const VT* vol, const drr::GridDev& g,
                            const double* frames, const drr::DetDev& det,
                            int n_poses, const GT* grad, void* img,
                            int img_dtype, double* partials, cudaStream_t st) {
  drr::DetDev d = det;
  const size_t smem = table_bytes(g, true);
  const int K = ray_split(d, n_poses);
  const dim3 grd = pose_grid(d, n_poses, K);
  DRR_DISPATCH_K(K,
    if (img_dtype == 1) {
      ensure_smem(drr::k_backward<VT, GT, double, kK>, smem);
      drr::k_backward<VT, GT, double, kK><<<grd, drr::kThreads, smem, st>>>(
          vol, g, frames, d, grad, static_cast<double*>(img), partials);
    } else {
      ensure_smem(drr::k_backward<VT, GT, float, kK>, smem);
      drr::k_backward<VT, GT, float, kK><<<grd, drr::kThreads, smem, st>>>(
          vol, g, frames, d, grad, static_cast<float*>(img), partials);
    })
}

}  // namespace

namespace {
template <typename ST, typename DT>
void launch_pack(const ST* src, int order, const int64_t* dims, int clamp, DT* dst,
                 cudaStream_t st) {
  const int64_t n = dims[0] * dims[1] * dims[2];
  if (order == DRR_ORDER_XFASTEST) {
    const int64_t blocks = (n + 255) / 256;
    drr::k_pack_linear<ST, DT><<<static_cast<unsigned>(blocks < 148 * 32 ? blocks : 148 * 32), 256,
                                 0, st>>>(src, n, clamp, dst);
  } else {
    const dim3 grd(static_cast<unsigned>((dims[2] + 31) / 32),
                   static_cast<unsigned>((dims[0] + 31) / 32), static_cast<unsigned>(dims[1]));
    drr::k_pack_zfastest<ST, DT><<<grd, dim3(32, 8), 0, st>>>(
        src, static_cast<int>(dims[0]), static_cast<int>(dims[1]), static_cast<int>(dims[2]),
        clamp, dst);
  }
}
template <typename DT>
void dispatch_pack(const void* src, int src_type, int order, const int64_t* dims, int clamp,
                   DT* dst, cudaStream_t st) {
  switch (src_type) {
    case DRR_SRC_F32: launch_pack(static_cast<const float*>(src), order, dims, clamp, dst, st); break;
    case DRR_SRC_F64: launch_pack(static_cast<const double*>(src), order, dims, clamp, dst, st); break;
    case DRR_SRC_I16: launch_pack(static_cast<const int16_t*>(src), order, dims, clamp, dst, st); break;
    default: launch_pack(static_cast<const uint8_t*>(src), order, dims, clamp, dst, st); break;
  }
}
}  // namespace

static int loss_step(const void* d_vol, int vol_dtype, const drr_grid* grid,
                     const double* d_frames, const double* d_eta, int32_t n_poses,
                     const drr_detector* det, const void* d_fixed, int64_t fixed_stride, int kind,
                     void* d_img, int img_dtype, double* d_value, int* d_status,
                     double* d_grad_frames, double* d_grad_eta, void* d_workspace,
                     size_t workspace_bytes, void* stream, const drr::RegStep& reg) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, true);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  if (kind != DRR_LOSS_NEG_ZNCC && kind != DRR_LOSS_L2)
    return fail(DRR_ERR_INVALID_ARGUMENT, "loss kind must be neg_zncc (0) or l2 (1), got %d", kind);
  const int64_t npix = static_cast<int64_t>(d.H) * d.W;
  if (fixed_stride != 0 && fixed_stride != npix)
    return fail(DRR_ERR_INVALID_ARGUMENT, "fixed_stride must be 0 or H*W");
  if (d_img == nullptr || d_fixed == nullptr || d_value == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "d_img, d_fixed and d_value must not be NULL");
  if (d_grad_eta != nullptr && d_eta == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "d_grad_eta needs d_eta");
  if ((vol_dtype != DRR_VOL_F32 && vol_dtype != DRR_VOL_F64) || (img_dtype != 0 && img_dtype != 1))
    return fail(DRR_ERR_INVALID_ARGUMENT, "bad dtypes vol=%d img=%d", vol_dtype, img_dtype);
  const size_t need = drr_loss_grad_workspace_size(n_poses, det);
  if (workspace_bytes < need || d_workspace == nullptr)
    return fail(DRR_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int K = ray_split(d, n_poses);
  const dim3 grd = pose_grid(d, n_poses, K);
  const int rows = static_cast<int>(grd.x * grd.y);  // one 36-sum row per CTA
  double* partials = static_cast<double*>(d_workspace);
  double* coef = partials + static_cast<size_t>(n_poses) * rows * drr::kLossSums;
  DRR_DISPATCH_K(K,
    if (vol_dtype == DRR_VOL_F32 && img_dtype == 0) {
      ensure_smem(drr::k_forward_loss<float, float, kK>, smem);
      drr::k_forward_loss<float, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<float*>(d_img),
          static_cast<const float*>(d_fixed), fixed_stride, partials);
    } else if (vol_dtype == DRR_VOL_F32) {
      ensure_smem(drr::k_forward_loss<float, double, kK>, smem);
      drr::k_forward_loss<float, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<double*>(d_img),
          static_cast<const double*>(d_fixed), fixed_stride, partials);
    } else if (img_dtype == 1) {
      ensure_smem(drr::k_forward_loss<double, double, kK>, smem);
      drr::k_forward_loss<double, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<double*>(d_img),
          static_cast<const double*>(d_fixed), fixed_stride, partials);
    } else {
      ensure_smem(drr::k_forward_loss<double, float, kK>, smem);
      drr::k_forward_loss<double, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<float*>(d_img),
          static_cast<const float*>(d_fixed), fixed_stride, partials);
    })
  rc = check_launch("drr_forward_loss_grad/walk");
  if (rc) return rc;
  for (int32_t i0 = 0; i0 < n_poses; i0 += 65535) {
    const int32_t n = n_poses - i0 < 65535 ? n_poses - i0 : 65535;
    const dim3 lg(drr::kLossCluster, n);
    const int64_t fo = fixed_stride * i0, io = npix * i0;
    int* sts = d_status ? d_status + i0 : nullptr;
    if (img_dtype == 0)
      drr::k_image_loss<float><<<lg, drr::kLossThreads, 0, st>>>(
          static_cast<const float*>(d_img) + io, static_cast<const float*>(d_fixed) + fo,
          fixed_stride, npix, kind, d_value + i0, nullptr, sts, coef + 3 * i0);
    else
      drr::k_image_loss<double><<<lg, drr::kLossThreads, 0, st>>>(
          static_cast<const double*>(d_img) + io, static_cast<const double*>(d_fixed) + fo,
          fixed_stride, npix, kind, d_value + i0, nullptr, sts, coef + 3 * i0);
    rc = check_launch("drr_forward_loss_grad/loss");
    if (rc) return rc;
  }
  if (d_grad_frames == nullptr && d_grad_eta == nullptr && !reg.on) return DRR_OK;
  drr::k_reduce_loss_grad<<<n_poses, drr::kReduceLossThreads, 0, st>>>(
      partials, rows, coef, d_eta, d_grad_frames, d_grad_eta, reg);
  return check_launch("drr_forward_loss_grad/reduce");
}


extern "C" {

const char* drr_last_error(void) { return g_err; }

int drr_version(void) { return 2; }

int drr_struct_sizes(size_t* grid, size_t* detector, size_t* reg_config, size_t* peer_handle) {
  if (grid) *grid = sizeof(drr_grid);
  if (detector) *detector = sizeof(drr_detector);
  if (reg_config) *reg_config = sizeof(drr_reg_config);
  if (peer_handle) *peer_handle = sizeof(drr_peer_handle);
  return DRR_OK;
}

int drr_raysum(const void* d_vol, int vol_dtype, const drr_grid* grid,
               const double* d_src, const double* d_pix, int64_t n_rays,
               double* d_out, void* stream) {
  drr::GridDev g;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, false);
  if (n_rays < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_rays < 0");
  if (n_rays == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned blocks = static_cast<unsigned>((n_rays + drr::kRayThreads - 1) / drr::kRayThreads);
  if (vol_dtype == DRR_VOL_F32) {
    ensure_smem(drr::k_raysum<float>, smem);
    drr::k_raysum<float><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const float*>(d_vol), g, d_src, d_pix, n_rays, d_out);
  }
  else if (vol_dtype == DRR_VOL_F64) {
    ensure_smem(drr::k_raysum<double>, smem);
    drr::k_raysum<double><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const double*>(d_vol), g, d_src, d_pix, n_rays, d_out);
  }
  else
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  return check_launch("drr_raysum");
}

int drr_raysum_endpoint_grad(const void* d_vol, int vol_dtype,
                             const drr_grid* grid, const double* d_src,
                             const double* d_pix, int64_t n_rays,
                             double* d_out, double* d_dEds, double* d_dEdp,
                             void* stream) {
  drr::GridDev g;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, true);
  if (n_rays < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_rays < 0");
  if (n_rays == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned blocks = static_cast<unsigned>((n_rays + drr::kRayThreads - 1) / drr::kRayThreads);
  if (vol_dtype == DRR_VOL_F32) {
    ensure_smem(drr::k_raysum_grad<float>, smem);
    drr::k_raysum_grad<float><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const float*>(d_vol), g, d_src, d_pix, n_rays, d_out, d_dEds, d_dEdp);
  }
  else if (vol_dtype == DRR_VOL_F64) {
    ensure_smem(drr::k_raysum_grad<double>, smem);
    drr::k_raysum_grad<double><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const double*>(d_vol), g, d_src, d_pix, n_rays, d_out, d_dEds, d_dEdp);
  }
  else
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  return check_launch("drr_raysum_endpoint_grad");
}

int drr_raysum_tangents(const void* d_vol, int vol_dtype, const drr_grid* grid,
                        const double* d_src, const double* d_dsrc, const double* d_pix,
                        const double* d_dpix, int64_t n_rays, int32_t n_tangents,
                        double* d_out, double* d_denergy, void* stream) {
  drr::GridDev g;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, true);
  if (n_rays < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_rays < 0");
  if (n_tangents < 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_tangents must be >= 1, got %d", n_tangents);
  if (n_rays == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const unsigned blocks = static_cast<unsigned>((n_rays + drr::kRayThreads - 1) / drr::kRayThreads);
  if (vol_dtype == DRR_VOL_F32) {
    ensure_smem(drr::k_raysum_grad<float>, smem);
    drr::k_raysum_grad<float><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const float*>(d_vol), g, d_src, d_pix, n_rays, d_out, nullptr, nullptr,
        n_tangents, d_dsrc, d_dpix, d_denergy);
  } else if (vol_dtype == DRR_VOL_F64) {
    ensure_smem(drr::k_raysum_grad<double>, smem);
    drr::k_raysum_grad<double><<<blocks, drr::kRayThreads, smem, st>>>(
        static_cast<const double*>(d_vol), g, d_src, d_pix, n_rays, d_out, nullptr, nullptr,
        n_tangents, d_dsrc, d_dpix, d_denergy);
  } else {
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  }
  return check_launch("drr_raysum_tangents");
}

int drr_forward(const void* d_vol, int vol_dtype, const drr_grid* grid,
                const double* d_frames, int32_t n_poses,
                const drr_detector* det, void* d_img, int img_dtype,
                void* stream) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, false);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int K = ray_split(d, n_poses);
  const dim3 grd = pose_grid(d, n_poses, K);
  if ((vol_dtype != DRR_VOL_F32 && vol_dtype != DRR_VOL_F64) || (img_dtype != 0 && img_dtype != 1))
    return fail(DRR_ERR_INVALID_ARGUMENT, "bad dtypes vol=%d img=%d", vol_dtype, img_dtype);
  DRR_DISPATCH_K(K,
    if (vol_dtype == DRR_VOL_F32 && img_dtype == 0) {
      ensure_smem(drr::k_forward<float, float, kK>, smem);
      drr::k_forward<float, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<float*>(d_img));
    } else if (vol_dtype == DRR_VOL_F32) {
      ensure_smem(drr::k_forward<float, double, kK>, smem);
      drr::k_forward<float, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<double*>(d_img));
    } else if (img_dtype == 1) {
      ensure_smem(drr::k_forward<double, double, kK>, smem);
      drr::k_forward<double, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<double*>(d_img));
    } else {
      ensure_smem(drr::k_forward<double, float, kK>, smem);
      drr::k_forward<double, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<float*>(d_img));
    })
  return check_launch("drr_forward");
}

size_t drr_backward_workspace_size(int32_t n_poses, const drr_detector* det) {
  drr::DetDev d;
  if (make_det(det, d) || n_poses < 0) return 0;
  // max over the re-walk tiling (K threads per ray) and the Jacobian
  // contraction's 16 x 8 tiles
  const dim3 grd = pose_grid(d, 1, ray_split(d, n_poses));
  const dim3 grd1 = pose_grid(d, 1, 1);
  const size_t tiles = grd.x * grd.y > grd1.x * grd1.y ? grd.x * grd.y : grd1.x * grd1.y;
  return static_cast<size_t>(n_poses) * tiles * drr::kFrameGrads * sizeof(double);
}

int drr_forward_jac(const void* d_vol, int vol_dtype, const drr_grid* grid,
                    const double* d_frames, int32_t n_poses, const drr_detector* det,
                    void* d_img, int img_dtype, double* d_jac, void* stream) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, true);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  if (d_jac == nullptr || d_img == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "d_img and d_jac must not be NULL");
  if ((vol_dtype != DRR_VOL_F32 && vol_dtype != DRR_VOL_F64) || (img_dtype != 0 && img_dtype != 1))
    return fail(DRR_ERR_INVALID_ARGUMENT, "bad dtypes vol=%d img=%d", vol_dtype, img_dtype);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int K = ray_split(d, n_poses);
  const dim3 grd = pose_grid(d, n_poses, K);
  const size_t npix = static_cast<size_t>(n_poses) * d.H * d.W;
  DRR_DISPATCH_K(K,
    if (vol_dtype == DRR_VOL_F32 && img_dtype == 0) {
      ensure_smem(drr::k_forward_jac<float, float, kK>, smem);
      drr::k_forward_jac<float, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<float*>(d_img), d_jac, npix);
    } else if (vol_dtype == DRR_VOL_F32) {
      ensure_smem(drr::k_forward_jac<float, double, kK>, smem);
      drr::k_forward_jac<float, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, static_cast<double*>(d_img), d_jac, npix);
    } else if (img_dtype == 1) {
      ensure_smem(drr::k_forward_jac<double, double, kK>, smem);
      drr::k_forward_jac<double, double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<double*>(d_img), d_jac, npix);
    } else {
      ensure_smem(drr::k_forward_jac<double, float, kK>, smem);
      drr::k_forward_jac<double, float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, static_cast<float*>(d_img), d_jac, npix);
    })
  return check_launch("drr_forward_jac");
}

int drr_backward_jac(const double* d_jac, int32_t n_poses, const drr_detector* det,
                     const void* d_grad_img, int grad_dtype, double* d_grad_frames,
                     void* d_workspace, size_t workspace_bytes, void* stream) {
  drr::DetDev d;
  int rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  const size_t need = drr_backward_workspace_size(n_poses, det);
  if (workspace_bytes < need || d_workspace == nullptr)
    return fail(DRR_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  if (grad_dtype != 0 && grad_dtype != 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "bad grad dtype %d", grad_dtype);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* partials = static_cast<double*>(d_workspace);
  const dim3 grd = pose_grid(d, n_poses, 1);
  const size_t npix = static_cast<size_t>(n_poses) * d.H * d.W;
  if (grad_dtype == 0)
    drr::k_backward_jac<float><<<grd, drr::kThreads, 0, st>>>(
        d_jac, npix, d, static_cast<const float*>(d_grad_img), partials);
  else
    drr::k_backward_jac<double><<<grd, drr::kThreads, 0, st>>>(
        d_jac, npix, d, static_cast<const double*>(d_grad_img), partials);
  rc = check_launch("drr_backward_jac");
  if (rc) return rc;
  drr::k_reduce_frames<<<n_poses, drr::kReduceThreads, 0, st>>>(
      partials, static_cast<int>(grd.x * grd.y), d_grad_frames);
  return check_launch("drr_backward_jac/reduce");
}

int drr_backward(const void* d_vol, int vol_dtype, const drr_grid* grid,
                 const double* d_frames, int32_t n_poses,
                 const drr_detector* det, const void* d_grad_img,
                 int grad_dtype, double* d_grad_frames, void* d_img,
                 int img_dtype, void* d_workspace, size_t workspace_bytes,
                 void* stream) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, true);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  const size_t need = drr_backward_workspace_size(n_poses, det);
  if (workspace_bytes < need || d_workspace == nullptr)
    return fail(DRR_ERR_WORKSPACE, "workspace needs %zu bytes, got %zu", need, workspace_bytes);
  if ((img_dtype != 0 && img_dtype != 1) || (grad_dtype != 0 && grad_dtype != 1))
    return fail(DRR_ERR_INVALID_ARGUMENT, "bad dtypes grad=%d img=%d", grad_dtype, img_dtype);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  double* partials = static_cast<double*>(d_workspace);
  if (vol_dtype == DRR_VOL_F32) {
    const float* vol = static_cast<const float*>(d_vol);
    if (grad_dtype == 0)
      launch_backward(vol, g, d_frames, d, n_poses, static_cast<const float*>(d_grad_img), d_img, img_dtype, partials, st);
    else
      launch_backward(vol, g, d_frames, d, n_poses, static_cast<const double*>(d_grad_img), d_img, img_dtype, partials, st);
  } else if (vol_dtype == DRR_VOL_F64) {
    const double* vol = static_cast<const double*>(d_vol);
    if (grad_dtype == 0)
      launch_backward(vol, g, d_frames, d, n_poses, static_cast<const float*>(d_grad_img), d_img, img_dtype, partials, st);
    else
      launch_backward(vol, g, d_frames, d, n_poses, static_cast<const double*>(d_grad_img), d_img, img_dtype, partials, st);
  } else {
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  }
  rc = check_launch("drr_backward");
  if (rc) return rc;
  const dim3 grd = pose_grid(d, 1, ray_split(d, n_poses));
  drr::k_reduce_frames<<<n_poses, drr::kReduceThreads, 0, st>>>(
      partials, static_cast<int>(grd.x * grd.y), d_grad_frames);
  return check_launch("drr_backward/reduce");
}

size_t drr_loss_grad_workspace_size(int32_t n_poses, const drr_detector* det) {
  drr::DetDev d;
  if (make_det(det, d) || n_poses < 0) return 0;
  const dim3 grd = pose_grid(d, 1, ray_split(d, n_poses));
  return static_cast<size_t>(n_poses) *
         (static_cast<size_t>(grd.x) * grd.y * drr::kLossSums + 3) * sizeof(double);
}

int drr_forward_loss_grad(const void* d_vol, int vol_dtype, const drr_grid* grid,
                          const double* d_frames, const double* d_eta, int32_t n_poses,
                          const drr_detector* det, const void* d_fixed, int64_t fixed_stride,
                          int kind, void* d_img, int img_dtype, double* d_value, int* d_status,
                          double* d_grad_frames, double* d_grad_eta, void* d_workspace,
                          size_t workspace_bytes, void* stream) {
  drr::RegStep off{};
  off.on = 0;
  return loss_step(d_vol, vol_dtype, grid, d_frames, d_eta, n_poses, det, d_fixed, fixed_stride,
                   kind, d_img, img_dtype, d_value, d_status, d_grad_frames, d_grad_eta,
                   d_workspace, workspace_bytes, stream, off);
}

int drr_register_step(const void* d_vol, int vol_dtype, const drr_grid* grid, double* d_frames,
                      double* d_eta, double* d_velocity, int32_t n_poses, const drr_detector* det,
                      const void* d_fixed, int64_t fixed_stride, int kind, void* d_img,
                      int img_dtype, double* d_value, int* d_status, const double* isocenter,
                      const drr_reg_config* cfg, int32_t iter, int* d_state, int* d_n_records,
                      double* d_trace_eta, double* d_trace_loss, void* d_workspace,
                      size_t workspace_bytes, void* stream) {
  if (cfg == nullptr || isocenter == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "cfg and isocenter must not be NULL");
  if (!(cfg->lr_rotation > 0) || !(cfg->lr_translation > 0))
    return fail(DRR_ERR_INVALID_ARGUMENT, "learning rates must be positive");
  if (!(cfg->momentum >= 0.0 && cfg->momentum < 1.0))
    return fail(DRR_ERR_INVALID_ARGUMENT, "momentum must be in [0, 1), got %g", cfg->momentum);
  if (cfg->max_iters < 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "max_iters must be >= 1, got %d", cfg->max_iters);
  if (iter < 0 || iter > cfg->max_iters)
    return fail(DRR_ERR_INVALID_ARGUMENT, "iter %d outside [0, max_iters]", iter);
  if (d_status == nullptr || d_eta == nullptr || d_velocity == nullptr || d_state == nullptr ||
      d_n_records == nullptr || d_trace_eta == nullptr || d_trace_loss == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "registration buffers must not be NULL");
  drr::RegStep reg{};
  reg.on = 1;
  reg.iter = iter;
  reg.cfg = drr::RegConfig{cfg->lr_rotation, cfg->lr_translation, cfg->momentum,
                           cfg->converged_threshold, cfg->max_iters};
  reg.eta = d_eta;
  reg.vel = d_velocity;
  reg.value = d_value;
  reg.status = d_status;
  reg.state = d_state;
  reg.n_rec = d_n_records;
  reg.trace_eta = d_trace_eta;
  reg.trace_loss = d_trace_loss;
  reg.frames = d_frames;
  reg.iso0 = isocenter[0];
  reg.iso1 = isocenter[1];
  reg.iso2 = isocenter[2];
  return loss_step(d_vol, vol_dtype, grid, d_frames, d_eta, n_poses, det, d_fixed, fixed_stride,
                   kind, d_img, img_dtype, d_value, d_status, nullptr, nullptr, d_workspace,
                   workspace_bytes, stream, reg);
}

int drr_volume_bounds(const void* d_vol, int vol_dtype, const drr_grid* grid,
                      int32_t* d_bounds, void* stream) {
  drr::GridDev g;
  const int rc = make_grid(grid, g);
  if (rc) return rc;
  if (d_vol == nullptr || d_bounds == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "drr_volume_bounds: NULL argument");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (static_cast<int64_t>(g.total) + 255) / 256;
  const unsigned grd = static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16);
  drr::k_bounds_init<<<1, 32, 0, st>>>(g, d_bounds);
  if (vol_dtype == DRR_VOL_F32)
    drr::k_volume_bounds<float><<<grd, 256, 0, st>>>(static_cast<const float*>(d_vol), g, d_bounds);
  else if (vol_dtype == DRR_VOL_F64)
    drr::k_volume_bounds<double><<<grd, 256, 0, st>>>(static_cast<const double*>(d_vol), g,
                                                      d_bounds);
  else
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  drr::k_bounds_finish<<<1, 32, 0, st>>>(d_bounds);
  return check_launch("drr_volume_bounds");
}

int drr_volume_hull_dirs(void) { return drr::kHullDirs; }

int drr_volume_hull(const void* d_vol, int vol_dtype, const drr_grid* grid, int32_t* d_hull,
                    void* stream) {
  drr::GridDev g;
  const int rc = make_grid(grid, g);
  if (rc) return rc;
  if (d_vol == nullptr || d_hull == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "drr_volume_hull: NULL argument");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int64_t blocks = (static_cast<int64_t>(g.total) + 255) / 256;
  const unsigned grd = static_cast<unsigned>(blocks < 148 * 16 ? blocks : 148 * 16);
  drr::k_hull_init<<<1, 32, 0, st>>>(d_hull);
  if (vol_dtype == DRR_VOL_F32)
    drr::k_volume_hull<float><<<grd, 256, 0, st>>>(static_cast<const float*>(d_vol), g, d_hull);
  else if (vol_dtype == DRR_VOL_F64)
    drr::k_volume_hull<double><<<grd, 256, 0, st>>>(static_cast<const double*>(d_vol), g, d_hull);
  else
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  return check_launch("drr_volume_hull");
}

static int signature_launch(const void* d_vol, int vol_dtype, const drr_grid* grid,
                            const double* d_frames, int32_t n_poses, const drr_detector* det,
                            uint64_t* d_sig, void* stream, bool per_ray) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  for (int a = 0; a < 3; ++a) {  // the reference's structure includes the zero margins
    g.tlo[a] = g.o[a];
    g.thi[a] = g.hi[a];
  }
  g.hull = 0;
  const size_t smem = table_bytes(g, false);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (!per_ray) cudaMemsetAsync(d_sig, 0, sizeof(uint64_t) * n_poses, st);
  const dim3 grd = pose_grid(d, n_poses, 1);
  auto* out = reinterpret_cast<unsigned long long*>(d_sig);
  auto launch = [&](auto kern, const auto* vol) {
    ensure_smem(kern, smem);
    kern<<<grd, drr::kThreads, smem, st>>>(vol, g, d_frames, d, out);
  };
  if (vol_dtype == DRR_VOL_F32) {
    const auto* v = static_cast<const float*>(d_vol);
    per_ray ? launch(drr::k_signature<float, true>, v) : launch(drr::k_signature<float, false>, v);
  } else if (vol_dtype == DRR_VOL_F64) {
    const auto* v = static_cast<const double*>(d_vol);
    per_ray ? launch(drr::k_signature<double, true>, v)
            : launch(drr::k_signature<double, false>, v);
  } else {
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  }
  return check_launch(per_ray ? "drr_ray_signatures" : "drr_signature");
}

int drr_signature(const void* d_vol, int vol_dtype, const drr_grid* grid,
                  const double* d_frames, int32_t n_poses, const drr_detector* det,
                  uint64_t* d_sig, void* stream) {
  return signature_launch(d_vol, vol_dtype, grid, d_frames, n_poses, det, d_sig, stream, false);
}

int drr_ray_signatures(const void* d_vol, int vol_dtype, const drr_grid* grid,
                       const double* d_frames, int32_t n_poses, const drr_detector* det,
                       uint64_t* d_sig, void* stream) {
  return signature_launch(d_vol, vol_dtype, grid, d_frames, n_poses, det, d_sig, stream, true);
}

int drr_volume_pack(const void* d_src, int src_type, int src_order, const int64_t* dims,
                    int clamp_negative, void* d_dst, int dst_dtype, void* stream) {
  if (d_src == nullptr || d_dst == nullptr || dims == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "drr_volume_pack: NULL argument");
  int64_t total = 1;
  for (int a = 0; a < 3; ++a) {
    if (dims[a] < 1)
      return fail(DRR_ERR_INVALID_ARGUMENT, "dims must be >= 1, got %lld on axis %d",
                  (long long)dims[a], a);
    total *= dims[a];
  }
  if (total >= (int64_t(1) << 31))
    return fail(DRR_ERR_INVALID_ARGUMENT, "volume has %lld voxels; limit is 2^31-1",
                (long long)total);
  if (src_type != DRR_SRC_F32 && src_type != DRR_SRC_F64 && src_type != DRR_SRC_I16 &&
      src_type != DRR_SRC_U8)
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown source type %d", src_type);
  if (src_order != DRR_ORDER_XFASTEST && src_order != DRR_ORDER_ZFASTEST)
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown source order %d", src_order);
  if (dims[1] > 65535 && src_order == DRR_ORDER_ZFASTEST)
    return fail(DRR_ERR_INVALID_ARGUMENT, "ny must be <= 65535 for a z-fastest source");
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (dst_dtype == DRR_VOL_F32)
    dispatch_pack(d_src, src_type, src_order, dims, clamp_negative, static_cast<float*>(d_dst), st);
  else if (dst_dtype == DRR_VOL_F64)
    dispatch_pack(d_src, src_type, src_order, dims, clamp_negative, static_cast<double*>(d_dst), st);
  else
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown dst_dtype %d", dst_dtype);
  return check_launch("drr_volume_pack");
}

int drr_loss_grad_jac(const double* d_jac, const void* d_img, const void* d_fixed, int img_dtype,
                      int64_t fixed_stride, int32_t n_images, const drr_detector* det, int kind,
                      double* d_value, int* d_status, double* d_grad_frames, const double* d_eta,
                      double* d_grad_eta, void* stream) {
  drr::DetDev d;
  int rc = make_det(det, d);
  if (rc) return rc;
  if (n_images < 0 || n_images > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_images must be in [0, 65535], got %d", n_images);
  if (n_images == 0) return DRR_OK;
  if (kind != DRR_LOSS_NEG_ZNCC && kind != DRR_LOSS_L2)
    return fail(DRR_ERR_INVALID_ARGUMENT, "loss kind must be neg_zncc (0) or l2 (1), got %d", kind);
  const int64_t npix = static_cast<int64_t>(d.H) * d.W;
  if (fixed_stride != 0 && fixed_stride != npix)
    return fail(DRR_ERR_INVALID_ARGUMENT, "fixed_stride must be 0 or H*W");
  if (d_jac == nullptr || d_img == nullptr || d_fixed == nullptr || d_value == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "d_jac, d_img, d_fixed and d_value must not be NULL");
  if (d_grad_eta != nullptr && d_eta == nullptr)
    return fail(DRR_ERR_INVALID_ARGUMENT, "d_grad_eta needs d_eta");
  if (img_dtype != 0 && img_dtype != 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown img_dtype %d", img_dtype);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const dim3 grd(drr::kLossCluster, n_images);
  const size_t npix_total = static_cast<size_t>(n_images) * npix;
  // TMA staging pays once the clusters fill the GPU twice (4 CTAs per SM)
  const bool tma = DRR_LGJ_TMA && static_cast<int64_t>(n_images) * drr::kLossCluster >=
                                      2 * 4 * static_cast<int64_t>(device_sms());
  auto launch = [&](auto kern, const auto* img, const auto* fx) {
    kern<<<grd, drr::kLossThreads, 0, st>>>(d_jac, npix_total, img, fx, fixed_stride, d, kind,
                                            d_value, d_status, d_grad_frames, d_eta, d_grad_eta);
  };
  if (img_dtype == 0) {
    const auto* im = static_cast<const float*>(d_img);
    const auto* fx = static_cast<const float*>(d_fixed);
    tma ? launch(drr::k_loss_grad_jac<float, true>, im, fx)
        : launch(drr::k_loss_grad_jac<float, false>, im, fx);
  } else {
    const auto* im = static_cast<const double*>(d_img);
    const auto* fx = static_cast<const double*>(d_fixed);
    tma ? launch(drr::k_loss_grad_jac<double, true>, im, fx)
        : launch(drr::k_loss_grad_jac<double, false>, im, fx);
  }
  return check_launch("drr_loss_grad_jac");
}

int drr_count_steps(const void* d_vol, int vol_dtype, const drr_grid* grid,
                    const double* d_frames, int32_t n_poses,
                    const drr_detector* det, int32_t* d_steps, void* stream) {
  drr::GridDev g;
  drr::DetDev d;
  int rc = make_grid(grid, g);
  if (rc) return rc;
  const size_t smem = table_bytes(g, false);
  rc = make_det(det, d);
  if (rc) return rc;
  if (n_poses < 0 || n_poses > 65535)
    return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses must be in [0, 65535], got %d", n_poses);
  if (n_poses == 0) return DRR_OK;
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int K = ray_split(d, n_poses);
  const dim3 grd = pose_grid(d, n_poses, K);
  if (vol_dtype != DRR_VOL_F32 && vol_dtype != DRR_VOL_F64)
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown vol_dtype %d", vol_dtype);
  DRR_DISPATCH_K(K,
    if (vol_dtype == DRR_VOL_F32) {
      ensure_smem(drr::k_count<float, kK>, smem);
      drr::k_count<float, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const float*>(d_vol), g, d_frames, d, d_steps);
    } else {
      ensure_smem(drr::k_count<double, kK>, smem);
      drr::k_count<double, kK><<<grd, drr::kThreads, smem, st>>>(
          static_cast<const double*>(d_vol), g, d_frames, d, d_steps);
    })
  return check_launch("drr_count_steps");
}

int drr_pose_frames(const double* d_eta, int32_t n_poses, const double* isocenter,
                    double* d_frames, void* stream) {
  if (n_poses < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses < 0");
  if (isocenter == nullptr) return fail(DRR_ERR_INVALID_ARGUMENT, "isocenter is NULL");
  if (n_poses == 0) return DRR_OK;
  const int th = 128;
  drr::k_pose_frames<<<(n_poses + th - 1) / th, th, 0, static_cast<cudaStream_t>(stream)>>>(
      d_eta, isocenter[0], isocenter[1], isocenter[2], n_poses, d_frames);
  return check_launch("drr_pose_frames");
}

int drr_pose_grad(const double* d_eta, const double* d_grad_frames, int32_t n_poses,
                  double* d_grad_eta, void* stream) {
  if (n_poses < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses < 0");
  if (n_poses == 0) return DRR_OK;
  const int th = 128;
  drr::k_pose_grad<<<(n_poses + th - 1) / th, th, 0, static_cast<cudaStream_t>(stream)>>>(
      d_eta, d_grad_frames, n_poses, d_grad_eta);
  return check_launch("drr_pose_grad");
}

int drr_image_loss(const void* d_img, const void* d_fixed, int img_dtype, int64_t fixed_stride,
                   int32_t n_images, int64_t npix, int kind, double* d_value, float* d_grad,
                   int* d_status, void* stream) {
  if (n_images < 0 || npix < 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "need n_images >= 0 and npix >= 1");
  if (kind != DRR_LOSS_NEG_ZNCC && kind != DRR_LOSS_L2)
    return fail(DRR_ERR_INVALID_ARGUMENT, "loss kind must be neg_zncc (0) or l2 (1), got %d", kind);
  if (fixed_stride != 0 && fixed_stride != npix)
    return fail(DRR_ERR_INVALID_ARGUMENT, "fixed_stride must be 0 or npix");
  if (n_images == 0) return DRR_OK;
  if (img_dtype != 0 && img_dtype != 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "unknown img_dtype %d", img_dtype);
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  // one cluster per image: grid (kLossCluster, images), images in launches of
  // at most 65535 (the grid's y limit)
  for (int32_t i0 = 0; i0 < n_images; i0 += 65535) {
    const int32_t n = n_images - i0 < 65535 ? n_images - i0 : 65535;
    const dim3 grd(drr::kLossCluster, n);
    const int64_t fo = fixed_stride * i0, io = npix * i0;
    double* val = d_value + i0;
    float* grad = d_grad ? d_grad + io : nullptr;
    int* sts = d_status ? d_status + i0 : nullptr;
    if (img_dtype == 0)
      drr::k_image_loss<float><<<grd, drr::kLossThreads, 0, st>>>(
          static_cast<const float*>(d_img) + io, static_cast<const float*>(d_fixed) + fo,
          fixed_stride, npix, kind, val, grad, sts, nullptr);
    else
      drr::k_image_loss<double><<<grd, drr::kLossThreads, 0, st>>>(
          static_cast<const double*>(d_img) + io, static_cast<const double*>(d_fixed) + fo,
          fixed_stride, npix, kind, val, grad, sts, nullptr);
    const int rc = check_launch("drr_image_loss");
    if (rc) return rc;
  }
  return DRR_OK;
}

int drr_register_update(double* d_eta, double* d_velocity, const double* d_grad_frames,
                        const double* d_value, const int* d_loss_status,
                        const drr_reg_config* cfg, int32_t iter, int* d_state, int* d_n_records,
                        double* d_trace_eta, double* d_trace_loss, int32_t n_poses,
                        void* stream) {
  if (cfg == nullptr) return fail(DRR_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (!(cfg->lr_rotation > 0) || !(cfg->lr_translation > 0))
    return fail(DRR_ERR_INVALID_ARGUMENT, "learning rates must be positive");
  if (!(cfg->momentum >= 0.0 && cfg->momentum < 1.0))
    return fail(DRR_ERR_INVALID_ARGUMENT, "momentum must be in [0, 1), got %g", cfg->momentum);
  if (cfg->max_iters < 1)
    return fail(DRR_ERR_INVALID_ARGUMENT, "max_iters must be >= 1, got %d", cfg->max_iters);
  if (iter < 0 || iter > cfg->max_iters)
    return fail(DRR_ERR_INVALID_ARGUMENT, "iter %d outside [0, max_iters]", iter);
  if (n_poses < 0) return fail(DRR_ERR_INVALID_ARGUMENT, "n_poses < 0");
  if (n_poses == 0) return DRR_OK;
  drr::RegConfig c{cfg->lr_rotation, cfg->lr_translation, cfg->momentum,
                   cfg->converged_threshold, cfg->max_iters};
  const int th = 128;
  drr::k_register_update<<<(n_poses + th - 1) / th, th, 0, static_cast<cudaStream_t>(stream)>>>(
      d_eta, d_velocity, d_grad_frames, d_value, d_loss_status, c, iter, d_state, d_n_records,
      d_trace_eta, d_trace_loss, n_poses);
  return check_launch("drr_register_update");
}

#include "peer_memory.cuh"

}  // extern "C"
#endif  // DRR_KERNELS_ONLY
