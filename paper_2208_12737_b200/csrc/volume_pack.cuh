// volume_pack.cuh -- one-time volume ingest into the walk's device layout
// (SURVEY 8(b) B2 drr_volume_pack; 8(f) row 4).
//
// The walk gathers from the reference's x-fastest flat order
// (flat = i + nx (j + ny k), volume.py:77-79) as fp32 (or f64 for the
// bit-identical plugin path).  Sources arrive either already x-fastest (the
// reference's flat_data(), .dvol payloads, raw files: volume.py:149-222) or
// as a C-ordered (nx, ny, nz) array indexed data[i, j, k] (numpy / torch
// default, z fastest).  One kernel converts, casts (f64 / f32 / i16 / u8 ->
// f32 or f64, no Hounsfield rescale, volume.py:211-218) and optionally clamps
// negatives (--clamp-negative), so no host transpose or extra
// device copy is needed.  HBM-bound: the z-fastest case is a per-j-slab 2-D
// transpose of (i, k) through 32 x 33 shared-memory tiles, so both the
// reads (k-contiguous) and the writes (i-contiguous) are coalesced.
//
// Layout study (DESIGN.md (d)): a bricked layout (4x4x4 / 8x4x2 / 2x2x2
// bricks) was evaluated against the linear one on the walk's own gather
// pattern at C2 (scripts/layout_sim.py): it cuts the 128-B lines a warp's
// gather touches by 37% but the 32-B sectors only by 9%, and the L1 data
// pipe -- the measured limiter -- moves ~4 sectors per wavefront, while the
// walk would need a per-axis step table lookup per voxel-step (+3
// instructions).  So the walk layout stays linear.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace drr {

template <typename ST>
__device__ __forceinline__ double pack_load(const ST* p, int64_t i) {
  return static_cast<double>(p[i]);
}

template <typename ST, typename DT>
__global__ void __launch_bounds__(256)
    k_pack_linear(const ST* __restrict__ src, int64_t n, int clamp, DT* __restrict__ dst) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = pack_load(src, i);
    if (clamp && v < 0.0) v = 0.0;
    dst[i] = static_cast<DT>(v);
  }
}

// src[(i * ny + j) * nz + k] -> dst[(k * ny + j) * nx + i]; grid (ceil(nz/32),
// ceil(nx/32), ny), block (32, 8).
template <typename ST, typename DT>
__global__ void __launch_bounds__(256)
    k_pack_zfastest(const ST* __restrict__ src, int nx, int ny, int nz, int clamp,
                    DT* __restrict__ dst) {
  __shared__ double tile[32][33];
  const int k0 = blockIdx.x * 32, i0 = blockIdx.y * 32, j = blockIdx.z;
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int i = i0 + r, k = k0 + threadIdx.x;
    if (i < nx && k < nz) {
      double v = pack_load(src, (static_cast<int64_t>(i) * ny + j) * nz + k);
      if (clamp && v < 0.0) v = 0.0;
      tile[r][threadIdx.x] = v;
    }
  }
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += 8) {
    const int k = k0 + r, i = i0 + threadIdx.x;
    if (i < nx && k < nz)
      dst[(static_cast<int64_t>(k) * ny + j) * nx + i] = static_cast<DT>(tile[threadIdx.x][r]);
  }
}

}  // namespace drr
