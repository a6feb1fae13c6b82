// Compiles only the walk kernels named below (no C ABI) so their SASS can be
// studied quickly: scripts/sass_count.sh
#define DRR_KERNELS_ONLY 1
#include "../paper_2208_12737_b200/csrc/drr_kernels.cu"
template __global__ void drr::k_forward_jac<float, float, 1>(const float*, const drr::GridDev,
                                                             const double*, const drr::DetDev,
                                                             float*, double*, size_t);
template __global__ void drr::k_forward<float, float, 1>(const float*, const drr::GridDev,
                                                         const double*, const drr::DetDev, float*);
template __global__ void drr::k_backward<float, float, float, 1>(const float*, const drr::GridDev,
                                                                 const double*, const drr::DetDev,
                                                                 const float*, float*, double*);
template __global__ void drr::k_forward_loss<float, float, 1>(const float*, const drr::GridDev,
                                                              const double*, const drr::DetDev,
                                                              float*, const float*, int64_t, double*);
