// pose_kernels.cuh -- the pose side of the hot path, on the device.
//
//   k_pose_frames      eta (rho, theta, phi, gamma, bx, by, bz) -> frame
//                      (s, c, e1, e2)            geometry.py:120-149,166-175
//   k_pose_grad        dL/dframe (12) -> dL/deta (7): the analytic tangents of
//                      the same map (the reference's dual numbers, dual.py)
//   k_register_update  one momentum gradient-descent iteration of
//                      registration.register (registration.py:89-125) with
//                      its convergence / failure bookkeeping kept on the
//                      device, so a whole registration step is capturable in
//                      a CUDA graph with no host round trip.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

namespace drr {

struct PoseTrig {
  double st, ct, sp, cp, sg, cg;
};

__device__ __forceinline__ PoseTrig pose_trig(const double* eta) {
  PoseTrig t;
  sincos(eta[1], &t.st, &t.ct);
  sincos(eta[2], &t.sp, &t.cp);
  sincos(eta[3], &t.sg, &t.cg);
  return t;
}

// The frame of one pose (geometry.py:120-149 + the isocenter offset).
__device__ __forceinline__ void pose_frame_one(const double* __restrict__ e, double iso0,
                                               double iso1, double iso2, double* __restrict__ f) {
  const PoseTrig t = pose_trig(e);
  const double rho = e[0];
  const double u[3] = {t.sp * t.ct, t.sp * t.st, t.cp};
  const double et[3] = {-t.st, t.ct, 0.0};
  const double ep[3] = {t.cp * t.ct, t.cp * t.st, -t.sp};
  const double iso[3] = {iso0, iso1, iso2};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    f[a] = iso[a] + (e[4 + a] + rho * u[a]);
    f[3 + a] = iso[a] + (e[4 + a] - rho * u[a]);
    f[6 + a] = t.cg * ep[a] - t.sg * et[a];
    f[9 + a] = t.cg * et[a] + t.sg * ep[a];
  }
}

__global__ void k_pose_frames(const double* __restrict__ eta, double iso0, double iso1,
                              double iso2, int n, double* __restrict__ frames) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  pose_frame_one(eta + 7 * b, iso0, iso1, iso2, frames + 12 * b);
}

// dL/deta = J^T dL/dframe with J = d frame / d eta (12 x 7).
__device__ __forceinline__ void pose_grad(const double* e, const double* gf, double* ge) {
  const PoseTrig t = pose_trig(e);
  const double rho = e[0];
  const double u[3] = {t.sp * t.ct, t.sp * t.st, t.cp};
  const double du_th[3] = {-t.sp * t.st, t.sp * t.ct, 0.0};
  const double du_ph[3] = {t.cp * t.ct, t.cp * t.st, -t.sp};
  const double et[3] = {-t.st, t.ct, 0.0};
  const double det_th[3] = {-t.ct, -t.st, 0.0};
  const double ep[3] = {t.cp * t.ct, t.cp * t.st, -t.sp};
  const double dep_th[3] = {-t.cp * t.st, t.cp * t.ct, 0.0};
  const double dep_ph[3] = {-t.sp * t.ct, -t.sp * t.st, -t.cp};
  double g[7] = {0, 0, 0, 0, 0, 0, 0};
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double gs = gf[a], gc = gf[3 + a], g1 = gf[6 + a], g2 = gf[9 + a];
    // s = shift + rho u ; c = shift - rho u
    g[0] += (gs - gc) * u[a];
    g[1] += (gs - gc) * rho * du_th[a];
    g[2] += (gs - gc) * rho * du_ph[a];
    g[4 + a] += gs + gc;
    // e1 = cg ep - sg et ; e2 = cg et + sg ep
    g[1] += g1 * (t.cg * dep_th[a] - t.sg * det_th[a]) + g2 * (t.cg * det_th[a] + t.sg * dep_th[a]);
    g[2] += g1 * (t.cg * dep_ph[a]) + g2 * (t.sg * dep_ph[a]);
    g[3] += g1 * (-t.sg * ep[a] - t.cg * et[a]) + g2 * (-t.sg * et[a] + t.cg * ep[a]);
  }
#pragma unroll
  for (int k = 0; k < 7; ++k) ge[k] = g[k];
}

__global__ void k_pose_grad(const double* __restrict__ eta, const double* __restrict__ gframes,
                            int n, double* __restrict__ geta) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  pose_grad(eta + 7 * b, gframes + 12 * b, geta + 7 * b);
}

// Registration states (registration.py:63-86 RegistrationTrace flags).
constexpr int kRegRunning = 0, kRegConverged = 1, kRegFailed = 2, kRegDone = 3;

struct RegConfig {
  double lr_rot, lr_trans, momentum, threshold;
  int max_iters;
};

// One iteration for each of n independent registrations.  `value`/`status`
// come from k_image_loss on the current pose; gframes from drr_backward.
// Trace rows are written at index `iter` (trace_eta n x (max_iters+1) x 6,
// trace_loss n x (max_iters+1)); n_rec counts recorded rows.
// One iteration of registration b (registration.py:89-125): records the
// trace row `iter`, sets the state on failure / convergence / the last
// iteration, else applies the momentum step with the pose gradient of
// dL/dframe `gf`.  Returns true when eta changed.
__device__ __forceinline__ bool register_update_one(int b, double* __restrict__ eta,
                                                    double* __restrict__ vel,
                                                    const double* __restrict__ gf, double value,
                                                    int loss_status, const RegConfig& cfg,
                                                    int iter, int* __restrict__ state,
                                                    int* __restrict__ n_rec,
                                                    double* __restrict__ trace_eta,
                                                    double* __restrict__ trace_loss) {
  if (state[b] != kRegRunning) return false;
  double* e = eta + 7 * b;
  const int row = iter;
  double* te = trace_eta + (static_cast<int64_t>(b) * (cfg.max_iters + 1) + row) * 6;
#pragma unroll
  for (int k = 0; k < 6; ++k) te[k] = e[1 + k];
  n_rec[b] = row + 1;
  // failure modes of loss_and_gradient (registration.py:106-113): metric
  // undefined (sigma == 0), gradient undefined (|sin phi| <= 1e-6,
  // gradients.py:39-42), invalid pose (non-finite or rho <= 0)
  bool finite = e[0] > 0.0;
#pragma unroll
  for (int k = 0; k < 7; ++k) finite = finite && isfinite(e[k]);
  const bool gimbal = !(fabs(sin(e[2])) > 1e-6);
  if (loss_status != 0 || gimbal || !finite) {
    trace_loss[static_cast<int64_t>(b) * (cfg.max_iters + 1) + row] = INFINITY;
    state[b] = kRegFailed;
    return false;
  }
  trace_loss[static_cast<int64_t>(b) * (cfg.max_iters + 1) + row] = value;
  if (value < cfg.threshold) { state[b] = kRegConverged; return false; }
  if (iter == cfg.max_iters) { state[b] = kRegDone; return false; }
  double g[7];
  pose_grad(e, gf, g);
  double* vb = vel + 6 * b;
#pragma unroll
  for (int k = 0; k < 6; ++k) {
    const double beta = k < 3 ? cfg.lr_rot : cfg.lr_trans;
    vb[k] = cfg.momentum * vb[k] - beta * g[1 + k];
    e[1 + k] += vb[k];
  }
  return true;
}

// One iteration for each of n independent registrations.  `value`/`status`
// come from k_image_loss on the current pose; gframes from drr_backward.
// Trace rows are written at index `iter` (trace_eta n x (max_iters+1) x 6,
// trace_loss n x (max_iters+1)); n_rec counts recorded rows.
__global__ void k_register_update(double* __restrict__ eta, double* __restrict__ vel,
                                  const double* __restrict__ gframes,
                                  const double* __restrict__ value,
                                  const int* __restrict__ loss_status, RegConfig cfg,
                                  int iter, int* __restrict__ state, int* __restrict__ n_rec,
                                  double* __restrict__ trace_eta,
                                  double* __restrict__ trace_loss, int n) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n) return;
  register_update_one(b, eta, vel, gframes + 12 * b, value[b], loss_status[b], cfg, iter, state,
                      n_rec, trace_eta, trace_loss);
}

}  // namespace drr
