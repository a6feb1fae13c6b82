/*
 * drr_b200.h -- C ABI of the B200-native vectorised-Siddon DRR renderer.
 *
 * Stateless, re-entrant, one device per call (the caller selects the device
 * with cudaSetDevice / torch.cuda.device).  Every pointer argument named
 * `d_*` is DEVICE memory; `stream` is a cudaStream_t passed as void*.  The
 * library never allocates device memory: the backward pass's workspace size is
 * queried with drr_backward_workspace_size and supplied by the caller.
 * Functions return DRR_OK (0) or a negative status; drr_last_error() gives the
 * message of the calling thread's last failure.
 *
 * What each entry point replaces in the reference (drrtrace, /root/reference):
 *   drr_raysum               <- _kernels/_native.pyx:140-193 siddon_raysum
 *                               (and jacobs_raysum, _native.pyx:285-382: the
 *                               GPU walk is already incremental)
 *   drr_raysum_endpoint_grad <- _kernels/_native.pyx:196-282 siddon_raysum_grad
 *                               (reverse-mode: dE/ds, dE/dp per ray)
 *   drr_raysum_tangents      <- the same function with its own contract:
 *                               energies + d_energy (N x T) from the caller's
 *                               source / pixel tangents
 *                               (reverse-mode form: dE/ds, dE/dp per ray; the
 *                               host shim contracts them with the T tangents)
 *   drr_forward              <- raytrace.py:132-142 render() fused with
 *                               geometry.py:152-175 detector_grid()
 *   drr_backward             <- gradients.py:45-69 render_with_gradient +
 *                               the pixel_grad @ d_image reduction, in reverse
 *                               mode down to the 12-number frame (s, c, e1, e2)
 *   drr_forward_jac          <- gradients.py:45-58 render_with_gradient (image and
 *                               per-ray derivatives from one walk, as
 *                               _native.pyx:196-282 does)
 *   drr_backward_jac         <- gradients.py:61-69 the pixel_grad @ d_image
 *                               contraction, down to the 12-number frame
 *   drr_count_steps          <- _kernels/python_ref.py:191-201 ray_structure
 *                               (number of used voxel-steps per ray)
 *   drr_signature            <- gradients.py:124-142 discrete_signature (the
 *                               traversal structure of every ray, hashed)
 *   drr_ray_signatures       <- the same, one hash per ray (per-ray
 *                               attribution of detect_fd_boundaries,
 *                               gradients.py:145-167)
 *   drr_pose_frames          <- geometry.py:120-149 _pose_frame (+ the
 *                               isocenter offset of geometry.py:166-175), batched
 *   drr_pose_grad            <- the tangent half of the same map (dual.py
 *                               duals seeded in geometry.py:130-131): dL/dframe
 *                               -> dL/d(rho, theta, phi, gamma, bx, by, bz)
 *   drr_image_loss           <- metrics.py:71-91 loss_value_and_pixel_grad
 *                               (neg_zncc, l2), batched, fused
 *   drr_loss_grad_jac        <- gradients.py:61-69's loss, pixel gradient and
 *                               pixel_grad @ d_image from stored Jacobians
 *   drr_forward_loss_grad    <- gradients.py:61-69 loss_and_gradient for the
 *                               two losses of metrics.py:71-91, batched: one
 *                               walk per ray, no stored Jacobian
 *   drr_register_update      <- one iteration of registration.py:89-125
 *                               register() (momentum GD + convergence state)
 *   drr_register_step        <- the same iteration with its loss and
 *                               gradient: three launches in all
 *   drr_volume_bounds        <- no counterpart: the occupied box and hull
 *   drr_volume_hull             that let the walks skip exactly-zero margins
 *   drr_volume_pack          <- volume.py:77-79 flat_data() (the x-fastest
 *                               layout) + volume.py:196-222 import_raw's cast
 *                               and clamp, as one device pass
 *   drr_peer_export / _open  <- no reference counterpart: the population
 *   / _close                    study runs independent registrations in
 *                               parallel processes and collects their traces
 *                               (cli.py:133-145); here the
 *                               collecting rank's output buffers are opened by
 *                               every rank so its kernels store results
 *                               straight into them over NVLink
 */
#ifndef DRR_B200_H
#define DRR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DRR_OK 0
#define DRR_ERR_INVALID_ARGUMENT -1   /* -> drrtrace InvalidArgumentError   */
#define DRR_ERR_CUDA -2               /* launch / runtime failure            */
#define DRR_ERR_GRADIENT_UNDEFINED -3 /* -> drrtrace GradientUndefinedError  */
#define DRR_ERR_WORKSPACE -4          /* workspace too small                 */

/* Volume element type of d_vol. */
#define DRR_VOL_F32 0 /* product layout: fp32 densities, x-fastest        */
#define DRR_VOL_F64 1 /* drop-in for the reference's float64 flat volume  */

/* Axis-aligned voxel grid: dims[a] voxels of spacing[a] mm, planes at
 * origin[a] + k*spacing[a], k = 0..dims[a]   (volume.py:24-60).
 * occ_lo / occ_hi (optional): the voxel-index box [occ_lo, occ_hi) outside of
 * which every voxel is exactly zero (drr_volume_bounds).  The walks then run
 * over that box only -- segments outside it add nothing to any sum, so every
 * image and gradient is bit-identical to the full walk.  All-zero occ_hi
 * means the whole volume.
 * hull_valid / hull_lo / hull_hi (optional, with the box): drr_volume_hull's
 * ranges of n . (i, j, k) over the non-zero voxels for its directions
 * n = (1,1,0) (1,-1,0) (1,0,1) (1,0,-1) (0,1,1) (0,1,-1) (1,1,1) (1,1,-1)
 * (1,-1,1) (-1,1,1) (2,1,0) (1,2,0) (2,-1,0) (1,-2,0); hull_valid = the
 * number of directions filled (drr_volume_hull_dirs()), 0 = no hull.  Each
 * ray is then also trimmed to that polytope (again bit-identical). */
typedef struct drr_grid {
  int64_t dims[3];
  double spacing[3];
  double origin[3];
  int64_t occ_lo[3];
  int64_t occ_hi[3];
  int32_t hull_valid;
  int32_t hull_lo[16];
  int32_t hull_hi[16];
} drr_grid;

/* Detector: H x W pixels, pitch_x along W, pitch_y along H (geometry.py:71-97,
 * 152-157).  Pixel (h, w) sits at c + a_h e1 + a_w e2.
 * ray_split: threads per ray for the batched kernels -- 1 = one thread walks
 * the whole ray (bit-identical to the reference's sequential sum), 2/4/8 =
 * the ray is cut at dominant-axis crossings and the chunk sums combined
 * (same segments, different summation order: ~1e-16 relative), 0 = auto
 * (split only when B*H*W rays cannot fill the GPU, e.g. one pose). */
typedef struct drr_detector {
  int32_t height;
  int32_t width;
  double pitch_x;
  double pitch_y;
  int32_t ray_split;
} drr_detector;

/* Frames: B x 12 float64, per pose (s[3], c[3], e1[3], e2[3]) in volume
 * coordinates (isocenter already added), geometry.py:120-149. */

const char *drr_last_error(void);
int drr_version(void);
/* sizeof the ABI structs as this library was compiled (a binding checks its
 * own layouts against them; any pointer may be NULL). */
int drr_struct_sizes(size_t *grid, size_t *detector, size_t *reg_config,
                     size_t *peer_handle);

/* Energies of explicit rays from one source: out[r] = |p_r - s| sum seg V.
 * d_src: 3 doubles, d_pix: N x 3 doubles, d_out: N doubles. */
int drr_raysum(const void *d_vol, int vol_dtype, const drr_grid *grid,
               const double *d_src, const double *d_pix, int64_t n_rays,
               double *d_out, void *stream);

/* Same walk, plus the reverse-mode endpoint derivatives dE/ds and dE/dp
 * (N x 3 each).  d_out is bitwise equal to drr_raysum's. */
int drr_raysum_endpoint_grad(const void *d_vol, int vol_dtype,
                             const drr_grid *grid, const double *d_src,
                             const double *d_pix, int64_t n_rays,
                             double *d_out, double *d_dEds, double *d_dEdp,
                             void *stream);

/* siddon_raysum_grad's own contract (_native.pyx:196-282): energies and
 * d_energy[r, t] = dE/ds . d_src[:, t] + dE/dp . d_pix[r, :, t], the
 * endpoint derivatives contracted in the walk's epilogue.  d_dsrc: 3 x T,
 * d_dpix: N x 3 x T, d_denergy: N x T (row-major doubles). */
int drr_raysum_tangents(const void *d_vol, int vol_dtype, const drr_grid *grid,
                        const double *d_src, const double *d_dsrc,
                        const double *d_pix, const double *d_dpix,
                        int64_t n_rays, int32_t n_tangents, double *d_out,
                        double *d_denergy, void *stream);

/* Batched DRR forward: pixel rays generated in-kernel from the frames.
 * d_img: B x H x W, float32 (img_dtype 0) or float64 (img_dtype 1). */
int drr_forward(const void *d_vol, int vol_dtype, const drr_grid *grid,
                const double *d_frames, int32_t n_poses,
                const drr_detector *det, void *d_img, int img_dtype,
                void *stream);

size_t drr_backward_workspace_size(int32_t n_poses, const drr_detector *det);

/* Batched backward: d_grad_img B x H x W (float32 or float64 per
 * grad_dtype) -> d_grad_frames B x 12 float64, reduced over pixels in a fixed
 * order (bit-reproducible; no atomics).  Optionally also writes the image
 * (d_img may be NULL; same dtype rule as drr_forward's img_dtype). */
int drr_backward(const void *d_vol, int vol_dtype, const drr_grid *grid,
                 const double *d_frames, int32_t n_poses,
                 const drr_detector *det, const void *d_grad_img,
                 int grad_dtype, double *d_grad_frames, void *d_img,
                 int img_dtype, void *d_workspace, size_t workspace_bytes,
                 void *stream);

/* Forward with the ray Jacobian: ONE walk per ray writes the image (as
 * drr_forward) and each ray's endpoint derivatives into d_jac, 6 x (B*H*W)
 * float64 structure-of-arrays: rows 0-2 dE/ds, rows 3-5 dE/dp.  Replaces
 * gradients.py:45-58 render_with_gradient, which also obtains energies and
 * tangents from one traversal (_native.pyx:196-282 siddon_raysum_grad). */
int drr_forward_jac(const void *d_vol, int vol_dtype, const drr_grid *grid,
                    const double *d_frames, int32_t n_poses,
                    const drr_detector *det, void *d_img, int img_dtype,
                    double *d_jac, void *stream);

/* Backward from stored ray Jacobians (no walk): d_grad_frames (B x 12) =
 * sum over pixels of grad_img * dE/d(s, c, e1, e2) in the same fixed order as
 * drr_backward -- the `pixel_grad @ d_image` contraction of
 * gradients.py:61-69.  Workspace: drr_backward_workspace_size. */
int drr_backward_jac(const double *d_jac, int32_t n_poses,
                     const drr_detector *det, const void *d_grad_img,
                     int grad_dtype, double *d_grad_frames, void *d_workspace,
                     size_t workspace_bytes, void *stream);

/* The occupied box of a device volume in the walk's layout: per axis the
 * voxel-index range [lo, hi) holding every voxel that is not exactly zero
 * (NaN counts as nonzero, -0.0 as zero).  An all-zero volume
 * gives lo = hi = 0.  d_bounds: 6 int32 device ints (lo[3], hi[3]). */
int drr_volume_bounds(const void *d_vol, int vol_dtype, const drr_grid *grid,
                      int32_t *d_bounds, void *stream);

/* The occupied hull of a device volume: for the drr_volume_hull_dirs()
 * directions of drr_grid, the min (d_hull[0..15]) and max (d_hull[16..31]) of
 * n . (i, j, k) over the voxels that are not exactly zero (NaN counts).
 * d_hull: 32 int32 device ints. */
int drr_volume_hull_dirs(void);
int drr_volume_hull(const void *d_vol, int vol_dtype, const drr_grid *grid,
                    int32_t *d_hull, void *stream);

/* One-time ingest of a device volume into the walk's layout: x-fastest
 * (flat = i + nx (j + ny k), volume.py:77-79), dst_dtype DRR_VOL_F32 / F64.
 * The source is either already x-fastest (DRR_ORDER_XFASTEST: flat_data(),
 * .dvol and raw payloads) or a C-ordered (nx, ny, nz) array data[i, j, k]
 * (DRR_ORDER_ZFASTEST: numpy / torch default); it is cast without rescaling
 * and, with clamp_negative, negatives become 0. */
#define DRR_SRC_F32 0
#define DRR_SRC_F64 1
#define DRR_SRC_I16 2
#define DRR_SRC_U8 3
#define DRR_ORDER_XFASTEST 0
#define DRR_ORDER_ZFASTEST 1
int drr_volume_pack(const void *d_src, int src_type, int src_order,
                    const int64_t *dims, int clamp_negative, void *d_dst,
                    int dst_dtype, void *stream);

/* Used voxel-steps per ray (segments longer than 1e-12), B x H x W int32. */
int drr_count_steps(const void *d_vol, int vol_dtype, const drr_grid *grid,
                    const double *d_frames, int32_t n_poses,
                    const drr_detector *det, int32_t *d_steps, void *stream);

/* Per-pose 64-bit signature of the discrete traversal structure of all its
 * rays (crossing labels in merge order, used segments, their voxels, the
 * exit selector; python_ref.py:191-201 ray_structure).  Equal signatures =
 * the same smooth branch of the energy map (detect_fd_boundaries,
 * gradients.py:145-167).  d_sig: B uint64. */
int drr_signature(const void *d_vol, int vol_dtype, const drr_grid *grid,
                  const double *d_frames, int32_t n_poses,
                  const drr_detector *det, uint64_t *d_sig, void *stream);

/* The per-ray terms of drr_signature: d_sig is B x H x W uint64, and each
 * pose's drr_signature is the wrapping sum of its rays' entries.  Used to
 * attribute finite-difference stencils ray by ray (fd.ray_fd_report). */
int drr_ray_signatures(const void *d_vol, int vol_dtype, const drr_grid *grid,
                       const double *d_frames, int32_t n_poses,
                       const drr_detector *det, uint64_t *d_sig, void *stream);

/* B x 7 pose vectors (rho, theta, phi, gamma, bx, by, bz) -> B x 12 frames.
 * isocenter: 3 doubles in HOST memory (the volume centre). */
int drr_pose_frames(const double *d_eta, int32_t n_poses,
                    const double *isocenter, double *d_frames, void *stream);

/* dL/dframe (B x 12) -> dL/deta (B x 7) at poses d_eta. */
int drr_pose_grad(const double *d_eta, const double *d_grad_frames,
                  int32_t n_poses, double *d_grad_eta, void *stream);

#define DRR_LOSS_NEG_ZNCC 0
#define DRR_LOSS_L2 1
/* Per-image loss value (B doubles) and optional fp32 pixel gradient
 * (B x npix) of img (B x npix) against fixed (fixed_stride = 0: one image
 * shared by all; = npix: one per image).  img_dtype 0 = float32, 1 = float64
 * (fixed has the same dtype).  d_status (optional, B ints) = 1 where the
 * metric is undefined (zero variance, metrics.py:29-30). */
int drr_image_loss(const void *d_img, const void *d_fixed, int img_dtype,
                   int64_t fixed_stride, int32_t n_images, int64_t npix,
                   int kind, double *d_value, float *d_grad, int *d_status,
                   void *stream);

/* A whole neg-ZNCC / L2 loss-and-gradient step for B poses with ONE walk per
 * ray and no stored ray Jacobian: the walk writes the image (img_dtype 0 =
 * float32, 1 = float64; d_fixed has the same dtype, fixed_stride 0 = one
 * fixed image for all, H*W = one per pose) and per-CTA sums of the ray
 * Jacobian weighted by 1, the image value and the fixed value; the loss
 * kernel gives value / status (as drr_image_loss) and the pixel gradient as an
 * affine map of the two images; a fixed-order reduction combines them into
 * d_grad_frames (B x 12) and, given d_eta, d_grad_eta (B x 7).  Either
 * gradient output may be NULL.  Undefined metrics (status 1) give NaN.
 * Workspace: drr_loss_grad_workspace_size. */
size_t drr_loss_grad_workspace_size(int32_t n_poses, const drr_detector *det);
int drr_forward_loss_grad(const void *d_vol, int vol_dtype, const drr_grid *grid,
                          const double *d_frames, const double *d_eta,
                          int32_t n_poses, const drr_detector *det,
                          const void *d_fixed, int64_t fixed_stride, int kind,
                          void *d_img, int img_dtype, double *d_value,
                          int *d_status, double *d_grad_frames,
                          double *d_grad_eta, void *d_workspace,
                          size_t workspace_bytes, void *stream);

/* The stored-Jacobian step's tail in one launch: per image (one 8-CTA
 * cluster) the neg-ZNCC / L2 value and status (as drr_image_loss), then the
 * float64 pixel gradient contracted with drr_forward_jac's d_jac (6 x
 * (B*H*W)) into d_grad_frames (B x 12, may be NULL) and, given d_eta,
 * d_grad_eta (B x 7) -- in place of drr_image_loss + drr_backward_jac +
 * drr_pose_grad.  img_dtype 0 / 1 as drr_forward_jac's image (d_fixed the
 * same dtype); fixed_stride 0 or H*W; n_images <= 65535. */
int drr_loss_grad_jac(const double *d_jac, const void *d_img, const void *d_fixed,
                      int img_dtype, int64_t fixed_stride, int32_t n_images,
                      const drr_detector *det, int kind, double *d_value,
                      int *d_status, double *d_grad_frames, const double *d_eta,
                      double *d_grad_eta, void *stream);

/* Momentum gradient descent settings (registration.py:41-58). */
typedef struct drr_reg_config {
  double lr_rotation;
  double lr_translation;
  double momentum;
  double converged_threshold;
  int32_t max_iters;
} drr_reg_config;

#define DRR_REG_RUNNING 0
#define DRR_REG_CONVERGED 1
#define DRR_REG_FAILED 2
#define DRR_REG_DONE 3

/* One registration iteration `iter` for B independent registrations: records
 * (pose[1:], loss) into the traces (B x (max_iters+1) x 6 and
 * B x (max_iters+1)), sets the state on convergence / failure / last
 * iteration, else applies v <- m v - beta * grad[1:], eta[1:] += v. */
int drr_register_update(double *d_eta, double *d_velocity,
                        const double *d_grad_frames, const double *d_value,
                        const int *d_loss_status, const drr_reg_config *cfg,
                        int32_t iter, int *d_state, int *d_n_records,
                        double *d_trace_eta, double *d_trace_loss,
                        int32_t n_poses, void *stream);

/* Peer-memory outputs (one node, one process per GPU).  drr_peer_export
 * describes a device buffer of the calling process (an IPC handle of its
 * allocation plus the buffer's offset in it); another process passes that
 * handle to drr_peer_open on its own device and gets a pointer its kernels may
 * store into (peer access over NVLink is enabled lazily).  drr_peer_close
 * takes the opened pointer and the handle's offset. */
typedef struct drr_peer_handle {
  unsigned char ipc[64];
  uint64_t offset; /* byte offset of the buffer inside the allocation */
  uint64_t bytes;  /* bytes from the buffer to the end of the allocation */
} drr_peer_handle;

int drr_peer_export(const void *d_ptr, drr_peer_handle *out);
int drr_peer_open(const drr_peer_handle *h, void **d_ptr);
int drr_peer_close(void *d_ptr, uint64_t offset);

/* One momentum-GD iteration `iter` for B registrations in three launches: the
 * Jacobian-free walk of drr_forward_loss_grad at d_frames, the loss, and a
 * reduction that also applies drr_register_update's bookkeeping and step and
 * writes the frames of the updated poses back into d_frames for the next
 * iteration (isocenter: 3 doubles in HOST memory).  d_frames must hold the
 * frames of d_eta on entry (drr_pose_frames once before the first
 * iteration).  Workspace: drr_loss_grad_workspace_size. */
int drr_register_step(const void *d_vol, int vol_dtype, const drr_grid *grid,
                      double *d_frames, double *d_eta, double *d_velocity,
                      int32_t n_poses, const drr_detector *det,
                      const void *d_fixed, int64_t fixed_stride, int kind,
                      void *d_img, int img_dtype, double *d_value,
                      int *d_status, const double *isocenter,
                      const drr_reg_config *cfg, int32_t iter, int *d_state,
                      int *d_n_records, double *d_trace_eta,
                      double *d_trace_loss, void *d_workspace,
                      size_t workspace_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* DRR_B200_H */
