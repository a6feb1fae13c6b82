/*
 * siddon_oracle.c -- TEST INFRASTRUCTURE ONLY (the parity checker, never the
 * product path).  A plain-C restatement of the reference's vectorised Siddon
 * kernels and pose geometry (drrtrace, /root/reference/pkg), written from the
 * reference's documented behaviour.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load it.
 *
 * Build: oracle/Makefile (gcc -O2 -ffp-contract=off, no -march, so no FMA is
 * contracted: the reference extension is built the same way,
 * pkg/setup.py:18-25).  Every arithmetic expression keeps the reference's
 * operation order so results are bit-identical to the reference's native
 * backend (pinned by tests/test_oracle.py against tests/golden/).
 *
 * Volume: flat x-fastest float64, idx = i + nx*(j + ny*k)   (volume.py:77-79)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SEGMENT_EPS 1e-12 /* _native.pyx:16, python_ref.py:23 */
#define CONST_LABEL 3     /* _native.pyx:17 */

/* Slab entry/exit clipped to [0,1] with first-max / first-min labels over
 * (x, y, z, clip).  Follows _native.pyx:20-65 (== python_ref.py:47-68). */
static int entry_exit(const double *s, const double *d, const double *o,
                      const double *sp, const int64_t *n, double *amin,
                      double *amax, int *lab_min, int *lab_max) {
  double cmin[4], cmax[4];
  for (int ax = 0; ax < 3; ++ax) {
    double hi = o[ax] + (double)n[ax] * sp[ax];
    if (d[ax] == 0.0) {
      if (o[ax] <= s[ax] && s[ax] <= hi) {
        cmin[ax] = -INFINITY;
        cmax[ax] = INFINITY;
      } else {
        cmin[ax] = INFINITY;
        cmax[ax] = -INFINITY;
      }
      continue;
    }
    double a0 = (o[ax] - s[ax]) / d[ax];
    double a1 = (hi - s[ax]) / d[ax];
    if (a0 > a1) { double t = a0; a0 = a1; a1 = t; }
    cmin[ax] = a0;
    cmax[ax] = a1;
  }
  cmin[3] = 0.0;
  cmax[3] = 1.0;
  int best = 0;
  for (int ax = 1; ax < 4; ++ax) if (cmin[ax] > cmin[best]) best = ax;
  *lab_min = best;
  *amin = cmin[best];
  best = 0;
  for (int ax = 1; ax < 4; ++ax) if (cmax[ax] < cmax[best]) best = ax;
  *lab_max = best;
  *amax = cmax[best];
  return *amin < *amax;
}

/* Midpoint -> clamped flat voxel index.  _native.pyx:68-82. */
static int64_t voxel_at(const double *s, const double *d, double mid,
                        const double *o, const double *sp, const int64_t *n) {
  int64_t idx[3];
  for (int ax = 0; ax < 3; ++ax) {
    int64_t i = (int64_t)floor((s[ax] + mid * d[ax] - o[ax]) / sp[ax]);
    if (i < 0) i = 0;
    else if (i >= n[ax]) i = n[ax] - 1;
    idx[ax] = i;
  }
  return idx[0] + n[0] * (idx[1] + n[1] * idx[2]);
}

/* Ascending crossings of one axis inside [amin, amax].  _native.pyx:85-112
 * (scans from plane 0 / n exactly like the reference). */
static int fill_axis(const double *s, const double *d, const double *o,
                     const double *sp, const int64_t *n, int ax, double amin,
                     double amax, double *buf) {
  if (d[ax] == 0.0) return 0;
  int64_t i, i1, step;
  if (d[ax] > 0.0) { i = 0; i1 = n[ax] + 1; step = 1; }
  else { i = n[ax]; i1 = -1; step = -1; }
  int cnt = 0;
  for (; i != i1; i += step) {
    double a = (o[ax] + (double)i * sp[ax] - s[ax]) / d[ax];
    if (a > amax) break;
    if (a >= amin) buf[cnt++] = a;
  }
  return cnt;
}

/* One ray: walks the merged crossing list and calls back per segment.  The
 * merge picks the smallest head with strict '<' over x, y, z so ties go to the
 * lowest axis (_native.pyx:177-191; python_ref.py:105 stable argsort). */
typedef struct {
  double amin, amax;
  int lab_min, lab_max, hit;
} ray_info;

static int64_t max_dim(const int64_t *n) {
  int64_t m = n[0];
  if (n[1] > m) m = n[1];
  if (n[2] > m) m = n[2];
  return m;
}

/* out[r] = |d| * sum_m seg_m V[vox(mid_m)]  -- _native.pyx:140-193.
 * steps (optional) receives the number of used segments per ray. */
void orc_raysum(const double *vol, const int64_t *n, const double *sp,
                const double *o, const double *src, const double *pix,
                int64_t nrays, double *out, int64_t *steps) {
  int64_t m = max_dim(n) + 1;
  double *buf = (double *)malloc(sizeof(double) * 3 * m);
  double s[3] = {src[0], src[1], src[2]};
  for (int64_t r = 0; r < nrays; ++r) {
    double d[3];
    for (int ax = 0; ax < 3; ++ax) d[ax] = pix[3 * r + ax] - s[ax];
    double amin, amax;
    int lmin, lmax;
    out[r] = 0.0;
    if (steps) steps[r] = 0;
    if (!entry_exit(s, d, o, sp, n, &amin, &amax, &lmin, &lmax)) continue;
    int cnt[3], p[3] = {0, 0, 0};
    for (int ax = 0; ax < 3; ++ax)
      cnt[ax] = fill_axis(s, d, o, sp, n, ax, amin, amax, buf + ax * m);
    double acc = 0.0, prev = amin;
    int64_t used = 0;
    for (;;) {
      int sel = -1;
      double best = INFINITY;
      for (int ax = 0; ax < 3; ++ax)
        if (p[ax] < cnt[ax] && buf[ax * m + p[ax]] < best) {
          best = buf[ax * m + p[ax]];
          sel = ax;
        }
      double cur = sel < 0 ? amax : best;
      double seg = cur - prev;
      if (seg > SEGMENT_EPS) {
        acc += seg * vol[voxel_at(s, d, 0.5 * (prev + cur), o, sp, n)];
        ++used;
      }
      prev = cur;
      if (sel < 0) break;
      p[sel] += 1;
    }
    out[r] = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) * acc;
    if (steps) steps[r] = used;
  }
  free(buf);
}

/* Tangent of a crossing parameter given its selecting label.
 * _native.pyx:115-129: d_alpha = (-ds_a - alpha (dp_a - ds_a)) / d_a. */
static void alpha_tangent(int label, double alpha, const double *d,
                          const double *dsrc, const double *dpix_r, int T,
                          double *out) {
  if (label >= CONST_LABEL) {
    for (int t = 0; t < T; ++t) out[t] = 0.0;
    return;
  }
  double inv = 1.0 / d[label];
  for (int t = 0; t < T; ++t)
    out[t] = (-dsrc[label * T + t] -
              alpha * (dpix_r[label * T + t] - dsrc[label * T + t])) * inv;
}

/* Forward-mode energies + T tangents -- _native.pyx:196-282.
 * dsrc (3,T), dpix (N,3,T), dout (N,T). */
void orc_raysum_grad(const double *vol, const int64_t *n, const double *sp,
                     const double *o, const double *src, const double *dsrc,
                     const double *pix, const double *dpix, int64_t nrays,
                     int T, double *out, double *dout) {
  int64_t m = max_dim(n) + 1;
  double *buf = (double *)malloc(sizeof(double) * 3 * m);
  double *prev_t = (double *)malloc(sizeof(double) * T);
  double *cur_t = (double *)malloc(sizeof(double) * T);
  double *dacc = (double *)malloc(sizeof(double) * T);
  double s[3] = {src[0], src[1], src[2]};
  for (int64_t r = 0; r < nrays; ++r) {
    const double *dp = dpix + r * 3 * T;
    double d[3];
    for (int ax = 0; ax < 3; ++ax) d[ax] = pix[3 * r + ax] - s[ax];
    double amin, amax;
    int lmin, lmax;
    out[r] = 0.0;
    for (int t = 0; t < T; ++t) dout[r * T + t] = 0.0;
    if (!entry_exit(s, d, o, sp, n, &amin, &amax, &lmin, &lmax)) continue;
    int cnt[3], p[3] = {0, 0, 0};
    for (int ax = 0; ax < 3; ++ax)
      cnt[ax] = fill_axis(s, d, o, sp, n, ax, amin, amax, buf + ax * m);
    double acc = 0.0, prev = amin;
    for (int t = 0; t < T; ++t) dacc[t] = 0.0;
    alpha_tangent(lmin, amin, d, dsrc, dp, T, prev_t);
    for (;;) {
      int sel = -1;
      double best = INFINITY;
      for (int ax = 0; ax < 3; ++ax)
        if (p[ax] < cnt[ax] && buf[ax * m + p[ax]] < best) {
          best = buf[ax * m + p[ax]];
          sel = ax;
        }
      double cur;
      int lab;
      if (sel < 0) { cur = amax; lab = lmax; }
      else { cur = best; lab = sel; }
      alpha_tangent(lab, cur, d, dsrc, dp, T, cur_t);
      double seg = cur - prev;
      if (seg > SEGMENT_EPS) {
        double v = vol[voxel_at(s, d, 0.5 * (prev + cur), o, sp, n)];
        acc += seg * v;
        for (int t = 0; t < T; ++t) dacc[t] += v * (cur_t[t] - prev_t[t]);
      }
      prev = cur;
      memcpy(prev_t, cur_t, sizeof(double) * T);
      if (sel < 0) break;
      p[sel] += 1;
    }
    double length = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    out[r] = length * acc;
    for (int t = 0; t < T; ++t) {
      double dlen = (d[0] * (dp[0 * T + t] - dsrc[0 * T + t]) +
                     d[1] * (dp[1 * T + t] - dsrc[1 * T + t]) +
                     d[2] * (dp[2 * T + t] - dsrc[2 * T + t])) / length;
      dout[r * T + t] = dlen * acc + length * dacc[t];
    }
  }
  free(buf); free(prev_t); free(cur_t); free(dacc);
}

/* Reverse-mode restatement of the same derivative (the form the GPU backward
 * kernel computes): per ray, dE/ds (3) and dE/dp (3).  With c_k the
 * coefficient of crossing k (V of the used segment ending at k minus V of the
 * used segment starting at k), a crossing on axis a has
 *   d alpha/ds_a = (alpha - 1)/d_a,  d alpha/dp_a = -alpha/d_a
 * (the T-tangent formula of _native.pyx:115-129 with ds/dp unit seeds), and
 * the length term contributes -+ (d/|d|) acc (_native.pyx:275-281). */
void orc_raysum_endpoint_grad(const double *vol, const int64_t *n,
                              const double *sp, const double *o,
                              const double *src, const double *pix,
                              int64_t nrays, double *out, double *dEds,
                              double *dEdp) {
  int64_t m = max_dim(n) + 1;
  double *buf = (double *)malloc(sizeof(double) * 3 * m);
  double s[3] = {src[0], src[1], src[2]};
  for (int64_t r = 0; r < nrays; ++r) {
    double d[3];
    for (int ax = 0; ax < 3; ++ax) d[ax] = pix[3 * r + ax] - s[ax];
    double amin, amax;
    int lmin, lmax;
    out[r] = 0.0;
    for (int ax = 0; ax < 3; ++ax) dEds[3 * r + ax] = dEdp[3 * r + ax] = 0.0;
    if (!entry_exit(s, d, o, sp, n, &amin, &amax, &lmin, &lmax)) continue;
    int cnt[3], p[3] = {0, 0, 0};
    for (int ax = 0; ax < 3; ++ax)
      cnt[ax] = fill_axis(s, d, o, sp, n, ax, amin, amax, buf + ax * m);
    double acc = 0.0, prev = amin;
    double G[3] = {0, 0, 0}, H[3] = {0, 0, 0}; /* sum c_k, sum c_k alpha_k */
    int prev_lab = lmin;
    for (;;) {
      int sel = -1;
      double best = INFINITY;
      for (int ax = 0; ax < 3; ++ax)
        if (p[ax] < cnt[ax] && buf[ax * m + p[ax]] < best) {
          best = buf[ax * m + p[ax]];
          sel = ax;
        }
      double cur;
      int lab;
      if (sel < 0) { cur = amax; lab = lmax; }
      else { cur = best; lab = sel; }
      double seg = cur - prev;
      if (seg > SEGMENT_EPS) {
        double v = vol[voxel_at(s, d, 0.5 * (prev + cur), o, sp, n)];
        acc += seg * v;
        if (lab < CONST_LABEL) { G[lab] += v; H[lab] += v * cur; }
        if (prev_lab < CONST_LABEL) { G[prev_lab] -= v; H[prev_lab] -= v * prev; }
      }
      prev = cur;
      prev_lab = lab;
      if (sel < 0) break;
      p[sel] += 1;
    }
    double L = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
    out[r] = L * acc;
    for (int ax = 0; ax < 3; ++ax) {
      double g_s = 0.0, g_p = 0.0;
      if (d[ax] != 0.0) {
        g_s = L * (H[ax] - G[ax]) / d[ax];
        g_p = -L * H[ax] / d[ax];
      }
      dEds[3 * r + ax] = g_s - d[ax] / L * acc;
      dEdp[3 * r + ax] = g_p + d[ax] / L * acc;
    }
  }
  free(buf);
}

/* Pose 7-vector (rho, theta, phi, gamma, bx, by, bz) + isocenter -> the
 * 12-number frame (s, c, e1, e2).  Values of geometry.py:120-149 (with the
 * isocenter added as in geometry.py:166-175). */
void orc_pose_frame(const double *eta, const double *iso, double *frame) {
  double rho = eta[0], th = eta[1], ph = eta[2], ga = eta[3];
  double st = sin(th), ct = cos(th), sph = sin(ph), cph = cos(ph);
  double sg = sin(ga), cg = cos(ga);
  double u[3] = {sph * ct, sph * st, cph};
  double et[3] = {-st, ct, 0.0};
  double ep[3] = {cph * ct, cph * st, -sph};
  for (int a = 0; a < 3; ++a) {
    double source = eta[4 + a] + rho * u[a];
    double center = eta[4 + a] - rho * u[a];
    frame[0 + a] = iso[a] + source;
    frame[3 + a] = iso[a] + center;
    frame[6 + a] = cg * ep[a] - sg * et[a];
    frame[9 + a] = cg * et[a] + sg * ep[a];
  }
}

/* Detector pixel positions p[h,w] = (c + a_h e1) + a_w e2 with
 * a_h = (h - (H-1)/2) pitch_y, a_w = (w - (W-1)/2) pitch_x
 * (geometry.py:152-157,171-174; numpy evaluates left to right). */
void orc_detector_grid(const double *frame, int64_t H, int64_t W,
                       double pitch_x, double pitch_y, double *pix) {
  for (int64_t h = 0; h < H; ++h) {
    double ah = ((double)h - (double)(H - 1) / 2.0) * pitch_y;
    for (int64_t w = 0; w < W; ++w) {
      double aw = ((double)w - (double)(W - 1) / 2.0) * pitch_x;
      for (int a = 0; a < 3; ++a)
        pix[(h * W + w) * 3 + a] =
            frame[3 + a] + ah * frame[6 + a] + aw * frame[9 + a];
    }
  }
}

/* render(): one DRR from a frame (raytrace.py:132-142). */
void orc_render(const double *vol, const int64_t *n, const double *sp,
                const double *o, const double *frame, int64_t H, int64_t W,
                double pitch_x, double pitch_y, double *img, int64_t *steps) {
  double *pix = (double *)malloc(sizeof(double) * 3 * H * W);
  orc_detector_grid(frame, H, W, pitch_x, pitch_y, pix);
  orc_raysum(vol, n, sp, o, frame, pix, H * W, img, steps);
  free(pix);
}

/* Backward of render() w.r.t. the 12-number frame for an upstream pixel
 * gradient g: dL/ds = sum g dE/ds, dL/dc = sum g dE/dp,
 * dL/de1 = sum g a_h dE/dp, dL/de2 = sum g a_w dE/dp   (p = c + a_h e1 + a_w e2,
 * geometry.py:171-174).  Sequential pixel order. */
void orc_render_backward(const double *vol, const int64_t *n, const double *sp,
                         const double *o, const double *frame, int64_t H,
                         int64_t W, double pitch_x, double pitch_y,
                         const double *grad_img, double *img,
                         double *grad_frame) {
  int64_t N = H * W;
  double *pix = (double *)malloc(sizeof(double) * 3 * N);
  double *dEds = (double *)malloc(sizeof(double) * 3 * N);
  double *dEdp = (double *)malloc(sizeof(double) * 3 * N);
  orc_detector_grid(frame, H, W, pitch_x, pitch_y, pix);
  orc_raysum_endpoint_grad(vol, n, sp, o, frame, pix, N, img, dEds, dEdp);
  for (int k = 0; k < 12; ++k) grad_frame[k] = 0.0;
  for (int64_t h = 0; h < H; ++h) {
    double ah = ((double)h - (double)(H - 1) / 2.0) * pitch_y;
    for (int64_t w = 0; w < W; ++w) {
      double aw = ((double)w - (double)(W - 1) / 2.0) * pitch_x;
      int64_t r = h * W + w;
      double g = grad_img[r];
      for (int a = 0; a < 3; ++a) {
        grad_frame[0 + a] += g * dEds[3 * r + a];
        grad_frame[3 + a] += g * dEdp[3 * r + a];
        grad_frame[6 + a] += g * ah * dEdp[3 * r + a];
        grad_frame[9 + a] += g * aw * dEdp[3 * r + a];
      }
    }
  }
  free(pix); free(dEds); free(dEdp);
}
