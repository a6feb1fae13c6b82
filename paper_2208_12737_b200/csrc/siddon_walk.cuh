// siddon_walk.cuh -- grid / ray types, the per-ray setup (slab entry and
// exit, first crossings, crossing count, fast-voxel certificate, ray
// splitting) and the select-based walk (v4) with its visitors.  The kernels
// walk with siddon_lean.cuh; the v4 walk here serves rays whose direction has
// a subnormal-scale component (Ray::safe), which need IEEE division.
//
// Semantics are those of the reference's vectorised Siddon kernel
// (_native.pyx:140-193 / python_ref.py:130-138): the ray R(a) = s + a (p - s),
// a in [amin, amax] from the slab rule clipped to [0, 1]; all plane crossings
// a_k = (o + k sp - s) / d inside [amin, amax] are visited in ascending order
// (ties -> lowest axis first); segments with seg <= 1e-12 are skipped; each
// used segment adds seg * V[voxel(midpoint)]; E = |p - s| * sum.
//
// B200 design (not a port of the reference's sort-and-merge):
//  * no crossing list is materialised -- each axis keeps only its NEXT plane
//    index and crossing parameter, so a ray is O(1) registers and the walk is
//    one pass over the voxels it touches;
//  * every crossing parameter is bit-identical to the reference's
//    (o + k*sp - s)/d: the division is replaced by one multiply by the
//    correctly-rounded reciprocal plus one Markstein FMA correction, which is
//    the correctly rounded quotient (checked against IEEE division);
//  * the voxel of a segment comes from the next-plane indices (pure integer
//    bookkeeping).  The reference floors the midpoint instead; the two agree
//    whenever the midpoint is farther than the rounding noise from every
//    plane, which `seg > T` certifies (T per ray, see ray_setup).  Segments
//    that fail the test (near-ties, grazing and near-parallel rays) take the
//    reference's exact floor/clamp path, so results stay bit-identical.
//
// The translation unit is compiled with --fmad=false: every a*b+c written
// below rounds twice, exactly like the reference's C (built without -march,
// so without FMA contraction).  FMAs that are wanted are explicit __fma_rn.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace drr {

constexpr double kSegEps = 1e-12;  // _native.pyx:16
constexpr int kConstLabel = 3;     // _native.pyx:17

struct GridDev {
  int n[3];
  int stride[3];   // 1, nx, nx*ny
  int total;       // nx*ny*nz (< 2^31, checked on the host)
  double sp[3];
  double o[3];
  double hi[3];    // o + n*sp, as _native.pyx:34 computes it
  // faces of the occupied box (every voxel outside it is exactly zero):
  // P(lo) and P(hi) with P(k) = o + k*sp rounded as the plane table rounds it,
  // so the trimmed entry / exit parameters are the walk's own crossing
  // parameters of those planes; the whole volume gives tlo = o, thi = hi
  double tlo[3], thi[3];
  // optional occupied hull (hull != 0): in voxel-index coordinates u_a =
  // (x_a - o_a) / sp_a every voxel that is not exactly zero lies inside
  // hlo[q] <= n_q . u <= hhi[q] for the kHullDirs directions n_q of
  // hull_dir (the box covers the axis directions); the supports are of the
  // voxels' whole boxes, widened by 1/16 voxel against rounding (the fp32 slab
  // tests err by ~1e-4 voxel, the reference's midpoints by ~1e-12)
  int hull;
  float isp[3];  // 1 / sp
  double ispd[3];  // 1 / sp in double (setup estimates)
  float hlo[16], hhi[16];
};
// A/B (scripts/gpu_ab_trim.sh, 256 C2 poses): unrolled 10.70 ms, rolled 12.71
// (its runtime direction table); box-only trimming 11.31 / 11.78.
#ifndef DRR_HULL_UNROLL
#define DRR_HULL_UNROLL 1
#endif
// Hull directions (integer components, voxel-index space): the 10 diagonals
// of the cube, then 4 in-plane (x, y) directions that round the octagonal
// cross-section to a 16-gon (a patient's body is a prism along z).  The ABI
// carries 16 slots (drr_grid::hull_lo / hull_hi).
#ifndef DRR_HULL_DIRS
#define DRR_HULL_DIRS 14
#endif
constexpr int kHullDirs = DRR_HULL_DIRS;
__host__ __device__ __forceinline__ int hull_dir(int q, int a) {
  constexpr int kDir[16][3] = {{1, 1, 0}, {1, -1, 0}, {1, 0, 1}, {1, 0, -1}, {0, 1, 1},
                               {0, 1, -1}, {1, 1, 1}, {1, 1, -1}, {1, -1, 1}, {-1, 1, 1},
                               {2, 1, 0}, {1, 2, 0}, {2, -1, 0}, {1, -2, 0},
                               {0, 0, 0}, {0, 0, 0}};
  return kDir[q][a];
}

template <typename VT>
__device__ __forceinline__ double load_voxel(const VT* __restrict__ vol, int i) {
  return static_cast<double>(__ldg(vol + i));
}

// Setup divisions (entry / exit, first crossings, counts) by the walk's
// Markstein form instead of IEEE '/' -- both correctly rounded, so the same
// bits (all GPU parity tests); A/B (scripts/gpu_ab_var.sh, 256 C2 poses):
// fwd+jac 10.35 -> 9.97 ms.
#ifndef DRR_SETUP_DIVRN
#define DRR_SETUP_DIVRN 1
#endif

// Correctly rounded num / d given inv = RN(1/d) (Markstein correction).
__device__ __forceinline__ double div_rn(double num, double d, double inv) {
  const double q0 = __dmul_rn(num, inv);
  const double r = __fma_rn(-q0, d, num);
  return __fma_rn(r, inv, q0);
}

// Crossing parameter of plane k on one axis, reference operation order:
// (o + k*sp - s) / d   (_native.pyx:105).
__device__ __forceinline__ double plane_alpha(double o, double sp, int k,
                                              double s, double d, double inv,
                                              bool safe) {
  const double num = (o + static_cast<double>(k) * sp) - s;
  if (safe) return num / d;  // subnormal-scale direction: plain IEEE division
  return div_rn(num, d, inv);
}

// The reference's midpoint voxel lookup, exactly (_native.pyx:68-82).
__device__ __forceinline__ int exact_index(double s, double d, double mid,
                                           double o, double sp, int n) {
  const double f = floor((s + mid * d - o) / sp);
  if (!(f >= 0.0)) return 0;  // also maps NaN to 0 like the reference's cast
  if (f >= static_cast<double>(n)) return n - 1;
  return static_cast<int>(f);
}

__device__ __forceinline__ int exact_voxel(const GridDev& g, double s0, double s1,
                                        double s2, double d0, double d1,
                                        double d2, double mid) {
  const int i = exact_index(s0, d0, mid, g.o[0], g.sp[0], g.n[0]);
  const int j = exact_index(s1, d1, mid, g.o[1], g.sp[1], g.n[1]);
  const int k = exact_index(s2, d2, mid, g.o[2], g.sp[2], g.n[2]);
  return i + g.n[0] * (j + g.n[1] * k);
}

// ---- plane table ---------------------------------------------------------
// Per CTA, shared memory holds every plane coordinate P_a(k) = o_a + k*sp_a
// (the reference's expression, _native.pyx:105) for k = 0..n_a, bracketed by
// kPad sentinel slots on each side whose crossing parameter is a huge positive
// number in the walking direction, so an exhausted axis never wins the merge
// (and the lookahead walk may read up to kPad slots past the last plane).
// Axis a's P_a(0) sits at index plane_base(g, a).
constexpr double kSentinel = 1e280;
constexpr int kPad = 3;

__host__ __device__ __forceinline__ int plane_table_len(const GridDev& g) {
  return g.n[0] + g.n[1] + g.n[2] + 3 * (2 * kPad + 1);
}
// Start of the per-thread area after the plane table, in doubles: rounded up
// to an even count so 16-byte shared-memory vector loads stay aligned.
__host__ __device__ __forceinline__ int plane_table_span(const GridDev& g) {
  return (plane_table_len(g) + 1) & ~1;
}
__host__ __device__ __forceinline__ int plane_base(const GridDev& g, int a) {
  return a == 0 ? kPad
                : (a == 1 ? g.n[0] + 1 + 3 * kPad : g.n[0] + g.n[1] + 2 + 5 * kPad);
}

// The table is source-relative: entry k of axis a holds the numerator of the
// crossing parameter, (o_a + k*sp_a) - s_a -- the reference's two roundings in
// its order (_native.pyx:105), so num / d is the same division.  Every ray of
// a CTA shares the source (one pose per CTA; one source per explicit-ray
// call), so the walk reads the numerator instead of P and s: one shared-memory
// load and one add fewer per voxel-step.  Sentinels stay +-1e280 (|s| is far
// below their ulp).
__device__ __forceinline__ void build_plane_table(const GridDev& g, const double* __restrict__ src,
                                                  double* tab) {
  const int l0 = g.n[0] + 1 + 2 * kPad, l1 = g.n[1] + 1 + 2 * kPad,
            l2 = g.n[2] + 1 + 2 * kPad;
  for (int i = threadIdx.x; i < l0 + l1 + l2; i += blockDim.x) {
    int j, n;
    double o, sp, s;
    if (i < l0) { j = i; n = g.n[0]; o = g.o[0]; sp = g.sp[0]; s = __ldg(src); }
    else if (i < l0 + l1) { j = i - l0; n = g.n[1]; o = g.o[1]; sp = g.sp[1]; s = __ldg(src + 1); }
    else { j = i - l0 - l1; n = g.n[2]; o = g.o[2]; sp = g.sp[2]; s = __ldg(src + 2); }
    const int k = j - kPad;
    double v;
    if (k < 0) v = -kSentinel;
    else if (k > n) v = kSentinel;
    else v = (o + static_cast<double>(k) * sp) - s;
    tab[i] = v;
  }
}

struct Ray {
  double s[3], d[3], inv[3];
  double an[3];     // crossing parameter of the next plane per axis
  int q[3];         // plane-table index of that plane
  int st[3];        // +1 / -1 walking direction, 0 for a parallel axis
  double amin, amax;  // start / end crossing of this walk (whole ray or chunk)
  double T;         // fast-voxel threshold on seg (see ray_setup)
  int lab_min, lab_max;
  int end_lab;      // chunked walk: crossings tied with amax on axes >= end_lab
                    // belong to the next chunk (kNoEndLab for a ray's real exit)
  int flat;         // flat voxel index of the segment after amin
  int count;        // crossings this walk takes (the counted walk, siddon_lean.cuh)
  int D;            // dominant axis: largest |d_a| / sp_a
  bool hit;
  bool safe;        // some |d_a| tiny: use IEEE '/' instead of the Markstein form
};
constexpr int kNoEndLab = 4;

// Slab entry/exit, first-max/first-min labels over (x, y, z, clip):
// _native.pyx:20-65.  The slab is the occupied box [tlo, thi] (GridDev): a
// walk over it is the reference's walk over the whole volume with its
// exactly-zero margins left out.  Every segment outside the box has value 0
// and every crossing outside it coefficient 0 (value before = after = 0), so
// acc, G and H receive the same nonzero terms in the same order; at the box
// faces the entry / exit semantics (a virtual crossing at amin with the
// first-max label, then every plane crossing with amin <= alpha <= amax,
// ties to the lowest axis) put the same coefficient on the same crossing as
// the full walk does.  Bit-identical results (tests/test_gpu_trim.py).
__device__ __forceinline__ void entry_exit(const GridDev& g, Ray& r) {
  double cmin[3], cmax[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (r.d[a] == 0.0) {
      const bool inside = (g.tlo[a] <= r.s[a]) && (r.s[a] <= g.thi[a]);
      cmin[a] = inside ? -INFINITY : INFINITY;
      cmax[a] = inside ? INFINITY : -INFINITY;
    } else {
#if DRR_SETUP_DIVRN
      // correctly rounded like IEEE '/', by the walk's Markstein form (r.inv
      // and r.safe are set before entry_exit in this build)
      double a0 = r.safe ? (g.tlo[a] - r.s[a]) / r.d[a] : div_rn(g.tlo[a] - r.s[a], r.d[a], r.inv[a]);
      double a1 = r.safe ? (g.thi[a] - r.s[a]) / r.d[a] : div_rn(g.thi[a] - r.s[a], r.d[a], r.inv[a]);
#else
      double a0 = (g.tlo[a] - r.s[a]) / r.d[a];
      double a1 = (g.thi[a] - r.s[a]) / r.d[a];
#endif
      if (a0 > a1) { const double t = a0; a0 = a1; a1 = t; }
      cmin[a] = a0;
      cmax[a] = a1;
    }
  }
  // First-max over (x, y, z, clip=0) and first-min over (x, y, z, clip=1):
  // strict comparisons keep the lowest label on ties.
  double bmin = cmin[0], bmax = cmax[0];
  int lmin = 0, lmax = 0;
#pragma unroll
  for (int a = 1; a < 3; ++a) {
    if (cmin[a] > bmin) { bmin = cmin[a]; lmin = a; }
    if (cmax[a] < bmax) { bmax = cmax[a]; lmax = a; }
  }
  if (0.0 > bmin) { bmin = 0.0; lmin = kConstLabel; }
  if (1.0 < bmax) { bmax = 1.0; lmax = kConstLabel; }
  r.lab_min = lmin;
  r.amin = bmin;
  r.lab_max = lmax;
  r.amax = bmax;
  r.hit = r.amin < r.amax;
}

// Axis parameters by (possibly runtime) axis index.
__device__ __forceinline__ void axis_params(const GridDev& g, const Ray& r, int a,
                                            double& o, double& sp, double& s, double& d,
                                            double& inv, int& st, int& n) {
  if (a == 0) { o = g.o[0]; sp = g.sp[0]; s = r.s[0]; d = r.d[0]; inv = r.inv[0]; st = r.st[0]; n = g.n[0]; }
  else if (a == 1) { o = g.o[1]; sp = g.sp[1]; s = r.s[1]; d = r.d[1]; inv = r.inv[1]; st = r.st[1]; n = g.n[1]; }
  else { o = g.o[2]; sp = g.sp[2]; s = r.s[2]; d = r.d[2]; inv = r.inv[2]; st = r.st[2]; n = g.n[2]; }
}

// First plane k (in walking order, may be -1 / n+1 = none) on axis a whose
// crossing parameter is after a_s: alpha > a_s (strict) or alpha >= a_s.
// Estimate, then fix up with exact crossing parameters (monotone in k).
__device__ __forceinline__ int first_plane_after(const GridDev& g, const Ray& r, int a,
                                                 double a_s, bool strict) {
  double o, sp, s, d, inv;
  int st, n;
  axis_params(g, r, a, o, sp, s, d, inv, st, n);
  const double t = (s + a_s * d - o) * g.ispd[a];  // an estimate: fixed up exactly below
  double kf = st > 0 ? ceil(t) : floor(t);
  kf = fmin(fmax(kf, -1.0), (double)n + 1.0);
  int k = (int)kf;
  for (int it = 0; it < 64; ++it) {
    const int kb = k - st;
    if (kb >= 0 && kb <= n) {
      const double ab = plane_alpha(o, sp, kb, s, d, inv, !DRR_SETUP_DIVRN || r.safe);
      if (strict ? ab > a_s : ab >= a_s) { k = kb; continue; }
    }
    if (k >= 0 && k <= n) {
      const double ak = plane_alpha(o, sp, k, s, d, inv, !DRR_SETUP_DIVRN || r.safe);
      if (!(strict ? ak > a_s : ak >= a_s)) { k += st; continue; }
    }
    break;
  }
  return k;
}

__device__ __forceinline__ double axis_alpha(const GridDev& g, const Ray& r, int a, int k) {
  double o, sp, s, d, inv;
  int st, n;
  axis_params(g, r, a, o, sp, s, d, inv, st, n);
  return plane_alpha(o, sp, k, s, d, inv, !DRR_SETUP_DIVRN || r.safe);
}

// Trim [amin, amax] to the occupied hull (GridDev::hull), exactly.  fp32 slab
// tests against the kHullDirs hull directions give the approximate parameters where
// the ray enters and leaves the hull; since the hull holds the non-zero
// voxels' whole boxes (widened against rounding), everything the exact ray
// meets before the entry -- midpoint rounding included -- is an exactly-zero
// voxel.  The walk then starts at the last dominant-axis plane crossing at
// least 1/16 voxel before the entry (its
// exact parameter, the walk's own) with entry_exit's semantics (a virtual
// crossing, then every crossing >= amin on every axis, ties to the lowest
// axis), and stops symmetrically after the exit: the skipped segments add
// +0 and the skipped crossings carry coefficient 0, so images and sums keep
// the full walk's bits.  A ray that misses the hull is a miss (its full walk
// sums zeros).
__device__ __forceinline__ void hull_trim(const GridDev& g, Ray& r) {
  float us[3], ud[3];
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    us[a] = static_cast<float>((r.s[a] - g.o[a]) * static_cast<double>(g.isp[a]));
    ud[a] = static_cast<float>(r.d[a] * static_cast<double>(g.isp[a]));
  }
  float tin = static_cast<float>(r.amin), tout = static_cast<float>(r.amax);
#if DRR_HULL_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
  for (int q = 0; q < kHullDirs; ++q) {
    float ns = 0.f, nd = 0.f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      ns += hull_dir(q, a) * us[a];
      nd += hull_dir(q, a) * ud[a];
    }
    if (nd != 0.f) {
      const float inv = 1.0f / nd;
      const float t1 = (g.hlo[q] - ns) * inv, t2 = (g.hhi[q] - ns) * inv;
      tin = fmaxf(tin, fminf(t1, t2));
      tout = fminf(tout, fmaxf(t1, t2));
    } else if (ns < g.hlo[q] || ns > g.hhi[q]) {
      tin = 1.f;
      tout = 0.f;
    }
  }
  if (!(tin < tout)) {
    r.hit = false;
    return;
  }
  const int D = r.D;
  const double udD = D == 0 ? ud[0] : (D == 1 ? ud[1] : ud[2]);
  const double usD = D == 0 ? us[0] : (D == 1 ? us[1] : us[2]);
  const int stD = udD > 0.0 ? 1 : -1;
  const double half = 0.0625 / fabs(udD);  // 1/16 dominant-axis voxel, in alpha
  const int nD = g.n[D];
  if (static_cast<double>(tin) - half > r.amin) {
    const double target = static_cast<double>(tin) - half;
    const double u = usD + target * udD;
    int k = static_cast<int>(stD > 0 ? floor(u) : ceil(u));  // last D-plane before target
    k = k < 0 ? 0 : (k > nD ? nD : k);
    double ak = axis_alpha(g, r, D, k);
    if (!(ak < target)) {
      k -= stD;
      ak = (k >= 0 && k <= nD) ? axis_alpha(g, r, D, k) : r.amin;
    }
    if (ak > r.amin && ak < target) {
      r.amin = ak;
      r.lab_min = D;
    }
  }
  if (static_cast<double>(tout) + half < r.amax) {
    const double target = static_cast<double>(tout) + half;
    const double u = usD + target * udD;
    int k = static_cast<int>(stD > 0 ? ceil(u) : floor(u));  // first D-plane after target
    k = k < 0 ? 0 : (k > nD ? nD : k);
    double ak = axis_alpha(g, r, D, k);
    if (!(ak > target)) {
      k += stD;
      ak = (k >= 0 && k <= nD) ? axis_alpha(g, r, D, k) : r.amax;
    }
    if (ak < r.amax && ak > target) {
      r.amax = ak;
      r.lab_max = D;
    }
  }
  r.hit = r.amin < r.amax;
}

// Per-ray setup for chunk `chunk` of `nchunks` (one ray split
// across threads by dominant-axis plane index ranges).  The crossing sequence
// of the whole ray, ordered by (alpha, axis) like the reference's merge, is
// cut at dominant-axis crossings B_j = (alpha_D(b_j), D); chunk j walks the
// segments between B_j and B_{j+1}, so every segment (and every crossing's
// reverse-mode coefficient) is counted exactly once across the chunks.
// nchunks = 1 is the whole ray with the reference's entry/exit semantics.
__device__ __forceinline__ void ray_setup(const GridDev& g, const double* s,
                                          const double* p, Ray& r,
                                          int nchunks = 1, int chunk = 0) {
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.s[a] = s[a];
    r.d[a] = p[a] - s[a];
  }
#if DRR_SETUP_DIVRN
  r.safe = false;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    r.inv[a] = r.d[a] == 0.0 ? 0.0 : __drcp_rn(r.d[a]);
    if (r.d[a] != 0.0 && !(fabs(r.d[a]) > 1e-20)) r.safe = true;
  }
#endif
  entry_exit(g, r);
#if !DRR_SETUP_DIVRN
  r.safe = false;
#endif
  r.end_lab = kNoEndLab;
  if (!r.hit) return;
  double T = 0.0, wmax = -1.0;
  int D = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double d = r.d[a];
    if (d == 0.0) {
      r.st[a] = 0;
      r.inv[a] = 0.0;
      continue;
    }
    const double inv = __drcp_rn(d);
    if (!(fabs(d) > 1e-20)) r.safe = true;
    r.inv[a] = inv;
    r.st[a] = d > 0.0 ? 1 : -1;
    // Fast-voxel certificate.  The reference's midpoint position and our
    // crossing parameters carry rounding error below ~2^-50 * M voxels, with
    // M the coordinate magnitude in voxel units.  A used segment's midpoint
    // sits at least seg/2 * |d|/sp voxels from every a-plane, so
    // seg > 2^-39 * (M + 1) * sp / |d| guarantees floor(midpoint) equals the
    // next-plane bookkeeping with a 2^10 safety factor.
    const double M = fabs(r.s[a]) + fabs(d) + fabs(g.o[a]) + fabs(g.hi[a]) + g.sp[a];
#if DRR_SETUP_DIVRN
    T = fmax(T, 0x1.0p-39 * M * fabs(inv));  // a threshold: any rounding is fine (2^10 margin)
#else
    T = fmax(T, 0x1.0p-39 * M / fabs(d));
#endif
    const double w = fabs(d) * g.ispd[a];
    if (w > wmax) { wmax = w; D = a; }
  }
  r.T = T;
  r.D = D;
  if (g.hull) {
    hull_trim(g, r);
    if (!r.hit) return;
  }
  // Start event per axis: (amin, entry) for chunk 0, else (alpha_D(b_j), D).
  double a_s = r.amin;
  int lab_s = -1;  // -1: entry semantics (every crossing with alpha >= amin)
  if (nchunks > 1) {
    const int stD = D == 0 ? r.st[0] : (D == 1 ? r.st[1] : r.st[2]);
    const int kf = first_plane_after(g, r, D, r.amin, false);
    const int kl = first_plane_after(g, r, D, r.amax, true) - stD;
    const int nD = (kl - kf) * stD + 1;
    bool split = nD >= 2 * nchunks;
    // boundaries must be strictly increasing crossings (always true unless
    // |d_D| / sp_D exceeds ~2^52; then fall back to one thread per ray)
    for (int j = 1; split && j < nchunks; ++j) {
      const int b = kf + stD * ((j * nD) / nchunks);
      split = axis_alpha(g, r, D, b) > axis_alpha(g, r, D, b - stD);
    }
    if (!split) {
      if (chunk != 0) { r.hit = false; return; }
    } else {
      if (chunk > 0) {
        const int b = kf + stD * ((chunk * nD) / nchunks);
        a_s = axis_alpha(g, r, D, b);
        lab_s = D;
        r.amin = a_s;
        r.lab_min = D;
      }
      if (chunk < nchunks - 1) {
        const int b = kf + stD * (((chunk + 1) * nD) / nchunks);
        r.amax = axis_alpha(g, r, D, b);
        r.lab_max = D;
        r.end_lab = D;
      }
    }
  }
  int vox[3];
  r.count = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    if (r.st[a] == 0) {
      // Constant index along a parallel axis: the reference evaluates
      // floor(((s + mid*0) - o)/sp) = floor((s - o)/sp), then clamps.
      r.q[a] = plane_base(g, a);
      r.an[a] = INFINITY;
      const double f = floor((r.s[a] - g.o[a]) / g.sp[a]);
      vox[a] = !(f >= 0.0) ? 0 : (f >= (double)g.n[a] ? g.n[a] - 1 : (int)f);
      continue;
    }
    int k;
    if (lab_s < 0) k = first_plane_after(g, r, a, a_s, false);
    else if (a == lab_s) k = first_plane_after(g, r, a, a_s, false) + r.st[a];
    else k = first_plane_after(g, r, a, a_s, a < lab_s);
    // (a == D: the plane after b_j -- b_j is the first plane with
    //  alpha >= a_s, the split test excludes an exact tie with b_j - st;
    //  a < D: ties at a_s came before B_j; a > D: ties at a_s come after it)
    const int n = g.n[a];
    r.q[a] = plane_base(g, a) + k;
    r.an[a] = (k >= 0 && k <= n) ? axis_alpha(g, r, a, k) : kSentinel;
    vox[a] = r.st[a] > 0 ? k - 1 : k;
    // crossings of axis a this walk takes: after the start event (k on) and
    // up to the end event -- alpha <= amax, or alpha < amax for axes >= end_lab
    const int k_end = first_plane_after(g, r, a, r.amax, a < r.end_lab);
    const int c = (k_end - k) * r.st[a];
    r.count += c > 0 ? c : 0;
  }
  r.flat = vox[0] + g.stride[1] * vox[1] + g.stride[2] * vox[2];
}

// Gather pipeline depth of the v4 walk (segment i's voxel load is consumed in
// iteration i + DRR_PIPE).
#ifndef DRR_PIPE
#define DRR_PIPE 1
#endif

template <typename VT>
struct PipeStage {
  bool used;
  double seg, a;
  int lab;
  VT v;
};

template <typename VT, bool kChunked, typename Visitor>
__device__ __forceinline__ void walk_select(const VT* __restrict__ vol,
                                            const GridDev& g,
                                            const double* __restrict__ tab,
                                            const Ray& r, Visitor& vis) {
  double an0 = r.an[0], an1 = r.an[1], an2 = r.an[2];
  int q0 = r.q[0], q1 = r.q[1], q2 = r.q[2];
  const double s0 = r.s[0], s1 = r.s[1], s2 = r.s[2];
  const double d0 = r.d[0], d1 = r.d[1], d2 = r.d[2];
  const double i0 = r.inv[0], i1 = r.inv[1], i2 = r.inv[2];
  const int st0 = r.st[0], st1 = r.st[1], st2 = r.st[2];
  const int df0 = st0, df1 = st1 * g.stride[1], df2 = st2 * g.stride[2];
  const double amax = r.amax, T = r.T;
  const bool safe = r.safe;
  const unsigned total = static_cast<unsigned>(g.total);
  int flat = r.flat;
  double prev = r.amin;
  int lab = r.lab_min;
  // pipe[0] is the oldest in-flight segment; empty stages are unused zero
  // segments (harmless to every visitor, see GradVisitor::segment).
  PipeStage<VT> pipe[DRR_PIPE];
#pragma unroll
  for (int k = 0; k < DRR_PIPE; ++k) pipe[k] = PipeStage<VT>{false, 0.0, 0.0, 0, VT(0)};
  for (;;) {
    const bool c1 = an1 < an0;
    double best = c1 ? an1 : an0;
    const bool c2 = an2 < best;
    best = c2 ? an2 : best;
    bool last = !(best <= amax);
    if (kChunked)  // chunk end B_{j+1} = (amax, end_lab): ties on axes >= end_lab come after it
      last = last || (best == amax && (c2 ? 2 : (c1 ? 1 : 0)) >= r.end_lab);
    const double cur = last ? amax : best;
    const double seg = cur - prev;
    const bool used = seg > kSegEps;
    int idx = flat;
    if (used && (!(seg > T) || static_cast<unsigned>(flat) >= total))
      idx = exact_voxel(g, s0, s1, s2, d0, d1, d2, 0.5 * (prev + cur));
    VT v = VT(0);
    if (used) v = __ldg(vol + idx);
    if constexpr (Visitor::kIndex) vis.index(used, idx, lab);
    vis.segment(pipe[0].used, pipe[0].seg, static_cast<double>(pipe[0].v), pipe[0].lab,
                pipe[0].a);
#pragma unroll
    for (int k = 0; k + 1 < DRR_PIPE; ++k) pipe[k] = pipe[k + 1];
    pipe[DRR_PIPE - 1] = PipeStage<VT>{used, seg, prev, lab, v};
    prev = cur;
    if (last) break;
    const double d = c2 ? d2 : (c1 ? d1 : d0);
    const double inv = c2 ? i2 : (c1 ? i1 : i0);
    const int q = (c2 ? q2 : (c1 ? q1 : q0)) + (c2 ? st2 : (c1 ? st1 : st0));
    const double num = tab[q];  // (o + q*sp) - s: the source-relative table
    const double an = safe ? num / d : div_rn(num, d, inv);
    const bool a0 = !(c1 || c2), a1 = c1 && !c2;
    an0 = a0 ? an : an0;
    an1 = a1 ? an : an1;
    an2 = c2 ? an : an2;
    q0 = a0 ? q : q0;
    q1 = a1 ? q : q1;
    q2 = c2 ? q : q2;
    flat += c2 ? df2 : (c1 ? df1 : df0);
    lab = c2 ? 2 : (c1 ? 1 : 0);
  }
#pragma unroll
  for (int k = 0; k < DRR_PIPE; ++k)
    vis.segment(pipe[k].used, pipe[k].seg, static_cast<double>(pipe[k].v), pipe[k].lab,
                pipe[k].a);
  vis.finish(r.lab_max, amax);
}

// ---- visitors ----------------------------------------------------------

struct SumVisitor {
  static constexpr bool kIndex = false;
  double acc = 0.0;
  __device__ __forceinline__ void segment(bool used, double seg, double v, int,
                                          double) {
    // _native.pyx:187 (TU built --fmad=false).  Unused segments arrive with
    // v = 0 and seg >= 0, so adding seg*v = +0 leaves acc bit-identical.
    (void)used;
    acc = acc + seg * v;
  }
  __device__ __forceinline__ void finish(int, double) {}
};

struct CountVisitor {
  static constexpr bool kIndex = false;
  int steps = 0;
  __device__ __forceinline__ void segment(bool used, double, double, int, double) {
    steps += used ? 1 : 0;
  }
  __device__ __forceinline__ void finish(int, double) {}
};

// Reverse mode: each crossing k on axis a carries the coefficient
// c_k = v(segment ending at k) - v(segment starting at k) (0 for skipped
// segments); with d alpha_k/ds_a = (alpha_k - 1)/d_a and
// d alpha_k/dp_a = -alpha_k/d_a the ray's endpoint gradients need only
// G_a = sum c_k and H_a = sum c_k alpha_k.  Label 3 (clip) has no tangent.
struct GradVisitor {
  static constexpr bool kIndex = false;
  double acc = 0.0;
  double pend = 0.0;  // value of the used segment ending at the next crossing
  double G0 = 0.0, G1 = 0.0, G2 = 0.0, H0 = 0.0, H1 = 0.0, H2 = 0.0;
  __device__ __forceinline__ void apply(int label, double alpha, double c) {
    // per-axis accumulation via selects (label 3 = clip: no tangent); measured
    // faster than predicated branches (profiles/r01_v2 A/B)
    const double c0 = label == 0 ? c : 0.0;
    const double c1 = label == 1 ? c : 0.0;
    const double c2 = label == 2 ? c : 0.0;
    G0 += c0; G1 += c1; G2 += c2;
    H0 = __fma_rn(c0, alpha, H0);
    H1 = __fma_rn(c1, alpha, H1);
    H2 = __fma_rn(c2, alpha, H2);
  }
  __device__ __forceinline__ void segment(bool used, double seg, double v,
                                          int lab_start, double a_start) {
    const double vv = used ? v : 0.0;
    acc = acc + seg * vv;
    apply(lab_start, a_start, pend - vv);
    pend = vv;
  }
  __device__ __forceinline__ void finish(int lab_end, double a_end) {
    apply(lab_end, a_end, pend);
  }
};

// Discrete structure of a traversal (python_ref.py:191-201 ray_structure:
// crossing labels in merge order, the used set, the voxel of each used
// segment, the exit selector) folded into a 64-bit hash.  Two poses whose
// rays hash alike share the piecewise-smooth branch of the energy map, so a
// finite-difference stencil between them is kink-free (gradients.py:124-167).
__host__ __device__ __forceinline__ uint64_t sig_mix(uint64_t h, uint64_t x) {
  h ^= x + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
  h ^= h >> 29;
  h *= 0xBF58476D1CE4E5B9ull;
  return h ^ (h >> 32);
}
struct SigVisitor {
  static constexpr bool kIndex = true;
  uint64_t h = 0x6A09E667F3BCC908ull;
  __device__ __forceinline__ void index(bool used, int idx, int lab) {
    h = sig_mix(h, (static_cast<uint64_t>(used ? static_cast<uint32_t>(idx) : 0xFFFFFFFFu) << 8) |
                       static_cast<uint64_t>(lab & 0xFF));
  }
  __device__ __forceinline__ void segment(bool, double, double, int, double) {}
  __device__ __forceinline__ void finish(int lab_end, double) {
    h = sig_mix(h, 0x100u | static_cast<uint64_t>(lab_end & 0xFF));
  }
};

}  // namespace drr
