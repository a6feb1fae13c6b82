// siddon_lean.cuh -- the counted, select-light Siddon walk (walk v5).
//
// Same segments, same arithmetic, same order as walk_select in
// siddon_walk.cuh (and therefore as the reference, _native.pyx:140-193);
// what changes is the instruction budget per voxel-step, which is what bounds
// the kernel (ncu r01: issue-bound, ALU and FP64 pipes busiest, DRAM below
// the algorithmic bytes):
//  * the number of crossings of the ray (or chunk) is counted at setup
//    (Ray::count, exact with the reference's [amin, amax] filter and the
//    chunk tie rule), so the loop has no end-of-ray compare/select;
//  * the winning axis is carried as one-hot 0/1 integers: the per-axis state
//    updates are integer multiply-adds (FMA pipe) instead of ALU selects, and
//    the reverse-mode sums (G_a, H_a) are FMAs by 0.0/1.0 masks;
//  * the winner's ray constants (d, 1/d) come from a per-thread record in
//    shared memory indexed by the axis (one LDS.128) instead of a select tree,
//    and the numerator o + k*sp - s from the source-relative plane table; the
//    exact-voxel path reads s, d from the record too, so the Ray itself is
//    dead inside the loop;
//  * each axis keeps the shared-memory byte address of its next-next plane;
//  * seg > max(T, 1e-12) is the single fast-path test (used and certified
//    voxel); everything else takes the reference's exact path out of line;
//  * the gather is a predicated load into a zeroed register, consumed one
//    iteration later, so no instruction waits on it in the issuing iteration.
#pragma once
#include "siddon_walk.cuh"

namespace drr {

// Per-thread shared-memory record: {d_a, 1/d_a} (16 B) and s_a (8 B, exact
// path only) per axis, structure-of-arrays over the CTA's threads
// (conflict-free LDS.128).  The plane table is source-relative
// (build_plane_table), so a voxel-step reads {d, 1/d} and the numerator.
// Walk tuning, per mode (A/B on C2, see profiles/):
//  * kQ: the record also holds each axis's plane-table cursor and voxel byte
//    step, so the winner's bookkeeping is two record loads and one store
//    instead of per-axis selects (fewer ALU/issue slots, more shared-memory
//    wavefronts): the gradient walks use it, the forward does not;
//  * PD: gather pipeline depth -- a segment's voxel value is consumed PD steps
//    after its load is issued (ncu lean1: 45% of stall samples waited on the
//    gather when it was consumed one step later).
#ifndef DRR_LEAN_PIPE_FWD
#define DRR_LEAN_PIPE_FWD 4
#endif
#ifndef DRR_LEAN_PIPE_GRAD
#define DRR_LEAN_PIPE_GRAD 3
#endif
// rays split over K > 1 lanes (few-pose launches: one wave or less, so latency
// matters more than occupancy) -- with 5 CTAs/SM (DRR_SPLIT_MINB_GRAD)
#ifndef DRR_LEAN_PIPE_GRAD_SPLIT
#define DRR_LEAN_PIPE_GRAD_SPLIT 4
#endif
#ifndef DRR_LEAN_Q_FWD
#define DRR_LEAN_Q_FWD 0
#endif
#ifndef DRR_LEAN_Q_GRAD
#define DRR_LEAN_Q_GRAD 1
#endif
// kQ record words per axis: the table cursor and the voxel byte step, each
// contiguous over the CTA's threads (qw below); the table step (+-8) follows
// from the voxel step's sign.  A/B on C2 fwd+jac: 2.08 ms, vs 2.14 for one
// 8-byte {cursor, step} word per thread (its cursor store is 8-byte strided:
// bank conflicts) and 2.16 for {table step, voxel step} beside the cursor.
constexpr int kLeanRecDoublesPerThread = 15;  // the largest record (gradient walk)
// Record doubles per thread a walk mode uses: {d, 1/d} x 3 and s x 3, plus
// (kQ) the cursor and voxel-step words, plus (gradient walk) the walk's end
// parameter and labels, parked there for the loop's duration.
__host__ __device__ constexpr int lean_rec_doubles(bool grad_walk) {
  return grad_walk ? 15 : (DRR_LEAN_Q_FWD ? 14 : 9);
}
constexpr int kLeanThreads = 128;  // threads per CTA of every kernel using the walk
#ifndef DRR_LEAN_UNROLL
#define DRR_LEAN_UNROLL 1
#endif
constexpr int kLeanUnroll = DRR_LEAN_UNROLL;  // pipeline blocks per loop iteration

enum LeanMode { kLeanSum = 0, kLeanCount = 1, kLeanGrad = 2 };

struct LeanSums {
  double acc = 0.0;
  double G0 = 0.0, G1 = 0.0, G2 = 0.0, H0 = 0.0, H1 = 0.0, H2 = 0.0;
  int steps = 0;
};

// Derived dominant axis (gradient walk, DRR_LEAN_DERIVE): over all crossings
// of a walk -- entry and exit included -- the coefficients telescope,
// sum_k c_k = 0, and sum_k c_k alpha_k = sum_m V_m seg_m = acc (Abel
// summation).  So only the two non-dominant axes A, B are accumulated per
// step (masks A, B; slots G0/H0, G1/H1) and the dominant axis D follows at the
// end: G_D = -(G_A + G_B + G_clip), H_D = acc - H_A - H_B - H_clip, where the
// clip terms come from a clip-labelled exit (a clip entry takes the 3-axis
// walk).  |d_D| >= |d| / sqrt(3), so the rounding of the derived H_D (a few
// ulps of acc) is not amplified by the 1/d_D of the endpoint formula.
#ifndef DRR_LEAN_DERIVE
#define DRR_LEAN_DERIVE 1
#endif

// Label of a crossing as the high words of three 0.0/1.0 doubles (one-hot over
// the axes; label 3 = clip: all zero, no tangent).  With DRR_LEAN_LAB1 the
// derived-axis walk keeps the bare axis id in h0 instead and forms the two
// masks where they are used (one register per stage, no mask copies).
#ifndef DRR_LEAN_LAB1
#define DRR_LEAN_LAB1 1
#endif
struct LabMask {
  int h0, h1, h2;
};
constexpr int kOneHi = 0x3FF00000;  // high word of 1.0
__device__ __forceinline__ LabMask lab_mask(int lab) {
  return LabMask{lab == 0 ? kOneHi : 0, lab == 1 ? kOneHi : 0, lab == 2 ? kOneHi : 0};
}

// A segment whose gather is in flight: in the gradient walk the parameter of
// its starting crossing (its length is the next stage's parameter minus this
// one -- the same subtraction the walk made, so bit-identical), in the sum walk
// its length; the value (0 if skipped), the starting crossing's label and, for
// counting, the used flag.
template <typename VT>
struct LeanStage {
  double a = 0.0;
  VT v = VT(0);
  LabMask m{0, 0, 0};
  int used = 0;
};

// G_lab += c and H_lab += c * alpha as FMAs by 0.0/1.0 masks: no per-lane
// branch and no select tree (c * 1 and c * 0 are exact; H rounds c * alpha
// once before the add, ~1 ulp of one term; the oracle bar is 1e-10 relative).
template <bool kDerive>
__device__ __forceinline__ void lean_apply(LeanSums& o, const LabMask& m, double a, double c,
                                           int axA = 0, int axB = 0) {
  const double ca = c * a;
  constexpr bool kLab1 = kDerive && DRR_LEAN_LAB1;
  const int h0 = kLab1 ? (m.h0 == axA ? kOneHi : 0) : m.h0;
  const int h1 = kLab1 ? (m.h0 == axB ? kOneHi : 0) : m.h1;
  const double k0 = __hiloint2double(h0, 0), k1 = __hiloint2double(h1, 0);
  o.G0 = __fma_rn(c, k0, o.G0);
  o.G1 = __fma_rn(c, k1, o.G1);
  o.H0 = __fma_rn(ca, k0, o.H0);
  o.H1 = __fma_rn(ca, k1, o.H1);
  if constexpr (!kDerive) {
    const double k2 = __hiloint2double(m.h2, 0);
    o.G2 = __fma_rn(c, k2, o.G2);
    o.H2 = __fma_rn(ca, k2, o.H2);
  }
}

// Consume one segment: [a, a_next) with value v.
template <int kMode, bool kDerive, typename VT>
__device__ __forceinline__ void lean_consume(LeanSums& o, double& pend, const LeanStage<VT>& st,
                                             double a_next, int axA = 0, int axB = 0) {
  if (kMode == kLeanCount) {
    o.steps += st.used;
    return;
  }
  const double vv = static_cast<double>(st.v);  // 0 for skipped segments
  // the gradient walk re-derives the length (its stage holds the start
  // parameter, needed for H); the sum walk's stage holds the length itself
  const double seg = kMode == kLeanGrad ? a_next - st.a : st.a;
  o.acc = o.acc + seg * vv;                       // _native.pyx:187 (TU is --fmad=false)
  if (kMode == kLeanGrad) {
    lean_apply<kDerive>(o, st.m, st.a, pend - vv, axA, axB);
    pend = vv;
  }
}

__device__ __forceinline__ double lds_f64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ void lds_2f64(uint32_t addr, double& a, double& b) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(a), "=d"(b) : "r"(addr));
}

// Skipped segments gather from here (a zero, so they add nothing and need no
// predicate on the load).
__device__ const double g_zero_voxel = 0.0;

// The voxel gather: read-only path; DRR_GATHER_HINT selects a cache-policy
// qualifier (0 = plain ld.global.nc).  A/B on C2 (scripts/gpu_ab_fast.sh):
// the 256-byte L2 prefetch hint (5) is ~1% faster than plain; L1 evict-first
// or no-allocate lose 8-19%; evict-last and 128-byte prefetch are neutral.
#ifndef DRR_GATHER_HINT
#define DRR_GATHER_HINT 5
#endif
__device__ __forceinline__ float gather_voxel(const float* p) {
#if DRR_GATHER_HINT == 1
  float v; asm volatile("ld.global.nc.L1::evict_last.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v;
#elif DRR_GATHER_HINT == 2
  float v; asm volatile("ld.global.nc.L1::no_allocate.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v;
#elif DRR_GATHER_HINT == 3
  float v; asm volatile("ld.global.nc.L2::128B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v;
#elif DRR_GATHER_HINT == 4
  float v; asm volatile("ld.global.nc.L1::evict_first.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v;
#elif DRR_GATHER_HINT == 5
  float v; asm volatile("ld.global.nc.L2::256B.f32 %0, [%1];" : "=f"(v) : "l"(p)); return v;
#else
  return __ldg(p);
#endif
}
__device__ __forceinline__ double gather_voxel(const double* p) { return __ldg(p); }

// Exact path (out of the fast path): the used test and the reference's
// floored midpoint (_native.pyx:68-82, 186), with s and d from the record.
// Returns the address to gather (the zero voxel for a skipped segment).
template <typename VT>
__device__ __forceinline__ const VT* lean_exact(const VT* __restrict__ vol, const GridDev& g,
                                                uint32_t dv_s, uint32_t dv_stride, uint32_t sv_s,
                                                uint32_t sv_stride, double prev, double cur,
                                                double seg, int& used) {
  used = seg > kSegEps;
  if (!used) return reinterpret_cast<const VT*>(&g_zero_voxel);
  double d0, d1, d2, i0, i1, i2;
  lds_2f64(dv_s, d0, i0);
  lds_2f64(dv_s + dv_stride, d1, i1);
  lds_2f64(dv_s + 2 * dv_stride, d2, i2);
  const double s0 = lds_f64(sv_s), s1 = lds_f64(sv_s + sv_stride),
               s2 = lds_f64(sv_s + 2 * sv_stride);
  return vol + exact_voxel(g, s0, s1, s2, d0, d1, d2, 0.5 * (prev + cur));
}

template <typename VT, int kMode, int kLeanPipe, bool kQ, bool kDerive>
__device__ __forceinline__ void lean_walk_impl(const VT* __restrict__ vol, const GridDev& g,
                                               const double* __restrict__ tab,
                                               double* __restrict__ rec, const Ray& r,
                                               LeanSums& o) {
  // next crossing parameter and smem byte address of the plane after it
  double an0 = r.an[0], an1 = r.an[1], an2 = r.an[2];
  const uint32_t tab_s = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
  const uint32_t qa_init[3] = {tab_s + 8u * static_cast<uint32_t>(r.q[0] + r.st[0]),
                               tab_s + 8u * static_cast<uint32_t>(r.q[1] + r.st[1]),
                               tab_s + 8u * static_cast<uint32_t>(r.q[2] + r.st[2])};
  const int db_init[3] = {r.st[0] * static_cast<int>(sizeof(VT)),
                          r.st[1] * g.stride[1] * static_cast<int>(sizeof(VT)),
                          r.st[2] * g.stride[2] * static_cast<int>(sizeof(VT))};
  // voxel bookkeeping as a byte pointer (a certified segment's voxel is in
  // range: its midpoint is more than the rounding noise inside every slab)
  const char* bp = reinterpret_cast<const char*>(vol + r.flat);
  // record layout (structure of arrays over the CTA's threads, in doubles
  // of nt): dv[a][tid] = {d_a, 1/d_a} (the winner's division constants: one
  // LDS.128) at 0; sv[a][tid] = s_a (exact path only) at 6; (kQ) qw[a][tid]
  // = table cursor, qw[3 + a][tid] = voxel byte step (4-byte words) at 9;
  // (gradient walk) the parked exit labels at 13.5 and end parameter at 14
  constexpr int nt = kLeanThreads;
  double* dv = rec + 2 * threadIdx.x;
  double* sv = rec + 6 * nt + threadIdx.x;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dv[2 * a * nt] = r.d[a];
    dv[2 * a * nt + 1] = r.inv[a];
    sv[a * nt] = r.s[a];
  }
  const uint32_t dv_s = static_cast<uint32_t>(__cvta_generic_to_shared(dv));
  const uint32_t sv_s = static_cast<uint32_t>(__cvta_generic_to_shared(sv));
  constexpr uint32_t dv_stride = 16u * nt, sv_stride = 8u * nt;
  // (!kQ) cursors and steps in registers
  uint32_t qa0 = qa_init[0], qa1 = qa_init[1], qa2 = qa_init[2];
  const int qs0 = 8 * r.st[0], qs1 = 8 * r.st[1], qs2 = 8 * r.st[2];
  const int db0 = db_init[0], db1 = db_init[1], db2 = db_init[2];
  uint32_t* qw = reinterpret_cast<uint32_t*>(rec + 9 * nt) + threadIdx.x;
  if constexpr (kQ) {
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      qw[a * nt] = qa_init[a];
      qw[(3 + a) * nt] = static_cast<uint32_t>(db_init[a]);
    }
  }
  const uint32_t qw_s = static_cast<uint32_t>(__cvta_generic_to_shared(qw));
  constexpr uint32_t qw_stride = 4u * nt;
  // (gradient walk) the end parameter and labels are only needed after the
  // loop: park them in the record instead of holding registers across it
  double* park_a = rec + 14 * nt + threadIdx.x;
  uint32_t* park_l = reinterpret_cast<uint32_t*>(rec + 12 * nt) + 3 * nt + threadIdx.x;
  if constexpr (kMode == kLeanGrad) {
    *park_a = r.amax;
    *park_l = static_cast<uint32_t>(r.lab_max) | (static_cast<uint32_t>(r.D) << 8);
  }
  asm volatile("" ::: "memory");  // the record stores precede every record load
  const double T2 = fmax(r.T, kSegEps);
  double prev = r.amin;
  // non-dominant axes (kDerive): masks h0 = [axis == A], h1 = [axis == B]
  const int axA = r.D == 0 ? 1 : 0, axB = r.D == 2 ? 1 : 2;
  auto derive_mask = [&](int lab) {
    if (DRR_LEAN_LAB1) return LabMask{lab, 0, 0};
    return LabMask{lab == axA ? kOneHi : 0, lab == axB ? kOneHi : 0, 0};
  };
  LabMask lm = kDerive ? derive_mask(r.lab_min) : lab_mask(r.lab_min);  // crossing at prev
  double pend = 0.0;
  // Ring of kLeanPipe in-flight segments (gather issued, value consumed
  // kLeanPipe steps later).  Steps run in blocks of kLeanPipe with the ring
  // slot fixed at compile time, so stages never move between registers.
  // Initially every slot is an empty segment [amin, amin) (adds nothing).
  LeanStage<VT> st[kLeanPipe];
#pragma unroll
  for (int j = 0; j < kLeanPipe; ++j) st[j].a = kMode == kLeanGrad ? prev : 0.0;
  // one step: consume ring slot j (the segment issued kLeanPipe steps ago;
  // it ends where slot j+1's segment starts), pick the winning crossing,
  // issue this segment's gather into slot j
  auto step = [&](int j) {
    lean_consume<kMode, kDerive, VT>(o, pend, st[j], st[(j + 1) % kLeanPipe].a, axA, axB);
    const bool c1 = an1 < an0;  // ties go to the lowest axis (_native.pyx:180-183)
    const double b01 = c1 ? an1 : an0;
    const bool c2 = an2 < b01;
    const double cur = c2 ? an2 : b01;
    const int m2 = c2, m1 = c1 && !c2, m0 = !(c1 || c2);
    // advance the winning axis
    const uint32_t k = m1 + 2 * m2;
    double d, inv;
    lds_2f64(dv_s + k * dv_stride, d, inv);
    double num;  // (o + k*sp) - s from the source-relative plane table
    int db;
    if constexpr (kQ) {
      uint32_t qa;
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(qa) : "r"(qw_s + k * qw_stride));
      asm volatile("ld.shared.u32 %0, [%1];" : "=r"(db) : "r"(qw_s + (3 + k) * qw_stride));
      num = lds_f64(qa);
      const uint32_t qs = 8u + (static_cast<uint32_t>(db >> 31) << 4);  // +-8 by the walk's sign
      asm volatile("st.shared.u32 [%0], %1;" :: "r"(qw_s + k * qw_stride), "r"(qa + qs) : "memory");
    } else {
      num = lds_f64(m0 * qa0 + m1 * qa1 + m2 * qa2);
      qa0 += m0 * qs0;
      qa1 += m1 * qs1;
      qa2 += m2 * qs2;
      db = m0 * db0 + m1 * db1 + m2 * db2;
    }
    const double an = div_rn(num, d, inv);
    an0 = m0 ? an : an0;
    an1 = m1 ? an : an1;
    an2 = m2 ? an : an2;
    // segment [prev, cur] in the bookkeeping voxel
    const VT* gp = reinterpret_cast<const VT*>(bp);
    int used = 1;
    const double seg = cur - prev;
    if (!(seg > T2)) gp = lean_exact(vol, g, dv_s, dv_stride, sv_s, sv_stride, prev, cur, seg, used);
    bp += db;
    st[j].v = gather_voxel(gp);
    st[j].used = used;
    st[j].a = kMode == kLeanGrad ? prev : seg;
    st[j].m = lm;
    if constexpr (kDerive)
      lm = derive_mask(static_cast<int>(k));
    else
      lm = LabMask{m0 * kOneHi, m1 * kOneHi, m2 * kOneHi};
    prev = cur;
  };
  const int n = r.count;
#pragma unroll(kLeanUnroll)
  for (int blk = n / kLeanPipe; blk > 0; --blk) {
#pragma unroll
    for (int j = 0; j < kLeanPipe; ++j) step(j);
  }
  const int rem = n % kLeanPipe;
#pragma unroll
  for (int j = 0; j + 1 < kLeanPipe; ++j)
    if (j < rem) step(j);
  // drain oldest first: slots rem..PD-1 (previous block), then 0..rem-1; each
  // ends where the next-younger one starts, the youngest at prev
#pragma unroll
  for (int j = 0; j < kLeanPipe; ++j)
    if (j >= rem)
      lean_consume<kMode, kDerive, VT>(o, pend, st[j],
                              j + 1 < kLeanPipe ? st[j + 1].a : (rem > 0 ? st[0].a : prev), axA,
                              axB);
#pragma unroll
  for (int j = 0; j + 1 < kLeanPipe; ++j)
    if (j < rem)
      lean_consume<kMode, kDerive, VT>(o, pend, st[j], j + 1 < rem ? st[j + 1].a : prev, axA, axB);
  // final segment [last crossing, amax]
  double amax = r.amax;
  int lab_max = r.lab_max, Dax = r.D;
  if constexpr (kMode == kLeanGrad) {
    uint32_t pl;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(amax)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(park_a))));
    asm volatile("ld.shared.u32 %0, [%1];" : "=r"(pl)
                 : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(park_l))));
    lab_max = static_cast<int>(pl & 0xFFu);
    Dax = static_cast<int>(pl >> 8);
  }
  {
    const double cur = amax;
    const double seg = cur - prev;
    const VT* gp = reinterpret_cast<const VT*>(bp);
    int used = 1;
    if (!(seg > T2)) gp = lean_exact(vol, g, dv_s, dv_stride, sv_s, sv_stride, prev, cur, seg, used);
    LeanStage<VT> last;
    last.a = kMode == kLeanGrad ? prev : seg;
    last.v = gather_voxel(gp);
    last.used = used;
    last.m = lm;
    lean_consume<kMode, kDerive, VT>(o, pend, last, cur, axA, axB);
  }
  if constexpr (kMode == kLeanGrad) {
    if constexpr (kDerive) {
      lean_apply<true>(o, derive_mask(lab_max), amax, pend, axA, axB);
      const double gc = lab_max == kConstLabel ? pend : 0.0;
      const double hc = lab_max == kConstLabel ? pend * amax : 0.0;
      const double gA = o.G0, gB = o.G1, hA = o.H0, hB = o.H1;
      const double gD = -((gA + gB) + gc), hD = ((o.acc - hA) - hB) - hc;
      o.G0 = Dax == 0 ? gD : gA;
      o.H0 = Dax == 0 ? hD : hA;
      o.G1 = Dax == 1 ? gD : (Dax == 0 ? gA : gB);
      o.H1 = Dax == 1 ? hD : (Dax == 0 ? hA : hB);
      o.G2 = Dax == 2 ? gD : gB;
      o.H2 = Dax == 2 ? hD : hB;
    } else {
      lean_apply<false>(o, lab_mask(lab_max), amax, pend);
    }
  }
}

// Rays with a subnormal-scale direction component (Ray::safe: |d_a| <= 1e-20,
// never produced by a detector pose in practice) need IEEE division for their
// crossing parameters; they take the v4 visitor walk, which has that path.
template <typename VT, int kMode>
__device__ __forceinline__ void safe_walk(const VT* __restrict__ vol, const GridDev& g,
                                          const double* __restrict__ tab, const Ray& r,
                                          LeanSums& o) {
  if (kMode == kLeanSum) {
    SumVisitor v;
    walk_select<VT, true>(vol, g, tab, r, v);
    o.acc = v.acc;
  } else if (kMode == kLeanCount) {
    CountVisitor v;
    walk_select<VT, true>(vol, g, tab, r, v);
    o.steps = v.steps;
  } else {
    GradVisitor v;
    walk_select<VT, true>(vol, g, tab, r, v);
    o.acc = v.acc;
    o.G0 = v.G0; o.G1 = v.G1; o.G2 = v.G2;
    o.H0 = v.H0; o.H1 = v.H1; o.H2 = v.H2;
  }
}

template <typename VT, int kMode, bool kSplit = false>
__device__ __forceinline__ void lean_walk(const VT* __restrict__ vol, const GridDev& g,
                                          const double* __restrict__ tab, double* rec,
                                          const Ray& r, LeanSums& o) {
  constexpr int kPipeGrad = kSplit ? DRR_LEAN_PIPE_GRAD_SPLIT : DRR_LEAN_PIPE_GRAD;
  if (r.safe)
    safe_walk<VT, kMode>(vol, g, tab, r, o);
  else if (kMode == kLeanGrad && DRR_LEAN_DERIVE && r.lab_min != kConstLabel)
    lean_walk_impl<VT, kMode, kPipeGrad, DRR_LEAN_Q_GRAD, true>(vol, g, tab, rec, r, o);
  else
    lean_walk_impl<VT, kMode, kMode == kLeanGrad ? kPipeGrad : DRR_LEAN_PIPE_FWD,
                   kMode == kLeanGrad ? DRR_LEAN_Q_GRAD : DRR_LEAN_Q_FWD, false>(vol, g, tab, rec,
                                                                                 r, o);
}

}  // namespace drr
