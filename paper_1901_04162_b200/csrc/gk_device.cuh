// gk_device.cuh -- device data layout and FP64 math shared by the sm_100a
// kernels of libgk (table build, fill, standalone evaluation).
//
// Layout in HBM:
//   Green interval records, one per plan interval j = 0..n-2 plus a sentinel
//   record n-1 for r = r_max, stride 2 + 2(d+1) doubles:
//     { a_j, a_{j+1}, c0.re, c0.im, c1.re, c1.im, ..., cd.re, cd.im }
//   where P_j(u) = sum_k c_k u^k, u = r - a_j, is the degree-d Lagrange
//   interpolant through the reference's stencil for interval j
//   (evaluator.hpp:40-95, 237-272; same nodes, so the same polynomial up to
//   rounding) and c0 is the node value itself (exact node reproduction).
//   Exp interval records (linear, evaluator.hpp:22-30), 6 doubles:
//     { a_j, a_{j+1}, e_j.re, e_j.im, slope.re, slope.im }.
//   Lookup buckets (uint32, width dr_min/2, so at most one node per bucket):
//     lk[b] = max(0, #{nodes with bucket < b} - 1); the interval holding r is
//     j = lk[b] + (r >= a_{lk[b]+1}), exactly the reference's locate()
//     (table.hpp:87-102) without clamping: r = r_max lands on the sentinel.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

// GK_DASSERT: device-side index/contract checks, compiled in only for the
// assert build (scripts/build_variant.sh asserts -DGK_DEVICE_ASSERTS), which
// stands in for compute-sanitizer (closed on the GPU pool): a failure traps
// the kernel and the ABI call returns GK_ERR_RUNTIME.
#ifdef GK_DEVICE_ASSERTS
#include <cstdio>
#define GK_DASSERT(c)                                                                 \
  do {                                                                                \
    if (!(c)) {                                                                       \
      printf("GK_DASSERT failed: %s (%s:%d) block %d thread %d\n", #c, __FILE__, __LINE__, \
             blockIdx.x, threadIdx.x);                                                \
      __trap();                                                                       \
    }                                                                                 \
  } while (0)
#else
#define GK_DASSERT(c) ((void)0)
#endif

namespace gk {

constexpr double kPi = 3.14159265358979323846;
constexpr double kMagic52 = 4503599627370496.0;   // 2^52
constexpr double kMagicRint = 6755399441055744.0; // 1.5 * 2^52

// Direct-mode phase table size: e^{-j theta} = e^{-j 2pi idx/M} e^{-j delta},
// |delta| <= D = pi/M = 3.8e-4 (128 KB of shared memory).  sin delta =
// delta - delta^3/6 (dropped delta^5/120 < 7e-20); cos delta - 1 = c delta^2
// with c the minimax constant on [0, D^2] (kCosMinimax): max error
// 0.00715 D^4 = 1.5e-16 (0.7 ulp of 1) for one DMUL instead of FMA + DMUL.
#ifndef GK_PHASE_COPYLOG2
#define GK_PHASE_COPYLOG2 0
#endif
constexpr int kPhaseLog2 = 13 - GK_PHASE_COPYLOG2;
constexpr int kPhaseM = 1 << kPhaseLog2;
// table entries per angle (1: one table).  Tried: 8 lane-interleaved copies of
// a 1024-entry table (conflict-free LDS.128, 2 more FP64 ops for the longer
// polynomials) -- C5 K4e 502 vs 468 ms, K4 883 vs 799 ms: not adopted
constexpr int kPhaseCopyLog2 = GK_PHASE_COPYLOG2;
constexpr int kPhaseSlots = kPhaseM << kPhaseCopyLog2;  // table entries (double2)
// c = -1/2 + b D^2, b = (sqrt 2 - 1)/12: the error x(-1/2 - c) + x^2/24,
// x = delta^2, equioscillates at x = D^2 and x = -12(-1/2 - c)
constexpr double kPhaseD = kPi / kPhaseM;
constexpr double kCosMinimax = -0.5 + (1.4142135623730951 - 1.0) / 12.0 * kPhaseD * kPhaseD;


struct TableDev {
  const double* grec;  // Green interval records
  const double* erec;  // Exp interval records
  const uint32_t* lk;  // lookup buckets
  double r_min, r_max;
  double inv_w, bias;  // bucket map: x = fma(r, inv_w, bias), b = floor(x)
  uint32_t nlk;
  uint32_t nrec;  // interval records (= plan nodes; record n-1 is the r_max sentinel)
  int degree;
  int grs;  // Green record stride in doubles = 2 + 2 (degree + 1)
  double k_re, k_im;
  // arithmetic locate on the uniform base grid (arith_locate): base point i is
  // r_min + i t_eff; coarse[c] = plan index - i for the 65 base points
  // 64 c .. 64 c + 64 when they are consecutive plan nodes, else -1
  const int32_t* coarse;
  uint32_t ncoarse;  // 0: off
  double t_eff, inv_t;
  // table sweep (K3s): node values on the base grid -- bg[i] / be[i] is the
  // Green / Exp value of plan node r_min + i t_eff (zero where that base point
  // is not a plan node), i = 0 .. nbase-1 -- and one bit per base interval i,
  // set where the reference's degree-3 stencil of the interval is base points
  // i-1 .. i+2 as consecutive plan nodes (equally spaced: the Lagrange
  // weights are the uniform ones)
  const double2* bg;
  const double2* be;
  const uint32_t* bclean;  // nbase / 32 + 8 words (zero-padded)
  uint32_t nbase;
  // the plan intervals overlapping a base interval whose bit is clear (and the
  // tail [a_{nbase-1}, r_max] with the r_max sentinel): pj[k] = plan interval,
  // pa[k] = its left node, ascending -- the sweep stages their records so
  // that non-uniform stencils are read from shared memory too
  const uint32_t* pj;
  const double* pa;
  uint32_t npatch;
};

// Shared-edge fills (direct_edge_kernel, table_edge_kernel; edges.cu): a
// block is the range [tb, te) of block positions (a bisection order of the
// source triangles, or the mesh order) and the distinct edges its triangles
// use (ne <= the mesh's edge cap), whose points sit at ep[c0 * n * 64 ...] as
// [chunk][point][(x, y) | (z, w)][32 lanes] double2.  (cx, cy, cz, rho) bounds every inner point of
// the block.
//
// Edge cap: 11 warp-wide chunks (352 edges) by default, 1..12 with
// GK_EDGE_CHUNKS at mesh creation.  12 warps x 352 edge sums + the 128 KB
// phase table stay under the 196 KB shared-memory carveout, leaving 60 KB of
// L1 for the block's points (12 chunks: 228 KB carveout, 28 KB of L1).
constexpr int kEdgeCap = 384;
constexpr int kEdgeChunksDefault = 11;
constexpr int kSweepChunksDefault = 2;  // the table sweep's block set (K3s)
constexpr int kSweepLeafPct = 50;      // its bisection leaves: 50 % of the edge cap
constexpr double kSweepRhoCap = 1.2;   // and no leaf wider than 1.2x the mean block radius
struct EdgeBlock {
  uint32_t tb, te, c0, ne;
  double cx, cy, cz, rho;
};

// ---------------------------------------------------------------- helpers

// squared distance; FMA form (pinned: all kernels share this one function so
// K1's range and the fills see bit-identical radii)
__device__ __forceinline__ double dist2(double ox, double oy, double oz, double ix, double iy,
                                        double iz) {
  const double dx = ox - ix, dy = oy - iy, dz = oz - iz;
  return __fma_rn(dz, dz, __fma_rn(dy, dy, __dmul_rn(dx, dx)));
}

// 1/sqrt(x) to ~1 ulp: MUFU.RSQ64H seed + one third-order correction
__device__ __forceinline__ double rsqrt_fast(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = __fma_rn(-x, __dmul_rn(y, y), 1.0);
  const double ye = __dmul_rn(y, e);
  return __fma_rn(ye, __fma_rn(0.375, e, 0.5), y);
}

// r = d2 * rsqrt(d2).  At a zero-distance pair rsqrt(0) = inf makes that
// NaN; the Exp kind is defined there (eval_analytic(PlainExp, k, 0) = (1, 0),
// kernel.hpp:58-60), so it takes r = 0 (Green stays NaN -> GK_ERR_DOMAIN,
// kernel.hpp:51-53).  Compile-time: no cost for the Green fills.
template <int KIND>
__device__ __forceinline__ double radius_of(double d2, double y) {
  const double r = __dmul_rn(d2, y);
  if constexpr (KIND == GK_KIND_EXP) return d2 > 0.0 ? r : 0.0;
  return r;
}

// bucket of r in the lookup hash (r >= r_min gives x >= 0); clamped so any
// input (out of range, NaN) yields a readable bucket
__device__ __forceinline__ uint32_t lookup_bucket(double r, const TableDev& t) {
  const double x = __fma_rn(r, t.inv_w, t.bias);
  const double y = __dadd_rd(x, kMagic52);
  const uint32_t b = static_cast<uint32_t>(__double2loint(y));
  return b < t.nlk ? b : t.nlk - 1;
}

// interval index of r (table.hpp:87-102 semantics, sentinel at r_max)
// base point i of the plan's uniform grid, rounded like build_plan
// (sampling.hpp:167, no contraction)
__device__ __forceinline__ double base_point(const TableDev& t, long long i) {
  return __dadd_rn(t.r_min, __dmul_rn(static_cast<double>(i), t.t_eff));
}

// Interval of r by arithmetic where r lies in a verified run of consecutive
// base-grid nodes (away from the refinement windows around zeros): no lookup
// bucket and no record header are read.  Returns false where the run
// structure does not hold (the caller takes the lookup path); when it
// returns true, j and a_j equal the lookup path's exactly.
__device__ __forceinline__ bool arith_locate(double r, const TableDev& t, uint32_t& j,
                                             double& aj) {
  if (t.ncoarse == 0 || !(r >= t.r_min)) return false;
  long long i = static_cast<long long>((r - t.r_min) * t.inv_t);  // guess, exact after the fix
  const long long imax = static_cast<long long>(t.ncoarse) * 64;
  if (i >= imax) return false;
  double a0 = base_point(t, i), a1 = base_point(t, i + 1);
  if (r < a0) {
    if (i == 0) return false;
    --i;
    a1 = a0;
    a0 = base_point(t, i);
  } else if (r >= a1) {
    ++i;
    if (i >= imax) return false;
    a0 = a1;
    a1 = base_point(t, i + 1);
  }
  if (!(a0 <= r && r < a1)) return false;
  const int32_t off = __ldg(t.coarse + (i >> 6));
  if (off < 0) return false;
  j = static_cast<uint32_t>(i + off);
  aj = a0;
  GK_DASSERT(j + 1 < t.nrec);  // a run never reaches the r_max sentinel
  return true;
}

__device__ __forceinline__ uint32_t locate_interval(double r, const TableDev& t,
                                                    const double* grec, int grs, double& aj) {
  {
    uint32_t j;
    if (arith_locate(r, t, j, aj)) return j;
  }
  const uint32_t base = __ldg(t.lk + lookup_bucket(r, t));
  GK_DASSERT(base < t.nrec);
  const double2 ab = __ldg(reinterpret_cast<const double2*>(grec + static_cast<size_t>(base) * grs));
  const bool hi = r >= ab.y;
  aj = hi ? ab.y : ab.x;
  // the located interval brackets r (table.hpp:87-102 contract) for r in range
  GK_DASSERT(!(r >= t.r_min && r <= t.r_max) || (aj <= r && base + (hi ? 1u : 0u) < t.nrec));
  return base + (hi ? 1u : 0u);
}

// Green kernel by table: degree-3 fast path
template <int DEG>
__device__ __forceinline__ double2 green_table(double r, const TableDev& t) {
  constexpr int RS = 2 + 2 * (DEG + 1);
  double aj;
  const uint32_t j = locate_interval(r, t, t.grec, RS, aj);
  const double2* c = reinterpret_cast<const double2*>(t.grec + static_cast<size_t>(j) * RS + 2);
  const double u = r - aj;
  double2 acc = __ldg(c + DEG);
#pragma unroll
  for (int k = DEG - 1; k >= 0; --k) {
    const double2 ck = __ldg(c + k);
    acc.x = __fma_rn(acc.x, u, ck.x);
    acc.y = __fma_rn(acc.y, u, ck.y);
  }
  return acc;
}

// runtime-degree variant (degrees other than the instantiated fast paths)
__device__ __forceinline__ double2 green_table_any(double r, const TableDev& t) {
  double aj;
  const uint32_t j = locate_interval(r, t, t.grec, t.grs, aj);
  const double2* c = reinterpret_cast<const double2*>(t.grec + static_cast<size_t>(j) * t.grs + 2);
  const double u = r - aj;
  double2 acc = __ldg(c + t.degree);
  for (int k = t.degree - 1; k >= 0; --k) {
    const double2 ck = __ldg(c + k);
    acc.x = __fma_rn(acc.x, u, ck.x);
    acc.y = __fma_rn(acc.y, u, ck.y);
  }
  return acc;
}

// Exp kernel by table (linear, evaluator.hpp:22-30)
__device__ __forceinline__ double2 exp_table(double r, const TableDev& t) {
  double aj;
  // Exp records carry the same {a_j, a_{j+1}} header as the Green records
  const uint32_t j = locate_interval(r, t, t.erec, 6, aj);
  const double2* c = reinterpret_cast<const double2*>(t.erec + static_cast<size_t>(j) * 6 + 2);
  const double u = r - aj;
  const double2 e0 = __ldg(c), s = __ldg(c + 1);
  return make_double2(__fma_rn(s.x, u, e0.x), __fma_rn(s.y, u, e0.y));
}

// Exp (linear) and Green (Lagrange) sharing one lookup: the Exp and Green
// records carry the same {a_j, a_{j+1}} header (fused pair fill)
template <int DEG>
__device__ __forceinline__ void pair_table(double r, const TableDev& t, double2& e, double2& g) {
  const int grs = DEG > 0 ? 2 + 2 * (DEG + 1) : t.grs;
  const int deg = DEG > 0 ? DEG : t.degree;
  double aj;
  const uint32_t j = locate_interval(r, t, t.grec, grs, aj);
  const double u = r - aj;
  const double2* ce = reinterpret_cast<const double2*>(t.erec + static_cast<size_t>(j) * 6 + 2);
  const double2 e0 = __ldg(ce), sl = __ldg(ce + 1);
  e = make_double2(__fma_rn(sl.x, u, e0.x), __fma_rn(sl.y, u, e0.y));
  const double2* c = reinterpret_cast<const double2*>(t.grec + static_cast<size_t>(j) * grs + 2);
  double2 acc = __ldg(c + deg);
#pragma unroll
  for (int k = deg - 1; k >= 0; --k) {
    const double2 ck = __ldg(c + k);
    acc.x = __fma_rn(acc.x, u, ck.x);
    acc.y = __fma_rn(acc.y, u, ck.y);
  }
  g = acc;
}

// ------------------------------------------- table window (shared memory)
//
// The fill's table path evaluates through a TableWin: a contiguous window of
// lookup buckets [b0, b0 + nb) and interval records [j0, j0 + nj), either the
// whole table in global memory (SMEM = false, read through L1 with __ldg) or
// the slice a tile needs, staged into shared memory by a TMA bulk copy
// (SMEM = true).  Indices are clamped into the window, so any input (out of
// range, NaN) reads valid memory; in-range radii of the tile are inside the
// window by construction (monotone bucket map, conservative tile bounds).
struct TableWin {
  const double* grec;
  const double* erec;
  const uint32_t* lk;
  uint32_t b0, nb, j0, nj;
};

template <bool SMEM, class T>
__device__ __forceinline__ T win_ld(const T* p) {
  if constexpr (SMEM) return *p;
  else return __ldg(p);
}

// used: the lane's value is kept (a valid, non-self pair) -- padding and self
// lanes also evaluate, their radii may lie outside the tile's window and
// their (clamped, meaningless) values are discarded
template <bool SMEM>
__device__ __forceinline__ uint32_t win_locate(double r, const TableDev& t, const TableWin& w,
                                               int grs, double& aj, bool used = true) {
  if constexpr (!SMEM) {  // in shared memory the lookup is cheaper than the arithmetic
    uint32_t j;
    if (arith_locate(r, t, j, aj) && j - w.j0 < w.nj) return j - w.j0;
  }
  uint32_t b = lookup_bucket(r, t) - w.b0;
  GK_DASSERT(!SMEM || !used || b < w.nb || !(r >= t.r_min && r <= t.r_max));  // window covers
  b = b < w.nb ? b : w.nb - 1;
  uint32_t base = win_ld<SMEM>(w.lk + b) - w.j0;
  GK_DASSERT(!SMEM || !used || base < w.nj || !(r >= t.r_min && r <= t.r_max));
  base = base < w.nj ? base : w.nj - 1;
  const double2 ab = win_ld<SMEM>(reinterpret_cast<const double2*>(w.grec + static_cast<size_t>(base) * grs));
  const bool hi = r >= ab.y;
  aj = hi ? ab.y : ab.x;
  const uint32_t j = base + (hi ? 1u : 0u);
  return j < w.nj ? j : w.nj - 1;
}

// Green (degree DEG, or runtime degree for DEG = 0), Exp, or both for one r
template <bool SMEM, int DEG, bool WANT_E, bool WANT_G>
__device__ __forceinline__ void win_eval(double r, const TableDev& t, const TableWin& w,
                                         double2& e, double2& g, bool used = true) {
  const int grs = DEG > 0 ? 2 + 2 * (DEG + 1) : t.grs;
  const int deg = DEG > 0 ? DEG : t.degree;
  double aj;
  const uint32_t j = win_locate<SMEM>(r, t, w, grs, aj, used);
  const double u = r - aj;
  if constexpr (WANT_E) {
    const double2* ce = reinterpret_cast<const double2*>(w.erec + static_cast<size_t>(j) * 6 + 2);
    const double2 e0 = win_ld<SMEM>(ce), sl = win_ld<SMEM>(ce + 1);
    e = make_double2(__fma_rn(sl.x, u, e0.x), __fma_rn(sl.y, u, e0.y));
  }
  if constexpr (WANT_G) {
    const double2* c = reinterpret_cast<const double2*>(w.grec + static_cast<size_t>(j) * grs + 2);
    double2 acc = win_ld<SMEM>(c + deg);
#pragma unroll
    for (int k = deg - 1; k >= 0; --k) {
      const double2 ck = win_ld<SMEM>(c + k);
      acc.x = __fma_rn(acc.x, u, ck.x);
      acc.y = __fma_rn(acc.y, u, ck.y);
    }
    g = acc;
  }
}

// --------------------------------------------------- TMA bulk-copy helpers

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t done = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(phase)
        : "memory");
  } while (!done);
}

constexpr int kKindPair = 2;  // fused Exp + Green sharing r

template <int KIND, int DEG>
__device__ __forceinline__ void table_values(double r, const TableDev& T, double2& v, double2& vg) {
  if constexpr (KIND == kKindPair) pair_table<DEG>(r, T, v, vg);
  else if constexpr (KIND == GK_KIND_EXP) v = exp_table(r, T);
  else if constexpr (DEG == 3) v = green_table<3>(r, T);
  else v = green_table_any(r, T);
}

// a staged window of base-grid node values (the table sweep K3s,
// fill_sweep.cuh, and the staged eval_batch, eval.cu)
struct SweepWin {
  const double2* g;      // Green node values of base points i0 .. i0 + wn - 1
  const double2* e;      // Exp node values
  const uint32_t* bits;  // clean bits, words w0 ..
  int i0, w0, wn;
  double x0, inv_t;  // x = fma(r, inv_t, x0) = (r - r_min) / t_eff
  // staged patch records (TableDev::pj / pa): np intervals with left nodes
  // pa[], Green records pg[] (10 doubles: a_j, a_j+1, c0..c3) and Exp records
  // pe[] (6 doubles: a_j, a_j+1, e_j, slope)
  const double* pa;
  const double* pg;
  const double* pe;
  int np;
};

// the staged record of the plan interval holding r, evaluated exactly like
// the global records (green_table<3> / exp_table / pair_table<3>: same
// record, same operations, so the same bits); false when no staged record
// holds r (the caller reads the global records)
template <int KIND>
__device__ __forceinline__ bool patch_values(double r, const SweepWin& W, double2& v, double2& vg) {
  constexpr bool WANT_G = KIND != GK_KIND_EXP, WANT_E = KIND != GK_KIND_GREEN;
  int lo = 0, hi = W.np;  // first staged record with pa > r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (W.pa[mid] <= r) lo = mid + 1;
    else hi = mid;
  }
  const int k = lo - 1;
  if (k < 0) return false;
  const double* rg = W.pg + 10 * k;
  const double* re = W.pe + 6 * k;
  if (!(r < (WANT_G ? rg[1] : re[1]))) return false;
  const double u = r - W.pa[k];
  double2 e = make_double2(0.0, 0.0), g = make_double2(0.0, 0.0);
  if constexpr (WANT_E) {
    e.x = __fma_rn(re[4], u, re[2]);
    e.y = __fma_rn(re[5], u, re[3]);
  }
  if constexpr (WANT_G) {
    g = make_double2(rg[8], rg[9]);
#pragma unroll
    for (int c = 2; c >= 0; --c) {
      g.x = __fma_rn(g.x, u, rg[2 + 2 * c]);
      g.y = __fma_rn(g.y, u, rg[3 + 2 * c]);
    }
  }
  if constexpr (KIND == kKindPair) {
    v = e;
    vg = g;
  } else if constexpr (KIND == GK_KIND_GREEN) {
    v = g;
  } else {
    v = e;
  }
  return true;
}

// stage the patch records a window of radii [a_lo, a_hi] can need (all of
// them, or none when they exceed cap) into pa / pg / pe; every thread of the CTA calls it, a __syncthreads
// follows before use.  Returns the count (the same in every thread).
template <bool WANT_G, bool WANT_E>
__device__ __forceinline__ int stage_patches(const TableDev& T, double a_lo, double a_hi, int cap,
                                             double* pa, double* pg, double* pe, int* s_k) {
  if (threadIdx.x == 0) {
    const int n = static_cast<int>(T.npatch);
    int lo = 0, hi = n;  // first k with pa > a_lo
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (T.pa[mid] <= a_lo) lo = mid + 1;
      else hi = mid;
    }
    const int k0 = lo > 0 ? lo - 1 : 0;
    hi = n;  // first k with pa > a_hi
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (T.pa[mid] <= a_hi) lo = mid + 1;
      else hi = mid;
    }
    const int cnt = lo - k0;
    s_k[0] = k0;
    s_k[1] = cnt <= cap ? cnt : 0;  // all or none: a partial list costs its misses a search
  }
  __syncthreads();
  const int k0 = s_k[0], cnt = s_k[1];
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) pa[i] = T.pa[k0 + i];
  if (WANT_G)
    for (int i = threadIdx.x; i < 10 * cnt; i += blockDim.x)
      pg[i] = T.grec[static_cast<size_t>(T.pj[k0 + i / 10]) * 10 + i % 10];
  if (WANT_E)
    for (int i = threadIdx.x; i < 6 * cnt; i += blockDim.x)
      pe[i] = T.erec[static_cast<size_t>(T.pj[k0 + i / 6]) * 6 + i % 6];
  return cnt;
}


// K(r) for the kind through the window, or the global records where the
// interval is not a uniform stencil inside the window
// EXACT: the interval and s from the rounded base points themselves (like
// arith_locate), so that s = 0 exactly at a node and nodes are reproduced
// exactly (evaluator.hpp:259-262; the standalone eval_batch); the fills
// need only the tolerance and take s from x = (r - r_min) / t_eff directly
// PATCH: non-uniform intervals first look for a staged record (the window
// stages them when they are few, S = 1e4); without it they go straight to
// the global records (dense zero windows, S = 1e3: the lookup would cost more
// than it saves -- C3 S = 1e3 102 vs 136 ms per 8192 rows)
template <int KIND, bool EXACT = false, bool PATCH = false>
__device__ __forceinline__ void sweep_values(double r, const SweepWin& W, const TableDev& T,
                                             double2& v, double2& vg) {
  constexpr bool WANT_G = KIND != GK_KIND_EXP, WANT_E = KIND != GK_KIND_GREEN;
  const double x = __fma_rn(r, W.inv_t, W.x0);
  const double yv = __dadd_rd(x, kMagic52);  // floor(x) + 2^52 (0 <= x < 2^31 in range)
  int i = __double2loint(yv);
  double s;
  if constexpr (EXACT) {
    double a0 = base_point(T, i), a1 = base_point(T, i + 1);
    if (r < a0) {
      --i;
      a0 = base_point(T, i);
    } else if (r >= a1) {
      ++i;
      a0 = a1;
    }
    s = (r - a0) * W.inv_t;
  } else {
    s = x - (yv - kMagic52);  // in [0, 1)
  }
  const int ii = i - W.i0;
  const bool win = static_cast<unsigned>(ii - 1) < static_cast<unsigned>(W.wn - 4);
  const int ic = win ? ii : 1;  // clamped: the window reads stay in bounds
  const int ia = W.i0 + ic;
  const bool ok = win && ((W.bits[(ia >> 5) - W.w0] >> (ia & 31)) & 1u);
  double2 g = make_double2(0.0, 0.0), e = make_double2(0.0, 0.0);
  if constexpr (WANT_G) {
    // uniform cubic Lagrange weights on nodes -1, 0, 1, 2
    const double2* f = W.g + (ic - 1);
    const double2 f0 = f[0], f1 = f[1], f2 = f[2], f3 = f[3];
    const double b = s - 1.0;
    const double sb = s * b;
    const double cm = __fma_rn(s, -1.0 / 6.0, 1.0 / 3.0);  // -(s - 2) / 6
    const double a6 = __fma_rn(s, 1.0 / 6.0, 1.0 / 6.0);   // (s + 1) / 6
    const double hb = __fma_rn(s, 0.5, -0.5);              // (s - 1) / 2
    const double h2 = __fma_rn(s, hb, -1.0);               // (s + 1)(s - 2) / 2
    const double w0 = sb * cm, w3 = sb * a6, w1 = h2 * b, w2 = -h2 * s;
    g.x = __fma_rn(w3, f3.x, __fma_rn(w2, f2.x, __fma_rn(w1, f1.x, w0 * f0.x)));
    g.y = __fma_rn(w3, f3.y, __fma_rn(w2, f2.y, __fma_rn(w1, f1.y, w0 * f0.y)));
  }
  if constexpr (WANT_E) {  // linear (evaluator.hpp:22-30)
    const double2 e0 = W.e[ic], e1 = W.e[ic + 1];
    e.x = __fma_rn(s, e1.x - e0.x, e0.x);
    e.y = __fma_rn(s, e1.y - e0.y, e0.y);
  }
  if constexpr (KIND == kKindPair) {
    v = e;
    vg = g;
  } else if constexpr (KIND == GK_KIND_GREEN) {
    v = g;
  } else {
    v = e;
  }
  if constexpr (PATCH) {
    if (!ok && !(win && patch_values<KIND>(r, W, v, vg))) table_values<KIND, 3>(r, T, v, vg);
  } else {
    if (!ok) table_values<KIND, 3>(r, T, v, vg);
  }
}

// ------------------------------------------------------------ direct math

// exp(-j k r) from a phase table tab[M] = (cos 2pi i/M, sin 2pi i/M) in
// shared memory: phi = r K1 (K1 = k M / 2pi), n = rint(phi) (1.5 2^52 magic
// add), f = phi - n in [-1/2, 1/2], delta = 2pi f / M;
//   cos(theta0 + delta) = C0 (1 + v) - S0 s,  sin(theta0 + delta) = S0 (1 + v) + C0 s
// with v = cos(delta) - 1 = kCosMinimax delta^2 and s = delta - delta^3/6.
// Returns (Re, -Im) of exp(-j k r) = (cos kr, sin kr): 11 FP64 ops + 1 LDS.128.
// table slot of angle index n (the lane's copy in the interleaved layout)
__device__ __forceinline__ unsigned phase_slot(unsigned n) {
  return ((n & (kPhaseM - 1)) << kPhaseCopyLog2) | (threadIdx.x & ((1u << kPhaseCopyLog2) - 1u));
}

// v = cos(delta) - 1 and s = sin(delta) for delta = 2 pi f / M
__device__ __forceinline__ void phase_poly(double f, double& v, double& s) {
  constexpr double C = 2.0 * kPi / kPhaseM;
  const double g = __dmul_rn(f, f);
  constexpr double s1 = C;
  constexpr double s3 = -C * C * C / 6.0;
  if constexpr (kPhaseM >= 8192) {
    constexpr double a1 = kCosMinimax * C * C;
    v = __dmul_rn(a1, g);
    s = __dmul_rn(f, __fma_rn(s3, g, s1));
  } else {  // coarser tables: one more term each (M = 1024: dropped < 1.2e-18)
    constexpr double a1 = -C * C / 2.0, a2 = C * C * C * C / 24.0;
    constexpr double s5 = C * C * C * C * C / 120.0;
    v = __dmul_rn(g, __fma_rn(a2, g, a1));
    s = __dmul_rn(f, __fma_rn(__fma_rn(s5, g, s3), g, s1));
  }
}

// The same rotation in the tan form (the fills' direct term): with
// tau = tan(delta) = delta + delta^3/3 (+ 2 delta^5/15 for coarser tables;
// dropped terms < 1.2e-18) and 1 + v = cos(delta),
//   cos(theta0 + delta) = (1 + v) (C0 - tau S0),  sin(theta0 + delta) = (1 + v) (S0 + tau C0):
// the caller folds 1 + v into the term's weight (Acc::add_tan), one FP64
// operation fewer per term than the sin/cos form (cis_phase below, kept for
// the ablation harnesses under scripts/).
__device__ __forceinline__ void phase_poly_tan(double f, double& v, double& tau) {
  constexpr double C = 2.0 * kPi / kPhaseM;
  constexpr double t1 = C, t3 = C * C * C / 3.0;
  const double g = __dmul_rn(f, f);
  if constexpr (kPhaseM >= 8192) {
    constexpr double a1 = kCosMinimax * C * C;
    v = __dmul_rn(a1, g);
    tau = __dmul_rn(f, __fma_rn(t3, g, t1));
  } else {
    constexpr double a1 = -C * C / 2.0, a2 = C * C * C * C / 24.0;
    constexpr double t5 = 2.0 * C * C * C * C * C / 15.0;
    v = __dmul_rn(g, __fma_rn(a2, g, a1));
    tau = __dmul_rn(f, __fma_rn(__fma_rn(t5, g, t3), g, t1));
  }
}

// (c, sn) = (cos kr, sin kr) / (1 + v): 8 FP64 ops + 1 LDS.128
__device__ __forceinline__ void cis_phase_tan(double r, double K1, const double2* tab, double& c,
                                              double& sn, double& v) {
  const double t = __fma_rn(r, K1, kMagicRint);
  const double nf = t - kMagicRint;
  const double f = __fma_rn(r, K1, -nf);
  const unsigned idx = phase_slot(static_cast<unsigned>(__double2loint(t)));
  double tau;
  phase_poly_tan(f, v, tau);
  const double2 T = tab[idx];
  c = __fma_rn(-tau, T.y, T.x);
  sn = __fma_rn(tau, T.x, T.y);
}

__device__ __forceinline__ double2 cis_phase(double r, double K1, const double2* tab) {
  const double t = __fma_rn(r, K1, kMagicRint);
  const double nf = t - kMagicRint;
  const double f = __fma_rn(r, K1, -nf);
  const unsigned idx = phase_slot(static_cast<unsigned>(__double2loint(t)));
  double v, s;
  phase_poly(f, v, s);
  const double2 T = tab[idx];
  const double c = __fma_rn(-T.y, s, __fma_rn(T.x, v, T.x));
  const double sn = __fma_rn(T.x, s, __fma_rn(T.y, v, T.y));
  return make_double2(c, sn);
}

// Standalone evaluation (eval_batch, real k): the same reduction with a
// 1024-entry table read through L1 (16 KB, no shared-memory staging for a
// microsecond kernel): |delta| <= pi/1024, cos delta - 1 to delta^4 and
// sin delta to delta^5 (dropped terms < 1.2e-18).  13 FP64 ops.
constexpr int kPhaseSmall = 1024;
// SMEM_TAB: tab is the table staged in shared memory (a plain load; __ldg
// would issue a global load on a shared address)
template <bool SMEM_TAB = false>
__device__ __forceinline__ double2 cis_phase_small(double r, double K1s, const double2* tab) {
  constexpr double C = 2.0 * kPi / kPhaseSmall;
  constexpr double a1 = -C * C / 2.0, a2 = C * C * C * C / 24.0;
  constexpr double s1 = C, s3 = -C * C * C / 6.0, s5 = C * C * C * C * C / 120.0;
  const double t = __fma_rn(r, K1s, kMagicRint);
  const double nf = t - kMagicRint;
  const double f = __fma_rn(r, K1s, -nf);
  const int idx = __double2loint(t) & (kPhaseSmall - 1);
  const double g = __dmul_rn(f, f);
  const double v = __dmul_rn(g, __fma_rn(a2, g, a1));
  const double s = __dmul_rn(f, __fma_rn(__fma_rn(s5, g, s3), g, s1));
  const double2 T = SMEM_TAB ? tab[idx] : __ldg(tab + idx);
  const double c = __fma_rn(-T.y, s, __fma_rn(T.x, v, T.x));
  const double sn = __fma_rn(T.x, s, __fma_rn(T.y, v, T.y));
  return make_double2(c, sn);
}

// Lossy media (complex k, k_im < 0), attenuation coupled to the phase
// reduction: with n + f = r K1 as in cis_phase, exp(k_im r) =
// exp(c lo) exp(c M hi) exp(c f), c = k_im / K1, n = hi M + lo.  The first
// factor is folded into the (per-fill) scaled phase table
// tab[lo] = (cos, sin)(2 pi lo / M) exp(c lo), the second is ahi[hi] (a few
// entries), the third a degree-4 polynomial in f (|c f| <= 1e-3 by
// construction: dropped term < 1e-17).  Gives the rotation like cis_phase_tan
// and the attenuation factor in att: 6 FP64 ops more than lossless
// (4 polynomial + 1 product, + 1 for the weight at the call site).
struct PhaseAtt {
  const double* ahi;
  int nhi;
  double q1, q2, q3, q4;  // c, c^2/2, c^3/6, c^4/24
};
// The rotation in the tan form (see cis_phase_tan): (c, sn) = (cos kr, sin kr)
// exp(c lo) / (1 + v), and the attenuation's remaining factor in att
__device__ __forceinline__ void cis_phase_att_tan(double r, double K1, const double2* tab,
                                                  const PhaseAtt& pa, double& att, double& c,
                                                  double& sn, double& v) {
  const double t = __fma_rn(r, K1, kMagicRint);
  const double nf = t - kMagicRint;
  const double f = __fma_rn(r, K1, -nf);
  const unsigned n = static_cast<unsigned>(__double2loint(t));
  const unsigned idx = phase_slot(n);
  unsigned hi = n >> kPhaseLog2;
  hi = hi < static_cast<unsigned>(pa.nhi) ? hi : static_cast<unsigned>(pa.nhi - 1);
  double tau;
  phase_poly_tan(f, v, tau);
  const double2 T = tab[idx];
  c = __fma_rn(-tau, T.y, T.x);
  sn = __fma_rn(tau, T.x, T.y);
  const double p = __fma_rn(__fma_rn(__fma_rn(__fma_rn(pa.q4, f, pa.q3), f, pa.q2), f, pa.q1), f, 1.0);
  att = __dmul_rn(pa.ahi[hi], p);
}

// exp(-x) for x = -k_im r >= 0 (lossy media) from a shared table
// E[n] = exp(-n/512): n = rint(512 x), f = 512 x - n in [-1/2, 1/2],
// exp(-f/512) by Taylor to f^4 (dropped term < 7.5e-18).  9 FP64 ops + 1 LDS.64.
constexpr double kAttenScale = 512.0;
__device__ __forceinline__ double atten_table(double r, double KA, const double* E, int nE) {
  constexpr double h = 1.0 / kAttenScale;
  constexpr double c1 = -h, c2 = h * h / 2.0, c3 = -h * h * h / 6.0, c4 = h * h * h * h / 24.0;
  const double t = __fma_rn(r, KA, kMagicRint);
  const double nf = t - kMagicRint;
  const double f = __fma_rn(r, KA, -nf);
  unsigned idx = static_cast<unsigned>(__double2loint(t));
  idx = idx < static_cast<unsigned>(nE) ? idx : static_cast<unsigned>(nE - 1);
  const double p = __fma_rn(__fma_rn(__fma_rn(__fma_rn(c4, f, c3), f, c2), f, c1), f, 1.0);
  return __dmul_rn(E[idx], p);
}


// reference-accuracy direct kernel via libdevice sincos (the accuracy oracle
// on the device side and the fallback of the table path, evaluator.hpp:199-205)
__device__ __forceinline__ double2 analytic_sincos(int kind, double k_re, double k_im, double r) {
  double s, c;
  sincos(k_re * r, &s, &c);
  double re = c, im = -s;
  if (k_im != 0.0) {
    const double a = exp(k_im * r);
    re *= a;
    im *= a;
  }
  if (kind == 1) {
    re = re / r;
    im = im / r;
  }
  return make_double2(re, im);
}

}  // namespace gk
