// fill_kernels.cuh -- K3 table fill and K4 direct fill kernels (templates),
// instantiated per outer-point count in fill_mo{1,3,4,6,7}.cu (parallel
// compilation) and launched by launch_fill (fill.cu).
//
// The fill replaces fill_matrix's fill_rows loop (matfill.hpp:169-203) with
// AnalyticKernel::accumulate (DIRECT, kernel.hpp:48-61) or
// TableKernel::accumulate -> accumulate_green (TABLE, evaluator.hpp:150-194).
//
// Work decomposition: a CTA of 8 warps owns a tile of 8 observation rows x
// 128 source columns; warp w takes row p = tile_row*8 + w, lane l takes the
// columns q = tile_col*128 + 32 b + l (b = 0..3), so every warp store is one
// coalesced 512-byte complex128 row segment.  The m outer points of p live in
// registers; the 3n inner points of q stream from a [3n][N] plane layout
// (coalesced 32-byte loads, L1/L2 resident).  Each lane keeps one complex
// accumulator per outer point (sum_i w_i K(r_oi)) and finishes the entry with
// sum_o w_o acc_o -- the reference's double sum regrouped (same terms).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <math_constants.h>

#include "gk_internal.h"

namespace gk {

constexpr int kRowsPerTile = 8;  // one row per warp
constexpr int kMaxColBlocks = 32;  // 32-column blocks per tile (adaptive, see launch_fill)
constexpr int kThreads = 32 * kRowsPerTile;
#ifndef GK_TABLE_WARPS
#define GK_TABLE_WARPS 8  // table_kernel (L1 path): rows per CTA
#endif
#ifndef GK_TABLE_CTAS
#define GK_TABLE_CTAS 2   // table_kernel: resident CTAs per SM
#endif

// per-entry accumulators: one complex per outer point, two for the fused pair
template <int MO, bool PAIR>
struct Acc {
  double2 e[MO], g[PAIR ? MO : 1];
  __device__ __forceinline__ void zero() {
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      e[o] = make_double2(0.0, 0.0);
      if constexpr (PAIR) g[o] = make_double2(0.0, 0.0);
    }
  }
  // acc += w (1 + v) (c - j s) for kind KIND (the tan form of the rotation,
  // cis_phase_tan: cos(delta) = 1 + v goes into the weight); y = 1/r
  template <int KIND>
  __device__ __forceinline__ void add_tan(int o, double w, double y, double c, double s, double v) {
    if constexpr (KIND == kKindPair) {
      const double we = __fma_rn(w, v, w);
      e[o].x = __fma_rn(we, c, e[o].x);
      e[o].y = __fma_rn(-we, s, e[o].y);
      const double b = __dmul_rn(w, y);
      const double wg = __fma_rn(b, v, b);
      g[o].x = __fma_rn(wg, c, g[o].x);
      g[o].y = __fma_rn(-wg, s, g[o].y);
    } else {
      const double b = KIND == GK_KIND_GREEN ? __dmul_rn(w, y) : w;
      const double wk = __fma_rn(b, v, b);
      e[o].x = __fma_rn(wk, c, e[o].x);
      e[o].y = __fma_rn(-wk, s, e[o].y);
    }
  }
  // acc += w * v (table values: v = K(r) for the kind, vg = Green for the pair)
  __device__ __forceinline__ void add_values(int o, double w, double2 v, double2 vg) {
    e[o].x = __fma_rn(w, v.x, e[o].x);
    e[o].y = __fma_rn(w, v.y, e[o].y);
    if constexpr (PAIR) {
      g[o].x = __fma_rn(w, vg.x, g[o].x);
      g[o].y = __fma_rn(w, vg.y, g[o].y);
    }
  }
  // finish sum_o w_o acc_o and store (self pairs stay zero, matfill.hpp:178).
  // A non-finite entry can only come from a zero-distance point pair, which
  // the reference rejects (eval_analytic, kernel.hpp:51-53): counted in *bad.
  template <class W>
  __device__ __forceinline__ void finish(const W& wo, bool self, bool valid, double2* z,
                                         double2* z2, size_t off, unsigned long long* bad) {
    double2 re = make_double2(0.0, 0.0), rg = make_double2(0.0, 0.0);
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double w = wo(o);
      re.x = __fma_rn(w, e[o].x, re.x);
      re.y = __fma_rn(w, e[o].y, re.y);
      if constexpr (PAIR) {
        rg.x = __fma_rn(w, g[o].x, rg.x);
        rg.y = __fma_rn(w, g[o].y, rg.y);
      }
    }
    if (self) re = rg = make_double2(0.0, 0.0);
    if (valid && !(isfinite(re.x) && isfinite(re.y) && isfinite(rg.x) && isfinite(rg.y)))
      atomicAdd(bad, 1ull);
    if (valid) {
      __stcs(z + off, re);
      if constexpr (PAIR) __stcs(z2 + off, rg);
    }
  }
};

__global__ void atten_kernel(double* E, int n);

struct FillArgs {
  const double4* outer;
  const double4* inner;
  size_t N;
  int ipt;
  size_t row_begin, row_end;
  size_t ncb, ntiles;
  int cpt;  // column blocks per tile
  double2* z;   // Exp or Green (or Exp for the fused pair fill)
  double2* z2;  // fused pair fill: Green
  size_t ldz;
  TableDev T;
  const double2* phase;
  double K1, k_re, k_im;
  const double4* bounds;  // per-triangle (centroid, rho_outer), for tile radius bounds
  const double* binner;   // per-triangle rho_inner
  double window_est;      // estimated radius spread of a 16 x 64 tile (staging heuristic)
  // lossy media: ATT 1 = attenuation coupled to the phase reduction
  // (cis_phase_att: phase = the per-fill scaled table, ahi[nhi], q = c^j/j!),
  // ATT 2 = the legacy table exp(-n / 512), n < natten (|k_im| > 2.6 k_re)
  const double* ahi;
  int nhi;
  double q1, q2, q3, q4;
  const double* atten;
  int natten;
  double KA;            // -k_im * 512
  unsigned long long* counters;  // [0] fallbacks (r < r_min), [1] r > r_max, [2] non-finite entries,
                                 // [3] kernel evaluations performed
  // shared-edge fill (direct_edge_kernel, edges.cu)
  const EdgeBlock* eblk;
  const double2* ep;  // [chunk][n][2][32]: (x, y) and (z, w) planes
  const uint4* ecol;  // per block position: (triangle q, e0 | e1 << 16, e2, 0)
  size_t nblk;
  int ecap;  // edge-sum slots per warp (>= every block's edge count)
  double r_far;
  // table sweep (K3s, fill_sweep.cuh): the mesh's small-block edge set (put
  // in eblk / ep / ecol / nblk / ecap when K3s runs), the in-range rows in
  // its spatial order (clusters of s_rc), the staged window's capacity in
  // base nodes
  const EdgeBlock* s_eblk;
  const double2* s_ep;
  const uint4* s_ecol;
  size_t s_nblk;
  int s_ecap;
  double s_rho_max;   // largest block radius of the sweep set
  double s_rho_rows;  // largest outer-point radius of a row triangle
  const uint32_t* s_rows;
  int s_rc;
  uint32_t s_wn;
  double s_delta;     // band width of the tile keys
  uint32_t* s_list;   // per-CTA tile lists [grid][s_rc * nblk] (scratch)
  unsigned long long* s_next_cluster;  // dynamic cluster counter (zeroed per launch)
  size_t s_full;      // clusters of s_rc rows; the rest hold s_rc / 2
};

// Column-block walk shared by both kernels: the (column block, inner point)
// iterations of a tile are flattened into one loop so the next inner point is
// always in flight (register double buffer) while the current one is used.
struct InnerWalk {
  const double4* inner;
  size_t N, q0base;
  int ipt, ncb;
  __device__ __forceinline__ void load(int cb, int i, int lane, double2& xy, double2& zw,
                                       size_t& q, bool& valid) const {
    const size_t qr = q0base + 32 * static_cast<size_t>(cb) + lane;
    valid = qr < N;
    q = valid ? qr : N - 1;
    const double2* p = reinterpret_cast<const double2*>(inner + static_cast<size_t>(i) * N + q);
    xy = __ldg(p);
    zw = __ldg(p + 1);
  }
};

// one-shot copy of `bytes` (multiple of 16, 16 B aligned) global -> shared,
// issued by thread 0 as a TMA bulk copy; every thread waits on the mbarrier
__device__ __forceinline__ void stage_bulk(void* dst, const void* src, uint32_t bytes,
                                          uint64_t* bar) {
  if (threadIdx.x == 0) {
    mbar_init(bar);
    mbar_expect_tx(bar, bytes);
    tma_load_1d(dst, src, bytes, bar);
  }
  __syncthreads();  // barrier initialised before anyone polls it
  mbar_wait(bar, 0);
}

// K4: direct evaluation.  Per eval: 6 (r^2) + 6 (rsqrt, r) + 8 (phase, table
// lookup, rotation in the tan form) + 4 (weight with cos(delta), accumulate)
// = 25 FP64 ops.
// The warp's outer points sit in shared memory (broadcast loads, one
// wavefront each) instead of registers, so ~80 registers per thread allow 3
// CTAs (24 warps) per SM to hide the FP64 dependency latency.
template <int MO, int KIND, int ATT, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) direct_kernel(const FillArgs A) {
  extern __shared__ double2 tab[];  // kPhaseM phase entries (128 KB) [+ attenuation table]
  __shared__ double so[kRowsPerTile][MO][4];
  __shared__ uint64_t bar;
  stage_bulk(tab, A.phase, kPhaseSlots * sizeof(double2), &bar);
  double* att = reinterpret_cast<double*>(tab + kPhaseSlots);
  if constexpr (ATT == 1)
    for (int i = threadIdx.x; i < A.nhi; i += blockDim.x) att[i] = A.ahi[i];
  if constexpr (ATT == 2)
    for (int i = threadIdx.x; i < A.natten; i += blockDim.x) att[i] = A.atten[i];
  const PhaseAtt pa{att, A.nhi, A.q1, A.q2, A.q3, A.q4};
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t N = A.N;
  double (*my)[4] = so[warp];

  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.ncb, tc = tile - tr * A.ncb;
    const size_t p = A.row_begin + tr * kRowsPerTile + warp;
    if (p >= A.row_end) continue;  // warp-uniform
    __syncwarp();
    if (lane < MO) {
      const double4 P = A.outer[p * MO + lane];
      my[lane][0] = P.x;
      my[lane][1] = P.y;
      my[lane][2] = P.z;
      my[lane][3] = P.w;
    }
    __syncwarp();
    const size_t q0base = tc * (32 * static_cast<size_t>(A.cpt));
    int ncb = static_cast<int>((N - q0base + 31) / 32);
    if (ncb > A.cpt) ncb = A.cpt;
    const InnerWalk W{A.inner, N, q0base, A.ipt, ncb};
    const int iters = ncb * A.ipt;
    double2 nxy, nzw;
    size_t q;
    bool valid;
    W.load(0, 0, lane, nxy, nzw, q, valid);
    Acc<MO, KIND == kKindPair> acc;
    acc.zero();
    int ncb_next = 0, ni = 0;  // (column block, inner point) of the prefetch
    for (int it = 0; it < iters; ++it) {
      const double2 pxy = nxy, pzw = nzw;
      const size_t qc = q;
      const bool vc = valid;
      if (++ni == A.ipt) {
        ni = 0;
        ++ncb_next;
      }
      const bool block_done = ni == 0;
      if (it + 1 < iters) W.load(ncb_next, ni, lane, nxy, nzw, q, valid);
#pragma unroll
      for (int o = 0; o < MO; ++o) {
        const double2 oxy = *reinterpret_cast<const double2*>(&my[o][0]);
        const double oz = my[o][2];
        const double d2 = dist2(oxy.x, oxy.y, oz, pxy.x, pxy.y, pzw.x);
        const double y = rsqrt_fast(d2);
        const double r = radius_of<KIND>(d2, y);
        double w = pzw.y;
        double c, sn, v;  // (cos kr, sin kr) / (1 + v)
        if constexpr (ATT == 1) {
          double a;
          cis_phase_att_tan(r, A.K1, tab, pa, a, c, sn, v);
          w = __dmul_rn(w, a);
        } else {
          cis_phase_tan(r, A.K1, tab, c, sn, v);
          if constexpr (ATT == 2) w = __dmul_rn(w, atten_table(r, A.KA, att, A.natten));
        }
        acc.template add_tan<KIND>(o, w, y, c, sn, v);
      }
      if (block_done) {  // column block complete: finish the entry
        acc.finish([&](int o) { return my[o][3]; }, qc == p, vc, A.z, A.z2,
                   (p - A.row_begin) * A.ldz + qc, A.counters + 2);
        acc.zero();
      }
    }
  }
}

// K4 fast path (IPT = 3n known at compile time, n = 1..5): the inner-point
// loop of a column block is fully unrolled with a one-point register
// prefetch, the outer points live in registers and 12 warps x 1 CTA per SM
// (~160 registers each) keep the FP64 pipe fed.  Non-FP64 instructions cost
// an issue cycle each while an FP64 warp instruction holds the 16-lane pipe
// for two, so this variant's ~9 non-FP64 instructions/eval (vs ~16 in the
// runtime-IPT kernel) are worth ~12% (ablations: scripts/direct_variants.cu).
// (The fused pair fill carries twice the accumulators: 8 warps, ~200 registers.)
#ifndef GK_WARPS_V4
#define GK_WARPS_V4 12  // scripts/build_variant.sh experiments override it
#endif
template <int KIND>
__host__ __device__ constexpr int warps_v4() { return KIND == kKindPair ? 8 : GK_WARPS_V4; }

template <int MO, int IPT, int KIND, int ATT>
__global__ void __launch_bounds__(32 * warps_v4<KIND>(), 1) direct_kernel_v4(const FillArgs A) {
  constexpr int kWarpsV4 = warps_v4<KIND>();
  extern __shared__ double2 tab[];  // kPhaseM phase entries (128 KB) [+ attenuation table]
  __shared__ double sw[kWarpsV4][MO];
  __shared__ uint64_t bar;
  stage_bulk(tab, A.phase, kPhaseSlots * sizeof(double2), &bar);
  double* att = reinterpret_cast<double*>(tab + kPhaseSlots);
  if constexpr (ATT == 1)
    for (int i = threadIdx.x; i < A.nhi; i += blockDim.x) att[i] = A.ahi[i];
  if constexpr (ATT == 2)
    for (int i = threadIdx.x; i < A.natten; i += blockDim.x) att[i] = A.atten[i];
  const PhaseAtt pa{att, A.nhi, A.q1, A.q2, A.q3, A.q4};
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t N = A.N;
  const double4* last = A.inner + (N - 1);

  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.ncb, tc = tile - tr * A.ncb;
    const size_t p = A.row_begin + tr * kWarpsV4 + warp;
    if (p >= A.row_end) continue;  // warp-uniform
    double ox[MO], oy[MO], oz[MO];
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double2 xy = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o));
      const double2 zw = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o) + 1);
      ox[o] = xy.x;
      oy[o] = xy.y;
      oz[o] = zw.x;
      if (lane == 0) sw[warp][o] = zw.y;
    }
    __syncwarp();
    const size_t q0 = tc * (32 * static_cast<size_t>(A.cpt));
    int nblk = static_cast<int>((N - q0 + 31) / 32);
    if (nblk > A.cpt) nblk = A.cpt;
    const double4* colp = A.inner + q0 + lane;  // column block 0, inner point 0
    double2 cxy, czw;
    {
      const double2* ptr = reinterpret_cast<const double2*>(colp <= last ? colp : last);
      cxy = __ldg(ptr);
      czw = __ldg(ptr + 1);
    }
    for (int cb = 0; cb < nblk; ++cb) {
      const double4* cp = colp <= last ? colp : last;
      Acc<MO, KIND == kKindPair> acc;
      acc.zero();
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const double2 pxy = cxy, pzw = czw;
        const double4* np = (i + 1 < IPT) ? cp + (i + 1) * N : (colp + 32 <= last ? colp + 32 : last);
        cxy = __ldg(reinterpret_cast<const double2*>(np));
        czw = __ldg(reinterpret_cast<const double2*>(np) + 1);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          const double d2 = dist2(ox[o], oy[o], oz[o], pxy.x, pxy.y, pzw.x);
          const double y = rsqrt_fast(d2);
          const double r = radius_of<KIND>(d2, y);
          double w = pzw.y;
          double c, sn, v;  // (cos kr, sin kr) / (1 + v)
          if constexpr (ATT == 1) {
            double a;
            cis_phase_att_tan(r, A.K1, tab, pa, a, c, sn, v);
            w = __dmul_rn(w, a);
          } else {
            cis_phase_tan(r, A.K1, tab, c, sn, v);
            if constexpr (ATT == 2) w = __dmul_rn(w, atten_table(r, A.KA, att, A.natten));
          }
          acc.template add_tan<KIND>(o, w, y, c, sn, v);
        }
      }
      const size_t q = q0 + 32 * static_cast<size_t>(cb) + lane;
      acc.finish([&](int o) { return sw[warp][o]; }, q == p, q < N, A.z, A.z2,
                 (p - A.row_begin) * A.ldz + q, A.counters + 2);
      colp += 32;
    }
    __syncwarp();
  }
}

// One direct term w K(|o - P|) into acc[o] (the v4 loop body).
// r_floor: the shared-edge far path asserts its precondition r >= r_far
template <int MO, int KIND, int ATT>
__device__ __forceinline__ void direct_term(Acc<MO, KIND == kKindPair>& acc, int o, double ox, double oy,
                                            double oz, double2 pxy, double2 pzw,
                                            const FillArgs& A, const double2* tab,
                                            const PhaseAtt& pa, const double* att,
                                            double r_floor = 0.0) {
  const double d2 = dist2(ox, oy, oz, pxy.x, pxy.y, pzw.x);
  const double y = rsqrt_fast(d2);
  const double r = radius_of<KIND>(d2, y);
  GK_DASSERT(r >= r_floor * (1.0 - 1e-12));
  double w = pzw.y;
  double c, sn, v;  // (cos kr, sin kr) / (1 + v)
  if constexpr (ATT == 1) {
    double a;
    cis_phase_att_tan(r, A.K1, tab, pa, a, c, sn, v);
    w = __dmul_rn(w, a);
  } else {
    cis_phase_tan(r, A.K1, tab, c, sn, v);
    if constexpr (ATT == 2) w = __dmul_rn(w, atten_table(r, A.KA, att, A.natten));
  }
  acc.template add_tan<KIND>(o, w, y, c, sn, v);
}

// K4e: the direct fill with shared edges (edges.cu).  A tile is 12 rows x one
// edge block.  Where every pair of (row p, block) is at least r_far apart, the
// warp evaluates each distinct edge of the block once (lane = edge, the n
// points fully unrolled: m x n terms per lane), keeps the edge sums
// E[e] = sum_o w_o sum_i w_i K(r_oi) in shared memory and writes
// Z[p][q] = E[e0(q)] + E[e1(q)] + E[e2(q)] for the block's triangles
// (coalesced streaming stores).  Nearer tiles take the per-triangle loop on
// the reference's own points.  On a closed mesh the far path performs ~0.55
// of the reference's evaluations.
#ifndef GK_EDGE_WARPS
#define GK_EDGE_WARPS 12
#endif
#ifndef GK_EDGE_ALLNEAR
#define GK_EDGE_ALLNEAR 0  // A/B: every tile through the near path
#endif
#ifndef GK_EDGE_GUNROLL
#define GK_EDGE_GUNROLL 5  // unroll of the edge-point loop (n <= 5: full)
#endif
#ifndef GK_EDGE_NEAR_UNROLL
#define GK_EDGE_NEAR_UNROLL 1  // unroll of the near tiles' point loop (A/B)
#endif
#define GK_PRAGMA(x) _Pragma(#x)
#define GK_UNROLL(n) GK_PRAGMA(unroll n)

// the fused Exp + Green pair carries two sums per edge: 8 warps (as v4's pair)
template <int KIND>
__host__ __device__ constexpr int edge_warps() { return KIND == kKindPair ? 8 : GK_EDGE_WARPS; }

template <int MO, int NPE, int KIND, int ATT>
__global__ void __launch_bounds__(32 * edge_warps<KIND>(), 1) direct_edge_kernel(const FillArgs A) {
  constexpr int W = edge_warps<KIND>();
  constexpr bool PAIR = KIND == kKindPair;
  constexpr int NS = PAIR ? 2 : 1;  // edge sums per edge
  constexpr int IPT = 3 * NPE;
  extern __shared__ double2 tab[];  // phase [kPhaseM] | edge sums [W][NS][ecap] | attenuation
  __shared__ double sw[W][MO];
  __shared__ uint64_t bar;
  stage_bulk(tab, A.phase, kPhaseSlots * sizeof(double2), &bar);
  double2* const sE = tab + kPhaseSlots;
  double* att = reinterpret_cast<double*>(sE + W * NS * A.ecap);
  if constexpr (ATT == 1)
    for (int i = threadIdx.x; i < A.nhi; i += blockDim.x) att[i] = A.ahi[i];
  const PhaseAtt pa{att, A.nhi, A.q1, A.q2, A.q3, A.q4};
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t N = A.N;
  double2* const myE = sE + warp * NS * A.ecap;  // [NS][ecap]: Exp (or the kind), Green
  unsigned long long nev = 0;

  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.nblk, b = tile - tr * A.nblk;
    const size_t p = A.row_begin + tr * W + warp;
    if (p >= A.row_end) continue;  // warp-uniform
    double ox[MO], oy[MO], oz[MO];
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double2 xy = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o));
      const double2 zw = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o) + 1);
      ox[o] = xy.x;
      oy[o] = xy.y;
      oz[o] = zw.x;
      if (lane == 0) sw[warp][o] = zw.y;
    }
    const EdgeBlock B = A.eblk[b];
    const double4 bp = A.bounds[p];
    // far: |c_p - c_B| - rho_p - rho_B >= r_far, compared squared (both
    // sides >= 0) with a margin far above the rounding of either side
    const double dx = bp.x - B.cx, dy = bp.y - B.cy, dz = bp.z - B.cz;
    const double reach = A.r_far + bp.w + B.rho;
    const bool far = !GK_EDGE_ALLNEAR && dx * dx + dy * dy + dz * dz >= reach * reach * (1.0 + 1e-12);
    double2* const zrow = A.z + (p - A.row_begin) * A.ldz;
    const uint4* const cols = A.ecol + B.tb;
    const uint32_t nb = B.te - B.tb;
    __syncwarp();
    if (far) {
      const int nch = static_cast<int>((B.ne + 31) >> 5);
      GK_DASSERT(B.ne <= static_cast<uint32_t>(A.ecap) && B.tb < B.te && B.te <= N);
      const double2* ep = A.ep + static_cast<size_t>(B.c0) * NPE * 64 + lane;
      double2 cxy = __ldg(ep);
      double2 czw = __ldg(ep + 32);
      for (int c = 0; c < nch; ++c) {
        Acc<MO, PAIR> acc;
        acc.zero();
        GK_UNROLL(GK_EDGE_GUNROLL)
        for (int g = 0; g < NPE; ++g) {
          const double2 pxy = cxy, pzw = czw;
          const double2* np = ep + (g + 1 < NPE ? (c * NPE + g + 1) * 64
                                                : (c + 1 < nch ? (c + 1) * NPE * 64 : 0));
          cxy = __ldg(np);
          czw = __ldg(np + 32);
#pragma unroll
          for (int o = 0; o < MO; ++o)
            direct_term<MO, KIND, ATT>(acc, o, ox[o], oy[o], oz[o], pxy, pzw, A, tab, pa, att,
                                       A.r_far);
        }
        double2 e = make_double2(0.0, 0.0), eg = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          const double w = sw[warp][o];
          e.x = __fma_rn(w, acc.e[o].x, e.x);
          e.y = __fma_rn(w, acc.e[o].y, e.y);
          if constexpr (PAIR) {
            eg.x = __fma_rn(w, acc.g[o].x, eg.x);
            eg.y = __fma_rn(w, acc.g[o].y, eg.y);
          }
        }
        myE[c * 32 + lane] = e;
        if constexpr (PAIR) myE[A.ecap + c * 32 + lane] = eg;
      }
      nev += static_cast<unsigned long long>(B.ne) * NPE * MO * NS;
      __syncwarp();
      // Z[p][q] = sum of q's three edge sums.  Far tiles never hold the self
      // pair (p's centroid lies inside its own block's sphere) nor a
      // zero distance (every pair is >= r_far > 0 apart): no checks needed.
      for (uint32_t jb = 0; jb < nb; jb += 32) {
        const uint32_t j = jb + lane;
        if (j < nb) {
          const uint4 col = __ldg(cols + j);  // (q, e0 | e1 << 16, e2)
          GK_DASSERT(col.x < N && (col.y & 0xffffu) < B.ne && (col.y >> 16) < B.ne && col.z < B.ne);
          const double2 e0 = myE[col.y & 0xffffu], e1 = myE[col.y >> 16], e2 = myE[col.z];
          __stcs(zrow + col.x, make_double2(e0.x + e1.x + e2.x, e0.y + e1.y + e2.y));
          if constexpr (PAIR) {
            const double2* G = myE + A.ecap;
            const double2 g0 = G[col.y & 0xffffu], g1 = G[col.y >> 16], g2 = G[col.z];
            __stcs(A.z2 + (p - A.row_begin) * A.ldz + col.x,
                   make_double2(g0.x + g1.x + g2.x, g0.y + g1.y + g2.y));
          }
        }
      }
      __syncwarp();  // myE is rewritten by the next tile
    } else {
      // near tile: the reference's own points of each source triangle
      unsigned nq = 0;
      for (uint32_t jb = 0; jb < nb; jb += 32) {
        const uint32_t j = jb + lane;
        const bool valid = j < nb;
        const size_t q = __ldg(cols + (valid ? j : nb - 1)).x;
        nq += __popc(__ballot_sync(0xffffffffu, valid && q != p));
        Acc<MO, PAIR> acc;
        acc.zero();
        GK_UNROLL(GK_EDGE_NEAR_UNROLL)
        for (int i = 0; i < IPT; ++i) {
          const double2* ptr = reinterpret_cast<const double2*>(A.inner + static_cast<size_t>(i) * N + q);
          const double2 pxy = __ldg(ptr), pzw = __ldg(ptr + 1);
#pragma unroll
          for (int o = 0; o < MO; ++o)
            direct_term<MO, KIND, ATT>(acc, o, ox[o], oy[o], oz[o], pxy, pzw, A, tab, pa, att);
        }
        acc.finish([&](int o) { return sw[warp][o]; }, q == p, valid, A.z, A.z2,
                   (p - A.row_begin) * A.ldz + q, A.counters + 2);
      }
      nev += static_cast<unsigned long long>(nq) * IPT * MO * NS;
    }
    __syncwarp();
  }
  if (lane == 0 && nev) atomicAdd(A.counters + 3, nev);
}

// K3: table evaluation (the paper's method) with the reference's fallback.
template <int MO, int KIND, int DEG>
__global__ void __launch_bounds__(32 * GK_TABLE_WARPS, GK_TABLE_CTAS) table_kernel(const FillArgs A) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t N = A.N;
  unsigned long long n_low = 0, n_high = 0;

  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.ncb, tc = tile - tr * A.ncb;
    const size_t p = A.row_begin + tr * GK_TABLE_WARPS + warp;
    if (p >= A.row_end) continue;  // warp-uniform
    double ox[MO], oy[MO], oz[MO];
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double2 xy = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o));
      const double zz = __ldg(reinterpret_cast<const double*>(A.outer + p * MO + o) + 2);
      ox[o] = xy.x;
      oy[o] = xy.y;
      oz[o] = zz;
    }
    const size_t q0base = tc * (32 * static_cast<size_t>(A.cpt));
    int ncb = static_cast<int>((N - q0base + 31) / 32);
    if (ncb > A.cpt) ncb = A.cpt;
    const InnerWalk W{A.inner, N, q0base, A.ipt, ncb};
    const int iters = ncb * A.ipt;
    double2 nxy, nzw;
    size_t q;
    bool valid;
    W.load(0, 0, lane, nxy, nzw, q, valid);
    Acc<MO, KIND == kKindPair> acc;
    acc.zero();
    int ncb_next = 0, ni = 0;  // (column block, inner point) of the prefetch
    for (int it = 0; it < iters; ++it) {
      const double2 pxy = nxy, pzw = nzw;
      const size_t qc = q;
      const bool vc = valid;
      if (++ni == A.ipt) {
        ni = 0;
        ++ncb_next;
      }
      const bool block_done = ni == 0;
      const bool self = qc == p;
      if (it + 1 < iters) W.load(ncb_next, ni, lane, nxy, nzw, q, valid);
#pragma unroll
      for (int o = 0; o < MO; ++o) {
        const double d2 = dist2(ox[o], oy[o], oz[o], pxy.x, pxy.y, pzw.x);
        const double r = radius_of<KIND>(d2, rsqrt_fast(d2));
        double2 v, vg = make_double2(0.0, 0.0);
        if constexpr (KIND == kKindPair) pair_table<DEG>(r, A.T, v, vg);
        else if constexpr (KIND == GK_KIND_EXP) v = exp_table(r, A.T);
        else if constexpr (DEG == 3) v = green_table<3>(r, A.T);
        else v = green_table_any(r, A.T);
        const bool oob = !(r >= A.T.r_min && r <= A.T.r_max);
        if (__any_sync(0xffffffffu, oob)) {
          if (oob) {
            if (!self && vc) {
              // the reference's eval_kernel fallback (evaluator.hpp:199-205)
              const unsigned calls = KIND == kKindPair ? 2u : 1u;
              if constexpr (KIND == kKindPair) {
                v = analytic_sincos(GK_KIND_EXP, A.T.k_re, A.T.k_im, r);
                vg = analytic_sincos(GK_KIND_GREEN, A.T.k_re, A.T.k_im, r);
              } else {
                v = analytic_sincos(KIND, A.T.k_re, A.T.k_im, r);
              }
              if (r > A.T.r_max) n_high += calls; else n_low += calls;
            } else {
              v = vg = make_double2(0.0, 0.0);
            }
          }
        }
        acc.add_values(o, pzw.y, v, vg);
      }
      if (block_done) {
        acc.finish([&](int o) { return __ldg(reinterpret_cast<const double*>(A.outer + p * MO + o) + 3); },
                   self, vc, A.z, A.z2, (p - A.row_begin) * A.ldz + qc, A.counters + 2);
        acc.zero();
      }
    }
  }
  for (int o = 16; o; o >>= 1) {
    n_low += __shfl_xor_sync(0xffffffffu, n_low, o);
    n_high += __shfl_xor_sync(0xffffffffu, n_high, o);
  }
  if (lane == 0 && n_low) atomicAdd(A.counters, n_low);
  if (lane == 0 && n_high) atomicAdd(A.counters + 1, n_high);
}

// ------------------------------------------- K3e: table fill with shared edges
//
// The paper's method on K4e's blocks (edges.cu): far tiles evaluate each
// distinct edge of a block once through the table (read through L1, as
// table_kernel does); near tiles run the per-triangle loop with the
// reference's fallback (evaluator.hpp:199-205).  launch_fill takes this path
// only when r_min <= r_far, so a far pair never falls back below the table:
// the fallback counts stay the reference's.
// 16 warps with the edge-point loop unrolled by 2 (128 registers, a few
// spilled): the L1/L2 gathers are latency-bound, so warps beat unrolling --
// C5 S = 1e4, 4096 rows: 12 warps fully unrolled 219 ms, 12 x 1 200 ms,
// 16 x 5 192 ms, 16 x 1 176 ms, 16 x 2 175 ms, 20 x 1 180 ms, 24 x 1 181 ms,
// 32 x 1 193 ms, 14 x 2 191 ms, 18 x 1 190 ms (scripts/build_variant.sh)
#ifndef GK_TEDGE_WARPS
#define GK_TEDGE_WARPS 16
#endif
#ifndef GK_TEDGE_GUNROLL
#define GK_TEDGE_GUNROLL 2  // unroll of the edge-point loop
#endif

// the kind's table value v (the fused pair: Exp in v, Green in vg)

// the fused pair carries two sums per edge: 8 warps
template <int KIND>
__host__ __device__ constexpr int tedge_warps() { return KIND == kKindPair ? 8 : GK_TEDGE_WARPS; }

// One (row p, edge block b) tile of the table fill on shared edges (K3e,
// K3s): the far path evaluates each distinct edge of the block once and
// combines Z[p][q] from the edge sums in myE; a near tile runs the
// per-triangle loop on the reference's own points.  `vals(r, v, vg)` is the
// table lookup (K3e: global records through L1; K3s: the staged window).
template <int MO, int NPE, int KIND, class Vals>
__device__ __forceinline__ void table_edge_tile(const FillArgs& A, size_t p, size_t b,
                                                double2* myE, double* sww, const Vals& vals,
                                                unsigned long long& nev,
                                                unsigned long long& n_low,
                                                unsigned long long& n_high) {
  constexpr bool PAIR = KIND == kKindPair;
  constexpr int NS = PAIR ? 2 : 1;
  constexpr int IPT = 3 * NPE;
  const int lane = threadIdx.x & 31;
  const size_t N = A.N;
  double ox[MO], oy[MO], oz[MO];
#pragma unroll
  for (int o = 0; o < MO; ++o) {
    const double2 xy = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o));
    const double2 zw = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o) + 1);
    ox[o] = xy.x;
    oy[o] = xy.y;
    oz[o] = zw.x;
    if (lane == 0) sww[o] = zw.y;
  }
  const EdgeBlock B = A.eblk[b];
  const double4 bp = A.bounds[p];
  const double dx = bp.x - B.cx, dy = bp.y - B.cy, dz = bp.z - B.cz;
  const double reach = A.r_far + bp.w + B.rho;
  const bool far = dx * dx + dy * dy + dz * dz >= reach * reach * (1.0 + 1e-12);
  double2* const zrow = A.z + (p - A.row_begin) * A.ldz;
  const uint4* const cols = A.ecol + B.tb;
  const uint32_t nb = B.te - B.tb;
  __syncwarp();
  if (far) {
    const int nch = static_cast<int>((B.ne + 31) >> 5);
    GK_DASSERT(B.ne <= static_cast<uint32_t>(A.ecap) && B.tb < B.te && B.te <= N);
    const double2* ep = A.ep + static_cast<size_t>(B.c0) * NPE * 64 + lane;
    double2 cxy = __ldg(ep);
    double2 czw = __ldg(ep + 32);
    for (int c = 0; c < nch; ++c) {
      Acc<MO, PAIR> acc;
      acc.zero();
      GK_UNROLL(GK_TEDGE_GUNROLL)
      for (int g = 0; g < NPE; ++g) {
        const double2 pxy = cxy, pzw = czw;
        const double2* np = ep + (g + 1 < NPE ? (c * NPE + g + 1) * 64
                                              : (c + 1 < nch ? (c + 1) * NPE * 64 : 0));
        cxy = __ldg(np);
        czw = __ldg(np + 32);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          const double d2 = dist2(ox[o], oy[o], oz[o], pxy.x, pxy.y, pzw.x);
          const double r = radius_of<KIND>(d2, rsqrt_fast(d2));
          GK_DASSERT(r >= A.r_far * (1.0 - 1e-12));
          n_high += (r > A.T.r_max) ? NS : 0;  // out_of_range (the reference's accumulate_green)
          double2 v, vg = make_double2(0.0, 0.0);
          vals(r, v, vg);
          acc.add_values(o, pzw.y, v, vg);
        }
      }
      double2 e = make_double2(0.0, 0.0), eg = make_double2(0.0, 0.0);
#pragma unroll
      for (int o = 0; o < MO; ++o) {
        const double w = sww[o];
        e.x = __fma_rn(w, acc.e[o].x, e.x);
        e.y = __fma_rn(w, acc.e[o].y, e.y);
        if constexpr (PAIR) {
          eg.x = __fma_rn(w, acc.g[o].x, eg.x);
          eg.y = __fma_rn(w, acc.g[o].y, eg.y);
        }
      }
      myE[c * 32 + lane] = e;
      if constexpr (PAIR) myE[A.ecap + c * 32 + lane] = eg;
    }
    nev += static_cast<unsigned long long>(B.ne) * NPE * MO * NS;
    __syncwarp();
    for (uint32_t jb = 0; jb < nb; jb += 32) {
      const uint32_t j = jb + lane;
      if (j < nb) {
        const uint4 col = __ldg(cols + j);  // (q, e0 | e1 << 16, e2)
        GK_DASSERT(col.x < N && (col.y & 0xffffu) < B.ne && (col.y >> 16) < B.ne && col.z < B.ne);
        const double2 e0 = myE[col.y & 0xffffu], e1 = myE[col.y >> 16], e2 = myE[col.z];
        __stcs(zrow + col.x, make_double2(e0.x + e1.x + e2.x, e0.y + e1.y + e2.y));
        if constexpr (PAIR) {
          const double2* G = myE + A.ecap;
          const double2 g0 = G[col.y & 0xffffu], g1 = G[col.y >> 16], g2 = G[col.z];
          __stcs(A.z2 + (p - A.row_begin) * A.ldz + col.x,
                 make_double2(g0.x + g1.x + g2.x, g0.y + g1.y + g2.y));
        }
      }
    }
    __syncwarp();
  } else {
    unsigned nq = 0;
    for (uint32_t jb = 0; jb < nb; jb += 32) {
      const uint32_t j = jb + lane;
      const bool valid = j < nb;
      const size_t q = __ldg(cols + (valid ? j : nb - 1)).x;
      const bool self = q == p;
      nq += __popc(__ballot_sync(0xffffffffu, valid && !self));
      Acc<MO, PAIR> acc;
      acc.zero();
#pragma unroll 1
      for (int i = 0; i < IPT; ++i) {
        const double2* ptr = reinterpret_cast<const double2*>(A.inner + static_cast<size_t>(i) * N + q);
        const double2 pxy = __ldg(ptr), pzw = __ldg(ptr + 1);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          const double d2 = dist2(ox[o], oy[o], oz[o], pxy.x, pxy.y, pzw.x);
          const double r = radius_of<KIND>(d2, rsqrt_fast(d2));
          double2 v, vg = make_double2(0.0, 0.0);
          vals(r, v, vg);
          const bool oob = !(r >= A.T.r_min && r <= A.T.r_max);
          if (__any_sync(0xffffffffu, oob)) {
            if (oob) {
              if (!self && valid) {
                // the reference's eval_kernel fallback (evaluator.hpp:199-205)
                if constexpr (PAIR) {
                  v = analytic_sincos(GK_KIND_EXP, A.T.k_re, A.T.k_im, r);
                  vg = analytic_sincos(GK_KIND_GREEN, A.T.k_re, A.T.k_im, r);
                } else {
                  v = analytic_sincos(KIND, A.T.k_re, A.T.k_im, r);
                }
                if (r > A.T.r_max) n_high += NS; else n_low += NS;
              } else {
                v = vg = make_double2(0.0, 0.0);
              }
            }
          }
          acc.add_values(o, pzw.y, v, vg);
        }
      }
      acc.finish([&](int o) { return sww[o]; }, self, valid, A.z, A.z2,
                 (p - A.row_begin) * A.ldz + q, A.counters + 2);
    }
    nev += static_cast<unsigned long long>(nq) * IPT * MO * NS;
  }
  __syncwarp();
}

// per-warp counters -> the fill's global counters (one atomic per warp)
__device__ __forceinline__ void flush_counters(const FillArgs& A, unsigned long long nev,
                                               unsigned long long n_low,
                                               unsigned long long n_high) {
  for (int o = 16; o; o >>= 1) {
    n_low += __shfl_xor_sync(0xffffffffu, n_low, o);
    n_high += __shfl_xor_sync(0xffffffffu, n_high, o);
  }
  const int lane = threadIdx.x & 31;
  if (lane == 0 && n_low) atomicAdd(A.counters, n_low);
  if (lane == 0 && n_high) atomicAdd(A.counters + 1, n_high);
  if (lane == 0 && nev) atomicAdd(A.counters + 3, nev);
}

template <int MO, int NPE, int KIND, int DEG>
__global__ void __launch_bounds__(32 * tedge_warps<KIND>(), 1) table_edge_kernel(const FillArgs A) {
  constexpr int W = tedge_warps<KIND>();
  constexpr int NS = KIND == kKindPair ? 2 : 1;
  extern __shared__ double2 sE[];  // edge sums [W][NS][ecap]
  __shared__ double sw[W][MO];
  const int warp = threadIdx.x >> 5;
  double2* const myE = sE + warp * NS * A.ecap;
  unsigned long long nev = 0, n_low = 0, n_high = 0;
  const auto vals = [&](double r, double2& v, double2& vg) { table_values<KIND, DEG>(r, A.T, v, vg); };
  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.nblk, b = tile - tr * A.nblk;
    const size_t p = A.row_begin + tr * W + warp;
    if (p >= A.row_end) continue;  // warp-uniform
    table_edge_tile<MO, NPE, KIND>(A, p, b, myE, sw[warp], vals, nev, n_low, n_high);
  }
  flush_counters(A, nev, n_low, n_high);
}

}  // namespace gk

#include "fill_sweep.cuh"

namespace gk {

// ------------------------------------------------ K3 with a shared-memory table
//
// North star part (2): the table a tile needs is held in shared memory.  Per
// tile (16 rows x 32 cpt columns) the CTA bounds the tile's radii from the
// per-triangle centroids and radii (as K1 does), maps [r_lo, r_hi] to the
// lookup-bucket and record ranges it can touch, and stages exactly those
// slices with TMA bulk copies (cp.async.bulk + mbarrier).  A table that fits
// whole is staged once per CTA; a tile whose window exceeds the budget reads
// the global table through L1 instead (correct either way: same code path,
// different TableWin).

#ifndef GK_TILES_PER_CTA
#define GK_TILES_PER_CTA 16  // set_tiling: widest tiles leaving this many per resident CTA
#endif
#ifndef GK_STAGED_CPT
#define GK_STAGED_CPT 2  // 32-column blocks per staged tile (windowed mode)
#endif
#ifndef GK_STAGED_WARPS
#define GK_STAGED_WARPS 16
#endif
constexpr int kStagedWarps = GK_STAGED_WARPS;

struct StageArgs {
  uint32_t lk_cap, j_cap;  // shared-memory capacity in buckets / records
  int whole;               // the whole table fits: stage once
};


// the fill of one tile through a table window (shared or global)
template <bool SMEM, int MO, int KIND, int DEG>
__device__ __forceinline__ void table_tile(const FillArgs& A, const TableWin& win, size_t p0,
                                           size_t tc, unsigned long long& n_low,
                                           unsigned long long& n_high) {
  constexpr bool WANT_E = KIND == GK_KIND_EXP || KIND == kKindPair;
  constexpr bool WANT_G = KIND == GK_KIND_GREEN || KIND == kKindPair;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t N = A.N;
  const size_t p = p0 + warp;
  if (p >= A.row_end) return;  // warp-uniform
  double ox[MO], oy[MO], oz[MO];
#pragma unroll
  for (int o = 0; o < MO; ++o) {
    const double2 xy = __ldg(reinterpret_cast<const double2*>(A.outer + p * MO + o));
    const double zz = __ldg(reinterpret_cast<const double*>(A.outer + p * MO + o) + 2);
    ox[o] = xy.x;
    oy[o] = xy.y;
    oz[o] = zz;
  }
  const size_t q0base = tc * (32 * static_cast<size_t>(A.cpt));
  int ncb = static_cast<int>((N - q0base + 31) / 32);
  if (ncb > A.cpt) ncb = A.cpt;
  const InnerWalk W{A.inner, N, q0base, A.ipt, ncb};
  const int iters = ncb * A.ipt;
  double2 nxy, nzw;
  size_t q;
  bool valid;
  W.load(0, 0, lane, nxy, nzw, q, valid);
  Acc<MO, KIND == kKindPair> acc;
  acc.zero();
  int ncb_next = 0, ni = 0;
  for (int it = 0; it < iters; ++it) {
    const double2 pxy = nxy, pzw = nzw;
    const size_t qc = q;
    const bool vc = valid;
    if (++ni == A.ipt) {
      ni = 0;
      ++ncb_next;
    }
    const bool block_done = ni == 0;
    const bool self = qc == p;
    if (it + 1 < iters) W.load(ncb_next, ni, lane, nxy, nzw, q, valid);
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double d2 = dist2(ox[o], oy[o], oz[o], pxy.x, pxy.y, pzw.x);
      const double r = radius_of<KIND>(d2, rsqrt_fast(d2));
      double2 ve = make_double2(0.0, 0.0), vg = make_double2(0.0, 0.0);
      win_eval<SMEM, DEG, WANT_E, WANT_G>(r, A.T, win, ve, vg, vc && !self);
      const bool oob = !(r >= A.T.r_min && r <= A.T.r_max);
      if (__any_sync(0xffffffffu, oob)) {
        if (oob) {
          if (!self && vc) {
            // the reference's eval_kernel fallback (evaluator.hpp:199-205)
            if constexpr (WANT_E) ve = analytic_sincos(GK_KIND_EXP, A.T.k_re, A.T.k_im, r);
            if constexpr (WANT_G) vg = analytic_sincos(GK_KIND_GREEN, A.T.k_re, A.T.k_im, r);
            const unsigned calls = KIND == kKindPair ? 2u : 1u;
            if (r > A.T.r_max) n_high += calls; else n_low += calls;
          } else {
            ve = vg = make_double2(0.0, 0.0);
          }
        }
      }
      if constexpr (KIND == kKindPair) acc.add_values(o, pzw.y, ve, vg);
      else acc.add_values(o, pzw.y, KIND == GK_KIND_EXP ? ve : vg, vg);
    }
    if (block_done) {
      acc.finish([&](int o) { return __ldg(reinterpret_cast<const double*>(A.outer + p * MO + o) + 3); },
                 self, vc, A.z, A.z2, (p - A.row_begin) * A.ldz + qc, A.counters + 2);
      acc.zero();
    }
  }
}

template <int MO, int KIND, int DEG>
__global__ void __launch_bounds__(32 * kStagedWarps, 1)
    table_staged_kernel(const FillArgs A, const StageArgs S) {
  constexpr bool WANT_E = KIND == GK_KIND_EXP || KIND == kKindPair;
  const int grs = DEG > 0 ? 2 + 2 * (DEG + 1) : A.T.grs;
  extern __shared__ __align__(16) unsigned char smem[];
  uint32_t* s_lk = reinterpret_cast<uint32_t*>(smem);
  double* s_grec = reinterpret_cast<double*>(smem + static_cast<size_t>(S.lk_cap) * 4);
  double* s_erec = s_grec + static_cast<size_t>(S.j_cap) * grs;
  __shared__ uint64_t bar;
  __shared__ double red_lo[kStagedWarps], red_hi[kStagedWarps];
  __shared__ uint32_t cur[4];   // staged window: b0, nb, j0, nj (nb = 0: none)
  __shared__ uint32_t want[4];  // window this tile needs
  __shared__ int mode;          // 0: shared window, 1: global table
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n = static_cast<uint32_t>(A.T.nrec);
  if (threadIdx.x == 0) {
    mbar_init(&bar);
    cur[1] = 0;
  }
  __syncthreads();
  uint32_t phase = 0;
  unsigned long long n_low = 0, n_high = 0;
  const TableWin gwin{A.T.grec, A.T.erec, A.T.lk, 0u, A.T.nlk, 0u, n};
  const size_t N = A.N;

  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.ncb, tc = tile - tr * A.ncb;
    const size_t p0 = A.row_begin + tr * kStagedWarps;
    if (!S.whole) {
      // conservative radius range of the tile's pairs (centroid +- radii)
      const size_t q0 = tc * (32 * static_cast<size_t>(A.cpt));
      const size_t ncols = (N - q0) < 32 * static_cast<size_t>(A.cpt) ? N - q0 : 32 * static_cast<size_t>(A.cpt);
      double lo = CUDART_INF, hi = 0.0;
      for (size_t k = threadIdx.x; k < kStagedWarps * ncols; k += blockDim.x) {
        const size_t pp = p0 + k / ncols, qq = q0 + k % ncols;
        if (pp >= A.row_end || qq == pp) continue;
        const double4 bp = A.bounds[pp];
        const double4 bq = A.bounds[qq];
        const double dx = bp.x - bq.x, dy = bp.y - bq.y, dz = bp.z - bq.z;
        const double dc = sqrt(dx * dx + dy * dy + dz * dz);
        const double rho = bp.w + __ldg(A.binner + qq);
        lo = fmin(lo, (dc - rho) * (1.0 - 1e-12));
        hi = fmax(hi, (dc + rho) * (1.0 + 1e-12));
      }
      for (int o = 16; o; o >>= 1) {
        lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
      }
      if (lane == 0) {
        red_lo[warp] = lo;
        red_hi[warp] = hi;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        for (int w = 1; w < kStagedWarps; ++w) {
          lo = fmin(lo, red_lo[w]);
          hi = fmax(hi, red_hi[w]);
        }
        lo = fmax(lo, A.T.r_min);
        hi = fmin(hi, A.T.r_max);
        if (!(lo <= hi)) lo = hi = A.T.r_min;  // no in-range pair: any valid window
        const uint32_t b_lo = lookup_bucket(lo, A.T), b_hi = lookup_bucket(hi, A.T);
        const uint32_t b0 = b_lo & ~3u;
        const uint32_t nb = (b_hi + 1 - b0 + 3) & ~3u;
        const uint32_t j_lo = __ldg(A.T.lk + b_lo);
        uint32_t j_hi = __ldg(A.T.lk + b_hi) + 1;
        if (j_hi > n - 1) j_hi = n - 1;
        want[0] = b0;
        want[1] = nb;
        want[2] = j_lo;
        want[3] = j_hi - j_lo + 1;
        const bool covered = cur[1] != 0 && b0 >= cur[0] && b0 + nb <= cur[0] + cur[1] &&
                             j_lo >= cur[2] && j_hi < cur[2] + cur[3];
        mode = covered ? 0 : (nb <= S.lk_cap && want[3] <= S.j_cap ? 2 : 1);
      }
    } else if (threadIdx.x == 0) {
      want[0] = 0;
      want[1] = (A.T.nlk + 3) & ~3u;
      want[2] = 0;
      want[3] = n;
      mode = cur[1] != 0 ? 0 : 2;
    }
    __syncthreads();
    if (mode == 2) {  // stage the window with TMA bulk copies
      if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        cur[0] = want[0];
        cur[1] = want[1];
        cur[2] = want[2];
        cur[3] = want[3];
        const uint32_t lk_bytes = want[1] * 4;
        const uint32_t g_bytes = want[3] * grs * 8;
        const uint32_t e_bytes = WANT_E ? want[3] * 6 * 8 : 0;
        mbar_expect_tx(&bar, lk_bytes + g_bytes + e_bytes);
        tma_load_1d(s_lk, A.T.lk + want[0], lk_bytes, &bar);
        tma_load_1d(s_grec, A.T.grec + static_cast<size_t>(want[2]) * grs, g_bytes, &bar);
        if (WANT_E) tma_load_1d(s_erec, A.T.erec + static_cast<size_t>(want[2]) * 6, e_bytes, &bar);
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      __syncthreads();
    }
    if (mode != 1) {
      const TableWin swin{s_grec, s_erec, s_lk, cur[0], cur[1], cur[2], cur[3]};
      table_tile<true, MO, KIND, DEG>(A, swin, p0, tc, n_low, n_high);
    } else {
      table_tile<false, MO, KIND, DEG>(A, gwin, p0, tc, n_low, n_high);
    }
    __syncthreads();  // the window may be restaged for the next tile
  }
  for (int o = 16; o; o >>= 1) {
    n_low += __shfl_xor_sync(0xffffffffu, n_low, o);
    n_high += __shfl_xor_sync(0xffffffffu, n_high, o);
  }
  if (lane == 0 && n_low) atomicAdd(A.counters, n_low);
  if (lane == 0 && n_high) atomicAdd(A.counters + 1, n_high);
}

template <class K>
void launch_kernel(gk_ctx* ctx, K kernel, const FillArgs& a, size_t smem, int threads = kThreads) {
  // opt in whenever dynamic shared memory is used: the 48 KB default covers
  // static + dynamic together (48 KB of edge sums + 768 B of weights failed)
  if (smem > 0)
    GK_CUDA(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
  int per_sm = 0;
  GK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem));
  if (per_sm < 1) per_sm = 1;
  size_t grid = static_cast<size_t>(ctx->sm_count) * per_sm;
  if (grid > a.ntiles) grid = a.ntiles;
  if (grid < 1) grid = 1;
  kernel<<<static_cast<unsigned>(grid), threads, smem, ctx->stream>>>(a);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
}

// widest tiles (fewest cold starts) that still leave >= 16 tiles per
// resident CTA for load balance
inline void set_tiling(const gk_ctx* ctx, FillArgs& a, int rows_per_tile, int ctas_per_sm) {
  const size_t row_blocks = (a.row_end - a.row_begin + rows_per_tile - 1) / rows_per_tile;
  const size_t col_blocks = (a.N + 31) / 32;
  const size_t want = static_cast<size_t>(ctx->sm_count) * ctas_per_sm * GK_TILES_PER_CTA;
  int cpt = kMaxColBlocks;
  while (cpt > 1 && row_blocks * ((col_blocks + cpt - 1) / cpt) < want) cpt /= 2;
  a.cpt = cpt;
  a.ncb = (col_blocks + cpt - 1) / cpt;
  a.ntiles = row_blocks * a.ncb;
}

template <int MO, int IPT, int KIND, int ATT>
void launch_v4(gk_ctx* ctx, FillArgs a, size_t smem) {
  set_tiling(ctx, a, warps_v4<KIND>(), 1);
  launch_kernel(ctx, direct_kernel_v4<MO, IPT, KIND, ATT>, a, smem, 32 * warps_v4<KIND>());
}

// K3e launch (edge sums in shared memory, the table through L1)
template <int MO, int KIND, int DEG>
int launch_table_edge(gk_ctx* ctx, FillArgs a) {
  constexpr int W = tedge_warps<KIND>();
  const size_t esmem = static_cast<size_t>(W) * (KIND == kKindPair ? 2 : 1) * a.ecap * sizeof(double2);
  auto go = [&](auto kern) {
    a.ntiles = ((a.row_end - a.row_begin + W - 1) / W) * a.nblk;
    launch_kernel(ctx, kern, a, esmem, 32 * W);
    return static_cast<int>(GK_PATH_TABLE_EDGE);
  };
  switch (a.ipt) {
    case 3: return go(table_edge_kernel<MO, 1, KIND, DEG>);
    case 6: return go(table_edge_kernel<MO, 2, KIND, DEG>);
    case 9: return go(table_edge_kernel<MO, 3, KIND, DEG>);
    case 12: return go(table_edge_kernel<MO, 4, KIND, DEG>);
    case 15: return go(table_edge_kernel<MO, 5, KIND, DEG>);
    default: fail(GK_ERR_RUNTIME, "shared-edge fill: n must be 1..5");
  }
}

// K3s launch (fill_sweep.cuh): the window takes the shared memory the edge
// sums and the band table leave (smem_budget caps it: tests force small
// windows and many bands); false when the window cannot cover a tile's
// radius spread with room for a band, or the bands would be too many (the
// caller takes K3e)
template <int MO, int KIND>
bool launch_table_sweep(gk_ctx* ctx, FillArgs a, size_t budget) {
  constexpr int W = sweep_warps<KIND>();
  constexpr int NS = KIND == kKindPair ? 2 : 1;
  constexpr int NWIN = KIND == kKindPair ? 2 : 1;
  constexpr size_t patch_bytes = kSweepPatch * (8 + (KIND != GK_KIND_EXP ? 80 : 0) +
                                                (KIND != GK_KIND_GREEN ? 48 : 0));
  const size_t limit = 227 * 1024 - 3072;  // opt-in maximum less the static shared memory
  // window nodes for a shared-memory budget: 16 B per node and window, 1 bit
  const auto window_of = [&](size_t fixed) -> size_t {
    if (fixed + 4096 > limit) return 0;
    size_t avail = limit - fixed;
    if (budget >= 4096 && budget < avail) avail = budget;
    size_t wn = (avail * 8) / (128 * NWIN + 1);
    const size_t whole = (static_cast<size_t>(a.T.nbase) + kSweepMargin + 31) & ~size_t(31);
    if (wn > whole) wn = whole;
    return wn & ~size_t(31);
  };
  const size_t base_fixed = static_cast<size_t>(W) * NS * a.s_ecap * 16 +
                            (((2 * kSweepBands + 1) * 4 + 15) & ~size_t(15)) + 64;
  // the staged records of non-uniform intervals pay where a window holds at
  // most kSweepPatch of them (with room to spare)
  size_t wn = window_of(base_fixed + patch_bytes);
  const bool patch = a.T.npatch > 0 && wn > 0 &&
                     static_cast<double>(a.T.npatch) * wn / a.T.nbase <= 0.7 * kSweepPatch;
  if (!patch) wn = window_of(base_fixed);
  const size_t fixed = base_fixed + (patch ? patch_bytes : 0);
  const double cap_r = (static_cast<double>(wn) - kSweepMargin) * a.T.t_eff;
  const double spread = 2.0 * (a.s_rho_max + a.s_rho_rows) * (1.0 + 1e-9);
  const double delta = cap_r - spread;
  // keys lie in [-spread / 2, r_max]: the bands of any cluster
  if (wn < 64 || !(delta >= 0.05 * cap_r) ||
      (a.T.r_max + spread) / delta + 2.0 > static_cast<double>(kSweepBands))
    return false;
  const size_t nbw = ((wn >> 5) + 8) & ~size_t(3);
  const size_t smem = NWIN * wn * 16 + nbw * 4 + fixed - 64;
  a.s_wn = static_cast<uint32_t>(wn);
  a.s_delta = delta;
  a.eblk = a.s_eblk;
  a.ep = a.s_ep;
  a.ecol = a.s_ecol;
  a.nblk = a.s_nblk;
  a.ecap = a.s_ecap;
  const size_t clusters = (a.row_end - a.row_begin + a.s_rc - 1) / a.s_rc;
  size_t grid = static_cast<size_t>(ctx->sm_count);
  if (grid > clusters) grid = clusters;
  a.s_full = clusters > grid ? clusters - grid : 0;
  DevBuf<uint32_t> list;  // stream-ordered: freed after the launch completes
  const size_t nlist = (grid * a.s_rc * a.nblk + 1) & ~size_t(1);
  list.alloc(nlist + 2, ctx->stream);
  a.s_list = list.p;
  a.s_next_cluster = reinterpret_cast<unsigned long long*>(list.p + nlist);
  GK_CUDA(cudaMemsetAsync(a.s_next_cluster, 0, sizeof(unsigned long long), ctx->stream));
  auto go = [&](auto kern) {
    GK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    kern<<<static_cast<unsigned>(grid), 32 * W, smem, ctx->stream>>>(a);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    return true;
  };
  const auto pick = [&](auto with, auto without) { return patch ? go(with) : go(without); };
  switch (a.ipt) {
    case 3: return pick(table_sweep_kernel<MO, 1, KIND, true>, table_sweep_kernel<MO, 1, KIND, false>);
    case 6: return pick(table_sweep_kernel<MO, 2, KIND, true>, table_sweep_kernel<MO, 2, KIND, false>);
    case 9: return pick(table_sweep_kernel<MO, 3, KIND, true>, table_sweep_kernel<MO, 3, KIND, false>);
    case 12: return pick(table_sweep_kernel<MO, 4, KIND, true>, table_sweep_kernel<MO, 4, KIND, false>);
    case 15: return pick(table_sweep_kernel<MO, 5, KIND, true>, table_sweep_kernel<MO, 5, KIND, false>);
    default: return false;
  }
}

// K3s for a kind; the fused pair whose two windows do not fit runs as the
// two single-kind sweeps (Exp into z, Green into z2): the same bits as the
// separate fills, which keeps the pair bitwise equal to them
template <int MO, int KIND>
bool try_sweep(gk_ctx* ctx, const FillArgs& a, size_t budget) {
  if (launch_table_sweep<MO, KIND>(ctx, a, budget)) return true;
  if constexpr (KIND == kKindPair) {
    FillArgs ag = a;
    ag.z = a.z2;
    if (!launch_table_sweep<MO, GK_KIND_EXP>(ctx, a, budget)) return false;
    if (!launch_table_sweep<MO, GK_KIND_GREEN>(ctx, ag, budget))
      fail(GK_ERR_RUNTIME, "table sweep: the Green window does not fit where the Exp one does");
    return true;
  }
  return false;
}

// returns the gk_fill_path that ran (the shared-edge paths count their evaluations)
template <int MO, int MODE, int KIND, int DEG, int ATT>
int launch_one(gk_ctx* ctx, FillArgs a, const gk_fill_options& o) {
  if constexpr (MODE == GK_MODE_DIRECT) {
    const size_t smem = kPhaseSlots * sizeof(double2) +
                        (ATT == 1 ? a.nhi * sizeof(double) : 0) +
                        (ATT == 2 ? a.natten * sizeof(double) : 0);
    const bool use_v4 = o.unrolled != 0;
    // shared-edge path (edges.cu): single kind, lossless or phase-coupled
    // attenuation, n = 1..5; launch_fill leaves nblk = 0 where it does not pay
    if constexpr (ATT != 2) {
      constexpr int W = edge_warps<KIND>();
      const size_t esmem = kPhaseSlots * sizeof(double2) +
                           W * (KIND == kKindPair ? 2 : 1) * a.ecap * sizeof(double2) +
                           (ATT == 1 ? a.nhi * sizeof(double) : 0);
      // the 227 KB opt-in limit (the pair's two sums per edge at 12 chunks
      // with many attenuation entries would exceed it): per-triangle then
      if (a.nblk > 0 && esmem + 2048 <= 227 * 1024) {
        auto go = [&](auto kern) {
          a.ntiles = ((a.row_end - a.row_begin + W - 1) / W) * a.nblk;
          launch_kernel(ctx, kern, a, esmem, 32 * W);
          return static_cast<int>(GK_PATH_DIRECT_EDGE);
        };
        switch (a.ipt) {
          case 3: return go(direct_edge_kernel<MO, 1, KIND, ATT>);
          case 6: return go(direct_edge_kernel<MO, 2, KIND, ATT>);
          case 9: return go(direct_edge_kernel<MO, 3, KIND, ATT>);
          case 12: return go(direct_edge_kernel<MO, 4, KIND, ATT>);
          case 15: return go(direct_edge_kernel<MO, 5, KIND, ATT>);
          default: fail(GK_ERR_RUNTIME, "shared-edge fill: n must be 1..5");
        }
      }
    }
    if (use_v4) {
      switch (a.ipt) {  // n = 1..5 Gauss points per edge: fully unrolled fast path
        case 3: launch_v4<MO, 3, KIND, ATT>(ctx, a, smem); return static_cast<int>(GK_PATH_DIRECT);
        case 6: launch_v4<MO, 6, KIND, ATT>(ctx, a, smem); return static_cast<int>(GK_PATH_DIRECT);
        case 9: launch_v4<MO, 9, KIND, ATT>(ctx, a, smem); return static_cast<int>(GK_PATH_DIRECT);
        case 12: launch_v4<MO, 12, KIND, ATT>(ctx, a, smem); return static_cast<int>(GK_PATH_DIRECT);
        case 15: launch_v4<MO, 15, KIND, ATT>(ctx, a, smem); return static_cast<int>(GK_PATH_DIRECT);
        default: break;
      }
    }
    set_tiling(ctx, a, kRowsPerTile, 2);
    launch_kernel(ctx, direct_kernel<MO, KIND, ATT, 2>, a, smem);
    return static_cast<int>(GK_PATH_DIRECT);
  } else {
    // o.table_placement: GK_TABLE_GLOBAL = through L1 (K3e where the mesh's
    // shared-edge blocks are in use, else the per-triangle L1 kernel),
    // GK_TABLE_SHARED = always staged per triangle (whole or per-tile
    // windows; tests and A/B), GK_AUTO = by size.  o.smem_budget shrinks the
    // window budget (tests).
    const int placement = o.table_placement;
    const bool automatic = placement != GK_TABLE_GLOBAL && placement != GK_TABLE_SHARED &&
                           placement != GK_TABLE_SWEEP;
    // K3s where launch_fill found it eligible (degree 3 / Exp, shared edges):
    // on request here, and under GK_AUTO for the dense tables below
    constexpr bool kSweepable = DEG == 3 || KIND == GK_KIND_EXP;
    if constexpr (kSweepable) {
      if (a.s_nblk > 0 && placement == GK_TABLE_SWEEP &&
          try_sweep<MO, KIND>(ctx, a, o.smem_budget))
        return static_cast<int>(GK_PATH_TABLE_SWEEP);
    }
    if (placement == GK_TABLE_SWEEP && a.nblk > 0) return launch_table_edge<MO, KIND, DEG>(ctx, a);
    if (a.nblk > 0 && placement == GK_TABLE_GLOBAL) return launch_table_edge<MO, KIND, DEG>(ctx, a);
    if (placement == GK_TABLE_GLOBAL) {
      set_tiling(ctx, a, GK_TABLE_WARPS, GK_TABLE_CTAS);
      launch_kernel(ctx, table_kernel<MO, KIND, DEG>, a, 0, 32 * GK_TABLE_WARPS);
      return static_cast<int>(GK_PATH_TABLE_L1);
    }
    // shared-memory window sizing: whole table if it fits, else proportional caps
    constexpr bool want_e = KIND == GK_KIND_EXP || KIND == kKindPair;
    const size_t rec_bytes = static_cast<size_t>(a.T.grs) * 8 + (want_e ? 48 : 0);
    size_t budget = 200 * 1024;
    if (o.smem_budget >= 4096 && o.smem_budget < budget) budget = static_cast<size_t>(o.smem_budget);
    StageArgs S{};
    const size_t nlk4 = (static_cast<size_t>(a.T.nlk) + 3) & ~size_t(3);
    const bool whole = nlk4 * 4 + a.T.nrec * rec_bytes <= budget;
    // a table too large to stage whole but small enough to stay L1-resident
    // (<= 300 KB of records) goes to K3e: C4 at S = 1e3 (233 KB) 145 vs 180 ms
    // windowed-staged; C3 (548 KB) and C5 (1.1 MB) stay staged (343 vs 311,
    // 184 vs 158 ms per 4096 rows)
    if (a.nblk > 0 && automatic && !whole && a.T.nrec * rec_bytes <= 300 * 1024)
      return launch_table_edge<MO, KIND, DEG>(ctx, a);
    // every larger table: the sweep (K3s, the table in shared memory per
    // distance band on shared edges) where its window covers a tile.  Full
    // C5: S = 1e4 1.91 s (K3e 3.54 s), S = 1e3 2.53 s (staged per-triangle
    // windows 3.16 s); per 8192 rows C3 S = 1e3 102 vs 125 ms
    // (scripts/sweep_ab.py)
    if constexpr (kSweepable) {
      if (automatic && !whole && a.s_nblk > 0 && try_sweep<MO, KIND>(ctx, a, 0))
        return static_cast<int>(GK_PATH_TABLE_SWEEP);
    }
    if (whole) {
      S.whole = 1;
      S.lk_cap = static_cast<uint32_t>(nlk4);
      S.j_cap = a.T.nrec;
      set_tiling(ctx, a, kStagedWarps, 1);
    } else {
      const double per_rec = static_cast<double>(a.T.nlk) / a.T.nrec;  // buckets per record
      const size_t j_cap = static_cast<size_t>(budget / (rec_bytes + 4.0 * per_rec * 1.5));
      // records a typical tile window spans; when it clearly exceeds the
      // capacity (dense tables, e.g. S = 1e4 on large meshes) every tile would
      // fall back to global reads: use the L1 kernel with its wider tiles
      const double est = a.T.nrec * a.window_est / (a.T.r_max - a.T.r_min);
      if (automatic && est > 2.0 * static_cast<double>(j_cap)) {
        // shared edges (K3e) instead of the L1 kernel: both read the table
        // through L1; K3e 1.3-1.4x faster at S = 1e4 on C3/C4/C5.  Tables
        // staged in shared memory (whole or per tile window) stay per
        // triangle: faster than K3e through L1 (C5 S = 1e3: 158 vs 225 ms
        // per 4096 rows).  Not when a test forces a staging path.
        if (a.nblk > 0) return launch_table_edge<MO, KIND, DEG>(ctx, a);
        set_tiling(ctx, a, GK_TABLE_WARPS, GK_TABLE_CTAS);
        launch_kernel(ctx, table_kernel<MO, KIND, DEG>, a, 0, 32 * GK_TABLE_WARPS);
        return static_cast<int>(GK_PATH_TABLE_L1);
      }
      S.j_cap = static_cast<uint32_t>(j_cap);
      S.lk_cap = static_cast<uint32_t>(((budget - j_cap * rec_bytes) / 4) & ~size_t(3));
      set_tiling(ctx, a, kStagedWarps, 1);
      // narrow tiles keep each tile's radius window small
      a.cpt = GK_STAGED_CPT;
      a.ncb = (a.N + 32 * GK_STAGED_CPT - 1) / (32 * GK_STAGED_CPT);
      a.ntiles = ((a.row_end - a.row_begin + kStagedWarps - 1) / kStagedWarps) * a.ncb;
    }
    const size_t smem = static_cast<size_t>(S.lk_cap) * 4 + static_cast<size_t>(S.j_cap) * rec_bytes;
    auto k = table_staged_kernel<MO, KIND, DEG>;
    GK_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 static_cast<int>(smem)));
    size_t grid = static_cast<size_t>(ctx->sm_count);
    if (grid > a.ntiles) grid = a.ntiles;
    if (grid < 1) grid = 1;
    k<<<static_cast<unsigned>(grid), 32 * kStagedWarps, smem, ctx->stream>>>(a, S);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    return static_cast<int>(GK_PATH_TABLE_STAGED);
  }
}

template <int MO, int KIND>
int dispatch_att(gk_ctx* ctx, const FillArgs& a, int att, const gk_fill_options& o) {
  if (att == 1) return launch_one<MO, GK_MODE_DIRECT, KIND, 0, 1>(ctx, a, o);
  if (att == 2) return launch_one<MO, GK_MODE_DIRECT, KIND, 0, 2>(ctx, a, o);
  return launch_one<MO, GK_MODE_DIRECT, KIND, 0, 0>(ctx, a, o);
}

// returns the gk_fill_path that ran (launch_fill)
template <int MO>
int dispatch_mo(gk_ctx* ctx, const FillArgs& a, gk_mode mode, int kind, int degree, int att,
                 const gk_fill_options& o) {
  if (mode == GK_MODE_DIRECT) {
    if (kind == GK_KIND_GREEN) return dispatch_att<MO, GK_KIND_GREEN>(ctx, a, att, o);
    if (kind == GK_KIND_EXP) return dispatch_att<MO, GK_KIND_EXP>(ctx, a, att, o);
    return dispatch_att<MO, kKindPair>(ctx, a, att, o);
  }
  if (kind == GK_KIND_EXP) return launch_one<MO, GK_MODE_TABLE, GK_KIND_EXP, 0, 0>(ctx, a, o);
  if (kind == GK_KIND_GREEN && degree == 3)
    return launch_one<MO, GK_MODE_TABLE, GK_KIND_GREEN, 3, 0>(ctx, a, o);
  if (kind == GK_KIND_GREEN) return launch_one<MO, GK_MODE_TABLE, GK_KIND_GREEN, 0, 0>(ctx, a, o);
  if (degree == 3) return launch_one<MO, GK_MODE_TABLE, kKindPair, 3, 0>(ctx, a, o);
  return launch_one<MO, GK_MODE_TABLE, kKindPair, 0, 0>(ctx, a, o);
}

// one explicit instantiation per translation unit (fill_mo<m>.cu)
extern template int dispatch_mo<1>(gk_ctx*, const FillArgs&, gk_mode, int, int, int, const gk_fill_options&);
extern template int dispatch_mo<3>(gk_ctx*, const FillArgs&, gk_mode, int, int, int, const gk_fill_options&);
extern template int dispatch_mo<4>(gk_ctx*, const FillArgs&, gk_mode, int, int, int, const gk_fill_options&);
extern template int dispatch_mo<6>(gk_ctx*, const FillArgs&, gk_mode, int, int, int, const gk_fill_options&);
extern template int dispatch_mo<7>(gk_ctx*, const FillArgs&, gk_mode, int, int, int, const gk_fill_options&);

}  // namespace gk
