// fill_sweep.cuh -- K3s: the paper's table fill (TableKernel::accumulate,
// evaluator.hpp:150-194, 237-272) on shared edges with the table held in
// shared memory (north star part 2), included by fill_kernels.cuh.
//
// Why a sweep.  A tile (row p, source block b) meets radii in [key, key +
// 2 (rho_p + rho_b)], key = |c_p - c_b| - rho_p - rho_b (bounding spheres of
// p's outer points and of b's inner points), so the table slice it needs is
// ~2 (rho_p + rho_b) / t_eff nodes wide whatever the distance.  A CTA owns a
// cluster of up to 32 rows (consecutive in the sweep set's spatial order),
// sorts the cluster's tiles by band of key (width delta, a counting sort into
// a per-CTA list in global memory) and walks the bands: band k's tiles need
// radii in [K_k, K_k + delta + 2 (rho_p,max + rho_b,max)], which one staged
// window of s_wn base nodes covers by the choice of delta.  Each band stages
// its window once (TMA bulk copies, mbarrier) and every tile of the band
// reads the table from shared memory.
//
// What is staged.  Away from the refinement windows around the kernel's zeros
// the plan's nodes are the uniform base grid r_min + i t_eff (build_plan,
// sampling.hpp:212-213), and 99.6-99.9 % of the degree-3 stencils at S = 1e4
// are four consecutive base points (SURVEY §7 hard part 2).  The window holds
// the node values by base index (16 B per node: 4x smaller than interval
// records), plus one bit per base interval marking those stencils.  For such
// an interval the reference's Lagrange cubic through nodes i-1..i+2 is
// evaluated with the uniform weights in s = (r - a_i) / t_eff; every other
// radius (stencils touching refined points or zeros, the table ends, r
// outside [r_min, r_max]) takes the global interval records -- the same path
// as K3e (table_values).  Which path a radius takes depends on the radius
// alone (a band's window covers every pair radius of its tiles), so the
// result does not depend on the row clusters or the row partition.
//
// Parity.  The cubic through the same four node values is unique; the
// uniform weights differ from the reference's w_a = prod(r - a_b) inv_den[a]
// (evaluator.hpp:264-269) only by rounding: s carries an absolute error of
// ~u r / t_eff, which moves the value by ~u (1 + k r) |f|, inside the stated
// per-term rounding tolerance 64 u (1 + |k| r) / r; at s = 0
// the weights are exactly (0, 1, 0, 0), so nodes are reproduced exactly
// (evaluator.hpp:259-262).
#pragma once

namespace gk {

#ifndef GK_SWEEP_WARPS
#define GK_SWEEP_WARPS 24  // measured: 12 -> 24 warps (80 registers, 72 B spill) C5 S=1e4 253 -> 227 ms per 8192 rows
#endif
template <int KIND>
__host__ __device__ constexpr int sweep_warps() { return KIND == kKindPair ? 8 : GK_SWEEP_WARPS; }
#ifndef GK_SWEEP_RC
#define GK_SWEEP_RC 32
#endif
constexpr int kSweepRowsPerCluster = GK_SWEEP_RC;  // rows per cluster (<= 32: one warp's lanes)
#ifndef GK_SWEEP_ORDERED
#define GK_SWEEP_ORDERED 0  // 1: warp-aggregated scatter (a warp's tiles of a band stay in order)
#endif
#ifndef GK_SWEEP_CHUNK
#define GK_SWEEP_CHUNK 1  // largest claim (tiles) from a band's list
#endif
constexpr int kSweepBands = 512;  // bands per cluster (launch_table_sweep checks the bound)
// staged records of non-uniform intervals per band: S = 1e4 windows need
// ~100 (C5); sparser tables (S = 1e3: ~700 per window) read them globally
#ifndef GK_SWEEP_PATCH
#define GK_SWEEP_PATCH 128
#endif
constexpr int kSweepPatch = GK_SWEEP_PATCH;
constexpr int kSweepMargin = 16;  // base nodes of the window kept as margin (8 per side)

// lower end of the tile's radii: |c_p - c_b| - rho_p - rho_b
__device__ __forceinline__ double sweep_key(const EdgeBlock* eb, size_t b, double4 cp) {
  const EdgeBlock& B = eb[b];
  const double dx = B.cx - cp.x, dy = B.cy - cp.y, dz = B.cz - cp.z;
  return sqrt(dx * dx + dy * dy + dz * dz) - B.rho - cp.w;
}

template <int MO, int NPE, int KIND, bool PATCH>
__global__ void __launch_bounds__(32 * sweep_warps<KIND>(), 1) table_sweep_kernel(const FillArgs A) {
  constexpr int W = sweep_warps<KIND>();
  constexpr bool WANT_G = KIND != GK_KIND_EXP, WANT_E = KIND != GK_KIND_GREEN;
  constexpr int NS = KIND == kKindPair ? 2 : 1;
  constexpr int RC = kSweepRowsPerCluster;
  const int wn = static_cast<int>(A.s_wn);
  const int nbw = ((wn >> 5) + 8) & ~3;  // staged bit words (multiple of 4: 16 B)
  extern __shared__ __align__(16) unsigned char smem[];
  unsigned char* sp = smem;
  double2* const s_g = reinterpret_cast<double2*>(sp);
  if (WANT_G) sp += static_cast<size_t>(wn) * 16;
  double2* const s_e = reinterpret_cast<double2*>(sp);
  if (WANT_E) sp += static_cast<size_t>(wn) * 16;
  uint32_t* const s_bits = reinterpret_cast<uint32_t*>(sp);
  sp += static_cast<size_t>(nbw) * 4;
  double2* const sE = reinterpret_cast<double2*>(sp);
  sp += static_cast<size_t>(W) * NS * A.ecap * 16;
  int* const s_off = reinterpret_cast<int*>(sp);  // [kSweepBands + 1] band offsets
  int* const s_cur = s_off + kSweepBands + 1;     // [kSweepBands] scatter / claim cursors
  sp += ((2 * kSweepBands + 1) * 4 + 15) & ~15;
  // the non-uniform intervals' records (TableDev::pj)
  double* const s_pa = reinterpret_cast<double*>(sp);
  if (PATCH) sp += kSweepPatch * 8;
  double* const s_pg = reinterpret_cast<double*>(sp);
  if (PATCH && WANT_G) sp += kSweepPatch * 80;
  double* const s_pe = reinterpret_cast<double*>(sp);
  __shared__ int s_pk[2];
  __shared__ double sw[W][MO];
  __shared__ uint64_t bar;
  __shared__ double s_red[W][2];
  __shared__ double4 s_row[RC];  // the cluster's rows: outer-point spheres

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const myE = sE + warp * NS * A.ecap;
  const double delta = A.s_delta, inv_delta = 1.0 / delta;
  const int nbase = static_cast<int>(A.T.nbase);
  const int nwords = (((nbase + 31) >> 5) + 8) & ~3;  // allocated bit words
  uint32_t* const glist = A.s_list + static_cast<size_t>(blockIdx.x) * RC * A.nblk;
  SweepWin win{s_g, s_e, s_bits, 0, 0, wn, -A.T.r_min * A.T.inv_t, A.T.inv_t,
               s_pa, s_pg, s_pe, 0};
  const auto vals = [&](double r, double2& v, double2& vg) {
    sweep_values<KIND, false, PATCH>(r, win, A.T, v, vg);
  };
  unsigned long long nev = 0, n_low = 0, n_high = 0;
  if (threadIdx.x == 0) mbar_init(&bar);
  __syncthreads();
  uint32_t phase = 0;

  const size_t nrows = A.row_end - A.row_begin;
  // clusters 0 .. s_full-1 hold RC rows; the last round's rows go in clusters
  // of RC / 2 (a shorter tail when the dynamic schedule drains)
  const size_t nfull = A.s_full;
  const size_t ncl = nfull + (nrows - nfull * RC + RC / 2 - 1) / (RC / 2);
  __shared__ size_t s_cl;
  for (;;) {
    // clusters are taken dynamically (the last word of the list scratch)
    if (threadIdx.x == 0) s_cl = atomicAdd(A.s_next_cluster, 1ull);
    __syncthreads();
    const size_t cl = s_cl;
    if (cl >= ncl) break;
    const size_t rb = cl < nfull ? cl * RC : nfull * RC + (cl - nfull) * (RC / 2);
    const size_t rc = cl < nfull ? RC : RC / 2;
    const int nr = static_cast<int>(nrows - rb < rc ? nrows - rb : rc);
    const uint32_t* const rows = A.s_rows + rb;
    if (warp == 0 && lane < nr) s_row[lane] = A.bounds[rows[lane]];
    __syncthreads();
    // tile t = (block t / nr, row t % nr): block-major, so that a warp's
    // consecutive claims mostly share the block (its edge points stay in L1)
    const size_t nblk = A.nblk;
    const size_t ntile = static_cast<size_t>(nr) * nblk;
    // pass 1: key range
    double kmin = CUDART_INF, kmax = -CUDART_INF;
    for (size_t t = threadIdx.x; t < ntile; t += blockDim.x) {
      const double k = sweep_key(A.eblk, t / nr, s_row[t % nr]);
      kmin = fmin(kmin, k);
      kmax = fmax(kmax, k);
    }
    for (int o = 16; o; o >>= 1) {
      kmin = fmin(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
      kmax = fmax(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    }
    if (lane == 0) {
      s_red[warp][0] = kmin;
      s_red[warp][1] = kmax;
    }
    for (int b = threadIdx.x; b <= kSweepBands; b += blockDim.x) s_off[b] = 0;
    __syncthreads();
    kmin = s_red[0][0];
    kmax = s_red[0][1];
    for (int w = 1; w < W; ++w) {
      kmin = fmin(kmin, s_red[w][0]);
      kmax = fmax(kmax, s_red[w][1]);
    }
    int nbands = static_cast<int>((kmax - kmin) * inv_delta) + 1;
    GK_DASSERT(nbands <= kSweepBands);
    nbands = nbands < kSweepBands ? nbands : kSweepBands;
    const auto band_of = [&](double k) {
      const int b = static_cast<int>((k - kmin) * inv_delta);
      return b < nbands ? b : nbands - 1;
    };
    // pass 2: band histogram (counts at s_off[band + 1])
    for (size_t t = threadIdx.x; t < ntile; t += blockDim.x)
      atomicAdd(&s_off[band_of(sweep_key(A.eblk, t / nr, s_row[t % nr])) + 1], 1);
    __syncthreads();
    if (warp == 0) {  // inclusive scan of the counts -> offsets
      int carry = 0;
      for (int b0 = 1; b0 <= nbands; b0 += 32) {
        const int b = b0 + lane;
        int v = b <= nbands ? s_off[b] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const int u = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += u;
        }
        if (b <= nbands) s_off[b] = v + carry;
        carry += __shfl_sync(0xffffffffu, v, 31);
      }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nbands; b += blockDim.x) s_cur[b] = s_off[b];
    __syncthreads();
    // pass 3: scatter the tiles by band; a warp's 32 consecutive tiles of one
    // band stay consecutive (one atomic per band and warp)
    for (size_t t0 = static_cast<size_t>(warp) * 32; t0 < ntile; t0 += blockDim.x) {
      const size_t t = t0 + lane;
      const int band = t < ntile ? band_of(sweep_key(A.eblk, t / nr, s_row[t % nr])) : -1;
      if (!GK_SWEEP_ORDERED) {
        if (band >= 0) glist[atomicAdd(&s_cur[band], 1)] = static_cast<uint32_t>(t);
        continue;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, band);
      const int leader = __ffs(peers) - 1;
      const int rank = __popc(peers & ((1u << lane) - 1u));
      int base = 0;
      if (band >= 0 && lane == leader) base = atomicAdd(&s_cur[band], __popc(peers));
      base = __shfl_sync(0xffffffffu, base, leader);
      if (band >= 0) glist[base + rank] = static_cast<uint32_t>(t);
    }
    __syncthreads();  // s_cur[band] == s_off[band + 1]: the claim cursors (counting down)
    for (int kb = 0; kb < nbands; ++kb) {
      const int lo = s_off[kb];
      if (s_off[kb + 1] == lo) continue;  // uniform
      // window: base nodes [i0, i0 + wn) from 8 nodes below the band's lowest radius
      const double xlo = (kmin + kb * delta - A.T.r_min) * A.T.inv_t;
      int i0 = xlo > 8.0 ? static_cast<int>(fmin(xlo, 2.0e9)) - 8 : 0;
      if (i0 > nbase - 1) i0 = nbase - 1;
      const int w0 = (i0 >> 5) & ~3;
      win.i0 = i0;
      win.w0 = w0;
      // nodes past the table's end are not staged: no interval reaching them
      // passes the window test (>= 4 keeps the unsigned test meaningful)
      win.wn = nbase - i0 < wn ? (nbase - i0 > 4 ? nbase - i0 : 4) : wn;
      if (threadIdx.x == 0) {
        // the previous band's generic-proxy reads of the window are complete
        // (barrier below): order them before the async-proxy writes
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t nn = static_cast<uint32_t>(nbase - i0 < wn ? nbase - i0 : wn);
        const uint32_t nw = static_cast<uint32_t>(nwords - w0 < nbw ? nwords - w0 : nbw);
        mbar_expect_tx(&bar, nn * 16u * (WANT_G + WANT_E) + nw * 4u);
        if (WANT_G) tma_load_1d(s_g, A.T.bg + i0, nn * 16u, &bar);
        if (WANT_E) tma_load_1d(s_e, A.T.be + i0, nn * 16u, &bar);
        tma_load_1d(s_bits, A.T.bclean + w0, nw * 4u, &bar);
      }
      // the non-uniform intervals' records the window's radii can meet
      if (PATCH) {
        win.np = stage_patches<WANT_G, WANT_E>(
            A.T, A.T.r_min + i0 * A.T.t_eff,
            i0 + win.wn >= nbase ? A.T.r_max : A.T.r_min + (i0 + win.wn) * A.T.t_eff,
            kSweepPatch, s_pa, s_pg, s_pe, s_pk);
        __syncthreads();
      }
      mbar_wait(&bar, phase);
      phase ^= 1u;
      // guided claims from the top of the band's list: chunks of up to 8
      // tiles, shrinking as the band drains
      for (;;) {
        int hi = 0, take = 0;
        if (lane == 0) {
          const int left = *reinterpret_cast<volatile int*>(&s_cur[kb]) - lo;
          take = left / (2 * W);
          take = take < 1 ? 1 : (take > GK_SWEEP_CHUNK ? GK_SWEEP_CHUNK : take);
          hi = atomicSub(&s_cur[kb], take);
        }
        hi = __shfl_sync(0xffffffffu, hi, 0);
        take = __shfl_sync(0xffffffffu, take, 0);
        if (hi <= lo) break;
        const int end = hi - take > lo ? hi - take : lo;
        for (int idx = hi - 1; idx >= end; --idx) {
          const uint32_t t = glist[idx];
          const size_t b = t / nr;
          const size_t r = t - b * nr;
          table_edge_tile<MO, NPE, KIND>(A, rows[r], b, myE, sw[warp], vals, nev, n_low, n_high);
        }
      }
      __syncthreads();  // the window is restaged for the next band
    }
  }
  flush_counters(A, nev, n_low, n_high);
}

}  // namespace gk
