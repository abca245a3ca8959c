// fill.cu -- fill dispatch (launch_fill), K1 distance range, phase and
// attenuation tables.  The fill kernels live in fill_kernels.cuh.
//
// launch_fill is fill_matrix's fill_rows loop (matfill.hpp:169-203) for a row
// block [row_begin, row_end) -- the reference's per-thread chunk
// (matfill.hpp:206-221) -- with AnalyticKernel (DIRECT, kernel.hpp:48-61) or
// TableKernel (TABLE, evaluator.hpp:150-194); self pairs stay zero
// (matfill.hpp:178).  K1 (launch_range) replaces max_vertex_distance
// (mesh.hpp:62-68) x 1.01 (matfill.hpp:270) and the fixed r_min
// (gktab_main.cpp:62) by the exact min/max quadrature-pair distance, so a
// device table spans exactly the radii the fill meets.  Complex k (lossy
// media) follows eval_analytic's form exp(-jkr) with k -> k_re + j k_im
// (kernel.hpp:48-61 extended; no reference path, kernel.hpp:23-24).
#include <cmath>
#include <cstdint>
#include <cstdlib>

#include <cub/block/block_scan.cuh>

#include "fill_kernels.cuh"

namespace gk {

// the table sweep's rows: the triangles of [rb, re) in the sweep set's
// spatial order (block positions), compacted; one CTA, order-preserving
__global__ void __launch_bounds__(1024) sweep_rows_kernel(const uint4* __restrict__ ecol, size_t N,
                                                          size_t rb, size_t re,
                                                          uint32_t* __restrict__ out) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage ts;
  __shared__ int base;
  if (threadIdx.x == 0) base = 0;
  __syncthreads();
  for (size_t j0 = 0; j0 < N; j0 += 1024) {
    const size_t j = j0 + threadIdx.x;
    uint32_t q = 0;
    int f = 0;
    if (j < N) {
      q = ecol[j].x;
      f = q >= rb && q < re;
    }
    int off = 0, tot = 0;
    Scan(ts).ExclusiveSum(f, off, tot);
    if (f) out[base + off] = q;
    __syncthreads();
    if (threadIdx.x == 0) base += tot;
    __syncthreads();
  }
}

__global__ void lossy_phase_kernel(double2* tab, double* ahi, int nhi, double c);

int launch_fill(gk_ctx* ctx, const gk_mesh* mesh, gk_mode mode, const gk_table* table,
                 int kind, double k_re, double k_im, size_t row_begin, size_t row_end,
                 gk_c128* z, gk_c128* z2, size_t ldz, unsigned long long* counters,
                 const gk_fill_options& opts) {
  FillArgs a{};
  a.outer = mesh->outer.p;
  a.inner = mesh->inner.p;
  a.bounds = mesh->bounds.p;
  a.binner = mesh->binner.p;
  // 16 rows x 64 columns of spatially ordered triangles span ~ (4 + 8) edges each way
  a.window_est = 18.0 * mesh->mean_edge;
  a.N = mesh->N;
  a.ipt = 3 * mesh->n;
  a.row_begin = row_begin;
  a.row_end = row_end;
  a.z = reinterpret_cast<double2*>(z);
  a.z2 = reinterpret_cast<double2*>(z2);
  a.ldz = ldz;
  if (table) a.T = table->dev;
  if (opts.arith_locate == 0) a.T.ncoarse = 0;
  a.phase = ctx->phase.p;
  a.K1 = k_re * kPhaseM / (2.0 * kPi);
  a.k_re = k_re;
  a.k_im = k_im;
  a.counters = counters;
  if (row_end <= row_begin || mesh->N == 0) return 0;

  DevBuf<double> atten;
  DevBuf<double2> lossy_tab;
  int att = 0;
  const bool phase_att = opts.lossy_phase != 0;
  if (mode == GK_MODE_DIRECT && k_im != 0.0 && k_im < 0.0 && k_re > 0.0 && phase_att &&
      kPi * -k_im / (k_re * kPhaseM) <= 1e-3) {
    // attenuation coupled to the phase reduction (cis_phase_att): per-fill
    // scaled phase table + exp(c M hi) for the hi = n >> 13 that occur
    att = 1;
    const double c = k_im / a.K1;
    a.nhi = static_cast<int>(a.K1 * mesh->diameter / kPhaseM) + 2;
    const size_t nhi2 = (static_cast<size_t>(a.nhi) + 1) / 2;  // double2 slots
    lossy_tab.alloc(kPhaseSlots + nhi2, ctx->stream);
    const int nthreads = kPhaseSlots > a.nhi ? kPhaseSlots : a.nhi;
    lossy_phase_kernel<<<(nthreads + 255) / 256, 256, 0, ctx->stream>>>(
        lossy_tab.p, reinterpret_cast<double*>(lossy_tab.p + kPhaseSlots), a.nhi, c);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    a.phase = lossy_tab.p;
    a.ahi = reinterpret_cast<const double*>(lossy_tab.p + kPhaseSlots);
    a.q1 = c;
    a.q2 = c * c / 2.0;
    a.q3 = c * c * c / 6.0;
    a.q4 = c * c * c * c / 24.0;
  } else if (mode == GK_MODE_DIRECT && k_im != 0.0) {
    att = 2;
    if (!(k_im < 0.0)) fail(GK_ERR_INVALID_ARGUMENT, "lossy medium needs Im k < 0 (attenuation)");
    // radii are bounded by the mesh's bounding-box diagonal
    const double xmax = -k_im * mesh->diameter * kAttenScale;
    if (!(xmax < 8000.0))
      fail(GK_ERR_INVALID_ARGUMENT, "lossy fill: attenuation exp(Im k r) range too large for the device table");
    a.natten = static_cast<int>(xmax) + 3;
    a.KA = -k_im * kAttenScale;
    atten.alloc(a.natten, ctx->stream);
    atten_kernel<<<(a.natten + 255) / 256, 256, 0, ctx->stream>>>(atten.p, a.natten);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    a.atten = atten.p;
  }
  // shared edges (edges.cu) pay where the blocks share most edges (closed
  // meshes) and are small against the mesh (N >= 4096: on C2, 1280 triangles
  // in 6 blocks, most tiles are near and the fill is 1.4x slower); n = 1..5,
  // lossless or with the phase-coupled attenuation (its ahi entries, <= 512
  // for every kind so that the fused pair stays bitwise equal to the
  // separate fills, fit beside the edge sums)
  // table mode (K3e): far pairs are >= max(r_far, r_min) apart, so they
  // never fall back below the table (the fallback counts stay the
  // reference's); a far pair above r_max is still detected (the fill fails
  // with out_of_range as the reference's does, its count then covering the
  // shared evaluations).
  // opts.shared_edges = 0 keeps the per-triangle kernels; 1 takes the shared
  // edges for any mesh size
  const bool forced = opts.shared_edges == 1;
  const bool table_edges = mode == GK_MODE_TABLE && table;
  if ((mode == GK_MODE_DIRECT || table_edges) && opts.shared_edges != 0 &&
      mesh->es.nblk > 0 && mesh->es.edge_ratio < 0.85 && mesh->n <= 5 &&
      mesh->es.r_far < 0.25 * mesh->diameter &&  // else few far tiles (e.g. coordinates far from the origin)
      (att == 0 || (att == 1 && a.nhi <= 512)) && (mesh->N >= 4096 || forced)) {
    a.eblk = mesh->es.eblk.p;
    a.ep = mesh->es.ep.p;
    a.ecol = mesh->es.ecol.p;
    a.nblk = mesh->es.nblk;
    a.ecap = mesh->es.ecap;
    // table mode: far pairs must also stay >= r_min (no fallback there)
    a.r_far = table_edges ? std::fmax(mesh->es.r_far, table->dev.r_min) : mesh->es.r_far;
  }
  // the table sweep (K3s, fill_sweep.cuh): degree 3 (or the linear Exp
  // kind), the mesh's small-block set under the same conditions as K3e;
  // launch_one decides whether the window fits
  const int degree = table ? table->dev.degree : 3;
  const EdgeSet& sw = mesh->sweep;
  if (table_edges && a.nblk > 0 && sw.nblk > 0 && table->dev.nbase > 0 &&
      (degree == 3 || kind == GK_KIND_EXP) && opts.table_placement != GK_TABLE_GLOBAL &&
      opts.table_placement != GK_TABLE_SHARED) {
    a.s_eblk = sw.eblk.p;
    a.s_ep = sw.ep.p;
    a.s_ecol = sw.ecol.p;
    a.s_nblk = sw.nblk;
    a.s_ecap = sw.ecap;
    a.s_rho_max = sw.rho_max;
    a.s_rho_rows = mesh->rho_outer_max * (1.0 + 1e-12);
    a.s_rc = kSweepRowsPerCluster;
    if (mesh->srows.n < mesh->N || mesh->srows_begin != row_begin || mesh->srows_end != row_end) {
      if (mesh->srows.n < mesh->N) mesh->srows.alloc(mesh->N, ctx->stream);
      sweep_rows_kernel<<<1, 1024, 0, ctx->stream>>>(sw.ecol.p, mesh->N, row_begin, row_end,
                                                     mesh->srows.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
      mesh->srows_begin = row_begin;
      mesh->srows_end = row_end;
    }
    a.s_rows = mesh->srows.p;
  }
  switch (mesh->m) {
    case 1: return dispatch_mo<1>(ctx, a, mode, kind, degree, att, opts);
    case 3: return dispatch_mo<3>(ctx, a, mode, kind, degree, att, opts);
    case 4: return dispatch_mo<4>(ctx, a, mode, kind, degree, att, opts);
    case 6: return dispatch_mo<6>(ctx, a, mode, kind, degree, att, opts);
    case 7: return dispatch_mo<7>(ctx, a, mode, kind, degree, att, opts);
    default: fail(GK_ERR_INVALID_ARGUMENT, "QuadratureSpec: outer_points must be one of 1, 3, 4, 6, 7");
  }
}

// lossy_phase_kernel: tab[lo] = (cos, sin)(2 pi lo / M) exp(c lo) and
// ahi[h] = exp(c M h), c = k_im / K1 (cis_phase_att)
__global__ void lossy_phase_kernel(double2* tab, double* ahi, int nhi, double c) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < kPhaseSlots) {  // slot i holds angle index i >> kPhaseCopyLog2
    const int lo = i >> kPhaseCopyLog2;
    double s, co;
    sincospi(2.0 * lo / kPhaseM, &s, &co);
    const double e = exp(c * lo);
    tab[i] = make_double2(co * e, s * e);
  }
  if (i < nhi) ahi[i] = exp(c * (static_cast<double>(kPhaseM) * i));
}

__global__ void atten_kernel(double* E, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) E[i] = exp(-static_cast<double>(i) / kAttenScale);
}

// ------------------------------------------------------------------- K1

__device__ __forceinline__ unsigned long long bits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double unbits(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}

__device__ __forceinline__ void reduce_minmax(double lo, double hi, unsigned long long* wmin,
                                              unsigned long long* wmax) {
  unsigned long long l = bits(lo), h = bits(hi);  // non-negative: bit order == value order
  for (int o = 16; o; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, l, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, h, o);
    l = l2 < l ? l2 : l;
    h = h2 > h ? h2 : h;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(wmin, l);
    atomicMax(wmax, h);
  }
}

// pass 1: one sample pair distance (outer 0, inner 0) per (p, q): an upper
// bound of the true min and a lower bound of the true max
__global__ void range_sample_kernel(const double4* outer, const double4* inner, int m, size_t N,
                                    size_t row_begin, size_t row_end, unsigned long long* w) {
  double lo = CUDART_INF, hi = 0.0;
  for (size_t p = row_begin + blockIdx.x; p < row_end; p += gridDim.x) {
    const double4 o = outer[p * m];
    for (size_t q = threadIdx.x; q < N; q += blockDim.x) {
      if (q == p) continue;
      const double4 I = inner[q];
      const double d2 = dist2(o.x, o.y, o.z, I.x, I.y, I.z);
      lo = fmin(lo, d2);
      hi = fmax(hi, d2);
    }
  }
  reduce_minmax(lo, hi, w + 0, w + 1);
}

// pass 2: exact min/max over the pairs whose centroid bounds can beat the
// samples: |c_p - c_q| - rho_p - rho_q <= m0  or  |c_p - c_q| + rho_p + rho_q >= M0
__global__ void range_exact_kernel(const double4* outer, const double4* inner,
                                   const double4* bounds, const double* binner, int m, int ipt,
                                   size_t N, size_t row_begin, size_t row_end,
                                   unsigned long long* w) {
  const double m0 = sqrt(unbits(w[0])), M0 = sqrt(unbits(w[1]));
  double lo = CUDART_INF, hi = 0.0;
  for (size_t p = row_begin + blockIdx.x; p < row_end; p += gridDim.x) {
    const double4 bp = bounds[p];
    for (size_t q = threadIdx.x; q < N; q += blockDim.x) {
      if (q == p) continue;
      const double4 bq = bounds[q];
      const double dx = bp.x - bq.x, dy = bp.y - bq.y, dz = bp.z - bq.z;
      const double dc2 = dx * dx + dy * dy + dz * dz;
      const double rho = bp.w + binner[q];
      const double a = m0 + rho, b = M0 - rho;
      const bool cmin = dc2 <= a * a * (1.0 + 1e-12);
      const bool cmax = b <= 0.0 || dc2 >= b * b * (1.0 - 1e-12);
      if (!(cmin || cmax)) continue;
      for (int o = 0; o < m; ++o) {
        const double4 O = outer[p * m + o];
        for (int i = 0; i < ipt; ++i) {
          const double4 I = inner[static_cast<size_t>(i) * N + q];
          const double d2 = dist2(O.x, O.y, O.z, I.x, I.y, I.z);
          lo = fmin(lo, d2);
          hi = fmax(hi, d2);
        }
      }
    }
  }
  reduce_minmax(lo, hi, w + 2, w + 3);
}

void launch_range(gk_ctx* ctx, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                  double* d2min, double* d2max) {
  cudaStream_t st = ctx->stream;
  unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  unsigned long long* w = ctx->scratch.p + 8;
  GK_CUDA(cudaMemcpyAsync(w, init, sizeof(init), cudaMemcpyHostToDevice, st));
  const size_t rows = row_end - row_begin;
  const unsigned grid = static_cast<unsigned>(rows < 65535 ? rows : 65535);
  range_sample_kernel<<<grid, 256, 0, st>>>(mesh->outer.p, mesh->inner.p, mesh->m, mesh->N,
                                            row_begin, row_end, w);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  range_exact_kernel<<<grid, 256, 0, st>>>(mesh->outer.p, mesh->inner.p, mesh->bounds.p,
                                           mesh->binner.p, mesh->m, 3 * mesh->n, mesh->N,
                                           row_begin, row_end, w);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  unsigned long long out[4];
  GK_CUDA(cudaMemcpyAsync(out, w, sizeof(out), cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  const unsigned long long lo = out[0] < out[2] ? out[0] : out[2];
  const unsigned long long hi = out[1] > out[3] ? out[1] : out[3];
  double a, b;
  std::memcpy(&a, &lo, 8);
  std::memcpy(&b, &hi, 8);
  *d2min = a;
  *d2max = b;
}

// {min d2, -max d2} of a rank's rows as two doubles on the device (the
// 16 bytes the multi-GPU range all-reduces with MIN, comm.cu)
__global__ void range_pack_kernel(const unsigned long long* w, double* out2) {
  const unsigned long long lo = w[0] < w[2] ? w[0] : w[2];
  const unsigned long long hi = w[1] > w[3] ? w[1] : w[3];
  out2[0] = unbits(lo);
  out2[1] = -unbits(hi);
}

void launch_range_device(gk_ctx* ctx, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                         double* out2) {
  cudaStream_t st = ctx->stream;
  if (row_end <= row_begin) {  // no rows: the identity of the MIN reduction
    const double id[2] = {INFINITY, -0.0};
    GK_CUDA(cudaMemcpyAsync(out2, id, sizeof(id), cudaMemcpyHostToDevice, st));
    GK_CUDA(cudaStreamSynchronize(st));  // `id` is a host stack buffer
    return;
  }
  unsigned long long init[4] = {~0ull, 0ull, ~0ull, 0ull};
  unsigned long long* w = ctx->scratch.p + 8;
  GK_CUDA(cudaMemcpyAsync(w, init, sizeof(init), cudaMemcpyHostToDevice, st));
  const size_t rows = row_end - row_begin;
  const unsigned grid = static_cast<unsigned>(rows < 65535 ? rows : 65535);
  range_sample_kernel<<<grid, 256, 0, st>>>(mesh->outer.p, mesh->inner.p, mesh->m, mesh->N,
                                            row_begin, row_end, w);
  range_exact_kernel<<<grid, 256, 0, st>>>(mesh->outer.p, mesh->inner.p, mesh->bounds.p,
                                           mesh->binner.p, mesh->m, 3 * mesh->n, mesh->N,
                                           row_begin, row_end, w);
  range_pack_kernel<<<1, 1, 0, st>>>(w, out2);
  count_launches(3);
  GK_CUDA(cudaGetLastError());
  // `init` is read by the copy engine before this frame returns
  GK_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------- phase table

// tab[slot] = (cos, sin)(2 pi (slot >> copy_log2) / M)
__global__ void phase_kernel(double2* tab, int M, int copy_log2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (M << copy_log2)) return;
  double s, c;
  sincospi(2.0 * (i >> copy_log2) / M, &s, &c);
  tab[i] = make_double2(c, s);
}

void init_phase_table(gk_ctx* ctx) {
  ctx->phase.alloc(kPhaseSlots, ctx->stream);
  phase_kernel<<<(kPhaseSlots + 255) / 256, 256, 0, ctx->stream>>>(ctx->phase.p, kPhaseM,
                                                                    kPhaseCopyLog2);
  ctx->phase_small.alloc(kPhaseSmall, ctx->stream);
  phase_kernel<<<(kPhaseSmall + 255) / 256, 256, 0, ctx->stream>>>(ctx->phase_small.p,
                                                                  kPhaseSmall, 0);
  count_launches(2);
  GK_CUDA(cudaGetLastError());
}

}  // namespace gk
