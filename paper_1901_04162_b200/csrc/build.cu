// build.cu -- K0 quadrature points and K2 device table build.
//
// Compiled with -fmad=false: every expression here must round exactly like
// the reference's x86-64 build (no FMA contraction), so that
//   * quadrature points equal detail::outer_points / inner_points
//     (matfill.hpp:105-133) bit for bit, and
//   * the sampling plan and the reference-format hash equal build_plan /
//     build_hash (sampling.hpp:149-236, table.hpp:54-82) bit for bit.
// The lookup structures derived from them (gk_device.cuh) use explicit
// __fma_rn/__dadd_rd intrinsics, identical under either flag.
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cfloat>
#include <cmath>
#include <cstring>

#include "gk_internal.h"

namespace gk {

// ------------------------------------------------------------ quadrature

struct QuadConst {
  int m, n;
  double b0[7], b1[7], b2[7], w[7];
  double gx[32], gw[32];
};

__global__ void points_kernel(const double* __restrict__ V, const uint32_t* __restrict__ T,
                              size_t N, QuadConst q, double4* __restrict__ outer,
                              double4* __restrict__ inner, double4* __restrict__ bounds,
                              double* __restrict__ binner) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= N) return;
  const uint32_t t[3] = {T[3 * i], T[3 * i + 1], T[3 * i + 2]};
  double vx[3], vy[3], vz[3];
  for (int c = 0; c < 3; ++c) {
    vx[c] = V[3 * static_cast<size_t>(t[c])];
    vy[c] = V[3 * static_cast<size_t>(t[c]) + 1];
    vz[c] = V[3 * static_cast<size_t>(t[c]) + 2];
  }
  // TriangleMesh::triangle_area (mesh.hpp:39-44)
  const double e1x = vx[1] - vx[0], e1y = vy[1] - vy[0], e1z = vz[1] - vz[0];
  const double e2x = vx[2] - vx[0], e2y = vy[2] - vy[0], e2z = vz[2] - vz[0];
  const double cx = e1y * e2z - e1z * e2y;
  const double cy = e1z * e2x - e1x * e2z;
  const double cz = e1x * e2y - e1y * e2x;
  const double area = 0.5 * sqrt(cx * cx + cy * cy + cz * cz);
  // centroid only feeds K1's conservative pair bounds
  const double gxc = (vx[0] + vx[1] + vx[2]) / 3.0;
  const double gyc = (vy[0] + vy[1] + vy[2]) / 3.0;
  const double gzc = (vz[0] + vz[1] + vz[2]) / 3.0;
  double rho_o = 0.0, rho_i = 0.0;
  // outer_points (matfill.hpp:105-119): a*b0 + b*b1 + c*b2, weight w*area
  for (int o = 0; o < q.m; ++o) {
    const double px = vx[0] * q.b0[o] + vx[1] * q.b1[o] + vx[2] * q.b2[o];
    const double py = vy[0] * q.b0[o] + vy[1] * q.b1[o] + vy[2] * q.b2[o];
    const double pz = vz[0] * q.b0[o] + vz[1] * q.b1[o] + vz[2] * q.b2[o];
    outer[i * q.m + o] = make_double4(px, py, pz, q.w[o] * area);
    const double dx = px - gxc, dy = py - gyc, dz = pz - gzc;
    rho_o = fmax(rho_o, sqrt(dx * dx + dy * dy + dz * dz));
  }
  // inner_points (matfill.hpp:121-133): a + (b-a)*x on edges v0v1, v1v2, v2v0
  for (int e = 0; e < 3; ++e) {
    const int a = e, b = (e + 1) % 3;
    const double lx = vx[a] - vx[b], ly = vy[a] - vy[b], lz = vz[a] - vz[b];
    const double len = sqrt(lx * lx + ly * ly + lz * lz);
    for (int g = 0; g < q.n; ++g) {
      const double px = vx[a] + (vx[b] - vx[a]) * q.gx[g];
      const double py = vy[a] + (vy[b] - vy[a]) * q.gx[g];
      const double pz = vz[a] + (vz[b] - vz[a]) * q.gx[g];
      inner[static_cast<size_t>(e * q.n + g) * N + i] = make_double4(px, py, pz, q.gw[g] * len);
      const double dx = px - gxc, dy = py - gyc, dz = pz - gzc;
      rho_i = fmax(rho_i, sqrt(dx * dx + dy * dy + dz * dz));
    }
  }
  bounds[i] = make_double4(gxc, gyc, gzc, rho_o * (1.0 + 1e-12) + 1e-300);
  binner[i] = rho_i * (1.0 + 1e-12) + 1e-300;
}

void launch_points(gk_mesh* mesh, const double* d_verts, const uint32_t* d_tris, cudaStream_t s) {
  QuadConst q{};
  q.m = mesh->m;
  q.n = mesh->n;
  triangle_rule(mesh->m, q.b0, q.b1, q.b2, q.w);
  gauss_legendre_unit(mesh->n, q.gx, q.gw);
  const int threads = 128;
  const unsigned blocks = static_cast<unsigned>((mesh->N + threads - 1) / threads);
  points_kernel<<<blocks, threads, 0, s>>>(d_verts, d_tris, mesh->N, q, mesh->outer.p,
                                           mesh->inner.p, mesh->bounds.p, mesh->binner.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
}

// max_vertex_distance (mesh.hpp:62-68): thread i scans j > i; |a - b|^2 in the
// reference's order (dot(a - b, a - b), no contraction: this unit is built
// with -fmad=false) and one correctly rounded sqrt of the maximum on the host
// side reproduce max_ij sqrt(.) exactly (sqrt is monotone).  Vertices j are
// staged through shared memory in tiles.
__global__ void max_vertex_d2_kernel(const double* __restrict__ V, size_t nv,
                                     unsigned long long* __restrict__ out) {
  __shared__ double tx[256], ty[256], tz[256];
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double ax = 0.0, ay = 0.0, az = 0.0;
  if (i < nv) {
    ax = V[3 * i];
    ay = V[3 * i + 1];
    az = V[3 * i + 2];
  }
  double best = 0.0;
  const size_t first = blockIdx.x * static_cast<size_t>(blockDim.x);  // j > i >= first
  for (size_t j0 = first; j0 < nv; j0 += 256) {
    __syncthreads();
    const size_t jl = j0 + threadIdx.x;
    if (jl < nv) {
      tx[threadIdx.x] = V[3 * jl];
      ty[threadIdx.x] = V[3 * jl + 1];
      tz[threadIdx.x] = V[3 * jl + 2];
    }
    __syncthreads();
    const size_t cnt = nv - j0 < 256 ? nv - j0 : 256;
    if (i < nv)
      for (size_t t = 0; t < cnt; ++t) {
        if (j0 + t <= i) continue;
        const double dx = ax - tx[t], dy = ay - ty[t], dz = az - tz[t];
        const double d2 = dx * dx + dy * dy + dz * dz;
        best = best < d2 ? d2 : best;
      }
  }
  for (int o = 16; o; o >>= 1) {
    const double v = __shfl_xor_sync(0xffffffffu, best, o);
    best = best < v ? v : best;
  }
  if ((threadIdx.x & 31) == 0 && best > 0.0)
    atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(best)));
}

void launch_max_vertex_d2(const double* verts, size_t nv, unsigned long long* d2_bits,
                          cudaStream_t s) {
  const unsigned blocks = static_cast<unsigned>((nv + 255) / 256);
  if (blocks == 0) return;
  max_vertex_d2_kernel<<<blocks, 256, 0, s>>>(verts, nv, d2_bits);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
}

// arithmetic locate (TableDev::coarse): for run c, base points 64 c .. 64 c + 64
// (r_min + i t_eff, this unit has no FMA contraction, so the values are the
// plan's bits) must be consecutive plan nodes; verified by exact search
__global__ void coarse_runs_kernel(const double* __restrict__ absc, size_t n, double r_min,
                                   double t_eff, uint32_t ncoarse, int32_t* __restrict__ coarse) {
  const size_t c = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (c >= ncoarse) return;
  long long first = -1;
  for (int k = 0; k <= 64; ++k) {
    const long long i = static_cast<long long>(c) * 64 + k;
    const double a = r_min + static_cast<double>(i) * t_eff;
    size_t lo = 0, hi = n;  // lower bound of a
    while (lo < hi) {
      const size_t mid = (lo + hi) / 2;
      if (absc[mid] < a) lo = mid + 1;
      else hi = mid;
    }
    if (lo >= n || absc[lo] != a) {
      coarse[c] = -1;
      return;
    }
    if (k == 0) first = static_cast<long long>(lo);
    else if (static_cast<long long>(lo) != first + k) {
      coarse[c] = -1;
      return;
    }
  }
  coarse[c] = static_cast<int32_t>(first - static_cast<long long>(c) * 64);
}

// table sweep (TableDev::bg / be / bclean): b2p[i] = plan index of base
// point i (r_min + i t_eff, rounded like build_plan, sampling.hpp:212-213) or
// -1, and its node values
__global__ void base_nodes_kernel(const double* __restrict__ absc, size_t n, double r_min,
                                  double t_eff, long long nbase, const double2* __restrict__ ev,
                                  const double2* __restrict__ gv, int32_t* __restrict__ b2p,
                                  double2* __restrict__ bg, double2* __restrict__ be) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nbase;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double a = r_min + static_cast<double>(i) * t_eff;
    size_t lo = 0, hi = n;  // lower bound of a
    while (lo < hi) {
      const size_t mid = (lo + hi) / 2;
      if (absc[mid] < a) lo = mid + 1;
      else hi = mid;
    }
    const bool hit = lo < n && absc[lo] == a;
    b2p[i] = hit ? static_cast<int32_t>(lo) : -1;
    bg[i] = hit ? gv[lo] : make_double2(0.0, 0.0);
    be[i] = hit ? ev[lo] : make_double2(0.0, 0.0);
  }
}

// bit k of word w: base interval i = 32 w + k has the reference's degree-3
// stencil (start j - 1, evaluator.hpp:49-51, 251-252) on base points
// i-1 .. i+2 as consecutive plan nodes j-1 .. j+2; zero padding past nbase
__global__ void base_clean_kernel(const int32_t* __restrict__ b2p, long long nbase,
                                  uint32_t nwords, uint32_t* __restrict__ bits) {
  const uint32_t w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= nwords) return;
  uint32_t word = 0;
  for (int k = 0; k < 32; ++k) {
    const long long i = 32LL * w + k;
    if (i < 1 || i + 2 >= nbase) continue;
    const int32_t j0 = b2p[i - 1];
    if (j0 >= 0 && b2p[i] == j0 + 1 && b2p[i + 1] == j0 + 2 && b2p[i + 2] == j0 + 3)
      word |= 1u << k;
  }
  bits[w] = word;
}

// patch flags: every plan interval j overlapping a base interval i whose
// clean bit is clear (i = 0 .. nbase-2), or the tail [a_{nbase-1}, r_max]
// (i = nbase-1, with the r_max sentinel n-1), gets flag[j] = 1
__global__ void patch_flag_kernel(const double* __restrict__ absc, size_t n, double r_min,
                                  double t_eff, double r_max, long long nbase,
                                  const uint32_t* __restrict__ bits, uint8_t* __restrict__ flag) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < nbase;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const bool tail = i == nbase - 1;
    if (!tail && ((bits[i >> 5] >> (i & 31)) & 1u)) continue;
    const double lo = r_min + static_cast<double>(i) * t_eff;
    const double hi = tail ? r_max : r_min + static_cast<double>(i + 1) * t_eff;
    // jl: the last node <= lo (the interval holding lo); jh: the last node < hi
    size_t a = 0, b = n;
    while (a < b) {
      const size_t mid = (a + b) / 2;
      if (absc[mid] <= lo) a = mid + 1;
      else b = mid;
    }
    const size_t jl = a > 0 ? a - 1 : 0;
    a = jl;
    b = n;
    while (a < b) {
      const size_t mid = (a + b) / 2;
      if (absc[mid] < hi) a = mid + 1;
      else b = mid;
    }
    const size_t jh = a > 0 ? a - 1 : 0;
    for (size_t j = jl; j <= jh && j < n; ++j) flag[j] = 1;
    if (tail) flag[n - 1] = 1;
  }
}

__global__ void patch_left_kernel(const double* __restrict__ absc, const uint32_t* __restrict__ pj,
                                  const int* __restrict__ np, double* __restrict__ pa) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < *np; k += gridDim.x * blockDim.x)
    pa[k] = absc[pj[k]];
}

// ---------------------------------------------------------- plan (K2)

struct PlanScalars {
  double r_min, r_max, t_eff, refined, keep_gap, qp;
  long long steps;
  int side_steps, refine;
  long long n_lo, ncand;  // zero candidates n in [n_lo, n_lo + ncand)
};

// scratch words (unsigned long long) used by the build
enum : int {
  W_NZ = 0,        // valid zeros
  W_NKZ,           // kept (inserted) zeros
  W_ZMIN,          // a zero equals r_min (merged)
  W_ZMAX,          // a zero equals r_max (merged)
  W_GAPMIN,        // min gap bits
  W_GAPMAX,        // max gap bits
  W_BAD,           // non-increasing abscissae / >1 node per lookup bucket
  W_COUNT
};

// zero_crossings (sampling.hpp:127-141) and the zero pass of the priority
// insertion (sampling.hpp:210-211): zeros are > keep_gap apart, so each one
// only meets the endpoints.  Sequential: a few hundred iterations.
__global__ void zeros_kernel(PlanScalars S, double* zeros, double* kept_zeros,
                             unsigned long long* w) {
  unsigned long long nz = 0, nkz = 0, zmin = 0, zmax = 0;
  for (long long c = 0; c < S.ncand; ++c) {
    const double z = static_cast<double>(S.n_lo + c) * S.qp;
    if (z > S.r_max) break;
    if (!(z >= S.r_min)) continue;
    zeros[nz++] = z;
    if (z == S.r_min) { zmin = 1; continue; }  // lower_bound hits r_min: merge
    if (z == S.r_max) { zmax = 1; continue; }  // merge into r_max
    if (S.r_max - z < S.keep_gap) continue;    // next (r_max) too close
    if (z - S.r_min < S.keep_gap) continue;    // prev (r_min) too close
    kept_zeros[nkz++] = z;
  }
  w[W_NZ] = nz;
  w[W_NKZ] = nkz;
  w[W_ZMIN] = zmin;
  w[W_ZMAX] = zmax;
}

__device__ __forceinline__ long long lower_bound_d(const double* a, long long n, double x) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = lo + (hi - lo) / 2;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// try_insert outcome against the neighbours found so far (sampling.hpp:195-206)
struct Nbr {
  double next, prev;
  bool equal;
  __device__ void see(double v, double r) {
    if (v == r) equal = true;
    else if (v > r) next = v < next ? v : next;
    else prev = v > prev ? v : prev;
  }
  __device__ bool keep(double r, double keep_gap) const {
    if (equal) return false;
    if (next - r < keep_gap) return false;
    if (r - prev < keep_gap) return false;
    return true;
  }
};

__device__ __forceinline__ void see_zeros(Nbr& nb, const double* kz, long long nkz, double r) {
  const long long pos = lower_bound_d(kz, nkz, r);
  if (pos < nkz) nb.see(kz[pos], r);
  if (pos > 0) nb.see(kz[pos - 1], r);
}

// base grid pass (sampling.hpp:212-213): kept unless an endpoint or a kept
// zero is within keep_gap (earlier base points are > t_eff > keep_gap away)
__global__ void base_kernel(PlanScalars S, const double* kz, const unsigned long long* w,
                            double* vals, uint8_t* keep) {
  const long long nkz = static_cast<long long>(w[W_NKZ]);
  for (long long i = 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       i < S.steps; i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double g = S.r_min + static_cast<double>(i) * S.t_eff;
    vals[i] = g;
    if (!S.refine) {
      keep[i] = 1;
      continue;
    }
    Nbr nb{S.r_max, S.r_min, false};
    see_zeros(nb, kz, nkz, g);
    keep[i] = nb.keep(g, S.keep_gap) ? 1 : 0;
  }
}

// refined pass (sampling.hpp:214-220): candidates z -/+ s*refined of every
// zero, kept unless a kept point of a stronger class is within keep_gap
// (windows of different zeros are disjoint on this path, checked on the host)
__global__ void refined_kernel(PlanScalars S, const double* zeros, const double* kz,
                               const unsigned long long* w, const uint8_t* base_keep,
                               double* vals, uint8_t* keep) {
  const long long nz = static_cast<long long>(w[W_NZ]);
  const long long nkz = static_cast<long long>(w[W_NKZ]);
  const long long per_zero = 2LL * S.side_steps;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
       c < nz * per_zero; c += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long zi = c / per_zero;
    const int rem = static_cast<int>(c % per_zero);
    const int s = rem / 2 + 1;
    const bool plus = rem & 1;
    const double z = zeros[zi];
    const double off = static_cast<double>(s) * S.refined;
    const double r = plus ? z + off : z - off;
    const bool in_range = plus ? (r < S.r_max) : (r > S.r_min);
    vals[c] = r;
    if (!in_range) {
      keep[c] = 0;
      continue;
    }
    Nbr nb{S.r_max, S.r_min, false};
    see_zeros(nb, kz, nkz, r);
    const long long ic = static_cast<long long>(floor((r - S.r_min) / S.t_eff));
    for (long long i = ic - 1; i <= ic + 2; ++i) {
      if (i < 1 || i >= S.steps || !base_keep[i]) continue;
      nb.see(S.r_min + static_cast<double>(i) * S.t_eff, r);
    }
    keep[c] = nb.keep(r, S.keep_gap) ? 1 : 0;
  }
}

// The exact priority insertion of build_plan (sampling.hpp:194-220) on one
// thread, for configurations whose refinement windows may interact
// (qp < 2 side_steps refined + margin): small plans only.
__global__ void plan_sequential_kernel(PlanScalars S, const double* zeros,
                                       const unsigned long long* w, double* kept, uint8_t* isz,
                                       unsigned long long* out_n) {
  const long long nz = static_cast<long long>(w[W_NZ]);
  long long n = 2;
  kept[0] = S.r_min;
  kept[1] = S.r_max;
  isz[0] = isz[1] = 0;
  auto try_insert = [&](double r, uint8_t is_zero) {
    const long long it = lower_bound_d(kept, n, r);
    if (it != n) {
      if (kept[it] == r) {
        isz[it] = isz[it] || is_zero;
        return;
      }
      if (kept[it] - r < S.keep_gap) return;
    }
    if (it != 0 && r - kept[it - 1] < S.keep_gap) return;
    for (long long k = n; k > it; --k) {
      kept[k] = kept[k - 1];
      isz[k] = isz[k - 1];
    }
    kept[it] = r;
    isz[it] = is_zero;
    ++n;
  };
  for (long long i = 0; i < nz; ++i) try_insert(zeros[i], 1);
  for (long long i = 1; i < S.steps; ++i)
    try_insert(S.r_min + static_cast<double>(i) * S.t_eff, 0);
  for (long long i = 0; i < nz; ++i) {
    for (int s = 1; s <= S.side_steps; ++s) {
      const double off = static_cast<double>(s) * S.refined;
      if (zeros[i] - off > S.r_min) try_insert(zeros[i] - off, 0);
      if (zeros[i] + off < S.r_max) try_insert(zeros[i] + off, 0);
    }
  }
  *out_n = static_cast<unsigned long long>(n);
}

__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}

// consecutive gaps: min -> dr_min, max -> t (sampling.hpp:228-233)
__global__ void gaps_kernel(const double* a, long long n, unsigned long long* w) {
  unsigned long long lo = ~0ull, hi = 0ull;
  bool bad = false;
  for (long long i = 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double g = a[i] - a[i - 1];
    if (!(g > 0.0)) bad = true;
    const unsigned long long b = dbits(g);
    lo = b < lo ? b : lo;
    hi = b > hi ? b : hi;
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long l2 = __shfl_xor_sync(0xffffffffu, lo, o);
    const unsigned long long h2 = __shfl_xor_sync(0xffffffffu, hi, o);
    lo = l2 < lo ? l2 : lo;
    hi = h2 > hi ? h2 : hi;
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&w[W_GAPMIN], lo);
    atomicMax(&w[W_GAPMAX], hi);
  }
  if (bad) atomicOr(&w[W_BAD], 1ull);
}

// build_hash seed pass (table.hpp:74-78): greatest j wins a shared bucket
__global__ void hash_seed_kernel(const double* a, long long n, double r_min, double dr_min,
                                 double inv_dr_min, unsigned long long nb, uint32_t* buckets) {
  for (long long j = 1 + blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    unsigned long long b = static_cast<unsigned long long>((a[j] - r_min) * inv_dr_min);
    if (r_min + static_cast<double>(b) * dr_min < a[j]) ++b;
    if (b < nb) atomicMax(&buckets[b], static_cast<uint32_t>(j));
  }
}

struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const {
    return a < b ? b : a;
  }
};

// KernelTable values (table.hpp:24-34) via device sincos (+ lossy extension)
__global__ void values_kernel(const double* a, long long n, double k_re, double k_im,
                              double2* ev, double2* gv) {
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double r = a[j];
    ev[j] = analytic_sincos(0, k_re, k_im, r);
    gv[j] = analytic_sincos(1, k_re, k_im, r);
  }
}

// Interval records (see gk_device.cuh).  Green: coefficients of the
// degree-d Lagrange interpolant on the reference's stencil (start =
// clamp(j - (d-1)/2, 0, n-d-1), evaluator.hpp:49-51) expanded around a_j.
__global__ void records_kernel(const double* a, long long n, const double2* ev, const double2* gv,
                               int d, double* grec, double* erec) {
  const int grs = 2 + 2 * (d + 1);
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    double* g = grec + j * grs;
    double* e = erec + j * 6;
    const double aj = a[j];
    const double an = j + 1 < n ? a[j + 1] : CUDART_INF;
    g[0] = aj;
    g[1] = an;
    e[0] = aj;
    e[1] = an;
    if (j == n - 1) {  // sentinel: r == r_max reproduces the last node
      for (int k = 2; k < grs; ++k) g[k] = 0.0;
      g[2] = gv[j].x;
      g[3] = gv[j].y;
      e[2] = ev[j].x;
      e[3] = ev[j].y;
      e[4] = 0.0;
      e[5] = 0.0;
      continue;
    }
    // Exp, linear: e_j + u (e_{j+1} - e_j) / (a_{j+1} - a_j)
    const double h = an - aj;
    e[2] = ev[j].x;
    e[3] = ev[j].y;
    e[4] = (ev[j + 1].x - ev[j].x) / h;
    e[5] = (ev[j + 1].y - ev[j].y) / h;
    // Green, degree d
    const long long back = (d - 1) / 2;
    long long s = j > back ? j - back : 0;
    if (s + d + 1 > n) s = n - d - 1;
    double y[8];
    for (int q = 0; q <= d; ++q) y[q] = a[s + q] - aj;
    double cr[8] = {0}, ci[8] = {0};
    for (int q = 0; q <= d; ++q) {
      // N_q(u) = prod_{b != q} (u - y_b), D_q = prod_{b != q} (y_q - y_b)
      double poly[8] = {1.0, 0, 0, 0, 0, 0, 0, 0};
      int deg = 0;
      double den = 1.0;
      for (int b = 0; b <= d; ++b) {
        if (b == q) continue;
        for (int k = deg + 1; k >= 1; --k) poly[k] = poly[k - 1] - y[b] * poly[k];
        poly[0] = -y[b] * poly[0];
        ++deg;
        den *= y[q] - y[b];
      }
      const double fr = gv[s + q].x / den, fi = gv[s + q].y / den;
      for (int k = 0; k <= d; ++k) {
        cr[k] += fr * poly[k];
        ci[k] += fi * poly[k];
      }
    }
    cr[0] = gv[j].x;  // exact node value at u = 0
    ci[0] = gv[j].y;
    for (int k = 0; k <= d; ++k) {
      g[2 + 2 * k] = cr[k];
      g[3 + 2 * k] = ci[k];
    }
  }
}

// lookup buckets: count nodes per bucket (must be <= 1), then exclusive scan
__global__ void lookup_count_kernel(const double* a, long long n, TableDev t, uint32_t* cnt,
                                    unsigned long long* w) {
  for (long long j = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; j < n;
       j += static_cast<long long>(gridDim.x) * blockDim.x) {
    const uint32_t b = lookup_bucket(a[j], t);
    if (atomicAdd(&cnt[b], 1u) != 0u) atomicOr(&w[W_BAD], 2ull);
  }
}

__global__ void lookup_finish_kernel(const uint32_t* excl, uint32_t nlk, uint32_t* lk) {
  for (uint32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < nlk; b += gridDim.x * blockDim.x)
    lk[b] = excl[b] > 0 ? excl[b] - 1 : 0;
}

// ------------------------------------------------------------ orchestration

namespace {

unsigned grid_for(long long n, int threads = 256) {
  long long b = (n + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 4096) b = 4096;
  return static_cast<unsigned>(b);
}

double from_bits(unsigned long long b) {
  double d;
  std::memcpy(&d, &b, 8);
  return d;
}

}  // namespace

void build_table_device(gk_ctx* ctx, gk_table* t, const gk_sampling_config& cfg, double k_zero,
                        double t_nominal, double k_re, double k_im, int degree) {
  cudaStream_t st = ctx->stream;
  GK_CUDA(cudaEventRecord(ctx->ev0, st));

  // scalar prologue (sampling.hpp:150-193), IEEE double on the host
  PlanScalars S{};
  S.r_min = cfg.r_min;
  S.r_max = cfg.r_max;
  const double span = cfg.r_max - cfg.r_min;
  if (!(span >= 2.0 * t_nominal))
    fail(GK_ERR_INVALID_ARGUMENT, "build_plan: range must cover at least two base intervals");
  const double steps_d = std::ceil(span / t_nominal);
  if (!(steps_d < 2.0e9))
    fail(GK_ERR_INVALID_ARGUMENT, "build_plan: plan too large for the device table");
  S.steps = static_cast<long long>(steps_d);
  S.t_eff = span / static_cast<double>(S.steps);
  S.refine = cfg.refine ? 1 : 0;
  S.refined = S.t_eff / static_cast<double>(cfg.refine_interval_divisor);
  const double min_gap = cfg.dedup_fraction * S.refined;
  S.side_steps =
      static_cast<int>(std::floor(cfg.refine_halfwidth_in_t * cfg.refine_interval_divisor + 1e-9));
  S.keep_gap = min_gap - 8.0 * DBL_EPSILON * cfg.r_max;
  S.qp = kPi / (2.0 * k_zero);
  long long n_lo = static_cast<long long>(std::floor(cfg.r_min / S.qp));
  if (n_lo < 1) n_lo = 1;
  S.n_lo = n_lo;
  S.ncand = S.refine ? static_cast<long long>(std::floor(cfg.r_max / S.qp)) - n_lo + 3 : 0;
  if (S.ncand < 0) S.ncand = 0;
  if (S.ncand > (1LL << 24))
    fail(GK_ERR_INVALID_ARGUMENT, "build_plan: too many kernel zeros in range for the device plan");

  DevBuf<unsigned long long> w;
  w.alloc(W_COUNT, st);
  GK_CUDA(cudaMemsetAsync(w.p, 0, w.bytes(), st));
  const unsigned long long init_min = ~0ull;
  GK_CUDA(cudaMemcpyAsync(w.p + W_GAPMIN, &init_min, 8, cudaMemcpyHostToDevice, st));

  DevBuf<double> zeros, kz;
  zeros.alloc(static_cast<size_t>(S.ncand) + 1, st);
  kz.alloc(static_cast<size_t>(S.ncand) + 1, st);
  if (S.refine) {
    zeros_kernel<<<1, 1, 0, st>>>(S, zeros.p, kz.p, w.p);
    count_launches(1);
  }
  GK_CUDA(cudaGetLastError());
  unsigned long long hw[W_COUNT];
  GK_CUDA(cudaMemcpyAsync(hw, w.p, sizeof(hw), cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  const long long nz = static_cast<long long>(hw[W_NZ]);
  const long long nkz = static_cast<long long>(hw[W_NKZ]);

  // windows of distinct zeros disjoint (with margin) -> class-parallel path
  const bool parallel =
      !S.refine || nz < 2 ||
      S.qp * (1.0 - 1e-9) > 2.0 * S.side_steps * S.refined + 2.0 * std::fabs(S.keep_gap) +
                                 64.0 * DBL_EPSILON * cfg.r_max;

  DevBuf<double> absc;
  long long n = 0;
  if (parallel) {
    const long long nbase = S.steps;  // index 0 unused
    const long long nref = S.refine ? nz * 2LL * S.side_steps : 0;
    DevBuf<double> cand;
    DevBuf<uint8_t> flags;
    const long long ncand_total = 2 + nkz + nbase + nref;
    cand.alloc(static_cast<size_t>(ncand_total), st);
    flags.alloc(static_cast<size_t>(ncand_total), st);
    // layout: [r_min, r_max | kept zeros | base (index 0 dummy) | refined]
    double* c_end = cand.p;
    uint8_t* f_end = flags.p;
    const double ends[2] = {cfg.r_min, cfg.r_max};
    const uint8_t ones[2] = {1, 1};
    GK_CUDA(cudaMemcpyAsync(c_end, ends, sizeof(ends), cudaMemcpyHostToDevice, st));
    GK_CUDA(cudaMemcpyAsync(f_end, ones, sizeof(ones), cudaMemcpyHostToDevice, st));
    if (nkz) {
      GK_CUDA(cudaMemcpyAsync(cand.p + 2, kz.p, nkz * sizeof(double), cudaMemcpyDeviceToDevice, st));
      GK_CUDA(cudaMemsetAsync(flags.p + 2, 1, static_cast<size_t>(nkz), st));
    }
    double* bvals = cand.p + 2 + nkz;
    uint8_t* bkeep = flags.p + 2 + nkz;
    GK_CUDA(cudaMemsetAsync(bkeep, 0, 1, st));  // index 0 is not a base point
    base_kernel<<<grid_for(nbase), 256, 0, st>>>(S, kz.p, w.p, bvals, bkeep);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    if (nref) {
      refined_kernel<<<grid_for(nref), 256, 0, st>>>(S, zeros.p, kz.p, w.p, bkeep,
                                                     bvals + nbase, bkeep + nbase);
      count_launches(1);
    }
    GK_CUDA(cudaGetLastError());
    // compact + sort (all values positive: uint64 order == double order)
    DevBuf<double> sel;
    sel.alloc(static_cast<size_t>(ncand_total), st);
    DevBuf<int> nsel;
    nsel.alloc(1, st);
    size_t tmp_bytes = 0;
    GK_CUDA(cub::DeviceSelect::Flagged(nullptr, tmp_bytes, cand.p, flags.p, sel.p, nsel.p,
                                       static_cast<int>(ncand_total), st));
    DevBuf<char> tmp;
    tmp.alloc(tmp_bytes, st);
    GK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, cand.p, flags.p, sel.p, nsel.p,
                                       static_cast<int>(ncand_total), st));
    count_launches(2);  // compact-init + select-sweep
    int nh = 0;
    GK_CUDA(cudaMemcpyAsync(&nh, nsel.p, sizeof(int), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    n = nh;
    absc.alloc(static_cast<size_t>(n), st);
    size_t sort_bytes = 0;
    auto* kin = reinterpret_cast<unsigned long long*>(sel.p);
    auto* kout = reinterpret_cast<unsigned long long*>(absc.p);
    GK_CUDA(cub::DeviceRadixSort::SortKeys(nullptr, sort_bytes, kin, kout, static_cast<int>(n), 0,
                                           64, st));
    DevBuf<char> tmp2;
    tmp2.alloc(sort_bytes, st);
    GK_CUDA(cub::DeviceRadixSort::SortKeys(tmp2.p, sort_bytes, kin, kout, static_cast<int>(n), 0,
                                           64, st));
    count_launches(10);  // histogram + exclusive-sum + 8 onesweep passes (64-bit keys)
  } else {
    const long long cap = 2 + nz + S.steps + nz * 2LL * S.side_steps;
    DevBuf<double> kept;
    DevBuf<uint8_t> isz;
    DevBuf<unsigned long long> nout;
    kept.alloc(static_cast<size_t>(cap), st);
    isz.alloc(static_cast<size_t>(cap), st);
    nout.alloc(1, st);
    plan_sequential_kernel<<<1, 1, 0, st>>>(S, zeros.p, w.p, kept.p, isz.p, nout.p);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    unsigned long long nh = 0;
    GK_CUDA(cudaMemcpyAsync(&nh, nout.p, 8, cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    n = static_cast<long long>(nh);
    absc.alloc(static_cast<size_t>(n), st);
    GK_CUDA(cudaMemcpyAsync(absc.p, kept.p, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    // zero_locations from the flags
    std::vector<uint8_t> hz(static_cast<size_t>(n));
    std::vector<double> ha(static_cast<size_t>(n));
    GK_CUDA(cudaMemcpyAsync(hz.data(), isz.p, n, cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaMemcpyAsync(ha.data(), kept.p, n * sizeof(double), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    t->zeros.clear();
    for (long long i = 0; i < n; ++i)
      if (hz[static_cast<size_t>(i)]) t->zeros.push_back(ha[static_cast<size_t>(i)]);
  }

  if (parallel) {
    // zero_locations: merged endpoints + inserted zeros, ascending
    std::vector<double> hkz(static_cast<size_t>(nkz));
    if (nkz)
      GK_CUDA(cudaMemcpyAsync(hkz.data(), kz.p, nkz * sizeof(double), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaStreamSynchronize(st));
    t->zeros.clear();
    if (hw[W_ZMIN]) t->zeros.push_back(cfg.r_min);
    t->zeros.insert(t->zeros.end(), hkz.begin(), hkz.end());
    if (hw[W_ZMAX]) t->zeros.push_back(cfg.r_max);
  }
  if (n < 2) fail(GK_ERR_INVALID_ARGUMENT, "SamplingPlan: need at least two abscissae");
  if (static_cast<long long>(degree) + 1 > n)
    fail(GK_ERR_INVALID_ARGUMENT, "KernelEvaluator: table smaller than the Lagrange stencil");

  gaps_kernel<<<grid_for(n), 256, 0, st>>>(absc.p, n, w.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  GK_CUDA(cudaMemcpyAsync(hw, w.p, sizeof(hw), cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  if (hw[W_BAD]) fail(GK_ERR_INVALID_ARGUMENT, "SamplingPlan: abscissae must be strictly increasing");
  const double dr_min = from_bits(hw[W_GAPMIN]);
  const double tmax = from_bits(hw[W_GAPMAX]);

  // reference-format hash (table.hpp:54-82)
  const double inv_dr_min = 1.0 / dr_min;
  const double nb_d = std::ceil((cfg.r_max - cfg.r_min) / dr_min) + 1.0;
  if (!(nb_d < 1.0e9)) fail(GK_ERR_INVALID_ARGUMENT, "build_hash: hash array too large");
  const unsigned long long nb = static_cast<unsigned long long>(nb_d);
  t->hash.alloc(nb, st);
  GK_CUDA(cudaMemsetAsync(t->hash.p, 0, t->hash.bytes(), st));
  hash_seed_kernel<<<grid_for(n), 256, 0, st>>>(absc.p, n, cfg.r_min, dr_min, inv_dr_min, nb,
                                                t->hash.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  {
    DevBuf<uint32_t> seeds;
    seeds.alloc(nb, st);
    GK_CUDA(cudaMemcpyAsync(seeds.p, t->hash.p, t->hash.bytes(), cudaMemcpyDeviceToDevice, st));
    size_t bytes = 0;
    GK_CUDA(cub::DeviceScan::InclusiveScan(nullptr, bytes, seeds.p, t->hash.p, MaxU32(),
                                           static_cast<int>(nb), st));
    DevBuf<char> tmp;
    tmp.alloc(bytes, st);
    GK_CUDA(cub::DeviceScan::InclusiveScan(tmp.p, bytes, seeds.p, t->hash.p, MaxU32(),
                                           static_cast<int>(nb), st));
    count_launches(2);  // scan-init + scan
  }

  // node values and interval records
  t->exp_vals.alloc(static_cast<size_t>(n), st);
  t->green_vals.alloc(static_cast<size_t>(n), st);
  values_kernel<<<grid_for(n), 256, 0, st>>>(absc.p, n, k_re, k_im, t->exp_vals.p,
                                             t->green_vals.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  const int grs = 2 + 2 * (degree + 1);
  t->grec.alloc(static_cast<size_t>(n) * grs, st);
  t->erec.alloc(static_cast<size_t>(n) * 6, st);
  records_kernel<<<grid_for(n, 128), 128, 0, st>>>(absc.p, n, t->exp_vals.p, t->green_vals.p,
                                                    degree, t->grec.p, t->erec.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());

  // lookup buckets of width dr_min / 2
  TableDev& d = t->dev;
  d.r_min = cfg.r_min;
  d.r_max = cfg.r_max;
  d.inv_w = 2.0 / dr_min;
  d.bias = -(cfg.r_min * d.inv_w) * (1.0 - 0x1p-40);
  const double xmax = std::fma(cfg.r_max, d.inv_w, d.bias);
  if (!(xmax < 2.0e9)) fail(GK_ERR_INVALID_ARGUMENT, "lookup hash too large");
  d.nlk = static_cast<uint32_t>(std::floor(xmax)) + 2u;
  t->lk.alloc(d.nlk + 4, st);  // +4: 16-byte-granular TMA windows may read past nlk
  {
    DevBuf<uint32_t> cnt;
    cnt.alloc(d.nlk, st);
    GK_CUDA(cudaMemsetAsync(cnt.p, 0, cnt.bytes(), st));
    lookup_count_kernel<<<grid_for(n), 256, 0, st>>>(absc.p, n, d, cnt.p, w.p);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    size_t bytes = 0;
    GK_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, bytes, cnt.p, t->lk.p, static_cast<int>(d.nlk),
                                          st));
    DevBuf<char> tmp;
    tmp.alloc(bytes, st);
    GK_CUDA(cub::DeviceScan::ExclusiveSum(tmp.p, bytes, cnt.p, t->lk.p, static_cast<int>(d.nlk),
                                          st));
    count_launches(2);  // scan-init + scan
    lookup_finish_kernel<<<grid_for(d.nlk), 256, 0, st>>>(t->lk.p, d.nlk, t->lk.p);
    count_launches(1);
    GK_CUDA(cudaGetLastError());
    GK_CUDA(cudaMemcpyAsync(hw, w.p, sizeof(hw), cudaMemcpyDeviceToHost, st));
    GK_CUDA(cudaEventRecord(ctx->ev1, st));
    GK_CUDA(cudaStreamSynchronize(st));
  }
  if (hw[W_BAD] & 2ull) fail(GK_ERR_RUNTIME, "lookup hash: two nodes share a bucket");

  float ms = 0.f;
  GK_CUDA(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
  t->absc.reset();
  t->absc.p = absc.p;  // take ownership
  t->absc.n = absc.n;
  t->absc.s = absc.s;
  absc.p = nullptr;
  absc.n = 0;

  // arithmetic-locate runs: whole runs strictly inside the base grid (the last
  // base interval ends at r_max itself and is left to the lookup path)
  {
    const long long runs = (S.steps - 1) / 64;
    d.ncoarse = runs > 0 && runs < (1LL << 26) ? static_cast<uint32_t>(runs) : 0u;
    d.t_eff = S.t_eff;
    d.inv_t = 1.0 / S.t_eff;
    if (d.ncoarse) {
      t->coarse.alloc(d.ncoarse, st);
      coarse_runs_kernel<<<grid_for(d.ncoarse, 128), 128, 0, st>>>(absc.p ? absc.p : t->absc.p, n,
                                                                   S.r_min, S.t_eff, d.ncoarse,
                                                                   t->coarse.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
    }
    d.coarse = t->coarse.p;
  }
  // table sweep arrays: base points 0 .. steps (base_nodes_kernel)
  {
    const long long nbase = S.steps + 1;
    d.nbase = nbase < (1LL << 30) ? static_cast<uint32_t>(nbase) : 0u;
    if (d.nbase) {
      const uint32_t nwords = ((static_cast<uint32_t>((nbase + 31) >> 5)) + 8u) & ~3u;
      DevBuf<int32_t> b2p;
      b2p.alloc(static_cast<size_t>(nbase), st);
      t->base_g.alloc(static_cast<size_t>(nbase), st);
      t->base_e.alloc(static_cast<size_t>(nbase), st);
      t->base_clean.alloc(nwords, st);
      base_nodes_kernel<<<grid_for(nbase, 128), 128, 0, st>>>(
          absc.p ? absc.p : t->absc.p, static_cast<size_t>(n), S.r_min, S.t_eff, nbase,
          t->exp_vals.p, t->green_vals.p, b2p.p, t->base_g.p, t->base_e.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
      base_clean_kernel<<<(nwords + 127) / 128, 128, 0, st>>>(b2p.p, nbase, nwords,
                                                               t->base_clean.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
    }
    d.bg = t->base_g.p;
    d.be = t->base_e.p;
    d.bclean = t->base_clean.p;
    d.npatch = 0;
    if (d.nbase) {  // the non-uniform intervals' list (TableDev::pj / pa)
      const double* ab = absc.p ? absc.p : t->absc.p;
      DevBuf<uint8_t> flag;
      flag.alloc(static_cast<size_t>(n), st);
      GK_CUDA(cudaMemsetAsync(flag.p, 0, static_cast<size_t>(n), st));
      patch_flag_kernel<<<grid_for(nbase, 128), 128, 0, st>>>(ab, static_cast<size_t>(n), S.r_min,
                                                              S.t_eff, cfg.r_max, nbase,
                                                              t->base_clean.p, flag.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
      t->patch_j.alloc(static_cast<size_t>(n), st);
      DevBuf<int> np;
      np.alloc(1, st);
      size_t tb = 0;
      cub::CountingInputIterator<uint32_t> idx(0u);
      GK_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, idx, flag.p, t->patch_j.p, np.p,
                                         static_cast<int>(n), st));
      DevBuf<char> tmp;
      tmp.alloc(tb, st);
      GK_CUDA(cub::DeviceSelect::Flagged(tmp.p, tb, idx, flag.p, t->patch_j.p, np.p,
                                         static_cast<int>(n), st));
      count_launches(2);
      t->patch_a.alloc(static_cast<size_t>(n), st);
      patch_left_kernel<<<grid_for(n, 256), 256, 0, st>>>(ab, t->patch_j.p, np.p, t->patch_a.p);
      count_launches(1);
      GK_CUDA(cudaGetLastError());
      int hnp = 0;
      GK_CUDA(cudaMemcpyAsync(&hnp, np.p, sizeof(int), cudaMemcpyDeviceToHost, st));
      GK_CUDA(cudaStreamSynchronize(st));
      d.npatch = static_cast<uint32_t>(hnp);
    }
    d.pj = t->patch_j.p;
    d.pa = t->patch_a.p;
  }
  d.grec = t->grec.p;
  d.erec = t->erec.p;
  d.lk = t->lk.p;
  d.degree = degree;
  d.nrec = static_cast<uint32_t>(n);
  d.grs = grs;
  d.k_re = k_re;
  d.k_im = k_im;

  gk_table_info& info = t->info;
  info.nodes = static_cast<uint64_t>(n);
  info.zeros = t->zeros.size();
  info.hash_buckets = nb;
  info.lookup_buckets = d.nlk;
  info.r_min = cfg.r_min;
  info.r_max = cfg.r_max;
  info.t = tmax;
  info.dr_min = dr_min;
  info.inv_dr_min = inv_dr_min;
  info.k_re = k_re;
  info.k_im = k_im;
  info.degree = degree;
  info.device_bytes = t->absc.bytes() + t->exp_vals.bytes() + t->green_vals.bytes() +
                      t->hash.bytes() + t->grec.bytes() + t->erec.bytes() + t->lk.bytes() +
                      t->coarse.bytes() + t->base_g.bytes() + t->base_e.bytes() +
                      t->base_clean.bytes();
  info.build_ms = ms;
}

}  // namespace gk
