// edges.cu -- shared-edge blocks for the direct and table fills
// (direct_edge_kernel, table_edge_kernel in fill_kernels.cuh).
//
// The reference evaluates, for every source triangle q, the n Gauss points of
// each of its 3 edges (inner_points, matfill.hpp:121-133) against every outer
// point of p (fill_rows, matfill.hpp:185-198).  On a closed mesh every edge
// belongs to two triangles, traversed in opposite directions, so the same n
// points (up to the rounding of a + (b - a) x vs b + (a - b) x', with the
// Gauss-Legendre weights symmetric, quadrature.hpp:85-110) are evaluated
// twice per outer point.  A block groups a range of source triangles in a
// spatial (recursive-bisection) order, or in mesh order when that is about
// as compact; each distinct edge of the block is evaluated once per outer
// point, in the orientation of the first block triangle that uses it (those
// points are copied from the reference-exact inner points, so they are
// bit-identical for that triangle), and Z[p][q] is the sum of q's three edge
// sums.
//
// Parity: the other triangle's points differ from the evaluated ones by at
// most `edge_delta` (measured here on the device points).  For a term with
// weight w and distance r the value moves by at most |w| delta (1 + |k| r) /
// r^2, i.e. delta / (64 u r) of the stated per-term tolerance
// |w| 64 u (1 + |k| r) / r (u = 2^-53).  The kernel uses the
// shared points only where every pair of the (row, block) tile is at least
// r_far = delta / (32 u) apart -- at most half the tolerance -- and the
// reference's own per-triangle points everywhere else.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "gk_internal.h"

namespace gk {

namespace {

// owner slot code: (t << 3) | (side << 1) | pad
__global__ void edge_gather_kernel(const double4* __restrict__ inner, size_t N, int n,
                                   const unsigned long long* __restrict__ owner, size_t nslots,
                                   double2* __restrict__ ep) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i >= nslots * n) return;
  const size_t slot = i / n;
  const int g = static_cast<int>(i - slot * n);
  const unsigned long long o = owner[slot];
  const size_t t = static_cast<size_t>(o >> 3);
  const int s = static_cast<int>((o >> 1) & 3);
  double4 P = inner[static_cast<size_t>(s * n + g) * N + t];
  if (o & 1) P.w = 0.0;  // padding lane: a real point of the block, zero weight
  // two planes per point, (x, y) and (z, w): a warp's load of either is one
  // 512-byte run
  const size_t at = ((slot >> 5) * n + g) * 64 + (slot & 31);
  ep[at] = make_double2(P.x, P.y);
  ep[at + 32] = make_double2(P.z, P.w);
}

// max over the sides (t, s) that do not own their edge slot of
// |inner point g of (t, s) - its twin among the slot's evaluated points|: the
// reversed parameterisation pairs g with n-1-g (the weights are equal), a
// side running the owner's way (gslot bit 31) pairs g with g
__global__ void edge_delta_kernel(const double4* __restrict__ inner, size_t N, int n,
                                  const uint32_t* __restrict__ gslot,
                                  const unsigned long long* __restrict__ owner,
                                  const double2* __restrict__ ep, unsigned long long* dmax) {
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  double d = 0.0;
  if (i < 3 * N * static_cast<size_t>(n)) {
    const size_t ts = i / n;
    const int g = static_cast<int>(i - ts * n);
    const size_t t = ts / 3;
    const int s = static_cast<int>(ts - 3 * t);
    const uint32_t slot = gslot[ts] & 0x7fffffffu;
    const int gq = (gslot[ts] >> 31) ? g : n - 1 - g;  // the twin point of the edge's owner
    const unsigned long long mine = (static_cast<unsigned long long>(t) << 3) | (s << 1);
    if (owner[slot] != mine) {
      const double4 P = inner[static_cast<size_t>(s * n + g) * N + t];
      const size_t at = ((slot >> 5) * static_cast<size_t>(n) + gq) * 64 + (slot & 31);
      const double2 Qxy = ep[at], Qzw = ep[at + 32];
      const double dx = P.x - Qxy.x, dy = P.y - Qxy.y, dz = P.z - Qzw.x;
      d = sqrt(dx * dx + dy * dy + dz * dz);
      if (P.w != Qzw.y) d = INFINITY;  // weights must match exactly (symmetric rule)
    }
  }
  for (int off = 16; off > 0; off >>= 1) d = fmax(d, __shfl_xor_sync(0xffffffffu, d, off));
  if ((threadIdx.x & 31) == 0 && d > 0.0) atomicMax(dmax, __double_as_longlong(d));
}

}  // namespace

EdgePlan plan_edge_blocks(const double* verts, size_t nv, const uint32_t* tris, size_t N,
                          size_t cap, int order_mode, int leaf_pct, double rho_cap) {
  // global edge ids: edges bucketed by their lower vertex (CSR), distinct
  // upper vertices numbered within each bucket
  std::vector<uint32_t> start(nv + 1, 0);
  for (size_t t = 0; t < N; ++t)
    for (int s = 0; s < 3; ++s) {
      const uint32_t a = tris[3 * t + s], b = tris[3 * t + (s + 1) % 3];
      ++start[std::min(a, b) + 1];
    }
  for (size_t v = 0; v < nv; ++v) start[v + 1] += start[v];
  std::vector<uint32_t> fillp(start.begin(), start.end() - 1), hi(3 * N), side_of(3 * N);
  for (size_t t = 0; t < N; ++t)
    for (int s = 0; s < 3; ++s) {
      const uint32_t a = tris[3 * t + s], b = tris[3 * t + (s + 1) % 3];
      const uint32_t slot = fillp[std::min(a, b)]++;
      hi[slot] = std::max(a, b);
      side_of[slot] = static_cast<uint32_t>(3 * t + s);
    }
  std::vector<uint32_t> gid(3 * N);
  uint32_t nedges = 0;
  for (size_t v = 0; v < nv; ++v)
    for (uint32_t i = start[v]; i < start[v + 1]; ++i) {
      uint32_t id = nedges;
      for (uint32_t j = start[v]; j < i; ++j)
        if (hi[j] == hi[i]) {
          id = gid[side_of[j]];
          break;
        }
      if (id == nedges) ++nedges;
      gid[side_of[i]] = id;
    }

  double X = 0.0;
  for (size_t i = 0; i < 3 * nv; ++i) X = std::max(X, std::fabs(verts[i]));

  // Blocks: greedy over the triangles in traversal order `ord` (position j
  // holds triangle ord[j]), <= cap distinct edges each.  Identity order keeps
  // every warp store one 512-byte run; a bisection order of the centroids is
  // used instead when it gives much more compact blocks (the row-major plate,
  // and the icosphere, whose own order still spans ~0.4 m per block at C5):
  // the far test needs compact blocks.
  struct Blocks {
    std::vector<EdgeBlock> blocks;
    std::vector<unsigned long long> owner;
    std::vector<ushort4> eidx;   // by position
    std::vector<uint32_t> gslot; // by (triangle, side)
    uint64_t edges = 0;
    double rho_mean = 0.0;
  };
  std::vector<uint32_t> stamp(nedges), local(nedges);
  // cuts (optional): positions where a block must start (subtree leaves)
  auto make_blocks = [&](const std::vector<uint32_t>* ord, const std::vector<size_t>* cuts) {
    Blocks R;
    R.eidx.resize(N);
    R.gslot.resize(3 * N);
    std::fill(stamp.begin(), stamp.end(), UINT32_MAX);
    uint32_t tb = 0, ne = 0, bid = 0;
    size_t first_slot = 0;
    auto finish_block = [&](uint32_t te) {
      EdgeBlock B{};
      B.tb = tb;
      B.te = te;
      B.c0 = static_cast<uint32_t>(first_slot / 32);
      B.ne = ne;
      R.blocks.push_back(B);
      R.edges += ne;
      const unsigned long long first = R.owner[first_slot];
      while (R.owner.size() % 32) R.owner.push_back(first | 1ull);
      first_slot = R.owner.size();
    };
    size_t next_cut = 0;
    for (size_t j = 0; j < N; ++j) {
      const size_t t = ord ? (*ord)[j] : j;
      int fresh = 0;
      for (int s = 0; s < 3; ++s) fresh += stamp[gid[3 * t + s]] != bid;
      bool cut = false;
      if (cuts) {
        while (next_cut < cuts->size() && (*cuts)[next_cut] < j) ++next_cut;
        cut = next_cut < cuts->size() && (*cuts)[next_cut] == j;
      }
      if ((cut || ne + fresh > cap) && j > tb) {
        finish_block(static_cast<uint32_t>(j));
        ++bid;
        tb = static_cast<uint32_t>(j);
        ne = 0;
      }
      uint16_t li[3];
      for (int s = 0; s < 3; ++s) {
        const uint32_t e = gid[3 * t + s];
        if (stamp[e] != bid) {
          stamp[e] = bid;
          local[e] = ne++;
          R.owner.push_back((static_cast<unsigned long long>(t) << 3) | (static_cast<unsigned>(s) << 1));
        }
        li[s] = static_cast<uint16_t>(local[e]);
        // bit 31: this side runs the same way as the edge's owner (a mesh
        // without a consistent orientation): its points pair g with g
        const size_t slot = first_slot + local[e];
        const unsigned long long o = R.owner[slot];
        const uint32_t a_owner = tris[3 * (o >> 3) + ((o >> 1) & 3)];
        const bool same = a_owner == tris[3 * t + s] && (o >> 3) != t;
        R.gslot[3 * t + s] = static_cast<uint32_t>(slot) | (same ? 0x80000000u : 0u);
      }
      R.eidx[j] = make_ushort4(li[0], li[1], li[2], 0);
    }
    finish_block(static_cast<uint32_t>(N));
    // bounding sphere of each block's vertices (every inner point lies on a
    // segment between two of them); the margin covers the points' rounding
    for (EdgeBlock& B : R.blocks) {
      double c[3] = {0.0, 0.0, 0.0};
      for (uint32_t j = B.tb; j < B.te; ++j) {
        const size_t t = ord ? (*ord)[j] : j;
        for (int s = 0; s < 3; ++s)
          for (int d = 0; d < 3; ++d) c[d] += verts[3 * static_cast<size_t>(tris[3 * t + s]) + d];
      }
      const double cnt = 3.0 * (B.te - B.tb);
      for (double& x : c) x /= cnt;
      double rho = 0.0;
      for (uint32_t j = B.tb; j < B.te; ++j) {
        const size_t t = ord ? (*ord)[j] : j;
        for (int s = 0; s < 3; ++s) {
          const double* v = verts + 3 * static_cast<size_t>(tris[3 * t + s]);
          const double dx = v[0] - c[0], dy = v[1] - c[1], dz = v[2] - c[2];
          rho = std::max(rho, std::sqrt(dx * dx + dy * dy + dz * dz));
        }
      }
      B.cx = c[0];
      B.cy = c[1];
      B.cz = c[2];
      B.rho = rho * (1.0 + 1e-12) + 1e-12 * X;
      R.rho_mean += B.rho / static_cast<double>(R.blocks.size());
    }
    return R;
  };

  Blocks R = make_blocks(nullptr, nullptr);
  // spatial order: recursive coordinate bisection of the centroids (split on
  // the longest axis) whose leaves are the blocks: a leaf is a range of at
  // most T triangles with <= cap distinct edges, and splits fall on multiples
  // of T so that nearly all leaves are full
  std::vector<uint32_t> sorder(N);
  std::vector<size_t> cuts;
  {
    std::vector<double> cen(3 * N);
    for (size_t t = 0; t < N; ++t)
      for (int d = 0; d < 3; ++d) {
        double c = 0.0;
        for (int s = 0; s < 3; ++s) c += verts[3 * static_cast<size_t>(tris[3 * t + s]) + d];
        cen[3 * t + d] = c / 3.0;
      }
    for (size_t j = 0; j < N; ++j) sorder[j] = static_cast<uint32_t>(j);
    std::vector<uint32_t> seen(nedges, UINT32_MAX);
    uint32_t probe = 0;
    auto edges_of = [&](size_t lo, size_t hi) {
      size_t cnt = 0;
      ++probe;
      for (size_t j = lo; j < hi; ++j)
        for (int s = 0; s < 3; ++s) {
          const uint32_t e = gid[3 * static_cast<size_t>(sorder[j]) + s];
          if (seen[e] != probe) {
            seen[e] = probe;
            ++cnt;
          }
        }
      return cnt;
    };
    // bounding radius of the vertices of triangles sorder[lo, hi) about their
    // mean (the block radius of make_blocks, without its rounding margin)
    auto rho_of = [&](size_t lo, size_t hi) {
      double c[3] = {0.0, 0.0, 0.0};
      for (size_t j = lo; j < hi; ++j)
        for (int s = 0; s < 3; ++s)
          for (int d = 0; d < 3; ++d)
            c[d] += verts[3 * static_cast<size_t>(tris[3 * static_cast<size_t>(sorder[j]) + s]) + d];
      for (double& x : c) x /= 3.0 * static_cast<double>(hi - lo);
      double rho = 0.0;
      for (size_t j = lo; j < hi; ++j)
        for (int s = 0; s < 3; ++s) {
          const double* v = verts + 3 * static_cast<size_t>(tris[3 * static_cast<size_t>(sorder[j]) + s]);
          const double dx = v[0] - c[0], dy = v[1] - c[1], dz = v[2] - c[2];
          rho = std::max(rho, std::sqrt(dx * dx + dy * dy + dz * dz));
        }
      return rho;
    };
    // leaf triangles per edge slot, percent (~1.6 edges per triangle);
    // gk_mesh_options.leaf_pct for A/B
    const size_t tfrac = leaf_pct >= 30 && leaf_pct <= 100 ? static_cast<size_t>(leaf_pct) : 61;
    const size_t T = std::max<size_t>(1, (cap * tfrac) / 100);
    std::vector<std::pair<size_t, size_t>> stack{{0, N}};
    while (!stack.empty()) {
      const auto [lo, hi] = stack.back();
      stack.pop_back();
      const size_t c = hi - lo;
      size_t mid;
      if (c <= T) {
        if ((edges_of(lo, hi) <= cap && (rho_cap <= 0.0 || rho_of(lo, hi) <= rho_cap)) || c == 1) {
          cuts.push_back(lo);
          continue;
        }
        mid = lo + c / 2;
      } else {
        const size_t L = (c + T - 1) / T;
        mid = lo + (L / 2) * T;
      }
      double bl[3] = {INFINITY, INFINITY, INFINITY}, bh[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (size_t j = lo; j < hi; ++j)
        for (int d = 0; d < 3; ++d) {
          bl[d] = std::min(bl[d], cen[3 * sorder[j] + d]);
          bh[d] = std::max(bh[d], cen[3 * sorder[j] + d]);
        }
      int ax = 0;
      for (int d = 1; d < 3; ++d)
        if (bh[d] - bl[d] > bh[ax] - bl[ax]) ax = d;
      std::nth_element(sorder.begin() + lo, sorder.begin() + mid, sorder.begin() + hi,
                       [&](uint32_t u, uint32_t v) {
                         const double cu = cen[3 * u + ax], cv = cen[3 * v + ax];
                         return cu < cv || (cu == cv && u < v);
                       });
      stack.push_back({mid, hi});
      stack.push_back({lo, mid});
    }
    std::sort(cuts.begin(), cuts.end());
    // within a leaf the order is free: ascending triangle index, so that a
    // warp's 32 stores of one row fall on as few 128-byte lines of Z as the
    // mesh numbering allows (subdivided meshes number siblings consecutively)
    for (size_t i = 0; i < cuts.size(); ++i) {
      const size_t lo = cuts[i], hi = i + 1 < cuts.size() ? cuts[i + 1] : N;
      std::sort(sorder.begin() + lo, sorder.begin() + hi);
    }
  }
  Blocks Rm = make_blocks(&sorder, &cuts);
  bool ordered = order_mode < 0 ? Rm.rho_mean < 0.75 * R.rho_mean : order_mode == 1;
  if (ordered) R = std::move(Rm);
  EdgePlan P;
  P.blocks = std::move(R.blocks);
  P.owner = std::move(R.owner);
  P.eidx = std::move(R.eidx);
  P.gslot = std::move(R.gslot);
  P.edges = R.edges;
  P.rho_mean = R.rho_mean;
  P.ordered = ordered;
  P.order.resize(N);
  for (size_t j = 0; j < N; ++j) P.order[j] = ordered ? sorder[j] : static_cast<uint32_t>(j);
  return P;
}

namespace {

// one block set of at most `cap` distinct edges per block into S
// rho_cap_rel > 0: leaves whose radius exceeds rho_cap_rel x the mean block
// radius of an uncapped plan are split (a second plan): the table sweep's
// window must cover the largest block's radius spread
void build_edge_set(const gk_mesh* mesh, const double* verts, const uint32_t* tris, size_t cap,
                    int order_mode, int leaf_pct, EdgeSet& S, double rho_cap_rel = 0.0) {
  const size_t N = mesh->N, nv = mesh->nv;
  const int n = mesh->n;
  S.ecap = static_cast<int>(cap);
  EdgePlan R = plan_edge_blocks(verts, nv, tris, N, cap, order_mode, leaf_pct);
  if (rho_cap_rel > 0.0 && R.ordered) {
    double rmax = 0.0;
    for (const EdgeBlock& B : R.blocks) rmax = std::max(rmax, B.rho);
    if (rmax > rho_cap_rel * R.rho_mean)
      R = plan_edge_blocks(verts, nv, tris, N, cap, order_mode, leaf_pct, rho_cap_rel * R.rho_mean);
  }
  const std::vector<EdgeBlock>& blocks = R.blocks;
  const std::vector<unsigned long long>& owner = R.owner;

  cudaStream_t st = mesh->ctx->stream;
  const size_t nslots = owner.size();
  DevBuf<unsigned long long> d_owner;
  DevBuf<uint32_t> d_gslot;
  d_owner.alloc(nslots, st);
  d_gslot.alloc(3 * N, st);
  S.eblk.alloc(blocks.size(), st);
  S.ecol.alloc(N, st);
  S.ep.alloc(nslots * n * 2, st);
  GK_CUDA(cudaMemcpyAsync(d_owner.p, owner.data(), nslots * sizeof(unsigned long long),
                          cudaMemcpyHostToDevice, st));
  GK_CUDA(cudaMemcpyAsync(d_gslot.p, R.gslot.data(), 3 * N * sizeof(uint32_t), cudaMemcpyHostToDevice, st));
  GK_CUDA(cudaMemcpyAsync(S.eblk.p, blocks.data(), blocks.size() * sizeof(EdgeBlock),
                          cudaMemcpyHostToDevice, st));
  std::vector<uint4> ecol(N);
  for (size_t j = 0; j < N; ++j) {
    const ushort4 e = R.eidx[j];
    ecol[j] = make_uint4(R.order[j],
                         static_cast<uint32_t>(e.x) | (static_cast<uint32_t>(e.y) << 16), e.z, 0u);
  }
  GK_CUDA(cudaMemcpyAsync(S.ecol.p, ecol.data(), N * sizeof(uint4), cudaMemcpyHostToDevice, st));
  const size_t work = nslots * n;
  edge_gather_kernel<<<static_cast<unsigned>((work + 255) / 256), 256, 0, st>>>(
      mesh->inner.p, N, n, d_owner.p, nslots, S.ep.p);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  unsigned long long* dmax = mesh->ctx->scratch.p + 30;
  GK_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), st));
  const size_t work2 = 3 * N * static_cast<size_t>(n);
  edge_delta_kernel<<<static_cast<unsigned>((work2 + 255) / 256), 256, 0, st>>>(
      mesh->inner.p, N, n, d_gslot.p, d_owner.p, S.ep.p, dmax);
  count_launches(1);
  GK_CUDA(cudaGetLastError());
  unsigned long long hbits = 0;
  GK_CUDA(cudaMemcpyAsync(&hbits, dmax, sizeof(hbits), cudaMemcpyDeviceToHost, st));
  GK_CUDA(cudaStreamSynchronize(st));
  double delta;
  std::memcpy(&delta, &hbits, sizeof(delta));
  S.nblk = blocks.size();
  S.edges = R.edges;
  S.rho_mean = R.rho_mean;
  S.rho_max = 0.0;
  for (const EdgeBlock& B : blocks) S.rho_max = std::max(S.rho_max, B.rho);
  S.ordered = R.ordered;
  S.edge_delta = delta;
  S.edge_ratio = static_cast<double>(nslots) / (3.0 * static_cast<double>(N));
  // delta / r_far = 32 u: the reversed-edge rounding stays under half the
  // per-term tolerance (u = 2^-53); a tiny floor keeps r_far > 0
  S.r_far = std::isfinite(delta) ? std::max(delta * 0x1p48, 1e-300) : INFINITY;
}

}  // namespace

void build_edge_blocks(gk_mesh* mesh, const double* verts, const uint32_t* tris,
                       const gk_mesh_options& opts) {
  const size_t N = mesh->N;
  mesh->es.nblk = mesh->sweep.nblk = 0;
  if (opts.shared_edges == 0) return;
  size_t cap = 32 * kEdgeChunksDefault;
  if (opts.edge_chunks >= 1 && opts.edge_chunks * 32 <= kEdgeCap)  // block size (tests, A/B)
    cap = static_cast<size_t>(opts.edge_chunks) * 32;
  mesh->es.ecap = static_cast<int>(cap);
  // the edge kernels unroll the n points of an edge (n = 1..5)
  if (N > (size_t(1) << 30) || mesh->n > 5) return;
  // -1: the more compact of mesh and bisection order; 0 / 1 forced (A/B)
  const int order_mode = opts.edge_order == 0 || opts.edge_order == 1 ? opts.edge_order : -1;
  build_edge_set(mesh, verts, tris, cap, order_mode, opts.leaf_pct, mesh->es);
  // the table sweep's set: small blocks (a band's window spans 2 (rho_rows +
  // rho_block) of radius), always in the spatial order (its row clusters
  // follow the same order)
  size_t scap = 32 * kSweepChunksDefault;
  if (opts.sweep_chunks >= 1 && opts.sweep_chunks * 32 <= kEdgeCap)
    scap = static_cast<size_t>(opts.sweep_chunks) * 32;
  build_edge_set(mesh, verts, tris, scap, 1, kSweepLeafPct, mesh->sweep, kSweepRhoCap);
}

}  // namespace gk
