// gk_internal.h -- host-side objects behind the C ABI (include/gk/gk.h).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gk/gk.h"
#include "gk_device.cuh"

namespace gk {

struct Error {
  gk_status status;
  std::string what;
};

[[noreturn]] inline void fail(gk_status s, const std::string& what) { throw Error{s, what}; }

inline void need(bool ok, gk_status s, const char* what) {
  if (!ok) fail(s, what);
}

// the thread-local message behind gk_last_error (abi.cu)
std::string& last_error_buffer();

// run an entry point's body: exceptions -> gk_status + gk_last_error message
template <class F>
gk_status guarded(F&& f) {
  try {
    f();
    return GK_OK;
  } catch (const Error& e) {
    last_error_buffer() = e.what;
    return e.status;
  } catch (const std::bad_alloc&) {
    last_error_buffer() = "out of host memory";
    return GK_ERR_RUNTIME;
  } catch (const std::exception& e) {
    last_error_buffer() = e.what();
    return GK_ERR_RUNTIME;
  }
}

// rethrow a failed entry point's status (composing entry points)
inline void ok(gk_status s) {
  if (s != GK_OK) fail(s, last_error_buffer());
}

#define GK_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t gk_e_ = (call);                                                         \
    if (gk_e_ != cudaSuccess)                                                           \
      ::gk::fail(GK_ERR_RUNTIME, std::string(#call) + ": " + cudaGetErrorString(gk_e_)); \
  } while (0)

// device buffer owned by a gk object.  Allocated stream-ordered from the
// device's default memory pool (release threshold = max, set at context
// creation) so the temporaries of a table build cost no device-wide syncs.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  cudaStream_t s = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { reset(); }
  void reset() {
    if (p) cudaFreeAsync(p, s);
    p = nullptr;
    n = 0;
  }
  void alloc(size_t count, cudaStream_t stream = nullptr) {
    reset();
    if (count == 0) count = 1;
    s = stream;
    GK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), count * sizeof(T), stream));
    n = count;
  }
  size_t bytes() const { return n * sizeof(T); }
};

// One set of shared-edge blocks over a mesh (edges.cu): every distinct edge
// of a block of source triangles is evaluated once and serves the (usually
// two) triangles that share it; used for (row, block) pairs at least r_far
// apart.  A mesh keeps two: `es` (11-chunk blocks: K4e / K3e) and `sweep`
// (small blocks: the table sweep K3s, whose shared-memory window must cover a
// block's radius spread).
struct EdgeSet {
  DevBuf<EdgeBlock> eblk;  // [nblk]
  DevBuf<double2> ep;      // [chunks][n][2][32] edge points (owner orientation): (x, y) and (z, w) planes
  DevBuf<uint4> ecol;      // [N] by block position: (triangle, e0 | e1 << 16, e2, 0)
  uint64_t edges = 0;
  int ecap = 0;  // edges per block (shared-memory slots per warp)
  double rho_mean = 0.0, rho_max = 0.0;
  bool ordered = false;
  size_t nblk = 0;
  double r_far = INFINITY;   // pairs this far apart absorb the reversed-edge rounding
  double edge_delta = 0.0;   // max |point - reversed-edge point| over shared sides
  double edge_ratio = 1.0;   // evaluated edge slots / (3 N): the far-path work fraction
};

}  // namespace gk

// gk_fill_rows_host's double-buffered fill -> D2H pipeline, kept by the
// context across calls (no per-call stream / event / buffer churn)
struct HostFillPipe {
  cudaStream_t copy = nullptr;
  cudaEvent_t filled[2] = {nullptr, nullptr}, copied[2] = {nullptr, nullptr};
  gk::DevBuf<gk_c128> buf[2];
};

struct gk_ctx {
  int device = 0;
  cudaStream_t own = nullptr;
  cudaStream_t stream = nullptr;
  int sm_count = 0;
  gk::DevBuf<unsigned long long> scratch;  // counters / reductions (64 words)
  gk::DevBuf<double2> phase;               // direct-mode phase table (kPhaseM)
  gk::DevBuf<double2> phase_small;         // eval_batch phase table (kPhaseSmall, L1-resident)
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  HostFillPipe pipe;
  gk_fill_options opts{};  // defaults for calls without options (gk_ctx_set_fill_options)
};

struct gk_table {
  gk_ctx* ctx = nullptr;
  gk_table_info info{};
  gk::TableDev dev{};
  gk::DevBuf<double> absc;
  gk::DevBuf<double2> exp_vals, green_vals;
  gk::DevBuf<uint32_t> hash;  // reference-format buckets (table.hpp:40-82)
  gk::DevBuf<double> grec, erec;
  gk::DevBuf<uint32_t> lk;
  gk::DevBuf<int32_t> coarse;  // arithmetic-locate runs (TableDev::coarse)
  gk::DevBuf<double2> base_g, base_e;  // table sweep: node values by base index (TableDev::bg / be)
  gk::DevBuf<uint32_t> base_clean;     // table sweep: uniform-stencil bits (TableDev::bclean)
  gk::DevBuf<uint32_t> patch_j;        // table sweep: non-uniform intervals (TableDev::pj)
  gk::DevBuf<double> patch_a;          // ... their left nodes (TableDev::pa)
  std::vector<double> zeros;  // zero_locations (host copy)
};

struct gk_mesh {
  gk_ctx* ctx = nullptr;
  size_t N = 0, nv = 0;
  int m = 0, n = 0;
  double diameter = 0.0;  // bounding-box diagonal of the vertices (bounds every pair distance)
  double mean_edge = 0.0; // edge of the mean-area equilateral triangle (tile window estimate)
  double rho_outer_max = 0.0;  // largest bounds[].w (a row's outer points about its centroid)
  gk::DevBuf<double4> outer;  // [N * m]    (x, y, z, w)
  gk::DevBuf<double4> inner;  // [3n][N]    (x, y, z, w), column-major in q
  gk::DevBuf<double4> bounds; // [N]        (cx, cy, cz, rho_outer), rho_inner in binner
  gk::DevBuf<double> binner;  // [N]
  gk::DevBuf<double> verts;   // [3 nv] vertices (max_vertex_distance)
  // shared-edge blocks (build_edge_blocks): the K4e / K3e set and the
  // table sweep's small blocks
  gk::EdgeSet es, sweep;
  // the table sweep's row clusters: in-range rows in the sweep set's spatial
  // order, cached for the last row range (gk_fill_rows)
  mutable gk::DevBuf<uint32_t> srows;
  mutable size_t srows_begin = 0, srows_end = 0, srows_n = 0;
};

namespace gk {

// library defaults of the kernel selection (gk_fill_options_init)
inline gk_fill_options default_fill_options() {
  gk_fill_options o;
  o.shared_edges = GK_AUTO;
  o.table_placement = GK_AUTO;
  o.arith_locate = GK_AUTO;
  o.lossy_phase = GK_AUTO;
  o.unrolled = GK_AUTO;
  o.eval_libdevice = GK_AUTO;
  o.smem_budget = 0;
  return o;
}

inline gk_mesh_options default_mesh_options() {
  gk_mesh_options o;
  o.shared_edges = GK_AUTO;
  o.edge_chunks = 0;
  o.edge_order = GK_AUTO;
  o.leaf_pct = 0;
  o.sweep_chunks = 0;
  return o;
}

inline bool path_counts_evaluations(int path) {
  return path == GK_PATH_DIRECT_EDGE || path == GK_PATH_TABLE_EDGE || path == GK_PATH_TABLE_SWEEP;
}

// launch accounting (gk_launch_count)
void count_launches(unsigned long long n);

// host-side quadrature rules (quadrature.hpp:35-110), bit-identical
void triangle_rule(int m, double* b0, double* b1, double* b2, double* w);
void gauss_legendre_unit(int n, double* x, double* w);
void sphere_mesh(double radius, int subdivisions, std::vector<double>& verts,
                 std::vector<uint32_t>& tris);
void plate_mesh(double side, int cells, std::vector<double>& verts, std::vector<uint32_t>& tris);
void jitter(double* v, size_t nv, uint64_t seed, double amp);
void validate_mesh(const double* v, size_t nv, const uint32_t* t, size_t nt);

// kernels launched by abi.cu (defined in build.cu / fill.cu / eval.cu)
void launch_points(gk_mesh* mesh, const double* d_verts, const uint32_t* d_tris,
                   cudaStream_t s);
// shared-edge blocks (edges.cu).  plan_edge_blocks is the host part: blocks
// of at most `cap` distinct edges over the triangles in mesh order or in a
// bisection order of the centroids (order_mode -1: the more compact, 0: mesh
// order, 1: bisection); order[j] is the triangle at block position j, eidx[j]
// its three block-local edge indices, owner[slot] = (t << 3) | (side << 1) |
// padding of every edge slot, gslot[3 t + s] the slot of side s of t.
struct EdgePlan {
  std::vector<EdgeBlock> blocks;
  std::vector<unsigned long long> owner;
  std::vector<ushort4> eidx;
  std::vector<uint32_t> gslot, order;
  uint64_t edges = 0;
  double rho_mean = 0.0;
  bool ordered = false;
};
EdgePlan plan_edge_blocks(const double* verts, size_t nv, const uint32_t* tris, size_t N,
                          size_t cap, int order_mode, int leaf_pct = 0, double rho_cap = 0.0);
// the device part for a mesh whose points launch_points has produced;
// synchronises the context stream
void build_edge_blocks(gk_mesh* mesh, const double* verts, const uint32_t* tris,
                       const gk_mesh_options& opts);
// max over vertex pairs of |a - b|^2 (reference summation order) -> *d2_bits
void launch_max_vertex_d2(const double* verts, size_t nv, unsigned long long* d2_bits,
                          cudaStream_t s);
// error_sweep (bounds.hpp:128-186): w[0..4] = max_rel_re, max_rel_im, max_abs,
// max_abs_at_exact_zero, max combined (double bits); w[5] = first probe index
// at the max combined; w[8..31] decade histogram.  `comb` scratch [probes].
void launch_sweep(gk_ctx* ctx, const gk_table* t, int kind, uint64_t probes, double* comb,
                  unsigned long long* w);
// Kernel::accumulate for nblocks blocks of block_len radii -> out[nblocks];
// w[0] fallbacks, w[1] first bad (flat index << 3 | code)
void launch_accumulate(gk_ctx* ctx, const gk_table* t, gk_kind kind, double k_re, double k_im,
                       const double* r, const double* wts, size_t block_len, size_t nblocks,
                       gk_c128* out, unsigned long long* w);
// compare_fills partial maxima (as non-negative double bits) -> w[0] (re), w[1] (im)
void launch_compare(gk_ctx* ctx, const gk_c128* test, const gk_c128* ref, size_t rows, size_t N,
                    size_t row_begin, size_t ld, unsigned long long* w);
void build_table_device(gk_ctx* ctx, gk_table* t, const gk_sampling_config& cfg, double k_zero,
                        double t_nominal, double k_re, double k_im, int degree);
// kind: GK_KIND_EXP, GK_KIND_GREEN, or 2 = fused pair (z = Exp, z2 = Green).
// Returns the gk_fill_path that ran (0: none); the shared-edge paths count
// the evaluations they performed into counters[3], elsewhere they equal the
// reference's calls (path_counts_evaluations).
int launch_fill(gk_ctx* ctx, const gk_mesh* mesh, gk_mode mode, const gk_table* table,
                 int kind, double k_re, double k_im, size_t row_begin, size_t row_end,
                 gk_c128* z, gk_c128* z2, size_t ldz, unsigned long long* d_fallbacks,
                 const gk_fill_options& opts);
void launch_range(gk_ctx* ctx, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                  double* d2min, double* d2max);
// the same on the device: out2 = {min d2, -max d2} over the rows ({inf, -0}
// for an empty range), ready for a MIN all-reduce
void launch_range_device(gk_ctx* ctx, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                         double* out2);
void launch_eval_batch(gk_ctx* ctx, const gk_table* table, gk_kind kind, double k_re,
                       double k_im, const double* r, size_t n, gk_c128* out,
                       unsigned long long* d_scratch);
void launch_locate(gk_ctx* ctx, const gk_table* t, const double* r, size_t n, uint32_t* out,
                   unsigned long long* w);
double run_fp64_peak(gk_ctx* ctx);
void init_phase_table(gk_ctx* ctx);

}  // namespace gk
