/*
 * gk.h -- C ABI of the B200-native MoM Green-function fill (arXiv 1901.04162
 * hot path).  libgk.so implements it with hand-written sm_100a CUDA kernels.
 *
 * The ABI is the drop-in boundary for the reference `gktab` library
 * (/root/reference/proj/include/gktab/, header-only C++20).  The reference
 * has no ABI of its own; every entry point below names the reference
 * interface it replaces (file:line, relative to proj/include/gktab/).
 *
 * Conventions (mirroring the reference):
 *  - errors: gk_status codes map 1:1 to the reference's exception types
 *    (invalid_argument, domain_error, out_of_range, overflow_error,
 *    runtime_error); gk_last_error() returns the message (thread-local).
 *  - gk_c128 is layout-compatible with std::complex<double>.
 *  - kinds use the reference's KernelKind values (kernel.hpp:14-17).
 *  - pointers documented "device" are CUDA device pointers on the context's
 *    device; "host" pointers are ordinary host memory.
 *  - a gk_ctx owns one CUDA stream (or borrows the caller's, see
 *    gk_ctx_set_stream); it is not re-entrant, but separate contexts may be
 *    driven from separate host threads.
 *  - there is no CPU fallback: without a usable sm_100 device every call
 *    fails with GK_ERR_RUNTIME.
 */
#ifndef GK_GK_H
#define GK_GK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GK_ABI_VERSION 3

typedef enum gk_status {
  GK_OK = 0,
  GK_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument */
  GK_ERR_DOMAIN = 2,           /* std::domain_error     */
  GK_ERR_OUT_OF_RANGE = 3,     /* std::out_of_range     */
  GK_ERR_OVERFLOW = 4,         /* std::overflow_error   */
  GK_ERR_RUNTIME = 5           /* std::runtime_error, CUDA failures */
} gk_status;

/* gktab::KernelKind (kernel.hpp:14-17) */
typedef enum gk_kind { GK_KIND_EXP = 0, GK_KIND_GREEN = 1 } gk_kind;

/* AnalyticKernel vs TableKernel (matfill.hpp:59-87) */
typedef enum gk_mode { GK_MODE_DIRECT = 0, GK_MODE_TABLE = 1 } gk_mode;

typedef struct gk_c128 { double re, im; } gk_c128;

typedef struct gk_ctx gk_ctx;
typedef struct gk_table gk_table;
typedef struct gk_mesh gk_mesh;

/* gktab::Medium (kernel.hpp:25-38).  eps_r_im != 0 is the lossy-medium
   extension (complex k = 2 pi sqrt(eps_r mu_r) / lambda0, principal root). */
typedef struct gk_medium {
  double lambda0, eps_r, mu_r, eps_r_im;
} gk_medium;

/* gktab::SamplingConfig (sampling.hpp:18-45), same defaults. */
typedef struct gk_sampling_config {
  double r_min, r_max;
  int samples_per_wavelength;
  int refine_interval_divisor;
  double refine_halfwidth_in_t;
  double dedup_fraction;
  int refine;
} gk_sampling_config;

/* gktab::FillReport (matfill.hpp:33-47), the fields fill_matrix sets. */
typedef struct gk_fill_report {
  uint64_t N;
  int m, n;
  uint64_t predicted_calls, actual_calls, fallback_calls;
  double wall_time_s; /* device time of the fill kernels (CUDA events) */
  /* kernel evaluations the device performed for these entries: actual_calls,
     or fewer where the fill evaluates each shared edge of a closed mesh once
     for both of its triangles (K4e direct, K3e table) */
  uint64_t evaluations;
  /* the fill kernel that ran (gk_fill_path) */
  int path;
} gk_fill_report;
/* The fill kernels; 0: nothing launched (empty row range). */
typedef enum gk_fill_path {
  GK_PATH_DIRECT = 1,        /* K4: direct, per triangle (the reference's order) */
  GK_PATH_DIRECT_EDGE = 2,   /* K4e: direct, shared edges */
  GK_PATH_TABLE_L1 = 3,      /* K3: table through L1, per triangle */
  GK_PATH_TABLE_STAGED = 4,  /* K3: table staged in shared memory, per triangle */
  GK_PATH_TABLE_EDGE = 5,    /* K3e: table through L1, shared edges */
  GK_PATH_TABLE_SWEEP = 6    /* K3s: distance-band windows in shared memory, shared edges */
} gk_fill_path;

/* ---------------------------------------------------- kernel selection
   Every choice the library makes between equivalent kernels, made explicit
   per call (no environment variable or other process-global state is read).
   The reference picks its kernel by type (AnalyticKernel / TableKernel,
   matfill.hpp:59-87); these only choose HOW the device evaluates it.  All
   choices give results within the same stated bound; the bit-identity
   classes are documented in DESIGN.md §3.  Initialise with
   gk_fill_options_init (every field GK_AUTO = the measured best). */
#define GK_AUTO (-1)
typedef enum gk_table_placement {
  GK_TABLE_GLOBAL = 0, /* table read through L1/L2 */
  GK_TABLE_SHARED = 1, /* table staged into shared memory: whole, or per-tile windows */
  GK_TABLE_SWEEP = 2   /* shared-edge sweep (K3s): per row cluster, source blocks by
                          distance band, each band's slice of the base-grid node values
                          staged into shared memory */
} gk_table_placement;
typedef struct gk_fill_options {
  /* GK_AUTO: shared-edge kernels (each mesh edge evaluated once for both of
     its triangles, DESIGN.md §5 K4e/K3e) where they pay: closed meshes of
     >= 4096 triangles with n <= 5;  0: never (the reference's per-triangle
     evaluation order, matfill.hpp:185-198);  1: whenever the mesh has
     shared-edge blocks (any mesh size; TABLE mode still picks by table
     size, GK_TABLE_GLOBAL takes them instead of staging) */
  int shared_edges;
  /* TABLE mode: GK_AUTO (staged whole when the table fits; a dense table
     through the sweep K3s where its window covers a tile, else K3e through
     L1), or a gk_table_placement (GK_TABLE_GLOBAL: the shared-edge K3e
     where the fill uses shared edges, else per triangle; GK_TABLE_SHARED:
     always staged, per triangle; GK_TABLE_SWEEP: K3s where it fits, else
     K3e) */
  int table_placement;
  /* TABLE mode: GK_AUTO / 1: arithmetic interval index on the plan's
     uniform runs (bit-identical lookup), 0: lookup buckets only */
  int arith_locate;
  /* lossy DIRECT fills: GK_AUTO / 1: attenuation coupled to the phase
     reduction, 0: separate attenuation table */
  int lossy_phase;
  /* DIRECT fills: GK_AUTO / 1: the n = 1..5 unrolled kernel, 0: the generic
     runtime-loop kernel */
  int unrolled;
  /* gk_eval_batch* (through gk_ctx_set_fill_options): GK_AUTO / 0: the
     phase-table direct evaluation, 1: libdevice sincos */
  int eval_libdevice;
  /* TABLE mode, staged: shared-memory bytes for a table window (0: 200 KB;
     smaller values force per-tile windows and their overflow path) */
  uint64_t smem_budget;
} gk_fill_options;
void gk_fill_options_init(gk_fill_options* opts);

/* Shared-edge block construction at gk_mesh_create_ex (DESIGN.md §5 K4e). */
typedef struct gk_mesh_options {
  int shared_edges;  /* GK_AUTO / 1: build the blocks, 0: do not */
  int edge_chunks;   /* warp-wide edge chunks per block, 1..12 (0 / GK_AUTO: 11) */
  int edge_order;    /* GK_AUTO: the more compact; 0: mesh order; 1: bisection order */
  int leaf_pct;      /* bisection leaf size in percent of the edge cap, 30..100 (0 / GK_AUTO: 61) */
  int sweep_chunks;  /* chunks per block of the table sweep's second, smaller block
                        set (DESIGN.md §5 K3s), 1..12 (0 / GK_AUTO: 2) */
} gk_mesh_options;
void gk_mesh_options_init(gk_mesh_options* opts);

typedef struct gk_table_info {
  uint64_t nodes, zeros, hash_buckets, lookup_buckets;
  double r_min, r_max, t, dr_min, inv_dr_min, k_re, k_im;
  int degree;
  uint64_t device_bytes;
  double build_ms; /* device time of gk_table_build */
} gk_table_info;

/* ---------------------------------------------------------------- context */
int gk_abi_version(void);
const char* gk_last_error(void);
gk_status gk_ctx_create(int device, gk_ctx** out);
/* Destroy a context after the tables and meshes created on it. */
gk_status gk_ctx_destroy(gk_ctx* ctx);
/* Run on the caller's cudaStream_t (e.g. torch.cuda.current_stream()), used
   as-is: 0 is the legacy default stream.  gk_ctx_use_own_stream restores the
   context's own (non-blocking) stream. */
gk_status gk_ctx_set_stream(gk_ctx* ctx, void* cuda_stream);
gk_status gk_ctx_use_own_stream(gk_ctx* ctx);
gk_status gk_ctx_synchronize(gk_ctx* ctx);
/* The context's default kernel selection, used where a call takes no
   gk_fill_options (or passes NULL): gk_fill_matrix_host, gk_bench_compare,
   gk_eval_batch*.  NULL restores the library defaults. */
gk_status gk_ctx_set_fill_options(gk_ctx* ctx, const gk_fill_options* opts);

/* ------------------------------------------------------------ kernel math */
/* gktab::wavenumber (kernel.hpp:41-44); complex for eps_r_im != 0 */
gk_status gk_wavenumber(const gk_medium* medium, double* k_re, double* k_im);

/* ------------------------------------------------------------------ table */
/* build_plan + KernelEvaluator ctor (sampling.hpp:149-236; evaluator.hpp:104-114:
   build_table x2, build_hash, pack_green_stencils), built on the device.
   The plan and the reference-format hash are bit-identical to the
   reference's; node values come from device sincos (ulp-level differences). */
gk_status gk_table_build(gk_ctx* ctx, const gk_sampling_config* cfg, const gk_medium* medium,
                         int lagrange_degree, gk_table** out);
gk_status gk_table_info_get(const gk_table* table, gk_table_info* info);
/* Host copies of the plan (abscissae[nodes], zeros[zeros]), node values
   (exp/green[nodes]) and the reference-format hash buckets[hash_buckets]
   (table.hpp:40-82).  Any pointer may be NULL. */
gk_status gk_table_download(const gk_table* table, double* abscissae, double* zeros,
                            gk_c128* exp_values, gk_c128* green_values, uint32_t* buckets);
gk_status gk_table_destroy(gk_table* table);
/* Wire formats of the reference, written from a device table:
   dump_table_binary (io.hpp:77-96): "GKTB", u32 version 1, u32 count, f64 k,
   u8 kind, count x (f64 r, f64 re, f64 im), little-endian -- readable by the
   reference's load_table_binary (io.hpp:105-132);
   dump_plan_csv (io.hpp:60-74): "index,r,is_zero,gap_to_next", %.17g. */
gk_status gk_table_dump_binary(const gk_table* table, gk_kind kind, const char* path);
gk_status gk_plan_dump_csv(const gk_table* table, const char* path);

/* KernelEvaluator::eval_batch (evaluator.hpp:209-221) when table != NULL
   (Exp: linear, Green: Lagrange; r < r_min -> analytic fallback, counted),
   eval_analytic (kernel.hpp:48-61) elementwise when table == NULL (k from
   k_re/k_im).  radii/out are device pointers.  On an invalid radius the call
   fails with the first failing index in the message, like the reference. */
gk_status gk_eval_batch(gk_ctx* ctx, const gk_table* table, gk_kind kind, double k_re,
                        double k_im, const double* radii, size_t n, gk_c128* out,
                        uint64_t* fallbacks);

/* The reference's plugin seam in batch: Kernel::accumulate (matfill.hpp:59-87;
   TableKernel -> KernelEvaluator::accumulate_green, evaluator.hpp:150-194, when
   table != NULL, AnalyticKernel{k} when NULL) for nblocks independent blocks:
   out[b] = sum_i K(radii[b*block_len + i]) * weights[b*block_len + i].
   Device buffers; one warp per block (lanes stride the block, warp-shuffle
   reduction).  For callers with their own quadrature.  Errors like
   eval_batch (the first failing flat index), fallbacks counted. */
gk_status gk_accumulate_batch(gk_ctx* ctx, const gk_table* table, gk_kind kind, double k_re,
                              double k_im, const double* radii, const double* weights,
                              size_t block_len, size_t nblocks, gk_c128* out,
                              uint64_t* fallbacks);

/* gk_accumulate_batch from HOST buffers (radii/weights[block_len * nblocks]
   in, out[nblocks] back): the FFI-friendly form of the Kernel seam. */
gk_status gk_accumulate_batch_host(gk_ctx* ctx, const gk_table* table, gk_kind kind,
                                   double k_re, double k_im, const double* radii,
                                   const double* weights, size_t block_len, size_t nblocks,
                                   gk_c128* out, uint64_t* fallbacks);

/* Stream-ordered form of gk_eval_batch for pipelines that launch many batches
   back to back (no host synchronisation per call).  `status` is a DEVICE
   array of 2 words that accumulates over calls: status[0] += fallbacks,
   status[1] = min over failing radii of (index << 3 | code).  Initialise it
   with gk_eval_status_reset and read it with gk_eval_status_read, which
   synchronises the context stream and fails like gk_eval_batch would have
   (the index is within the batch that failed). */
gk_status gk_eval_batch_async(gk_ctx* ctx, const gk_table* table, gk_kind kind, double k_re,
                              double k_im, const double* radii, size_t n, gk_c128* out,
                              uint64_t* status);
gk_status gk_eval_status_reset(gk_ctx* ctx, uint64_t* status);
gk_status gk_eval_status_read(gk_ctx* ctx, const uint64_t* status, uint64_t* fallbacks);

/* error_sweep (bounds.hpp:113-186) of a device table: probe_count uniformly
   spaced radii over [r_min, r_max] (endpoints included), the device
   interpolant against the device's analytic evaluation (libdevice sincos,
   within ~1 ulp of glibc).  The device tabulates Exp with linear and Green
   with Lagrange interpolation, so method must be GK_INTERP_LINEAR for Exp
   and GK_INTERP_LAGRANGE for Green (else GK_ERR_INVALID_ARGUMENT). */
typedef enum gk_interp { GK_INTERP_LINEAR = 0, GK_INTERP_LAGRANGE = 1 } gk_interp;
typedef struct gk_sweep_report {
  uint64_t probe_count;
  double max_rel_re, max_rel_im, max_abs, worst_r, max_abs_at_exact_zero;
  uint64_t decade_histogram[24]; /* slot d: relative modulus error in [1e(d-20), 1e(d-19)) */
} gk_sweep_report;
gk_status gk_error_sweep(gk_ctx* ctx, const gk_table* table, gk_kind kind, gk_interp method,
                         uint64_t probe_count, gk_sweep_report* out);

/* locate (table.hpp:87-102) on the device: for each radius the bracketing
   interval j with a_j <= r < a_{j+1} (r = r_max maps to nodes-2).  radii and
   out are device pointers; a radius outside [r_min, r_max] fails with
   GK_ERR_OUT_OF_RANGE naming the first such index. */
gk_status gk_locate(gk_ctx* ctx, const gk_table* table, const double* radii, size_t n,
                    uint32_t* out);

/* gk_eval_batch from HOST buffers (radii[n] in, out[n] back): the FFI-friendly
   form of KernelEvaluator::eval_batch; copies through device memory. */
gk_status gk_eval_batch_host(gk_ctx* ctx, const gk_table* table, gk_kind kind, double k_re,
                             double k_im, const double* radii, size_t n, gk_c128* out,
                             uint64_t* fallbacks);

/* ------------------------------------------------------------------- mesh */
/* Uploads a triangle mesh (host arrays: xyz-interleaved vertices[3 nv],
   triangles[3 nt]) and generates its quadrature points on the device:
   m outer points per triangle (triangle_rule, quadrature.hpp:35-76) and n
   Gauss points on each edge (gauss_legendre_unit, quadrature.hpp:85-110),
   exactly as detail::outer_points / inner_points (matfill.hpp:105-133).
   Validates like TriangleMesh::validate and QuadratureSpec::validate. */
gk_status gk_mesh_create(gk_ctx* ctx, const double* vertices, size_t nv,
                         const uint32_t* triangles, size_t nt, int outer_points,
                         int inner_points_per_edge, gk_mesh** out);
/* gk_mesh_create with explicit shared-edge block options (NULL: defaults) */
gk_status gk_mesh_create_ex(gk_ctx* ctx, const double* vertices, size_t nv,
                            const uint32_t* triangles, size_t nt, int outer_points,
                            int inner_points_per_edge, const gk_mesh_options* opts,
                            gk_mesh** out);
/* host copies: outer[4][nt*m] (x,y,z,w planes), inner[4][nt*3n] */
gk_status gk_mesh_points_download(const gk_mesh* mesh, double* outer, double* inner);
gk_status gk_mesh_destroy(gk_mesh* mesh);

/* Shared-edge blocks of a mesh (no reference counterpart: the direct fill's
   evaluation-sharing structure, DESIGN.md §5 K4e).  blocks = 0 when the mesh
   was created with gk_mesh_options.shared_edges = 0. */
typedef struct gk_mesh_edge_info {
  uint64_t blocks, edge_slots; /* evaluated edge slots incl. warp padding */
  double work_ratio;           /* edge_slots / (3 nt): far-tile work vs the reference */
  double delta;                /* max |point - reversed-edge point| over shared sides */
  double r_far;                /* the shared points serve tiles at least this far apart */
  uint64_t edges;              /* distinct edges summed over blocks (no padding) */
  double rho_mean;             /* mean bounding radius of a block */
  int ordered;                 /* 1: blocks follow a spatial (bisection) order of the triangles */
  double rho_max;              /* largest bounding radius of a block */
  /* the table sweep's block set (K3s; gk_mesh_options.sweep_chunks) */
  uint64_t sweep_blocks, sweep_edge_slots;
  double sweep_work_ratio, sweep_rho_max;
} gk_mesh_edge_info;
gk_status gk_mesh_edge_info_get(const gk_mesh* mesh, gk_mesh_edge_info* out);
/* The host part of the shared-edge blocks, without a device (tests): cut the
   nt triangles into blocks of at most 32 * chunks distinct edges, in mesh
   order (order_mode 0), in a bisection order of the centroids (1), or the
   more compact of the two (-1).  Outputs (caller-allocated):
   order[nt] = the triangle at each block position; edge_index[3 nt] = the
   block-local edge index of each side of the triangle at each position;
   block_start[nt + 1] = first position of each block followed by nt;
   block_edges[nt] = distinct edges of each block; *nblocks; *ordered.
   leaf_pct: bisection leaf size in percent of the edge cap (0: 61); rho_cap > 0:
   bisection leaves wider than rho_cap (vertex radius) are split too. */
gk_status gk_edge_blocks_plan(const double* vertices, size_t nv, const uint32_t* triangles,
                              size_t nt, int chunks, int order_mode, int leaf_pct,
                              double rho_cap, uint32_t* order,
                              uint32_t* edge_index, uint32_t* block_start,
                              uint32_t* block_edges, uint64_t* nblocks, int* ordered);

/* K1: min and max quadrature-point pair distance over observation rows
   [row_begin,row_end) and every source q != p (replaces max_vertex_distance
   + the fixed r_min of bench_compare, matfill.hpp:270 / mesh.hpp:62-68).
   The result is widened by 2^-49 relative on both sides so that every radius
   the fill (or the reference's glibc sqrt) computes lies inside it. */
gk_status gk_distance_range(gk_ctx* ctx, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                            double* r_min, double* r_max);

/* ------------------------------------------------------------------- fill */
/* fill_matrix's fill_rows (matfill.hpp:169-203) for rows [row_begin,row_end):
   z[(p-row_begin)*ldz + q] = sum_o sum_i w_o w_i K(|x_o - x_i|), self pairs 0.
   mode DIRECT = AnalyticKernel{k}, TABLE = TableKernel{table} (k from the
   table).  z is a device pointer.  report == NULL: asynchronous on the
   context stream; otherwise the call synchronizes and fills the report
   (actual_calls = 3 m n rows (N-1), exact fallback count, kernel time).
   opts selects between equivalent kernels (NULL: the context's defaults). */
gk_status gk_fill_rows(gk_ctx* ctx, const gk_mesh* mesh, gk_mode mode, const gk_table* table,
                       gk_kind kind, double k_re, double k_im, size_t row_begin, size_t row_end,
                       gk_c128* z, size_t ldz, const gk_fill_options* opts,
                       gk_fill_report* report);

/* Asynchronous fills (report == NULL) accumulate their fallback, out-of-range
   and zero-distance counts in the context; gk_fill_check synchronises, returns
   the accumulated fallbacks, resets the counts and fails like the synchronous
   call would have (GK_ERR_OUT_OF_RANGE / GK_ERR_DOMAIN) if any fill since the
   last check met such a pair. */
gk_status gk_fill_check(gk_ctx* ctx, uint64_t* fallbacks);

/* Fused Exp + Green fill sharing every radius (and, in TABLE mode, every
   lookup): z_exp gets the PlainExp matrix, z_green the GreenOverR matrix, each
   bit-identical to the separate gk_fill_rows result (both run on the shared
   edges when the separate fills do; with 12 edge chunks per block and more
   than ~200 attenuation entries the pair alone falls back to the
   per-triangle kernel, which agrees to rounding).  The EFIE-type use the
   paper's "several tables" serve.  Reported calls count
   both kernels. */
gk_status gk_fill_rows_pair(gk_ctx* ctx, const gk_mesh* mesh, gk_mode mode,
                            const gk_table* table, double k_re, double k_im, size_t row_begin,
                            size_t row_end, gk_c128* z_exp, gk_c128* z_green, size_t ldz,
                            const gk_fill_options* opts, gk_fill_report* report);

/* fill_matrix<Kernel> (matfill.hpp:144-228) end to end from HOST buffers:
   upload mesh, quadrature points, (TABLE) K1 range when cfg->r_min <= 0 or
   cfg->r_max <= 0, table build, fill, copy Z (nt x nt, row-major) back into
   z_host.  The reference-facing drop-in entry point. */
gk_status gk_fill_matrix_host(gk_ctx* ctx, const double* vertices, size_t nv,
                              const uint32_t* triangles, size_t nt, int outer_points,
                              int inner_points_per_edge, gk_mode mode,
                              const gk_sampling_config* cfg, const gk_medium* medium,
                              gk_kind kind, gk_c128* z_host, gk_fill_report* report);

/* fill_rows into HOST memory: rows [row_begin,row_end) land in
   z_host[(p-row_begin)*ldz_host + q], computed in <= 1 GiB row chunks whose
   device->host copies overlap the fill of the next chunk (double buffer, a
   second stream).  Pinned z_host gets full PCIe bandwidth.  For fills larger
   than host RAM (C5: 107 GB) call it per row range into a reused buffer. */
gk_status gk_fill_rows_host(gk_ctx* ctx, const gk_mesh* mesh, gk_mode mode,
                            const gk_table* table, gk_kind kind, double k_re, double k_im,
                            size_t row_begin, size_t row_end, gk_c128* z_host, size_t ldz_host,
                            const gk_fill_options* opts, gk_fill_report* report);

/* compare_fills (matfill.hpp:237-254) on DEVICE matrices: componentwise max
   relative error of test against ref over `rows` rows of an N-column block
   whose first row is matrix row row_begin (leading dimension ld), skipping
   the diagonal (p == q) and exactly-zero ref components, like the reference
   (NaN errors are ignored as std::max ignores them). */
gk_status gk_compare_fills(gk_ctx* ctx, const gk_c128* test, const gk_c128* ref, size_t rows,
                           size_t N, size_t row_begin, size_t ld, double* max_rel_re,
                           double* max_rel_im);

/* bench_compare (matfill.hpp:262-294) on the device, host mesh in: direct
   fill, then the table fill over a plan with r_max = 1.01 x
   max_vertex_distance (cfg->r_min kept) and the given Lagrange degree, the
   table build charged to the table side; with repeats > 1 the two fills
   interleave and the fastest device time per side counts; compare_fills of
   the two matrices.  Needs 2 N^2 x 16 B of device memory, like the
   reference's two host matrices. */
typedef struct gk_bench_report {
  gk_fill_report fill; /* the table fill's report (wall_time_s: its fastest) */
  double max_rel_re, max_rel_im;
  double speedup;         /* analytic_time_s / interp_time_s */
  double analytic_time_s; /* fastest direct fill (device time) */
  double interp_time_s;   /* fastest table fill + table build */
  double table_build_s;   /* device table build */
} gk_bench_report;
gk_status gk_bench_compare(gk_ctx* ctx, const double* vertices, size_t nv,
                           const uint32_t* triangles, size_t nt, int outer_points,
                           int inner_points_per_edge, const gk_medium* medium,
                           const gk_sampling_config* cfg, int lagrange_degree, gk_kind kind,
                           int repeats, gk_bench_report* out);

/* max_vertex_distance (mesh.hpp:62-68) of a device mesh: exact O(V^2) scan,
   bit-identical to the reference (its r_max convention in bench_compare,
   matfill.hpp:270, is 1.01 x this). */
gk_status gk_max_vertex_distance(gk_ctx* ctx, const gk_mesh* mesh, double* out);

/* ------------------------------------------- peer memory (fused fill+gather)
   The optional gather of Z fused into the fill: the destination
   rank allocates the full matrix with gk_shared_alloc and sends the 64-byte
   IPC handle to the other ranks (any transport), they map it with
   gk_ipc_open, and every rank's gk_fill_rows stores its row block straight
   into that matrix (NVLink peer stores on one node; no separate gather).
   gk_ipc_open'ed pointers are released with gk_ipc_close, the allocation
   with gk_shared_free after every rank has closed it. */
#define GK_IPC_HANDLE_BYTES 64
gk_status gk_shared_alloc(gk_ctx* ctx, size_t bytes, void** dptr,
                          unsigned char handle[GK_IPC_HANDLE_BYTES]);
gk_status gk_shared_free(gk_ctx* ctx, void* dptr);
gk_status gk_ipc_open(gk_ctx* ctx, const unsigned char handle[GK_IPC_HANDLE_BYTES], void** dptr);
gk_status gk_ipc_close(gk_ctx* ctx, void* dptr);

/* ------------------------------------------ multi-GPU row blocks (NCCL)
   The reference's row chunking (matfill.hpp:206-221: chunk = ceil(N /
   threads), contiguous) as one rank per GPU.  A gk_comm wraps an NCCL
   communicator on its context's device.  Either every process calls
   gk_comm_init with the same 128-byte id (made once by gk_comm_unique_id and
   shipped by the caller over any transport), or one process drives several
   GPUs with gk_comm_init_all (one context per device; then every per-rank
   call below must be issued from its own host thread, since NCCL
   collectives across ranks block until all ranks have joined). */
typedef struct gk_comm gk_comm;
#define GK_COMM_ID_BYTES 128
/* rows [begin, end) of `rank` out of `nranks` (host-only, no device) */
gk_status gk_rows_of(uint64_t N, int nranks, int rank, uint64_t* row_begin, uint64_t* row_end);
gk_status gk_comm_unique_id(unsigned char id[GK_COMM_ID_BYTES]);
gk_status gk_comm_init(gk_ctx* ctx, const unsigned char id[GK_COMM_ID_BYTES], int nranks,
                       int rank, gk_comm** out);
gk_status gk_comm_init_all(gk_ctx* const* ctxs, int n, gk_comm** comms);
gk_status gk_comm_destroy(gk_comm* comm);
gk_status gk_comm_info(const gk_comm* comm, int* nranks, int* rank);
/* K1 over this rank's rows + one 16-byte ncclAllReduce(MIN) of
   {min d^2, -max d^2} on the device: the global range of gk_distance_range
   (same widening), identical on every rank */
gk_status gk_distance_range_global(gk_ctx* ctx, gk_comm* comm, const gk_mesh* mesh,
                                   double* r_min, double* r_max);
/* One rank's share of fill_matrix (matfill.hpp:144-228) over the rows
   gk_rows_of gives it: TABLE mode computes the global range when cfg->r_min
   or cfg->r_max <= 0 (gk_distance_range_global), builds the table (identical
   on every rank) and fills; DIRECT fills.  z_rows (device) receives this
   rank's rows with leading dimension ldz; report (NULL: asynchronous) covers
   this rank's rows; r_range (may be NULL) receives the table range used. */
gk_status gk_fill_sharded(gk_ctx* ctx, gk_comm* comm, const gk_mesh* mesh, gk_mode mode,
                          const gk_sampling_config* cfg, const gk_medium* medium, gk_kind kind,
                          gk_c128* z_rows, size_t ldz, const gk_fill_options* opts,
                          gk_fill_report* report, double r_range[2]);
/* The optional gather: every rank's row block (z_rows,
   rows x N, leading dimension N, device) lands in its row slice of root's
   N x N device matrix z_full (grouped ncclSend / ncclRecv, no staging). */
gk_status gk_gather_rows(gk_ctx* ctx, gk_comm* comm, const gk_c128* z_rows, uint64_t N, int root,
                         gk_c128* z_full);

/* predicted_calls (matfill.hpp:50-56): 3 m n N^2 with the overflow guard */
gk_status gk_predicted_calls(uint64_t N, uint64_t m, uint64_t n, uint64_t* out);

/* ------------------------------------------------- workload generators (host)
   generate_sphere_mesh (mesh.hpp:154-202), bit-identical; two-call pattern:
   pass NULL arrays to get nv/nt first.  Plate and jitter are the benchmark's
   synthetic-workload generators (not in the reference). */
gk_status gk_sphere_mesh(double radius, int subdivisions, double* vertices, size_t* nv,
                         uint32_t* triangles, size_t* nt);
gk_status gk_plate_mesh(double side, int cells, double* vertices, size_t* nv,
                        uint32_t* triangles, size_t* nt);
/* splitmix64(seed) per coordinate, U(-amp, amp) from the top 53 bits */
gk_status gk_jitter(double* vertices, size_t nv, uint64_t seed, double amp);

/* ------------------------------------------------------------ measurement */
/* DFMA throughput microbenchmark on the context's device: FP64 TFLOP/s with
   an FMA counted as 2 flops (the fill's roofline denominator). */
gk_status gk_bench_fp64_peak(gk_ctx* ctx, double* tflops);
/* Number of kernels this library has launched in this process (its own
   kernels plus the CUB kernels of the table build), for launch accounting. */
uint64_t gk_launch_count(void);
/* SM count and clock of the context's device */
gk_status gk_device_info(gk_ctx* ctx, int* sm_count, int* sm_clock_khz, int* cc_major,
                         int* cc_minor);

#ifdef __cplusplus
}
#endif
#endif /* GK_GK_H */
