/*
 * gk_oracle.h -- CPU restatement of the gktab reference (arXiv 1901.04162).
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the parity checker for the
 * B200 product (libgk).  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load it.  The product
 * path never links, loads or calls anything under oracle/.
 *
 * Every function restates one reference function with the same IEEE
 * operation order (compiled with -ffp-contract=off, no FMA), so on x86-64 it
 * reproduces the reference bit for bit; tests/test_oracle_vs_ref.py pins that
 * against oracle/_ref/libgkref.so (the reference headers compiled in place)
 * and tests/golden/ (fixtures generated from the reference itself).
 *
 * Status codes mirror the reference's exception types:
 *   0 ok, 1 invalid_argument, 2 domain_error, 3 out_of_range,
 *   4 overflow_error, 5 runtime_error.
 */
#ifndef GK_ORACLE_H
#define GK_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { GO_OK = 0, GO_INVALID = 1, GO_DOMAIN = 2, GO_RANGE = 3, GO_OVERFLOW = 4, GO_RUNTIME = 5 };
enum { GO_EXP = 0, GO_GREEN = 1 };

typedef struct { double re, im; } go_c128;

/* kernel.hpp:25-44 */
typedef struct { double lambda0, eps_r, mu_r; } go_medium;
int go_wavenumber(const go_medium* m, double* k);
/* kernel.hpp:48-61 */
int go_eval_analytic(int kind, double k, double r, go_c128* out);
/* complex-k extension (C4; no reference counterpart): exp(-jkr), k = k_re + j k_im */
int go_eval_analytic_ck(int kind, double k_re, double k_im, double r, go_c128* out);

/* eval_analytic elementwise (test sweeps): status of the first failure */
int go_eval_analytic_batch(int kind, double k, double k_im, const double* r, size_t n,
                           go_c128* out);

/* sampling.hpp:18-45 */
typedef struct {
  double r_min, r_max;
  int samples_per_wavelength;
  int refine_interval_divisor;
  double refine_halfwidth_in_t;
  double dedup_fraction;
  int refine;
} go_sampling_cfg;
void go_sampling_cfg_default(go_sampling_cfg* c);
int go_sampling_cfg_validate(const go_sampling_cfg* c);

/* sampling.hpp:112-141 */
int go_base_interval(const go_medium* m, int S, double* t);
/* returns count; writes up to cap zeros */
int go_zero_crossings(double k, double r_min, double r_max, double* out, size_t cap, size_t* count);

/* sampling.hpp:48-105, 149-236.  Arrays are malloc'ed; free with go_plan_free. */
typedef struct {
  double* absc;
  size_t n;
  double* zeros;
  size_t nz;
  double t, dr_min;
} go_plan;
int go_build_plan(const go_sampling_cfg* c, const go_medium* m, go_plan* out);
/* core with explicit (k used for zeros, nominal t): the complex-k extension
   calls it with k_zero = Re k and t_nominal = lambda0/(S*Re sqrt(eps*mu)). */
int go_build_plan_core(const go_sampling_cfg* c, double k_zero, double t_nominal, go_plan* out);
int go_make_plan(const double* absc, size_t n, const double* zeros, size_t nz, go_plan* out);
int go_plan_copy_out(const go_plan* p, double* absc, double* zeros);
void go_plan_free(go_plan* p);

/* table.hpp:40-82 */
typedef struct {
  double r_min, r_max, dr_min, inv_dr_min;
  uint32_t* buckets;
  size_t nb;
} go_hash;
int go_build_hash(const go_plan* p, go_hash* out);
void go_hash_free(go_hash* h);
/* table.hpp:87-102 */
int go_locate(const go_hash* h, const go_plan* p, double r, size_t* j);

/* evaluator.hpp:102-309 (opaque) */
typedef struct go_evaluator go_evaluator;
/* k_im != 0 selects the complex-k table values (extension). */
go_evaluator* go_evaluator_create(const double* absc, size_t n, const double* zeros, size_t nz,
                                  double k, double k_im, int degree, int* status);
void go_evaluator_free(go_evaluator* ev);
size_t go_evaluator_size(const go_evaluator* ev);
const go_plan* go_evaluator_plan(const go_evaluator* ev);
const go_hash* go_evaluator_hash(const go_evaluator* ev);
int go_evaluator_tables(const go_evaluator* ev, go_c128* exp_vals, go_c128* green_vals);
uint64_t go_evaluator_fallbacks(const go_evaluator* ev);
int go_eval_exp(const go_evaluator* ev, double r, go_c128* out);
int go_eval_green(const go_evaluator* ev, double r, go_c128* out);
int go_eval_kernel(go_evaluator* ev, int kind, double r, go_c128* out);
/* evaluator.hpp:209-221; on failure *fail_index = failing radius index */
int go_eval_batch(go_evaluator* ev, int kind, const double* r, size_t n, go_c128* out,
                  size_t* fail_index);
/* evaluator.hpp:22-95 (generic paths used by sweeps and bounds) */
int go_interp_linear(const go_evaluator* ev, int kind, double r, go_c128* out);
int go_interp_lagrange(const go_evaluator* ev, int kind, int degree, double r, go_c128* out);
/* evaluator.hpp:150-194 */
int go_accumulate_green(go_evaluator* ev, const double* r, const double* w, size_t n, go_c128* out);

/* quadrature.hpp:35-110 */
int go_triangle_rule(int m, double* b0, double* b1, double* b2, double* w);
int go_gauss_legendre_unit(int n, double* x, double* w);

/* mesh.hpp:33-68, 154-202.  Vertices xyz-interleaved (3*nv), triangles (3*nt). */
int go_sphere_mesh(double radius, int subdivisions, double** verts, size_t* nv, uint32_t** tris,
                   size_t* nt);
/* workload generators (not in the reference; SURVEY 8c "portable jitter"):
   splitmix64(seed) per coordinate, U(-amp, amp) from the top 53 bits. */
void go_jitter(double* verts, size_t nv, uint64_t seed, double amp);
int go_plate_mesh(double side, int cells, double** verts, size_t* nv, uint32_t** tris, size_t* nt);
void go_mesh_free(double* verts, uint32_t* tris);
int go_mesh_validate(const double* verts, size_t nv, const uint32_t* tris, size_t nt);
double go_max_vertex_distance(const double* verts, size_t nv);
double go_triangle_area(const double* verts, const uint32_t* tri);

/* matfill.hpp:93-133: SoA points (x,y,z,w), sizes nt*m and nt*3n */
int go_outer_points(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                    double* x, double* y, double* z, double* w);
int go_inner_points(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int n,
                    double* x, double* y, double* z, double* w);

/* matfill.hpp:33-56 */
typedef struct {
  uint64_t N;
  int m, n;
  uint64_t predicted_calls, actual_calls, fallback_calls;
  double wall_time_s;
} go_fill_report;
int go_predicted_calls(uint64_t N, uint64_t m, uint64_t n, uint64_t* out);

/* matfill.hpp:144-228.  mode 0 = AnalyticKernel{k} (k_im extension),
   mode 1 = TableKernel{ev}.  Rows [row_begin,row_end) are filled into
   z[(p-row_begin)*ldz + q]; the reference fills all rows (0, N). */
enum { GO_MODE_DIRECT = 0, GO_MODE_TABLE = 1 };
int go_fill_rows(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m, int n,
                 int mode, double k, double k_im, go_evaluator* ev, int kind, int threads,
                 size_t row_begin, size_t row_end, go_c128* z, size_t ldz, go_fill_report* rep);

/* matfill.hpp:237-254 */
int go_compare_fills(const go_c128* test, const go_c128* ref, size_t n, double* max_rel_re,
                     double* max_rel_im);

/* bounds.hpp:37-111 */
int go_derivative_bound(int kind, double k, double r_low, int order, double* out);
int go_linear_bound(double h, int kind, double k, double r_low, double* out);
int go_lagrange_bound(const double* stencil, size_t n, double r, int kind, double k, double* out);
int go_pointwise_bound(const go_evaluator* ev, int kind, int method, double r, double* out);

/* Parity tolerance: for rows [row_begin,row_end),
   B[p][q] = sum_{o,i} |w_o w_i| (pw(r) + ulps * 2^-53 * (1 + |k| r) / r)
   where pw = pointwise_bound(ev, Green, Lagrange, r) when ev != NULL (table
   mode), 0 otherwise (direct mode).  k_abs = |k|. */
int go_entry_bounds(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m, int n,
                    const go_evaluator* ev, double k_abs, double ulps, size_t row_begin,
                    size_t row_end, double* bound, size_t ldb);

/* The same bound for an arbitrary list of rows (bound[r * ldb + q] for
   p = rows[r]), split over `threads` pthreads: full-size sampled-row parity. */
int go_entry_bounds_rows(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                         int n, const go_evaluator* ev, double k_abs, double ulps,
                         const uint64_t* rows, size_t nrows, int threads, double* bound,
                         size_t ldb);

/* Exact min / max quadrature-point pair distance over rows [row_begin,row_end)
   and all q != p (the K1 oracle; brute force). */
int go_distance_range(const double* verts, size_t nv, const uint32_t* tris, size_t nt, int m,
                      int n, size_t row_begin, size_t row_end, double* r_min, double* r_max);

#ifdef __cplusplus
}
#endif
#endif
