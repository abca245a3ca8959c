// ref_shim.cpp -- extern "C" wrappers around the UNMODIFIED gktab reference
// headers, compiled in place from /root/reference/proj/include by
// oracle/Makefile into oracle/_ref/libgkref.so.
//
// TEST INFRASTRUCTURE ONLY: the oracle's pin (tests/test_oracle_vs_ref.py),
// the golden-fixture generator (tests/golden/make_golden.py) and the
// reference arm of bench.py ("cpu_baseline.kind": "reference").  No reference
// source is copied; this file only calls into it.  Exceptions map to the
// status codes of oracle/gk_oracle.h.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <stdexcept>
#include <thread>
#include <vector>

#include "gktab/gktab.hpp"

using namespace gktab;

namespace {

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range&) {
    return 3;
  } catch (const std::domain_error&) {
    return 2;
  } catch (const std::invalid_argument&) {
    return 1;
  } catch (const std::overflow_error&) {
    return 4;
  } catch (const std::exception&) {
    return 5;
  }
}

struct Cfg {
  double r_min, r_max;
  int samples_per_wavelength, refine_interval_divisor;
  double refine_halfwidth_in_t, dedup_fraction;
  int refine;
};

SamplingConfig to_cfg(const Cfg* c) {
  SamplingConfig s;
  s.r_min = c->r_min;
  s.r_max = c->r_max;
  s.samples_per_wavelength = c->samples_per_wavelength;
  s.refine_interval_divisor = c->refine_interval_divisor;
  s.refine_halfwidth_in_t = c->refine_halfwidth_in_t;
  s.dedup_fraction = c->dedup_fraction;
  s.refine = c->refine != 0;
  return s;
}

TriangleMesh to_mesh(const double* v, size_t nv, const uint32_t* t, size_t nt) {
  TriangleMesh m;
  m.vertices.resize(nv);
  for (size_t i = 0; i < nv; ++i) m.vertices[i] = {v[3 * i], v[3 * i + 1], v[3 * i + 2]};
  m.triangles.resize(nt);
  for (size_t i = 0; i < nt; ++i) m.triangles[i] = {t[3 * i], t[3 * i + 1], t[3 * i + 2]};
  return m;
}

struct Report {
  uint64_t N;
  int m, n;
  uint64_t predicted_calls, actual_calls, fallback_calls;
  double wall_time_s;
};

void to_report(const FillReport& r, Report* out) {
  out->N = r.N;
  out->m = r.m;
  out->n = r.n;
  out->predicted_calls = r.predicted_calls;
  out->actual_calls = r.actual_calls;
  out->fallback_calls = r.fallback_calls;
  out->wall_time_s = r.wall_time_s;
}

}  // namespace

extern "C" {

int gr_wavenumber(const double* medium, double* k) {
  return guarded([&] { *k = wavenumber(Medium{medium[0], medium[1], medium[2]}); });
}

int gr_eval_analytic(int kind, double k, double r, double* out) {
  return guarded([&] {
    const Complex v = eval_analytic(static_cast<KernelKind>(kind), k, r);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int gr_base_interval(const double* medium, int S, double* t) {
  return guarded([&] { *t = base_interval(Medium{medium[0], medium[1], medium[2]}, S); });
}

int gr_zero_crossings(double k, double r_min, double r_max, double* out, size_t cap,
                      size_t* count) {
  return guarded([&] {
    const auto z = zero_crossings(k, r_min, r_max);
    *count = z.size();
    std::copy_n(z.begin(), std::min(cap, z.size()), out);
  });
}

// build_plan -> opaque handle
void* gr_plan_create(const Cfg* cfg, const double* medium, int* status) {
  SamplingPlan* p = nullptr;
  *status = guarded([&] {
    p = new SamplingPlan(build_plan(to_cfg(cfg), Medium{medium[0], medium[1], medium[2]}));
  });
  return p;
}

void* gr_make_plan(const double* absc, size_t n, const double* zeros, size_t nz, int* status) {
  SamplingPlan* p = nullptr;
  *status = guarded([&] {
    p = new SamplingPlan(make_plan(std::vector<double>(absc, absc + n),
                                   std::vector<double>(zeros, zeros + nz)));
  });
  return p;
}

void gr_plan_info(const void* h, size_t* n, size_t* nz, double* t, double* dr_min) {
  const auto* p = static_cast<const SamplingPlan*>(h);
  *n = p->abscissae.size();
  *nz = p->zero_locations.size();
  *t = p->t;
  *dr_min = p->dr_min;
}

void gr_plan_copy(const void* h, double* absc, double* zeros) {
  const auto* p = static_cast<const SamplingPlan*>(h);
  std::copy(p->abscissae.begin(), p->abscissae.end(), absc);
  std::copy(p->zero_locations.begin(), p->zero_locations.end(), zeros);
}

void gr_plan_free(void* h) { delete static_cast<SamplingPlan*>(h); }

int gr_build_hash(const void* h, size_t* nb, uint32_t* buckets, size_t cap, double* dr_min,
                  double* inv_dr_min) {
  return guarded([&] {
    const HashIndex hash = build_hash(*static_cast<const SamplingPlan*>(h));
    *nb = hash.buckets.size();
    *dr_min = hash.dr_min;
    *inv_dr_min = hash.inv_dr_min;
    if (buckets) std::copy_n(hash.buckets.begin(), std::min(cap, hash.buckets.size()), buckets);
  });
}

int gr_locate(const void* h, const double* r, size_t n, size_t* out) {
  return guarded([&] {
    const auto& plan = *static_cast<const SamplingPlan*>(h);
    const HashIndex hash = build_hash(plan);
    for (size_t i = 0; i < n; ++i) out[i] = locate(hash, plan, r[i]);
  });
}

// KernelEvaluator from explicit abscissae (make_plan) -> opaque handle
void* gr_evaluator_create(const double* absc, size_t n, const double* zeros, size_t nz, double k,
                          int degree, int* status) {
  KernelEvaluator* ev = nullptr;
  *status = guarded([&] {
    ev = new KernelEvaluator(make_plan(std::vector<double>(absc, absc + n),
                                       std::vector<double>(zeros, zeros + nz)),
                             k, degree);
  });
  return ev;
}

void gr_evaluator_free(void* h) { delete static_cast<KernelEvaluator*>(h); }

uint64_t gr_fallbacks(const void* h) {
  return static_cast<const KernelEvaluator*>(h)->fallback_count();
}

void gr_tables(const void* h, double* exp_vals, double* green_vals) {
  const auto* ev = static_cast<const KernelEvaluator*>(h);
  const size_t n = ev->plan().size();
  for (size_t i = 0; i < n; ++i) {
    exp_vals[2 * i] = ev->exp_table().values[i].real();
    exp_vals[2 * i + 1] = ev->exp_table().values[i].imag();
    green_vals[2 * i] = ev->green_table().values[i].real();
    green_vals[2 * i + 1] = ev->green_table().values[i].imag();
  }
}

int gr_eval_kernel(void* h, int kind, double r, double* out) {
  return guarded([&] {
    const Complex v =
        static_cast<const KernelEvaluator*>(h)->eval_kernel(static_cast<KernelKind>(kind), r);
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int gr_eval_batch(void* h, int kind, const double* r, size_t n, double* out) {
  return guarded([&] {
    const auto v = static_cast<const KernelEvaluator*>(h)->eval_batch(
        static_cast<KernelKind>(kind), std::span<const double>(r, n));
    std::memcpy(out, v.data(), v.size() * sizeof(Complex));
  });
}

int gr_eval_batch_threaded(void* h, int kind, const double* r, size_t n, double* out,
                           int threads) {
  std::vector<int> st(static_cast<size_t>(threads), 0);
  std::vector<std::thread> ws;
  const size_t chunk = (n + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    const size_t b = w * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    ws.emplace_back([&, b, e, w] {
      st[w] = gr_eval_batch(h, kind, r + b, e - b, out + 2 * b);
    });
  }
  for (auto& t : ws) t.join();
  for (int s : st)
    if (s) return s;
  return 0;
}

int gr_analytic_batch_threaded(int kind, double k, const double* r, size_t n, double* out,
                               int threads) {
  std::vector<int> st(static_cast<size_t>(threads), 0);
  std::vector<std::thread> ws;
  const size_t chunk = (n + threads - 1) / threads;
  for (int w = 0; w < threads; ++w) {
    const size_t b = w * chunk, e = std::min(n, b + chunk);
    if (b >= e) break;
    ws.emplace_back([&, b, e, w] {
      st[w] = guarded([&] {
        for (size_t i = b; i < e; ++i) {
          const Complex v = eval_analytic(static_cast<KernelKind>(kind), k, r[i]);
          out[2 * i] = v.real();
          out[2 * i + 1] = v.imag();
        }
      });
    });
  }
  for (auto& t : ws) t.join();
  for (int s : st)
    if (s) return s;
  return 0;
}

int gr_accumulate_green(void* h, const double* r, const double* w, size_t n, double* out) {
  return guarded([&] {
    const Complex v = static_cast<const KernelEvaluator*>(h)->accumulate_green(
        std::span<const double>(r, n), std::span<const double>(w, n));
    out[0] = v.real();
    out[1] = v.imag();
  });
}

int gr_pointwise_bound(void* h, int kind, int method, double r, double* out) {
  return guarded([&] {
    *out = pointwise_bound(*static_cast<const KernelEvaluator*>(h), static_cast<KernelKind>(kind),
                           method == 0 ? InterpMethod::Linear : InterpMethod::Lagrange, r);
  });
}

int gr_derivative_bound(int kind, double k, double r_low, int order, double* out) {
  return guarded(
      [&] { *out = derivative_bound(static_cast<KernelKind>(kind), k, r_low, order); });
}

int gr_triangle_rule(int m, double* b0, double* b1, double* b2, double* w) {
  return guarded([&] {
    const auto rule = triangle_rule(m);
    for (size_t i = 0; i < rule.size(); ++i) {
      b0[i] = rule[i].b0;
      b1[i] = rule[i].b1;
      b2[i] = rule[i].b2;
      w[i] = rule[i].w;
    }
  });
}

int gr_gauss_legendre_unit(int n, double* x, double* w) {
  return guarded([&] {
    const auto g = gauss_legendre_unit(n);
    for (size_t i = 0; i < g.size(); ++i) {
      x[i] = g[i].x;
      w[i] = g[i].w;
    }
  });
}

// generate_sphere_mesh: first call with verts == nullptr returns the counts
int gr_sphere_mesh(double radius, int subdivisions, double* verts, size_t* nv, uint32_t* tris,
                   size_t* nt) {
  return guarded([&] {
    const TriangleMesh m = generate_sphere_mesh(radius, subdivisions);
    *nv = m.vertices.size();
    *nt = m.triangles.size();
    if (!verts) return;
    for (size_t i = 0; i < m.vertices.size(); ++i) {
      verts[3 * i] = m.vertices[i].x;
      verts[3 * i + 1] = m.vertices[i].y;
      verts[3 * i + 2] = m.vertices[i].z;
    }
    for (size_t i = 0; i < m.triangles.size(); ++i)
      for (int c = 0; c < 3; ++c) tris[3 * i + c] = m.triangles[i][static_cast<size_t>(c)];
  });
}

double gr_max_vertex_distance(const double* v, size_t nv) {
  return max_vertex_distance(to_mesh(v, nv, nullptr, 0));
}

int gr_points(const double* v, size_t nv, const uint32_t* t, size_t nt, int m, int n,
              double* outer /*4 x nt*m*/, double* inner /*4 x nt*3n*/) {
  return guarded([&] {
    const TriangleMesh mesh = to_mesh(v, nv, t, nt);
    const auto o = detail::outer_points(mesh, m);
    const auto i = detail::inner_points(mesh, n);
    const size_t no = o.x.size(), ni = i.x.size();
    std::copy(o.x.begin(), o.x.end(), outer);
    std::copy(o.y.begin(), o.y.end(), outer + no);
    std::copy(o.z.begin(), o.z.end(), outer + 2 * no);
    std::copy(o.w.begin(), o.w.end(), outer + 3 * no);
    std::copy(i.x.begin(), i.x.end(), inner);
    std::copy(i.y.begin(), i.y.end(), inner + ni);
    std::copy(i.z.begin(), i.z.end(), inner + 2 * ni);
    std::copy(i.w.begin(), i.w.end(), inner + 3 * ni);
  });
}

// fill_matrix<AnalyticKernel|TableKernel> over the whole mesh (matfill.hpp:144-228)
int gr_fill_matrix(const double* v, size_t nv, const uint32_t* t, size_t nt, int m, int n,
                   int mode, double k, void* ev, int kind, int threads, double* z,
                   Report* report) {
  return guarded([&] {
    const TriangleMesh mesh = to_mesh(v, nv, t, nt);
    const QuadratureSpec spec{m, n};
    const auto kk = static_cast<KernelKind>(kind);
    auto res = mode == 0
                   ? fill_matrix(mesh, spec, AnalyticKernel{k}, kk, threads)
                   : fill_matrix(mesh, spec,
                                 TableKernel{static_cast<const KernelEvaluator*>(ev)}, kk, threads);
    std::memcpy(z, res.first.z.data(), res.first.z.size() * sizeof(Complex));
    to_report(res.second, report);
  });
}

// Row-sampled fill for configurations too large for a full CPU fill
// (SURVEY 8d): the given rows go through the reference's own
// AnalyticKernel/TableKernel::accumulate with fill_rows' staging loop
// (matfill.hpp:185-199) restated around them; rows are split over threads.
int gr_fill_sampled_rows(const double* v, size_t nv, const uint32_t* t, size_t nt, int m, int n,
                         int mode, double k, void* ev, int kind, int threads,
                         const uint64_t* rows, size_t nrows, double* z /*nrows x nt*/,
                         uint64_t* calls, double* wall_s) {
  return guarded([&] {
    const TriangleMesh mesh = to_mesh(v, nv, t, nt);
    QuadratureSpec{m, n}.validate();
    mesh.validate();
    const auto outer = detail::outer_points(mesh, m);
    const auto inner = detail::inner_points(mesh, n);
    const size_t N = nt, mm = static_cast<size_t>(m), ipt = static_cast<size_t>(3 * n);
    const auto kk = static_cast<KernelKind>(kind);
    const AnalyticKernel ak{k};
    const TableKernel tk{static_cast<const KernelEvaluator*>(ev)};
    std::vector<uint64_t> per(static_cast<size_t>(threads), 0);
    auto work = [&](size_t rb, size_t re, uint64_t& c) {
      const size_t block = mm * ipt;
      std::vector<double> br(block), bw(block);
      for (size_t ri = rb; ri < re; ++ri) {
        const size_t p = rows[ri];
        Complex* dst = reinterpret_cast<Complex*>(z) + ri * N;
        dst[p] = Complex(0.0, 0.0);
        for (size_t q = 0; q < N; ++q) {
          if (q == p) continue;
          size_t idx = 0;
          for (size_t o = 0; o < mm; ++o) {
            const size_t oi = p * mm + o;
            for (size_t i = 0; i < ipt; ++i) {
              const size_t ii = q * ipt + i;
              const double dx = outer.x[oi] - inner.x[ii];
              const double dy = outer.y[oi] - inner.y[ii];
              const double dz = outer.z[oi] - inner.z[ii];
              br[idx] = std::sqrt(dx * dx + dy * dy + dz * dz);
              bw[idx] = outer.w[oi] * inner.w[ii];
              ++idx;
            }
          }
          dst[q] = mode == 0 ? ak.accumulate(kk, br, bw) : tk.accumulate(kk, br, bw);
          c += block;
        }
      }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> ws;
    const size_t chunk = (nrows + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
      const size_t b = w * chunk, e = std::min(nrows, b + chunk);
      if (b >= e) break;
      ws.emplace_back(work, b, e, std::ref(per[static_cast<size_t>(w)]));
    }
    for (auto& th : ws) th.join();
    const auto t1 = std::chrono::steady_clock::now();
    *wall_s = std::chrono::duration<double>(t1 - t0).count();
    *calls = 0;
    for (auto c : per) *calls += c;
  });
}

// io.hpp wire formats through the reference's own writers / reader
int gr_dump_plan_csv(const double* absc, size_t n, const double* zeros, size_t nz,
                     const char* path) {
  return guarded([&] {
    const SamplingPlan plan = make_plan(std::vector<double>(absc, absc + n),
                                        std::vector<double>(zeros, zeros + nz));
    std::ofstream out(path);
    dump_plan_csv(plan, out);
  });
}

// write_bench_csv (io.hpp:147-156) of a report with the given fields -> path
int gr_write_bench_csv(const uint64_t* ints /* N,m,n,pred,actual,fallback */,
                       const double* dbls /* analytic,interp,speedup,re,im */, const char* path) {
  return guarded([&] {
    FillReport rep;
    rep.N = static_cast<std::size_t>(ints[0]);
    rep.m = static_cast<int>(ints[1]);
    rep.n = static_cast<int>(ints[2]);
    rep.predicted_calls = ints[3];
    rep.actual_calls = ints[4];
    rep.fallback_calls = ints[5];
    rep.analytic_time_s = dbls[0];
    rep.interp_time_s = dbls[1];
    rep.speedup = dbls[2];
    rep.max_rel_re = dbls[3];
    rep.max_rel_im = dbls[4];
    std::ofstream out(path);
    write_bench_csv(out, rep);
  });
}

// write_sweep_csv_header + _row (io.hpp:134-145) -> path
int gr_write_sweep_csv(int kind, int method, int degree, uint64_t probes,
                       const double* dbls /* re,im,abs,worst_r */, const char* path) {
  return guarded([&] {
    ErrorSweepReport rep;
    rep.probe_count = static_cast<std::size_t>(probes);
    rep.max_rel_re = dbls[0];
    rep.max_rel_im = dbls[1];
    rep.max_abs = dbls[2];
    rep.worst_r = dbls[3];
    std::ofstream out(path);
    write_sweep_csv_header(out);
    write_sweep_csv_row(out, kind == 0 ? KernelKind::PlainExp : KernelKind::GreenOverR,
                        method == 0 ? InterpMethod::Linear : InterpMethod::Lagrange, degree, rep);
  });
}

// error_sweep (bounds.hpp:128-186) of a reference evaluator: dbls[0..5] =
// max_rel_re, max_rel_im, max_abs, worst_r, max_abs_at_exact_zero; hist[24]
int gr_error_sweep(void* h, int kind, int method, uint64_t probes, double* dbls,
                   uint64_t* hist) {
  return guarded([&] {
    const auto* ev = static_cast<const KernelEvaluator*>(h);
    const ErrorSweepReport r =
        error_sweep(*ev, kind == 0 ? KernelKind::PlainExp : KernelKind::GreenOverR,
                    method == 0 ? InterpMethod::Linear : InterpMethod::Lagrange,
                    static_cast<std::size_t>(probes));
    dbls[0] = r.max_rel_re;
    dbls[1] = r.max_rel_im;
    dbls[2] = r.max_abs;
    dbls[3] = r.worst_r;
    dbls[4] = r.max_abs_at_exact_zero;
    for (int d = 0; d < 24; ++d) hist[d] = r.decade_histogram[d];
  });
}

int gr_dump_table_binary(void* h, int kind, const char* path) {
  return guarded([&] {
    const auto* ev = static_cast<const KernelEvaluator*>(h);
    std::ofstream out(path, std::ios::binary);
    dump_table_binary(kind == 0 ? ev->exp_table() : ev->green_table(), ev->plan(), out);
  });
}

// load_table_binary (io.hpp:105-132): counts first (radii == nullptr), then data
int gr_load_table_binary(const char* path, int* kind, double* k, size_t* count, double* radii,
                         double* values) {
  return guarded([&] {
    std::ifstream in(path, std::ios::binary);
    const TableDump d = load_table_binary(in);
    *kind = static_cast<int>(d.kind);
    *k = d.k;
    *count = d.radii.size();
    if (!radii) return;
    std::copy(d.radii.begin(), d.radii.end(), radii);
    std::memcpy(values, d.values.data(), d.values.size() * sizeof(Complex));
  });
}

int gr_compare_fills(const double* test, const double* ref, size_t n, double* re, double* im) {
  return guarded([&] {
    KernelMatrix a(n), b(n);
    std::memcpy(a.z.data(), test, n * n * sizeof(Complex));
    std::memcpy(b.z.data(), ref, n * n * sizeof(Complex));
    const auto s = compare_fills(a, b);
    *re = s.max_rel_re;
    *im = s.max_rel_im;
  });
}

int gr_predicted_calls(uint64_t N, uint64_t m, uint64_t n, uint64_t* out) {
  return guarded([&] { *out = predicted_calls(N, m, n); });
}

}  // extern "C"
