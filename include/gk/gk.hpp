// gk.hpp -- header-only C++20 adapter over the C ABI (gk.h), shaped like the
// reference library `gktab` (/root/reference/proj/include/gktab/) so code
// written against it switches by changing the namespace and the evaluator:
//
//   gktab::KernelEvaluator ev(build_plan(cfg, medium), k);      // CPU tables
//   auto [Z, rep] = gktab::fill_matrix(mesh, spec, gktab::TableKernel{&ev}, kind);
// becomes
//   gk::Context ctx;                                            // one B200
//   gk::DeviceEvaluator ev(ctx, cfg, medium);                   // tables built on the GPU
//   auto [Z, rep] = gk::fill_matrix(ctx, mesh, spec, gk::Mode::Table, medium, cfg, kind);
//
// Status codes are rethrown as the reference's exception types
// (std::invalid_argument, std::domain_error, std::out_of_range,
// std::overflow_error, std::runtime_error).  Link with -lgk.
#pragma once

#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <mutex>
#include <ostream>
#include <cstdint>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gk/gk.h"

namespace gk {

using Complex = std::complex<double>;
static_assert(sizeof(Complex) == sizeof(gk_c128), "gk_c128 must match std::complex<double>");

enum class KernelKind : std::uint8_t { PlainExp = GK_KIND_EXP, GreenOverR = GK_KIND_GREEN };
enum class Mode { Direct = GK_MODE_DIRECT, Table = GK_MODE_TABLE };

inline void check(gk_status s) {
  switch (s) {
    case GK_OK: return;
    case GK_ERR_INVALID_ARGUMENT: throw std::invalid_argument(gk_last_error());
    case GK_ERR_DOMAIN: throw std::domain_error(gk_last_error());
    case GK_ERR_OUT_OF_RANGE: throw std::out_of_range(gk_last_error());
    case GK_ERR_OVERFLOW: throw std::overflow_error(gk_last_error());
    default: throw std::runtime_error(gk_last_error());
  }
}

// gktab::Medium (kernel.hpp:25-38) + lossy extension
struct Medium {
  double lambda0 = 1.0, eps_r = 1.0, mu_r = 1.0, eps_r_im = 0.0;
  gk_medium c() const { return {lambda0, eps_r, mu_r, eps_r_im}; }
};

// gktab::SamplingConfig (sampling.hpp:18-45), same defaults
struct SamplingConfig {
  double r_min = 1e-4, r_max = 1.0;
  int samples_per_wavelength = 1000;
  int refine_interval_divisor = 2;
  double refine_halfwidth_in_t = 2.0;
  double dedup_fraction = 0.5;
  bool refine = true;
  gk_sampling_config c() const {
    return {r_min, r_max, samples_per_wavelength, refine_interval_divisor, refine_halfwidth_in_t,
            dedup_fraction, refine ? 1 : 0};
  }
};

// gktab::QuadratureSpec (quadrature.hpp:15-26)
struct QuadratureSpec {
  int outer_points = 4;
  int inner_points_per_edge = 3;
};

// gktab::TriangleMesh (mesh.hpp:33-58), flattened xyz / index triples
struct TriangleMesh {
  std::vector<double> vertices;
  std::vector<std::uint32_t> triangles;
  std::size_t triangle_count() const { return triangles.size() / 3; }
};

// gktab::KernelMatrix (matfill.hpp:24-31)
struct KernelMatrix {
  std::size_t n = 0;
  std::vector<Complex> z;
  explicit KernelMatrix(std::size_t size = 0) : n(size), z(size * size) {}
  Complex& at(std::size_t p, std::size_t q) { return z[p * n + q]; }
  const Complex& at(std::size_t p, std::size_t q) const { return z[p * n + q]; }
};

// gktab::FillReport (matfill.hpp:33-47); the last six fields are set by
// bench_compare only
struct FillReport {
  std::size_t N = 0;
  int m = 0, n = 0;
  std::uint64_t predicted_calls = 0, actual_calls = 0, fallback_calls = 0;
  double wall_time_s = 0.0;
  double max_rel_re = 0.0, max_rel_im = 0.0;
  double speedup = 0.0, analytic_time_s = 0.0, interp_time_s = 0.0, table_build_s = 0.0;
  std::uint64_t evaluations = 0;  // device evaluations (<= actual_calls: shared edges)
  static FillReport from(const gk_fill_report& r) {
    FillReport f;
    f.N = static_cast<std::size_t>(r.N);
    f.m = r.m;
    f.n = r.n;
    f.predicted_calls = r.predicted_calls;
    f.actual_calls = r.actual_calls;
    f.fallback_calls = r.fallback_calls;
    f.wall_time_s = r.wall_time_s;
    f.evaluations = r.evaluations;
    return f;
  }
};

// gktab::FillErrorStats / compare_fills (matfill.hpp:230-254), host matrices
struct FillErrorStats {
  double max_rel_re = 0.0;
  double max_rel_im = 0.0;
};
inline FillErrorStats compare_fills(const KernelMatrix& test, const KernelMatrix& ref) {
  if (test.n != ref.n) throw std::invalid_argument("compare_fills: size mismatch");
  FillErrorStats st;
  for (std::size_t p = 0; p < ref.n; ++p)
    for (std::size_t q = 0; q < ref.n; ++q) {
      if (p == q) continue;
      const Complex a = ref.at(p, q), b = test.at(p, q);
      if (a.real() != 0.0)
        st.max_rel_re = std::max(st.max_rel_re, std::abs(b.real() - a.real()) / std::abs(a.real()));
      if (a.imag() != 0.0)
        st.max_rel_im = std::max(st.max_rel_im, std::abs(b.imag() - a.imag()) / std::abs(a.imag()));
    }
  return st;
}

inline double wavenumber(const Medium& m) {
  double re = 0, im = 0;
  const gk_medium c = m.c();
  check(gk_wavenumber(&c, &re, &im));
  return re;
}

inline std::uint64_t predicted_calls(std::uint64_t N, std::uint64_t m, std::uint64_t n) {
  std::uint64_t out = 0;
  check(gk_predicted_calls(N, m, n, &out));
  return out;
}

// generate_sphere_mesh (mesh.hpp:154-202), bit-identical
inline TriangleMesh generate_sphere_mesh(double radius, int subdivisions) {
  std::size_t nv = 0, nt = 0;
  check(gk_sphere_mesh(radius, subdivisions, nullptr, &nv, nullptr, &nt));
  TriangleMesh m;
  m.vertices.resize(3 * nv);
  m.triangles.resize(3 * nt);
  check(gk_sphere_mesh(radius, subdivisions, m.vertices.data(), &nv, m.triangles.data(), &nt));
  return m;
}

// kernel selection (gk_fill_options), every field GK_AUTO by default
inline gk_fill_options default_fill_options() {
  gk_fill_options o;
  gk_fill_options_init(&o);
  return o;
}

// one B200 (RAII over gk_ctx).  A gk_ctx is not re-entrant: objects that may
// be called from several host threads (DeviceEvaluator as the reference's
// Kernel, whose fill_matrix calls accumulate from `threads` workers) take
// mutex() around every call on the context.
class Context {
 public:
  explicit Context(int device = 0) { check(gk_ctx_create(device, &h_)); }
  ~Context() { gk_ctx_destroy(h_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  gk_ctx* get() const { return h_; }
  void set_stream(void* cuda_stream) { check(gk_ctx_set_stream(h_, cuda_stream)); }
  void set_fill_options(const gk_fill_options& o) { check(gk_ctx_set_fill_options(h_, &o)); }
  std::mutex& mutex() const { return mu_; }

 private:
  gk_ctx* h_ = nullptr;
  mutable std::mutex mu_;
};

// gktab::KernelEvaluator (evaluator.hpp:102-309) with its tables on the GPU
// gktab::InterpMethod (bounds.hpp:15) and ErrorSweepReport (bounds.hpp:113-124)
enum class InterpMethod { Linear = GK_INTERP_LINEAR, Lagrange = GK_INTERP_LAGRANGE };
struct ErrorSweepReport {
  std::size_t probe_count = 0;
  double max_rel_re = 0.0, max_rel_im = 0.0, max_abs = 0.0, worst_r = 0.0;
  double max_abs_at_exact_zero = 0.0;
  std::uint64_t decade_histogram[24] = {};
};

class DeviceEvaluator {
 public:
  DeviceEvaluator(Context& ctx, const SamplingConfig& cfg, const Medium& medium = {},
                  int lagrange_degree = 3)
      : ctx_(&ctx) {
    const gk_sampling_config c = cfg.c();
    const gk_medium m = medium.c();
    check(gk_table_build(ctx.get(), &c, &m, lagrange_degree, &h_));
    check(gk_table_info_get(h_, &info_));
  }
  ~DeviceEvaluator() { gk_table_destroy(h_); }
  DeviceEvaluator(const DeviceEvaluator&) = delete;
  DeviceEvaluator& operator=(const DeviceEvaluator&) = delete;

  const gk_table_info& info() const { return info_; }
  gk_table* get() const { return h_; }
  double k() const { return info_.k_re; }
  int lagrange_degree() const { return info_.degree; }
  // relaxed atomic like the reference's counter (evaluator.hpp:100-101, 203)
  std::uint64_t fallback_count() const { return fallbacks_.load(std::memory_order_relaxed); }

  // eval_batch (evaluator.hpp:209-221): host in, host out.  Thread-safe: the
  // device call holds the context's mutex (the reference's evaluator is
  // shared by its fill's worker threads, evaluator.hpp:100-101).
  std::vector<Complex> eval_batch(KernelKind kind, std::span<const double> radii) const {
    std::vector<Complex> out(radii.size());
    std::uint64_t fb = 0;
    {
      std::lock_guard<std::mutex> lock(ctx_->mutex());
      check(gk_eval_batch_host(ctx_->get(), h_, static_cast<gk_kind>(kind), 0.0, 0.0,
                               radii.data(), radii.size(),
                               reinterpret_cast<gk_c128*>(out.data()), &fb));
    }
    fallbacks_.fetch_add(fb, std::memory_order_relaxed);
    return out;
  }
  // Kernel::accumulate of one block (sum_i K(r_i) w_i) on the device; thread-safe
  Complex accumulate(KernelKind kind, std::span<const double> radii,
                     std::span<const double> weights) const {
    Complex out{0.0, 0.0};
    std::uint64_t fb = 0;
    {
      std::lock_guard<std::mutex> lock(ctx_->mutex());
      check(gk_accumulate_batch_host(ctx_->get(), h_, static_cast<gk_kind>(kind), 0.0, 0.0,
                                     radii.data(), weights.data(), radii.size(), 1,
                                     reinterpret_cast<gk_c128*>(&out), &fb));
    }
    fallbacks_.fetch_add(fb, std::memory_order_relaxed);
    return out;
  }
  Complex eval_kernel(KernelKind kind, double r) const {
    return eval_batch(kind, std::span<const double>(&r, 1))[0];
  }
  Complex eval_exp(double r) const { return eval_kernel(KernelKind::PlainExp, r); }
  Complex eval_green(double r) const { return eval_kernel(KernelKind::GreenOverR, r); }

  // error_sweep (bounds.hpp:128-186) of this device table: Exp with Linear,
  // Green with Lagrange (the device's interpolants)
  ErrorSweepReport error_sweep(KernelKind kind, InterpMethod method, std::size_t probes) const {
    gk_sweep_report r{};
    std::lock_guard<std::mutex> lock(ctx_->mutex());
    check(gk_error_sweep(ctx_->get(), h_, static_cast<gk_kind>(kind),
                         static_cast<gk_interp>(method), probes, &r));
    ErrorSweepReport e;
    e.probe_count = static_cast<std::size_t>(r.probe_count);
    e.max_rel_re = r.max_rel_re;
    e.max_rel_im = r.max_rel_im;
    e.max_abs = r.max_abs;
    e.worst_r = r.worst_r;
    e.max_abs_at_exact_zero = r.max_abs_at_exact_zero;
    for (int d = 0; d < 24; ++d) e.decade_histogram[d] = r.decade_histogram[d];
    return e;
  }

  std::vector<double> abscissae() const {
    std::vector<double> a(info_.nodes);
    check(gk_table_download(h_, a.data(), nullptr, nullptr, nullptr, nullptr));
    return a;
  }
  std::vector<double> zero_locations() const {
    std::vector<double> z(info_.zeros);
    check(gk_table_download(h_, nullptr, z.data(), nullptr, nullptr, nullptr));
    return z;
  }
  std::vector<Complex> green_values() const {
    std::vector<Complex> g(info_.nodes);
    check(gk_table_download(h_, nullptr, nullptr, nullptr, reinterpret_cast<gk_c128*>(g.data()),
                            nullptr));
    return g;
  }

 private:
  Context* ctx_;
  gk_table* h_ = nullptr;
  gk_table_info info_{};
  mutable std::atomic<std::uint64_t> fallbacks_{0};
};

// fill_matrix<Kernel> (matfill.hpp:144-228) on the GPU, host mesh in, host
// matrix out.  Table mode: cfg.r_min / r_max <= 0 selects the device-computed
// quadrature-pair distance range.
inline std::pair<KernelMatrix, FillReport> fill_matrix(
    Context& ctx, const TriangleMesh& mesh, const QuadratureSpec& spec, Mode mode,
    const Medium& medium = {}, SamplingConfig cfg = SamplingConfig{0.0, 0.0},
    KernelKind kind = KernelKind::GreenOverR) {
  const std::size_t N = mesh.triangle_count();
  KernelMatrix z(N);
  gk_fill_report rep{};
  const gk_sampling_config c = cfg.c();
  const gk_medium m = medium.c();
  check(gk_fill_matrix_host(ctx.get(), mesh.vertices.data(), mesh.vertices.size() / 3,
                            mesh.triangles.data(), N, spec.outer_points,
                            spec.inner_points_per_edge, static_cast<gk_mode>(mode), &c, &m,
                            static_cast<gk_kind>(kind), reinterpret_cast<gk_c128*>(z.z.data()),
                            &rep));
  return {std::move(z), FillReport::from(rep)};
}

// The reference's plugin seam itself: a type satisfying gktab's duck-typed
// Kernel concept (matfill.hpp:59-87: accumulate(kind, radii, weights) and
// fallback_count()), backed by a device table.  It drops into the reference's
// own fill_matrix unchanged -- correct, but one device round trip per matrix
// entry, so it is for validation; the fast path replaces fill_matrix itself
// (gk::fill_matrix, one launch for the whole matrix).
class DeviceTableKernel {
 public:
  explicit DeviceTableKernel(const DeviceEvaluator* ev) : ev_(ev) {}
  // Kind: gk::KernelKind or the reference's own gktab::KernelKind (same values);
  // the sum runs on the device (gk_accumulate_batch_host, one block)
  template <class Kind>
  Complex accumulate(Kind kind, std::span<const double> radii,
                     std::span<const double> weights) const {
    if (radii.size() != weights.size())
      throw std::invalid_argument("accumulate: radii and weights differ in length");
    return ev_->accumulate(static_cast<KernelKind>(static_cast<int>(kind)), radii, weights);
  }
  template <class Kind>
  Complex operator()(Kind kind, double r) const {
    return ev_->eval_kernel(static_cast<KernelKind>(static_cast<int>(kind)), r);
  }
  std::uint64_t fallback_count() const { return ev_->fallback_count(); }

 private:
  const DeviceEvaluator* ev_;
};

// io.hpp:23-27, 134-156: the reference's report rows, %.17g numbers
inline std::string format_g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}
inline void write_bench_csv(std::ostream& out, const FillReport& r) {
  out << "N,m,n,predicted_calls,actual_calls,fallback_calls,analytic_s,interp_s,speedup,"
         "max_rel_re,max_rel_im\n";
  out << r.N << ',' << r.m << ',' << r.n << ',' << r.predicted_calls << ',' << r.actual_calls
      << ',' << r.fallback_calls << ',' << format_g17(r.analytic_time_s) << ','
      << format_g17(r.interp_time_s) << ',' << format_g17(r.speedup) << ','
      << format_g17(r.max_rel_re) << ',' << format_g17(r.max_rel_im) << '\n';
}
inline void write_sweep_csv_header(std::ostream& out) {
  out << "kernel,method,probes,max_rel_re,max_rel_im,max_abs,worst_r\n";
}
inline void write_sweep_csv_row(std::ostream& out, KernelKind kind, InterpMethod method,
                                int lagrange_degree, const ErrorSweepReport& r) {
  out << (kind == KernelKind::PlainExp ? "exp" : "green") << ','
      << (method == InterpMethod::Linear ? "linear" : "lagrange");
  if (method == InterpMethod::Lagrange) out << lagrange_degree;
  out << ',' << r.probe_count << ',' << format_g17(r.max_rel_re) << ','
      << format_g17(r.max_rel_im) << ',' << format_g17(r.max_abs) << ','
      << format_g17(r.worst_r) << '\n';
}

// bench_compare (matfill.hpp:262-294) on the GPU: direct vs table fill of the
// same mesh, table built over [cfg.r_min, 1.01 max_vertex_distance]
inline FillReport bench_compare(Context& ctx, const TriangleMesh& mesh, const QuadratureSpec& spec,
                                const Medium& medium, SamplingConfig cfg,
                                int lagrange_degree = 3,
                                KernelKind kind = KernelKind::GreenOverR, int repeats = 1) {
  gk_bench_report r{};
  const gk_sampling_config c = cfg.c();
  const gk_medium m = medium.c();
  check(gk_bench_compare(ctx.get(), mesh.vertices.data(), mesh.vertices.size() / 3,
                         mesh.triangles.data(), mesh.triangle_count(), spec.outer_points,
                         spec.inner_points_per_edge, &m, &c, lagrange_degree,
                         static_cast<gk_kind>(kind), repeats, &r));
  FillReport f = FillReport::from(r.fill);
  f.max_rel_re = r.max_rel_re;
  f.max_rel_im = r.max_rel_im;
  f.speedup = r.speedup;
  f.analytic_time_s = r.analytic_time_s;
  f.interp_time_s = r.interp_time_s;
  f.table_build_s = r.table_build_s;
  return f;
}

}  // namespace gk
