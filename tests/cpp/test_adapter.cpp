// C++ host-side test of the drop-in adapter (include/gk/gk.hpp) on a B200.
// Mirrors reference tests through the C ABI:
//   * CLI bench row prefix "20,4,3,14400,13680,0" (test_cli.cpp:176-189),
//   * reference-config zeros {0.25, 0.5, 0.75, 1} (test_sampling.cpp:42-49),
//   * node reproduction (test_evaluator.cpp:24-31),
//   * exception types (test_evaluator.cpp:83-91, test_matfill.cpp:23-26, 183-191),
//   * table fill vs direct fill agreement (acceptance criterion 5 gate, 1e-4),
//   * bench_compare report consistency (test_matfill.cpp:167-181).
// Built by __graft_entry__.build(); run by tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>
#include <sstream>
#include <stdexcept>
#include <vector>

#include "gk/gk.hpp"

static int failures = 0;
#define CHECK(c)                                                        \
  do {                                                                  \
    if (!(c)) {                                                         \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);          \
      ++failures;                                                       \
    }                                                                   \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  gk::Context ctx(0);

  // bench row prefix on the 20-triangle icosphere, m = 4, n = 3
  const auto mesh20 = gk::generate_sphere_mesh(0.5, 0);
  {
    auto [z, rep] = gk::fill_matrix(ctx, mesh20, {4, 3}, gk::Mode::Table, gk::Medium{});
    CHECK(rep.N == 20 && rep.m == 4 && rep.n == 3);
    CHECK(rep.predicted_calls == 14400 && rep.actual_calls == 13680 && rep.fallback_calls == 0);
    CHECK(z.at(0, 0) == gk::Complex(0.0, 0.0));
  }

  // reference configuration: forced zeros and node reproduction
  gk::DeviceEvaluator ev(ctx, gk::SamplingConfig{});
  {
    const auto z = ev.zero_locations();
    CHECK(z.size() == 4 && z[0] == 0.25 && z[1] == 0.5 && z[2] == 0.75 && z[3] == 1.0);
    const auto a = ev.abscissae();
    const auto g = ev.green_values();
    const auto v = ev.eval_batch(gk::KernelKind::GreenOverR, a);
    bool exact = true;
    for (std::size_t j = 0; j < a.size(); ++j) exact = exact && v[j] == g[j];
    CHECK(exact);
    CHECK(ev.eval_kernel(gk::KernelKind::GreenOverR, 5e-5) != gk::Complex(0, 0));
    CHECK(ev.fallback_count() == 1);  // r < r_min: analytic fallback, counted
  }

  // exception types
  CHECK(throws<std::invalid_argument>([&] { ev.eval_green(1.5); }));  // eval_batch rethrows
  CHECK(throws<std::overflow_error>([] { gk::predicted_calls(1ull << 32, 1ull << 16, 1ull << 16); }));
  CHECK(throws<std::invalid_argument>(
      [&] { gk::fill_matrix(ctx, mesh20, {5, 1}, gk::Mode::Direct, gk::Medium{}); }));
  CHECK(throws<std::invalid_argument>([] { gk::generate_sphere_mesh(1.0, 7); }));
  CHECK(throws<std::invalid_argument>([&] {
    gk::SamplingConfig bad;
    bad.r_min = 0.1;
    bad.r_max = 0.1 + 1.5e-3;
    gk::DeviceEvaluator e2(ctx, bad);
  }));

  // table fill vs direct fill, N = 320 (acceptance criterion 5 shape)
  {
    const auto mesh = gk::generate_sphere_mesh(0.5, 2);
    gk::SamplingConfig cfg{0.0, 0.0};
    cfg.samples_per_wavelength = 10000;
    auto [zt, rt] = gk::fill_matrix(ctx, mesh, {4, 3}, gk::Mode::Table, gk::Medium{}, cfg);
    auto [zd, rd] = gk::fill_matrix(ctx, mesh, {4, 3}, gk::Mode::Direct, gk::Medium{});
    double worst = 0.0;
    for (std::size_t p = 0; p < zt.n; ++p)
      for (std::size_t q = 0; q < zt.n; ++q) {
        if (p == q) continue;
        const gk::Complex a = zd.at(p, q), b = zt.at(p, q);
        if (a.real() != 0) worst = std::fmax(worst, std::fabs(b.real() - a.real()) / std::fabs(a.real()));
        if (a.imag() != 0) worst = std::fmax(worst, std::fabs(b.imag() - a.imag()) / std::fabs(a.imag()));
      }
    CHECK(worst <= 1e-4);
    CHECK(rt.actual_calls == 3ull * 4 * 3 * 320 * 319 && rd.actual_calls == rt.actual_calls);
    std::printf("N=320 table vs direct: max elementwise relative error %.3g\n", worst);
  }
  // BenchCompare.ReportConsistency (test_matfill.cpp:167-181)
  {
    const auto mesh80 = gk::generate_sphere_mesh(0.5, 1);
    gk::SamplingConfig cfg;
    cfg.samples_per_wavelength = 10000;
    const auto r = gk::bench_compare(ctx, mesh80, {4, 3}, gk::Medium{}, cfg);
    CHECK(r.N == 80u && r.actual_calls == 3ull * 4 * 3 * 80 * 79 && r.fallback_calls == 0u);
    CHECK(r.speedup > 0.0 && r.analytic_time_s > 0.0);
    CHECK(std::fabs(r.interp_time_s - (r.wall_time_s + r.table_build_s)) <= 1e-12);
    CHECK(r.max_rel_re <= 1e-4 && r.max_rel_im <= 1e-4);
    CHECK(throws<std::invalid_argument>(
        [&] { gk::bench_compare(ctx, mesh80, {4, 3}, gk::Medium{}, cfg, 3, gk::KernelKind::GreenOverR, 0); }));
    // host compare_fills of the two fills == the device report's statistic
    auto [zd, rd] = gk::fill_matrix(ctx, mesh80, {4, 3}, gk::Mode::Direct, gk::Medium{});
    const auto same = gk::compare_fills(zd, zd);
    CHECK(same.max_rel_re == 0.0 && same.max_rel_im == 0.0);
    (void)rd;
  }
  // the Kernel-concept adapter: accumulate == sum of w * eval_batch, fallbacks counted
  {
    gk::DeviceEvaluator e(ctx, gk::SamplingConfig{});
    const gk::DeviceTableKernel kern(&e);
    const std::vector<double> r = {5e-5, 0.25, 0.5, 0.75};  // the first is below r_min
    const std::vector<double> w = {0.5, 1.0, -2.0, 0.25};
    const gk::Complex a = kern.accumulate(gk::KernelKind::GreenOverR, r, w);
    const auto v = e.eval_batch(gk::KernelKind::GreenOverR, r);
    gk::Complex want{0.0, 0.0};
    double scale = 0.0;
    for (int i = 0; i < 4; ++i) {
      want += w[i] * v[i];
      scale += std::abs(w[i] * v[i]);
    }
    CHECK(std::abs(a - want) <= 1e-14 * scale);  // device shuffle-reduction order
    CHECK(kern.fallback_count() == 2);  // one per batch that met r < r_min
    CHECK(throws<std::invalid_argument>(
        [&] { kern.accumulate(gk::KernelKind::GreenOverR, r, std::span<const double>(w.data(), 3)); }));
  }

  // gk_fill_rows_host into a strided host window (ldz_host > N: the 2D-copy path)
  {
    const auto mesh = gk::generate_sphere_mesh(0.5, 1);  // N = 80
    const std::size_t N = mesh.triangle_count(), ld = N + 7, rows = 50;
    gk_mesh* m = nullptr;
    CHECK(gk_mesh_create(ctx.get(), mesh.vertices.data(), mesh.vertices.size() / 3,
                         mesh.triangles.data(), N, 4, 3, &m) == GK_OK);
    std::vector<gk::Complex> strided(rows * ld, gk::Complex(7.0, 7.0)), dense(rows * N);
    CHECK(gk_fill_rows_host(ctx.get(), m, GK_MODE_DIRECT, nullptr, GK_KIND_GREEN, 6.283185307179586,
                            0.0, 10, 10 + rows, reinterpret_cast<gk_c128*>(strided.data()), ld,
                            nullptr, nullptr) == GK_OK);
    CHECK(gk_fill_rows_host(ctx.get(), m, GK_MODE_DIRECT, nullptr, GK_KIND_GREEN, 6.283185307179586,
                            0.0, 10, 10 + rows, reinterpret_cast<gk_c128*>(dense.data()), N,
                            nullptr, nullptr) == GK_OK);
    bool same = true, pad_kept = true;
    for (std::size_t r = 0; r < rows; ++r) {
      for (std::size_t q = 0; q < N; ++q) same = same && strided[r * ld + q] == dense[r * N + q];
      for (std::size_t q = N; q < ld; ++q) pad_kept = pad_kept && strided[r * ld + q] == gk::Complex(7.0, 7.0);
    }
    CHECK(same && pad_kept);
    gk_mesh_destroy(m);
  }

  // error_sweep on the device + the reference's CSV row format
  {
    gk::DeviceEvaluator e(ctx, gk::SamplingConfig{});
    const auto rs = e.error_sweep(gk::KernelKind::GreenOverR, gk::InterpMethod::Lagrange, 10000);
    CHECK(rs.probe_count == 10000 && rs.max_rel_re > 0.0 && std::isfinite(rs.max_rel_re));
    CHECK(rs.max_abs > 0.0 && std::isfinite(rs.max_abs));
    CHECK(throws<std::invalid_argument>(
        [&] { e.error_sweep(gk::KernelKind::PlainExp, gk::InterpMethod::Lagrange, 10); }));
    std::ostringstream os;
    gk::write_sweep_csv_header(os);
    gk::write_sweep_csv_row(os, gk::KernelKind::GreenOverR, gk::InterpMethod::Lagrange, 3, rs);
    CHECK(os.str().rfind("kernel,method,probes,max_rel_re,max_rel_im,max_abs,worst_r\ngreen,lagrange3,10000,", 0) == 0);
    gk::FillReport fr;
    fr.N = 20;
    fr.m = 4;
    fr.n = 3;
    fr.predicted_calls = 14400;
    fr.actual_calls = 13680;
    fr.speedup = 0.1;
    std::ostringstream ob;
    gk::write_bench_csv(ob, fr);
    CHECK(ob.str() == "N,m,n,predicted_calls,actual_calls,fallback_calls,analytic_s,interp_s,"
                      "speedup,max_rel_re,max_rel_im\n20,4,3,14400,13680,0,0,0,"
                      "0.10000000000000001,0,0\n");
  }
  std::printf("%s (%d failure(s))\n", failures ? "FAILED" : "ALL OK", failures);
  return failures ? 1 : 0;
}
