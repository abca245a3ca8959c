// The drop-in at the reference's own plugin seam: gktab::fill_matrix (the
// UNMODIFIED reference header, compiled in place by oracle/Makefile) driven
// once with its CPU TableKernel and once with gk::DeviceTableKernel over a
// device table of the same (bit-identical) plan.  Same call counts, same
// fallback counts, entries equal to rounding.  Built as oracle/_ref/plug
// (test infrastructure: it links the reference); run on a B200 by
// tests/test_gpu_cpp.py.
#include <cmath>
#include <cstdio>

#include "gk/gk.hpp"
#include "gktab/gktab.hpp"

int main() {
  const auto mesh = gktab::generate_sphere_mesh(0.5, 1);  // N = 80
  const gktab::QuadratureSpec spec{4, 3};
  const gktab::Medium vac{1.0, 1.0, 1.0};
  gktab::SamplingConfig cfg;
  cfg.r_min = 0.3;  // a fat near field (test_matfill.cpp:152-165): fallbacks are exercised
  cfg.r_max = gktab::max_vertex_distance(mesh) * 1.01;
  cfg.samples_per_wavelength = 2000;
  const double k = gktab::wavenumber(vac);
  const gktab::KernelEvaluator ev(gktab::build_plan(cfg, vac), k, 3);
  auto [zc, rc] = gktab::fill_matrix(mesh, spec, gktab::TableKernel{&ev},
                                     gktab::KernelKind::GreenOverR);

  gk::Context ctx(0);
  gk::SamplingConfig gcfg;
  gcfg.r_min = cfg.r_min;
  gcfg.r_max = cfg.r_max;
  gcfg.samples_per_wavelength = cfg.samples_per_wavelength;
  const gk::DeviceEvaluator dev(ctx, gcfg, gk::Medium{1.0, 1.0, 1.0});
  auto [zg, rg] = gktab::fill_matrix(mesh, spec, gk::DeviceTableKernel{&dev},
                                     gktab::KernelKind::GreenOverR);

  double worst = 0.0;
  for (std::size_t i = 0; i < zc.z.size(); ++i) {
    const double d = std::abs(zg.z[i] - zc.z[i]);
    const double s = std::abs(zc.z[i]);
    if (s > 0) worst = std::fmax(worst, d / s);
  }
  bool same_plan = dev.info().nodes == ev.plan().size();
  if (same_plan) {
    const auto a = dev.abscissae();
    for (std::size_t i = 0; i < a.size(); ++i) same_plan = same_plan && a[i] == ev.plan().abscissae[i];
  }
  bool ok = same_plan && rg.actual_calls == rc.actual_calls &&
            rg.fallback_calls == rc.fallback_calls && rc.fallback_calls > 0 && worst < 1e-12;
  std::printf("plug: N=%zu calls %llu/%llu fallbacks %llu/%llu max rel diff %.3g -> %s\n",
              zc.n, (unsigned long long)rg.actual_calls, (unsigned long long)rc.actual_calls,
              (unsigned long long)rg.fallback_calls, (unsigned long long)rc.fallback_calls, worst,
              ok ? "OK" : "FAILED");

  // threads = 4: the reference's fill calls accumulate from 4 worker threads
  // at once (matfill.hpp:206-221); the device evaluator serialises its calls
  // on the shared context and counts fallbacks atomically, so the result is
  // the threads = 1 result and the fallback delta is the reference's
  const gk::DeviceEvaluator dev4(ctx, gcfg, gk::Medium{1.0, 1.0, 1.0});
  auto [z4, r4] = gktab::fill_matrix(mesh, spec, gk::DeviceTableKernel{&dev4},
                                     gktab::KernelKind::GreenOverR, 4);
  bool same4 = z4.z.size() == zg.z.size();
  for (std::size_t i = 0; same4 && i < zg.z.size(); ++i) same4 = z4.z[i] == zg.z[i];
  const bool ok4 = same4 && r4.actual_calls == rc.actual_calls &&
                   r4.fallback_calls == rc.fallback_calls && dev4.fallback_count() == rc.fallback_calls;
  std::printf("plug threads=4: calls %llu fallbacks %llu/%llu bitwise-equal to threads=1: %d -> %s\n",
              (unsigned long long)r4.actual_calls, (unsigned long long)r4.fallback_calls,
              (unsigned long long)rc.fallback_calls, same4 ? 1 : 0, ok4 ? "OK" : "FAILED");
  ok = ok && ok4;
  return ok ? 0 : 1;
}
