// abi.cu -- the extern "C" boundary (include/gk/gk.h) and the host-side
// orchestration behind it.  Every entry point converts exceptions into
// gk_status codes that mirror the reference's exception types; the message
// is kept in a thread-local buffer for gk_last_error().
#include <algorithm>
#include <atomic>
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "gk_internal.h"

namespace {

thread_local std::string g_last_error;

template <class F>
gk_status guarded(F&& f) {
  try {
    f();
    return GK_OK;
  } catch (const gk::Error& e) {
    g_last_error = e.what;
    return e.status;
  } catch (const std::bad_alloc&) {
    g_last_error = "out of host memory";
    return GK_ERR_RUNTIME;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return GK_ERR_RUNTIME;
  }
}

void need(bool ok, gk_status s, const char* what) {
  if (!ok) gk::fail(s, what);
}

// gktab::Medium::validate (kernel.hpp:30-37)
void validate_medium(const gk_medium& m) {
  need(std::isfinite(m.lambda0) && m.lambda0 > 0.0, GK_ERR_INVALID_ARGUMENT,
       "Medium: lambda0 must be finite and > 0");
  need(std::isfinite(m.eps_r) && m.eps_r > 0.0, GK_ERR_INVALID_ARGUMENT,
       "Medium: eps_r must be finite and > 0");
  need(std::isfinite(m.mu_r) && m.mu_r > 0.0, GK_ERR_INVALID_ARGUMENT,
       "Medium: mu_r must be finite and > 0");
  need(std::isfinite(m.eps_r_im) && m.eps_r_im <= 0.0, GK_ERR_INVALID_ARGUMENT,
       "Medium: eps_r_im must be finite and <= 0 (lossy medium)");
}

// gktab::SamplingConfig::validate (sampling.hpp:27-45)
void validate_cfg(const gk_sampling_config& c) {
  need(std::isfinite(c.r_min) && std::isfinite(c.r_max) && 0.0 < c.r_min && c.r_min < c.r_max,
       GK_ERR_INVALID_ARGUMENT, "SamplingConfig: need 0 < r_min < r_max, both finite");
  need(c.samples_per_wavelength >= 2, GK_ERR_INVALID_ARGUMENT,
       "SamplingConfig: samples_per_wavelength must be >= 2");
  need(c.refine_interval_divisor >= (c.refine ? 2 : 1), GK_ERR_INVALID_ARGUMENT,
       "SamplingConfig: refine_interval_divisor must be >= 2 when refinement is on");
  need(c.refine_halfwidth_in_t > 0.0, GK_ERR_INVALID_ARGUMENT,
       "SamplingConfig: refine_halfwidth_in_t must be > 0");
  need(c.dedup_fraction > 0.0 && c.dedup_fraction <= 1.0, GK_ERR_INVALID_ARGUMENT,
       "SamplingConfig: dedup_fraction must be in (0, 1]");
  need(!(c.refine && c.refine_halfwidth_in_t * c.refine_interval_divisor < 1.0),
       GK_ERR_INVALID_ARGUMENT,
       "SamplingConfig: refinement window narrower than one refined interval");
}

// k = 2 pi sqrt(eps_r mu_r) / lambda0 (kernel.hpp:41-44); complex when lossy
void wavenumber(const gk_medium& m, double& k_re, double& k_im) {
  validate_medium(m);
  if (m.eps_r_im == 0.0) {
    k_re = 2.0 * gk::kPi * std::sqrt(m.eps_r * m.mu_r) / m.lambda0;
    k_im = 0.0;
    return;
  }
  const std::complex<double> s = std::sqrt(std::complex<double>(m.eps_r * m.mu_r, m.eps_r_im * m.mu_r));
  const std::complex<double> k = 2.0 * gk::kPi * s / m.lambda0;
  k_re = k.real();
  k_im = k.imag();
}

// nominal base interval t = lambda0 / (S sqrt(eps_r mu_r)) (sampling.hpp:112-122);
// lossy: the real part of the refractive index sets the wavelength
double base_interval(const gk_medium& m, int S) {
  if (m.eps_r_im == 0.0)
    return m.lambda0 / (static_cast<double>(S) * std::sqrt(m.eps_r * m.mu_r));
  const std::complex<double> s = std::sqrt(std::complex<double>(m.eps_r * m.mu_r, m.eps_r_im * m.mu_r));
  return m.lambda0 / (static_cast<double>(S) * s.real());
}

void validate_spec(int m, int n) {
  need(m == 1 || m == 3 || m == 4 || m == 6 || m == 7, GK_ERR_INVALID_ARGUMENT,
       "QuadratureSpec: outer_points must be one of 1, 3, 4, 6, 7");
  need(n >= 1, GK_ERR_INVALID_ARGUMENT, "QuadratureSpec: inner_points_per_edge must be >= 1");
  need(n <= 32, GK_ERR_INVALID_ARGUMENT, "QuadratureSpec: device fill supports inner_points_per_edge <= 32");
}

uint64_t predicted(uint64_t N, uint64_t m, uint64_t n) {
  const unsigned __int128 wide =
      static_cast<unsigned __int128>(3) * m * n * (static_cast<unsigned __int128>(N) * N);
  need(wide <= static_cast<unsigned __int128>(UINT64_MAX), GK_ERR_OVERFLOW,
       "predicted_calls: 3*m*n*N^2 overflows 64 bits");
  return static_cast<uint64_t>(wide);
}

void check_ctx(const gk_ctx* c) { need(c != nullptr, GK_ERR_INVALID_ARGUMENT, "null gk_ctx"); }

// scratch words 32..34: counters accumulated by asynchronous fills
constexpr int kAsyncFillCounters = 32;

// the reference's exceptions for fill counters {fallbacks, > r_max, non-finite}
void raise_fill_errors(const unsigned long long* h) {
  if (h[1])
    gk::fail(GK_ERR_OUT_OF_RANGE,
             "accumulate_green: " + std::to_string(h[1]) + " radii above the tabulated r_max");
  if (h[2])
    gk::fail(GK_ERR_DOMAIN, "eval_analytic: exp(-jkr)/r is singular at r = 0 (" +
                                std::to_string(h[2]) + " entries meet a zero-distance point pair)");
}

void use_device(const gk_ctx* c) { GK_CUDA(cudaSetDevice(c->device)); }

}  // namespace

namespace gk {
std::string& last_error_buffer() { return g_last_error; }
static std::atomic<unsigned long long> g_launches{0};
void count_launches(unsigned long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }
}  // namespace gk

extern "C" {

uint64_t gk_launch_count(void) { return gk::g_launches.load(std::memory_order_relaxed); }

int gk_abi_version(void) { return GK_ABI_VERSION; }

const char* gk_last_error(void) { return g_last_error.c_str(); }

gk_status gk_ctx_create(int device, gk_ctx** out) {
  return guarded([&] {
    need(out != nullptr, GK_ERR_INVALID_ARGUMENT, "null output");
    int count = 0;
    GK_CUDA(cudaGetDeviceCount(&count));
    need(device >= 0 && device < count, GK_ERR_INVALID_ARGUMENT, "gk_ctx_create: no such device");
    GK_CUDA(cudaSetDevice(device));
    cudaDeviceProp prop{};
    GK_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
      gk::fail(GK_ERR_RUNTIME, "gk_ctx_create: libgk is built for sm_100a (B200); device is sm_" +
                                   std::to_string(prop.major) + std::to_string(prop.minor));
    auto* c = new gk_ctx();
    c->device = device;
    c->opts = gk::default_fill_options();
    c->sm_count = prop.multiProcessorCount;
    cudaMemPool_t pool;
    GK_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t keep = UINT64_MAX;
    GK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    try {
      GK_CUDA(cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking));
      c->stream = c->own;
      GK_CUDA(cudaEventCreate(&c->ev0));
      GK_CUDA(cudaEventCreate(&c->ev1));
      c->scratch.alloc(64, c->stream);
      GK_CUDA(cudaMemsetAsync(c->scratch.p, 0, c->scratch.bytes(), c->stream));
      gk::init_phase_table(c);
      GK_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
      gk_ctx_destroy(c);
      throw;
    }
    *out = c;
  });
}

gk_status gk_ctx_destroy(gk_ctx* c) {
  return guarded([&] {
    if (!c) return;
    cudaSetDevice(c->device);
    if (c->stream) cudaStreamSynchronize(c->stream);
    // every context-owned buffer is released on the stream before it goes away
    if (c->pipe.copy) cudaStreamSynchronize(c->pipe.copy);
    c->scratch.reset();
    c->phase.reset();
    c->phase_small.reset();
    for (int b = 0; b < 2; ++b) {
      c->pipe.buf[b].reset();
      if (c->pipe.filled[b]) cudaEventDestroy(c->pipe.filled[b]);
      if (c->pipe.copied[b]) cudaEventDestroy(c->pipe.copied[b]);
    }
    if (c->pipe.copy) cudaStreamDestroy(c->pipe.copy);
    if (c->ev0) cudaEventDestroy(c->ev0);
    if (c->ev1) cudaEventDestroy(c->ev1);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
  });
}

gk_status gk_ctx_set_stream(gk_ctx* c, void* s) {
  return guarded([&] {
    check_ctx(c);
    c->stream = static_cast<cudaStream_t>(s);
  });
}

void gk_fill_options_init(gk_fill_options* o) {
  if (o) *o = gk::default_fill_options();
}

void gk_mesh_options_init(gk_mesh_options* o) {
  if (o) *o = gk::default_mesh_options();
}

gk_status gk_ctx_set_fill_options(gk_ctx* c, const gk_fill_options* o) {
  return guarded([&] {
    check_ctx(c);
    c->opts = o ? *o : gk::default_fill_options();
  });
}

gk_status gk_ctx_use_own_stream(gk_ctx* c) {
  return guarded([&] {
    check_ctx(c);
    c->stream = c->own;
  });
}

gk_status gk_ctx_synchronize(gk_ctx* c) {
  return guarded([&] {
    check_ctx(c);
    use_device(c);
    GK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

gk_status gk_wavenumber(const gk_medium* m, double* k_re, double* k_im) {
  return guarded([&] {
    need(m && k_re && k_im, GK_ERR_INVALID_ARGUMENT, "null argument");
    wavenumber(*m, *k_re, *k_im);
  });
}

gk_status gk_table_build(gk_ctx* c, const gk_sampling_config* cfg, const gk_medium* med,
                         int degree, gk_table** out) {
  return guarded([&] {
    check_ctx(c);
    need(cfg && med && out, GK_ERR_INVALID_ARGUMENT, "null argument");
    validate_cfg(*cfg);  // build_plan validates before the medium (sampling.hpp:150-151)
    double k_re, k_im;
    wavenumber(*med, k_re, k_im);
    need(degree >= 1, GK_ERR_INVALID_ARGUMENT, "KernelEvaluator: lagrange_degree must be >= 1");
    need(degree <= 7, GK_ERR_INVALID_ARGUMENT, "device tables support lagrange_degree <= 7");
    const double t_nominal = base_interval(*med, cfg->samples_per_wavelength);
    use_device(c);
    auto* t = new gk_table();
    t->ctx = c;
    try {
      gk::build_table_device(c, t, *cfg, k_re, t_nominal, k_re, k_im, degree);
    } catch (...) {
      delete t;
      throw;
    }
    *out = t;
  });
}

gk_status gk_table_info_get(const gk_table* t, gk_table_info* info) {
  return guarded([&] {
    need(t && info, GK_ERR_INVALID_ARGUMENT, "null argument");
    *info = t->info;
  });
}

gk_status gk_table_download(const gk_table* t, double* absc, double* zeros, gk_c128* ev,
                            gk_c128* gv, uint32_t* buckets) {
  return guarded([&] {
    need(t != nullptr, GK_ERR_INVALID_ARGUMENT, "null table");
    use_device(t->ctx);
    cudaStream_t s = t->ctx->stream;
    const size_t n = t->info.nodes;
    if (absc) GK_CUDA(cudaMemcpyAsync(absc, t->absc.p, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (ev) GK_CUDA(cudaMemcpyAsync(ev, t->exp_vals.p, n * 16, cudaMemcpyDeviceToHost, s));
    if (gv) GK_CUDA(cudaMemcpyAsync(gv, t->green_vals.p, n * 16, cudaMemcpyDeviceToHost, s));
    if (buckets)
      GK_CUDA(cudaMemcpyAsync(buckets, t->hash.p, t->info.hash_buckets * 4, cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    if (zeros && !t->zeros.empty()) std::memcpy(zeros, t->zeros.data(), t->zeros.size() * 8);
  });
}

namespace {

void put_u32(std::FILE* f, uint32_t v) {
  unsigned char b[4];
  for (int i = 0; i < 4; ++i) b[i] = static_cast<unsigned char>((v >> (8 * i)) & 0xff);
  std::fwrite(b, 1, 4, f);
}

void put_f64(std::FILE* f, double v) {
  uint64_t bits;
  std::memcpy(&bits, &v, 8);
  unsigned char b[8];
  for (int i = 0; i < 8; ++i) b[i] = static_cast<unsigned char>((bits >> (8 * i)) & 0xff);
  std::fwrite(b, 1, 8, f);
}

std::string g17(double v) {
  char buf[40];
  std::snprintf(buf, sizeof(buf), "%.17g", v);
  return buf;
}

}  // namespace

gk_status gk_table_dump_binary(const gk_table* t, gk_kind kind, const char* path) {
  return guarded([&] {
    need(t && path, GK_ERR_INVALID_ARGUMENT, "null argument");
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    const size_t n = t->info.nodes;
    std::vector<double> a(n);
    std::vector<gk_c128> v(n);
    const gk_status s = gk_table_download(t, a.data(), nullptr,
                                          kind == GK_KIND_EXP ? v.data() : nullptr,
                                          kind == GK_KIND_GREEN ? v.data() : nullptr, nullptr);
    if (s != GK_OK) gk::fail(s, g_last_error);
    std::FILE* f = std::fopen(path, "wb");
    if (!f) gk::fail(GK_ERR_RUNTIME, std::string("dump_table_binary: cannot open '") + path + "'");
    std::fwrite("GKTB", 1, 4, f);
    put_u32(f, 1u);
    put_u32(f, static_cast<uint32_t>(n));
    put_f64(f, t->info.k_re);
    const unsigned char kb = static_cast<unsigned char>(kind);
    std::fwrite(&kb, 1, 1, f);
    for (size_t i = 0; i < n; ++i) {
      put_f64(f, a[i]);
      put_f64(f, v[i].re);
      put_f64(f, v[i].im);
    }
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) gk::fail(GK_ERR_RUNTIME, "dump_table_binary: write failed");
  });
}

gk_status gk_plan_dump_csv(const gk_table* t, const char* path) {
  return guarded([&] {
    need(t && path, GK_ERR_INVALID_ARGUMENT, "null argument");
    const size_t n = t->info.nodes;
    std::vector<double> a(n);
    const gk_status s = gk_table_download(t, a.data(), nullptr, nullptr, nullptr, nullptr);
    if (s != GK_OK) gk::fail(s, g_last_error);
    std::FILE* f = std::fopen(path, "w");
    if (!f) gk::fail(GK_ERR_RUNTIME, std::string("dump_plan_csv: cannot open '") + path + "'");
    std::fputs("index,r,is_zero,gap_to_next\n", f);
    size_t zi = 0;
    const std::vector<double>& z = t->zeros;
    for (size_t i = 0; i < n; ++i) {
      const double r = a[i];
      while (zi < z.size() && z[zi] < r) ++zi;
      const bool is_zero = zi < z.size() && z[zi] == r;
      const double gap = i + 1 < n ? a[i + 1] - r : 0.0;
      std::fprintf(f, "%zu,%s,%d,%s\n", i, g17(r).c_str(), is_zero ? 1 : 0, g17(gap).c_str());
    }
    const bool ok = std::ferror(f) == 0;
    std::fclose(f);
    if (!ok) gk::fail(GK_ERR_RUNTIME, "dump_plan_csv: write failed");
  });
}

gk_status gk_table_destroy(gk_table* t) {
  return guarded([&] {
    if (!t) return;
    cudaSetDevice(t->ctx->device);
    cudaStreamSynchronize(t->ctx->stream);
    delete t;
  });
}

namespace {

// validates and enqueues one eval_batch launch accumulating into w[2]
void enqueue_eval_batch(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re, double k_im,
                        const double* radii, size_t n, gk_c128* out, unsigned long long* w) {
  need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
  if (t) {
    k_re = t->dev.k_re;
    k_im = t->dev.k_im;
  }
  need(k_re >= 0.0, GK_ERR_INVALID_ARGUMENT, "eval_analytic: k must be >= 0");
  if (n == 0) return;
  need(radii && out, GK_ERR_INVALID_ARGUMENT, "null buffer");
  use_device(c);
  gk::launch_eval_batch(c, t, kind, k_re, k_im, radii, n, out, w);
}

// raises the reference's exception for a failing radius recorded in `word`
void raise_bad_radius(unsigned long long word, const double* radii) {
  if (word == ~0ull) return;
  const size_t idx = static_cast<size_t>(word >> 3);
  const unsigned code = static_cast<unsigned>(word & 7u);
  double r = 0.0;
  if (radii) GK_CUDA(cudaMemcpy(&r, radii + idx, sizeof(double), cudaMemcpyDeviceToHost));
  const char* why = code == 2 ? "exp(-jkr)/r is singular at r = 0"
                  : code == 3 ? "r outside the tabulated range"
                              : "r must be >= 0 (Exp) / > 0 (Green)";
  gk::fail(GK_ERR_INVALID_ARGUMENT, "eval_batch: radius [" + std::to_string(idx) + "]" +
                                        (radii ? " = " + std::to_string(r) : std::string()) +
                                        ": " + why);
}

}  // namespace

gk_status gk_eval_batch(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re, double k_im,
                        const double* radii, size_t n, gk_c128* out, uint64_t* fallbacks) {
  return guarded([&] {
    check_ctx(c);
    if (fallbacks) *fallbacks = 0;
    unsigned long long* w = c->scratch.p;  // [0] fallbacks, [1] first bad (index<<3 | code)
    if (n) {
      use_device(c);
      const unsigned long long init[2] = {0ull, ~0ull};
      GK_CUDA(cudaMemcpyAsync(w, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    }
    enqueue_eval_batch(c, t, kind, k_re, k_im, radii, n, out, w);
    if (n == 0) return;
    unsigned long long res[2];
    GK_CUDA(cudaMemcpyAsync(res, w, sizeof(res), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    if (fallbacks) *fallbacks = res[0];
    raise_bad_radius(res[1], radii);
  });
}

gk_status gk_compare_fills(gk_ctx* c, const gk_c128* test, const gk_c128* ref, size_t rows,
                           size_t N, size_t row_begin, size_t ld, double* max_rel_re,
                           double* max_rel_im) {
  return guarded([&] {
    check_ctx(c);
    need(ld >= N, GK_ERR_INVALID_ARGUMENT, "compare_fills: ld < N");
    need(rows == 0 || N == 0 || (test && ref), GK_ERR_INVALID_ARGUMENT, "null matrix");
    double re = 0.0, im = 0.0;
    if (rows && N) {
      use_device(c);
      unsigned long long* w = c->scratch.p + 24;
      GK_CUDA(cudaMemsetAsync(w, 0, 2 * sizeof(unsigned long long), c->stream));
      gk::launch_compare(c, test, ref, rows, N, row_begin, ld, w);
      unsigned long long h[2];
      GK_CUDA(cudaMemcpyAsync(h, w, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
      GK_CUDA(cudaStreamSynchronize(c->stream));
      std::memcpy(&re, &h[0], sizeof(double));
      std::memcpy(&im, &h[1], sizeof(double));
    }
    if (max_rel_re) *max_rel_re = re;
    if (max_rel_im) *max_rel_im = im;
  });
}

gk_status gk_error_sweep(gk_ctx* c, const gk_table* t, gk_kind kind, gk_interp method,
                         uint64_t probes, gk_sweep_report* out) {
  return guarded([&] {
    check_ctx(c);
    need(t != nullptr && out != nullptr, GK_ERR_INVALID_ARGUMENT, "null argument");
    need(probes >= 1, GK_ERR_INVALID_ARGUMENT, "error_sweep: need at least one probe");
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    need((kind == GK_KIND_EXP && method == GK_INTERP_LINEAR) ||
             (kind == GK_KIND_GREEN && method == GK_INTERP_LAGRANGE),
         GK_ERR_INVALID_ARGUMENT,
         "error_sweep: the device tabulates Exp with linear and Green with Lagrange "
         "interpolation");
    use_device(c);
    gk::DevBuf<unsigned long long> w;
    gk::DevBuf<double> comb;
    w.alloc(32, c->stream);
    comb.alloc(probes, c->stream);
    unsigned long long init[32] = {};
    init[5] = ~0ull;
    GK_CUDA(cudaMemcpyAsync(w.p, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    gk::launch_sweep(c, t, kind, probes, comb.p, w.p);
    unsigned long long h[32];
    GK_CUDA(cudaMemcpyAsync(h, w.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    auto dbl = [&](int i) {
      double v;
      std::memcpy(&v, &h[i], sizeof(double));
      return v;
    };
    gk_sweep_report r{};
    r.probe_count = probes;
    r.max_rel_re = dbl(0);
    r.max_rel_im = dbl(1);
    r.max_abs = dbl(2);
    r.max_abs_at_exact_zero = dbl(3);
    // the probe radius exactly as the kernel formed it (bounds.hpp:141-145)
    const uint64_t i = h[5] == ~0ull ? 0 : h[5];
    const double a = t->dev.r_min, b = t->dev.r_max;
    const double step = probes == 1 ? 0.0 : (b - a) / static_cast<double>(probes - 1);
    double rr = i + 1 == probes ? b : a + static_cast<double>(i) * step;
    rr = rr < a ? a : (rr > b ? b : rr);
    r.worst_r = rr;
    for (int d = 0; d < 24; ++d) r.decade_histogram[d] = h[8 + d];
    *out = r;
  });
}

gk_status gk_max_vertex_distance(gk_ctx* c, const gk_mesh* mesh, double* out) {
  return guarded([&] {
    check_ctx(c);
    need(mesh != nullptr && out != nullptr, GK_ERR_INVALID_ARGUMENT, "null argument");
    use_device(c);
    unsigned long long* w = c->scratch.p + 26;
    GK_CUDA(cudaMemsetAsync(w, 0, sizeof(unsigned long long), c->stream));
    gk::launch_max_vertex_d2(mesh->verts.p, mesh->nv, w, c->stream);
    unsigned long long h = 0;
    GK_CUDA(cudaMemcpyAsync(&h, w, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    double d2 = 0.0;
    std::memcpy(&d2, &h, sizeof(double));
    *out = std::sqrt(d2);
  });
}

gk_status gk_accumulate_batch(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re,
                              double k_im, const double* radii, const double* weights,
                              size_t len, size_t nblocks, gk_c128* out, uint64_t* fallbacks) {
  return guarded([&] {
    check_ctx(c);
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    if (t) {
      k_re = t->dev.k_re;
      k_im = t->dev.k_im;
    }
    need(k_re >= 0.0, GK_ERR_INVALID_ARGUMENT, "eval_analytic: k must be >= 0");
    if (fallbacks) *fallbacks = 0;
    if (nblocks == 0) return;
    need(out != nullptr, GK_ERR_INVALID_ARGUMENT, "null output");
    need(len == 0 || (radii && weights), GK_ERR_INVALID_ARGUMENT, "null buffer");
    use_device(c);
    unsigned long long* w = c->scratch.p;
    const unsigned long long init[2] = {0ull, ~0ull};
    GK_CUDA(cudaMemcpyAsync(w, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    gk::launch_accumulate(c, t, kind, k_re, k_im, radii, weights, len, nblocks, out, w);
    unsigned long long res[2];
    GK_CUDA(cudaMemcpyAsync(res, w, sizeof(res), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    if (fallbacks) *fallbacks = res[0];
    raise_bad_radius(res[1], radii);
  });
}

gk_status gk_eval_batch_async(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re,
                              double k_im, const double* radii, size_t n, gk_c128* out,
                              uint64_t* status) {
  return guarded([&] {
    check_ctx(c);
    need(status != nullptr, GK_ERR_INVALID_ARGUMENT, "null status");
    enqueue_eval_batch(c, t, kind, k_re, k_im, radii, n, out,
                       reinterpret_cast<unsigned long long*>(status));
  });
}

gk_status gk_eval_status_reset(gk_ctx* c, uint64_t* status) {
  return guarded([&] {
    check_ctx(c);
    need(status != nullptr, GK_ERR_INVALID_ARGUMENT, "null status");
    use_device(c);
    GK_CUDA(cudaMemsetAsync(status, 0, sizeof(uint64_t), c->stream));
    GK_CUDA(cudaMemsetAsync(status + 1, 0xff, sizeof(uint64_t), c->stream));
  });
}

gk_status gk_eval_status_read(gk_ctx* c, const uint64_t* status, uint64_t* fallbacks) {
  return guarded([&] {
    check_ctx(c);
    need(status != nullptr, GK_ERR_INVALID_ARGUMENT, "null status");
    use_device(c);
    uint64_t res[2];
    GK_CUDA(cudaMemcpyAsync(res, status, sizeof(res), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    if (fallbacks) *fallbacks = res[0];
    raise_bad_radius(res[1], nullptr);
  });
}

gk_status gk_locate(gk_ctx* c, const gk_table* t, const double* radii, size_t n, uint32_t* out) {
  return guarded([&] {
    check_ctx(c);
    need(t != nullptr, GK_ERR_INVALID_ARGUMENT, "locate needs a table");
    if (n == 0) return;
    need(radii && out, GK_ERR_INVALID_ARGUMENT, "null buffer");
    use_device(c);
    unsigned long long* w = c->scratch.p;
    const unsigned long long init[2] = {0ull, ~0ull};
    GK_CUDA(cudaMemcpyAsync(w, init, sizeof(init), cudaMemcpyHostToDevice, c->stream));
    gk::launch_locate(c, t, radii, n, out, w);
    unsigned long long res[2];
    GK_CUDA(cudaMemcpyAsync(res, w, sizeof(res), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    if (res[1] != ~0ull)
      gk::fail(GK_ERR_OUT_OF_RANGE,
               "locate: radius [" + std::to_string(res[1]) + "] outside the tabulated range");
  });
}

gk_status gk_eval_batch_host(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re,
                             double k_im, const double* radii, size_t n, gk_c128* out,
                             uint64_t* fallbacks) {
  double* dr = nullptr;
  gk_c128* dout = nullptr;
  gk_status st = guarded([&] {
    check_ctx(c);
    if (fallbacks) *fallbacks = 0;
    if (n == 0) return;
    need(radii && out, GK_ERR_INVALID_ARGUMENT, "null buffer");
    use_device(c);
    GK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dr), n * sizeof(double), c->stream));
    GK_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dout), n * sizeof(gk_c128), c->stream));
    GK_CUDA(cudaMemcpyAsync(dr, radii, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
  });
  if (st == GK_OK && n) {
    st = gk_eval_batch(c, t, kind, k_re, k_im, dr, n, dout, fallbacks);
    if (st == GK_OK)
      st = guarded([&] {
        GK_CUDA(cudaMemcpyAsync(out, dout, n * sizeof(gk_c128), cudaMemcpyDeviceToHost, c->stream));
        GK_CUDA(cudaStreamSynchronize(c->stream));
      });
  }
  if (dr) cudaFreeAsync(dr, c->stream);
  if (dout) cudaFreeAsync(dout, c->stream);
  return st;
}

gk_status gk_accumulate_batch_host(gk_ctx* c, const gk_table* t, gk_kind kind, double k_re,
                                   double k_im, const double* radii, const double* weights,
                                   size_t len, size_t nblocks, gk_c128* out,
                                   uint64_t* fallbacks) {
  gk::DevBuf<double> dr, dw;
  gk::DevBuf<gk_c128> dout;
  gk_status st = guarded([&] {
    check_ctx(c);
    if (fallbacks) *fallbacks = 0;
    if (nblocks == 0) return;
    need(out != nullptr && (len == 0 || (radii && weights)), GK_ERR_INVALID_ARGUMENT,
         "null buffer");
    use_device(c);
    const size_t n = len * nblocks;
    dr.alloc(n, c->stream);
    dw.alloc(n, c->stream);
    dout.alloc(nblocks, c->stream);
    if (n) {
      GK_CUDA(cudaMemcpyAsync(dr.p, radii, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      GK_CUDA(cudaMemcpyAsync(dw.p, weights, n * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    }
  });
  if (st == GK_OK && nblocks) {
    st = gk_accumulate_batch(c, t, kind, k_re, k_im, dr.p, dw.p, len, nblocks, dout.p, fallbacks);
    if (st == GK_OK)
      st = guarded([&] {
        GK_CUDA(cudaMemcpyAsync(out, dout.p, nblocks * sizeof(gk_c128), cudaMemcpyDeviceToHost,
                                c->stream));
        GK_CUDA(cudaStreamSynchronize(c->stream));
      });
  }
  return st;
}

gk_status gk_mesh_create(gk_ctx* c, const double* verts, size_t nv, const uint32_t* tris,
                         size_t nt, int m, int n, gk_mesh** out) {
  return gk_mesh_create_ex(c, verts, nv, tris, nt, m, n, nullptr, out);
}

gk_status gk_mesh_create_ex(gk_ctx* c, const double* verts, size_t nv, const uint32_t* tris,
                            size_t nt, int m, int n, const gk_mesh_options* opts,
                            gk_mesh** out) {
  return guarded([&] {
    const gk_mesh_options mo = opts ? *opts : gk::default_mesh_options();
    need(mo.edge_chunks == 0 || mo.edge_chunks == GK_AUTO ||
             (mo.edge_chunks >= 1 && mo.edge_chunks * 32 <= gk::kEdgeCap),
         GK_ERR_INVALID_ARGUMENT, "gk_mesh_options: edge_chunks must be 1..12");
    need(mo.sweep_chunks == 0 || mo.sweep_chunks == GK_AUTO ||
             (mo.sweep_chunks >= 1 && mo.sweep_chunks * 32 <= gk::kEdgeCap),
         GK_ERR_INVALID_ARGUMENT, "gk_mesh_options: sweep_chunks must be 1..12");
    check_ctx(c);
    need(out != nullptr, GK_ERR_INVALID_ARGUMENT, "null output");
    validate_spec(m, n);  // fill_matrix validates the spec first (matfill.hpp:148)
    need(nv == 0 || verts, GK_ERR_INVALID_ARGUMENT, "null vertices");
    need(nt == 0 || tris, GK_ERR_INVALID_ARGUMENT, "null triangles");
    gk::validate_mesh(verts, nv, tris, nt);
    need(nt >= 1, GK_ERR_INVALID_ARGUMENT, "gk_mesh_create: empty mesh");
    use_device(c);
    auto* mesh = new gk_mesh();
    try {
      mesh->ctx = c;
      mesh->N = nt;
      mesh->nv = nv;
      mesh->m = m;
      mesh->n = n;
      double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
      for (size_t i = 0; i < nv; ++i)
        for (int c3 = 0; c3 < 3; ++c3) {
          lo[c3] = std::fmin(lo[c3], verts[3 * i + c3]);
          hi[c3] = std::fmax(hi[c3], verts[3 * i + c3]);
        }
      double area = 0.0;
      for (size_t i = 0; i < nt; ++i) {
        const double* a = verts + 3 * static_cast<size_t>(tris[3 * i]);
        const double* b = verts + 3 * static_cast<size_t>(tris[3 * i + 1]);
        const double* c3v = verts + 3 * static_cast<size_t>(tris[3 * i + 2]);
        const double e1x = b[0] - a[0], e1y = b[1] - a[1], e1z = b[2] - a[2];
        const double e2x = c3v[0] - a[0], e2y = c3v[1] - a[1], e2z = c3v[2] - a[2];
        const double cx = e1y * e2z - e1z * e2y, cy = e1z * e2x - e1x * e2z, cz = e1x * e2y - e1y * e2x;
        area += 0.5 * std::sqrt(cx * cx + cy * cy + cz * cz);
      }
      mesh->mean_edge = std::sqrt(4.0 * (area / static_cast<double>(nt)) / std::sqrt(3.0));
      mesh->diameter = std::sqrt((hi[0] - lo[0]) * (hi[0] - lo[0]) + (hi[1] - lo[1]) * (hi[1] - lo[1]) +
                                 (hi[2] - lo[2]) * (hi[2] - lo[2])) * (1.0 + 1e-12);
      mesh->outer.alloc(nt * m, c->stream);
      mesh->inner.alloc(nt * 3 * static_cast<size_t>(n), c->stream);
      mesh->bounds.alloc(nt, c->stream);
      mesh->binner.alloc(nt, c->stream);
      gk::DevBuf<uint32_t> dt;
      mesh->verts.alloc(3 * nv, c->stream);
      dt.alloc(3 * nt, c->stream);
      GK_CUDA(cudaMemcpyAsync(mesh->verts.p, verts, 3 * nv * sizeof(double), cudaMemcpyHostToDevice, c->stream));
      GK_CUDA(cudaMemcpyAsync(dt.p, tris, 3 * nt * sizeof(uint32_t), cudaMemcpyHostToDevice, c->stream));
      gk::launch_points(mesh, mesh->verts.p, dt.p, c->stream);
      {
        std::vector<double4> hb(nt);
        GK_CUDA(cudaMemcpyAsync(hb.data(), mesh->bounds.p, nt * sizeof(double4),
                                cudaMemcpyDeviceToHost, c->stream));
        GK_CUDA(cudaStreamSynchronize(c->stream));
        for (const double4& b : hb) mesh->rho_outer_max = std::fmax(mesh->rho_outer_max, b.w);
      }
      gk::build_edge_blocks(mesh, verts, tris, mo);
      GK_CUDA(cudaStreamSynchronize(c->stream));
    } catch (...) {
      delete mesh;
      throw;
    }
    *out = mesh;
  });
}

gk_status gk_mesh_edge_info_get(const gk_mesh* mesh, gk_mesh_edge_info* out) {
  return guarded([&] {
    need(mesh != nullptr && out != nullptr, GK_ERR_INVALID_ARGUMENT, "null argument");
    out->blocks = mesh->es.nblk;
    out->edge_slots = mesh->es.nblk ? mesh->es.ep.n / (2 * static_cast<size_t>(mesh->n)) : 0;
    out->work_ratio = mesh->es.edge_ratio;
    out->delta = mesh->es.edge_delta;
    out->r_far = mesh->es.r_far;
    out->edges = mesh->es.edges;
    out->rho_mean = mesh->es.rho_mean;
    out->ordered = mesh->es.ordered ? 1 : 0;
    out->rho_max = mesh->es.rho_max;
    out->sweep_blocks = mesh->sweep.nblk;
    out->sweep_edge_slots = mesh->sweep.nblk ? mesh->sweep.ep.n / (2 * static_cast<size_t>(mesh->n)) : 0;
    out->sweep_work_ratio = mesh->sweep.edge_ratio;
    out->sweep_rho_max = mesh->sweep.rho_max;
  });
}

gk_status gk_edge_blocks_plan(const double* verts, size_t nv, const uint32_t* tris, size_t nt,
                              int chunks, int order_mode, int leaf_pct, double rho_cap,
                              uint32_t* order, uint32_t* edge_index,
                              uint32_t* block_start, uint32_t* block_edges, uint64_t* nblocks,
                              int* ordered) {
  return guarded([&] {
    need(verts && tris && order && edge_index && block_start && block_edges && nblocks && ordered,
         GK_ERR_INVALID_ARGUMENT, "null argument");
    need(chunks >= 1 && chunks * 32 <= gk::kEdgeCap, GK_ERR_INVALID_ARGUMENT,
         "gk_edge_blocks_plan: chunks must be 1..12");
    need(order_mode >= -1 && order_mode <= 1, GK_ERR_INVALID_ARGUMENT, "bad order_mode");
    gk::validate_mesh(verts, nv, tris, nt);
    need(nt >= 1, GK_ERR_INVALID_ARGUMENT, "empty mesh");
    const gk::EdgePlan P = gk::plan_edge_blocks(verts, nv, tris, nt, 32 * static_cast<size_t>(chunks),
                                                order_mode, leaf_pct, rho_cap);
    for (size_t j = 0; j < nt; ++j) {
      order[j] = P.order[j];
      edge_index[3 * j] = P.eidx[j].x;
      edge_index[3 * j + 1] = P.eidx[j].y;
      edge_index[3 * j + 2] = P.eidx[j].z;
    }
    for (size_t b = 0; b < P.blocks.size(); ++b) {
      block_start[b] = P.blocks[b].tb;
      block_edges[b] = P.blocks[b].ne;
    }
    block_start[P.blocks.size()] = static_cast<uint32_t>(nt);
    *nblocks = P.blocks.size();
    *ordered = P.ordered ? 1 : 0;
  });
}

gk_status gk_mesh_points_download(const gk_mesh* mesh, double* outer, double* inner) {
  return guarded([&] {
    need(mesh != nullptr, GK_ERR_INVALID_ARGUMENT, "null mesh");
    use_device(mesh->ctx);
    cudaStream_t s = mesh->ctx->stream;
    const size_t no = mesh->N * mesh->m, ni = mesh->N * 3 * static_cast<size_t>(mesh->n);
    std::vector<double4> ho(no), hi(ni);
    GK_CUDA(cudaMemcpyAsync(ho.data(), mesh->outer.p, no * sizeof(double4), cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaMemcpyAsync(hi.data(), mesh->inner.p, ni * sizeof(double4), cudaMemcpyDeviceToHost, s));
    GK_CUDA(cudaStreamSynchronize(s));
    if (outer)
      for (size_t k = 0; k < no; ++k) {
        outer[k] = ho[k].x;
        outer[no + k] = ho[k].y;
        outer[2 * no + k] = ho[k].z;
        outer[3 * no + k] = ho[k].w;
      }
    if (inner) {
      // device planes are [3n][N]; the reference order is q * 3n + i
      const size_t N = mesh->N, ipt = 3 * static_cast<size_t>(mesh->n);
      for (size_t i = 0; i < ipt; ++i)
        for (size_t q = 0; q < N; ++q) {
          const double4& v = hi[i * N + q];
          const size_t k = q * ipt + i;
          inner[k] = v.x;
          inner[ni + k] = v.y;
          inner[2 * ni + k] = v.z;
          inner[3 * ni + k] = v.w;
        }
    }
  });
}

gk_status gk_mesh_destroy(gk_mesh* mesh) {
  return guarded([&] {
    if (!mesh) return;
    cudaSetDevice(mesh->ctx->device);
    cudaStreamSynchronize(mesh->ctx->stream);
    delete mesh;
  });
}

gk_status gk_distance_range(gk_ctx* c, const gk_mesh* mesh, size_t row_begin, size_t row_end,
                            double* r_min, double* r_max) {
  return guarded([&] {
    check_ctx(c);
    need(mesh && r_min && r_max, GK_ERR_INVALID_ARGUMENT, "null argument");
    need(mesh->N >= 2, GK_ERR_INVALID_ARGUMENT, "gk_distance_range: need at least two triangles");
    need(row_begin < row_end && row_end <= mesh->N, GK_ERR_INVALID_ARGUMENT,
         "gk_distance_range: bad row range");
    use_device(c);
    double d2min = 0.0, d2max = 0.0;
    gk::launch_range(c, mesh, row_begin, row_end, &d2min, &d2max);
    *r_min = std::sqrt(d2min) * (1.0 - 0x1p-49);
    *r_max = std::sqrt(d2max) * (1.0 + 0x1p-49);
  });
}

namespace {

// fill_rows on the device for kind EXP / GREEN, or 2 = the fused pair (z: Exp, z2: Green)
void fill_rows_impl(gk_ctx* c, const gk_mesh* mesh, gk_mode mode, const gk_table* t, int kind,
                    double k_re, double k_im, size_t row_begin, size_t row_end, gk_c128* z,
                    gk_c128* z2, size_t ldz, const gk_fill_options* opts,
                    gk_fill_report* report) {
  check_ctx(c);
  need(mesh != nullptr, GK_ERR_INVALID_ARGUMENT, "null mesh");
  need(mode == GK_MODE_DIRECT || mode == GK_MODE_TABLE, GK_ERR_INVALID_ARGUMENT, "bad mode");
  need(row_begin <= row_end && row_end <= mesh->N, GK_ERR_INVALID_ARGUMENT,
       "gk_fill_rows: bad row range");
  need(ldz >= mesh->N, GK_ERR_INVALID_ARGUMENT, "gk_fill_rows: ldz < N");
  need(row_begin == row_end || (z && (kind != 2 || z2)), GK_ERR_INVALID_ARGUMENT, "null z");
  if (mode == GK_MODE_TABLE) {
    need(t != nullptr, GK_ERR_INVALID_ARGUMENT, "TABLE mode needs a table");
    k_re = t->dev.k_re;
    k_im = t->dev.k_im;
  }
  need(k_re >= 0.0, GK_ERR_INVALID_ARGUMENT, "eval_analytic: k must be >= 0");
  const uint64_t kinds = kind == 2 ? 2 : 1;
  const uint64_t pred = predicted(mesh->N, mesh->m, mesh->n);
  use_device(c);
  // synchronous fills count into their own words; asynchronous ones (report
  // == NULL) accumulate in the context until gk_fill_check reads them
  unsigned long long* cnt = c->scratch.p + (report ? 16 : kAsyncFillCounters);
  if (report) {
    GK_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c->stream));
    GK_CUDA(cudaEventRecord(c->ev0, c->stream));
  }
  const int path =
      gk::launch_fill(c, mesh, mode, t, kind, k_re, k_im, row_begin, row_end, z, z2, ldz, cnt,
                      opts ? *opts : c->opts);
  if (!report) return;
  GK_CUDA(cudaEventRecord(c->ev1, c->stream));
  unsigned long long h[4];
  GK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
  GK_CUDA(cudaStreamSynchronize(c->stream));
  float ms = 0.f;
  GK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
  report->N = mesh->N;
  report->m = mesh->m;
  report->n = mesh->n;
  report->predicted_calls = kinds * pred;
  const size_t rows = row_end - row_begin;
  report->actual_calls = kinds * 3ull * mesh->m * mesh->n * rows * (mesh->N - 1);
  report->fallback_calls = h[0] + h[1];
  report->wall_time_s = ms * 1e-3;
  report->evaluations = gk::path_counts_evaluations(path) ? h[3] : report->actual_calls;
  report->path = path;
  raise_fill_errors(h);
}

}  // namespace

gk_status gk_fill_check(gk_ctx* c, uint64_t* fallbacks) {
  return guarded([&] {
    check_ctx(c);
    use_device(c);
    unsigned long long* cnt = c->scratch.p + kAsyncFillCounters;
    unsigned long long h[4];
    GK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(h), c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    if (fallbacks) *fallbacks = h[0] + h[1];
    raise_fill_errors(h);
  });
}

gk_status gk_fill_rows(gk_ctx* c, const gk_mesh* mesh, gk_mode mode, const gk_table* t,
                       gk_kind kind, double k_re, double k_im, size_t row_begin, size_t row_end,
                       gk_c128* z, size_t ldz, const gk_fill_options* opts,
                       gk_fill_report* report) {
  return guarded([&] {
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    fill_rows_impl(c, mesh, mode, t, kind, k_re, k_im, row_begin, row_end, z, nullptr, ldz,
                   opts, report);
  });
}

gk_status gk_fill_rows_pair(gk_ctx* c, const gk_mesh* mesh, gk_mode mode, const gk_table* t,
                            double k_re, double k_im, size_t row_begin, size_t row_end,
                            gk_c128* z_exp, gk_c128* z_green, size_t ldz,
                            const gk_fill_options* opts, gk_fill_report* report) {
  return guarded([&] {
    fill_rows_impl(c, mesh, mode, t, 2, k_re, k_im, row_begin, row_end, z_exp, z_green, ldz,
                   opts, report);
  });
}

namespace {

// chunked, double-buffered device fill + D2H into host memory
void fill_rows_to_host(gk_ctx* c, const gk_mesh* mesh, gk_mode mode, const gk_table* table,
                       gk_kind kind, double k_re, double k_im, size_t row_begin, size_t row_end,
                       gk_c128* z_host, size_t ldz, const gk_fill_options& opts,
                       gk_fill_report* report) {
  const size_t nt = mesh->N;
  need(ldz >= nt, GK_ERR_INVALID_ARGUMENT, "ldz_host < N");
  need(row_begin <= row_end && row_end <= nt, GK_ERR_INVALID_ARGUMENT, "bad row range");
  need(row_begin == row_end || z_host, GK_ERR_INVALID_ARGUMENT, "null z_host");
  if (mode == GK_MODE_TABLE) {
    need(table != nullptr, GK_ERR_INVALID_ARGUMENT, "TABLE mode needs a table");
    k_re = table->dev.k_re;
    k_im = table->dev.k_im;
  }
  const size_t row_bytes = nt * sizeof(gk_c128);
  // chunk sizes grow geometrically from ~32 MB to 1 GiB: the copy engine
  // starts after a sub-millisecond first fill instead of a 1 GiB one, then
  // every copy overlaps the (faster) fill of the next chunk
  size_t chunk = (size_t(1) << 30) / row_bytes;
  if (chunk < 8) chunk = 8;
  if (chunk > row_end - row_begin) chunk = row_end - row_begin;
  if (chunk == 0) chunk = 1;
  size_t first = (size_t(32) << 20) / row_bytes;
  if (first < 8) first = 8;
  if (first > chunk) first = chunk;
  HostFillPipe& P = c->pipe;
  auto cleanup = [&] {  // leave both streams idle; the pipe itself is kept
    if (P.copy) cudaStreamSynchronize(P.copy);
    cudaStreamSynchronize(c->stream);
  };
  try {
    if (!P.copy) {
      GK_CUDA(cudaStreamCreateWithFlags(&P.copy, cudaStreamNonBlocking));
      for (int b = 0; b < 2; ++b) {
        GK_CUDA(cudaEventCreateWithFlags(&P.filled[b], cudaEventDisableTiming));
        GK_CUDA(cudaEventCreateWithFlags(&P.copied[b], cudaEventDisableTiming));
      }
    }
    for (int b = 0; b < 2; ++b)
      if (P.buf[b].n < chunk * nt) P.buf[b].alloc(chunk * nt, c->stream);
    cudaStream_t copy = P.copy;
    gk_c128* dz[2] = {P.buf[0].p, P.buf[1].p};
    cudaEvent_t* filled = P.filled;
    cudaEvent_t* copied = P.copied;
    unsigned long long* cnt = c->scratch.p + 16;
    GK_CUDA(cudaMemsetAsync(cnt, 0, 4 * sizeof(unsigned long long), c->stream));
    GK_CUDA(cudaEventRecord(c->ev0, c->stream));
    size_t idx = 0, step = first;
    int path = 0;
    for (size_t rb = row_begin; rb < row_end; rb += step, step = std::min(chunk, 2 * step), ++idx) {
      const size_t re = rb + step < row_end ? rb + step : row_end;
      const int b = static_cast<int>(idx & 1);
      if (idx >= 2) GK_CUDA(cudaStreamWaitEvent(c->stream, copied[b], 0));
      path = gk::launch_fill(c, mesh, mode, table, kind, k_re, k_im, rb, re, dz[b], nullptr, nt,
                             cnt, opts);
      GK_CUDA(cudaEventRecord(filled[b], c->stream));
      GK_CUDA(cudaStreamWaitEvent(copy, filled[b], 0));
      if (ldz == nt)  // contiguous rows on both sides: one linear copy
        GK_CUDA(cudaMemcpyAsync(z_host + (rb - row_begin) * ldz, dz[b], (re - rb) * row_bytes,
                                cudaMemcpyDeviceToHost, copy));
      else
        GK_CUDA(cudaMemcpy2DAsync(z_host + (rb - row_begin) * ldz, ldz * sizeof(gk_c128), dz[b],
                                  row_bytes, row_bytes, re - rb, cudaMemcpyDeviceToHost, copy));
      GK_CUDA(cudaEventRecord(copied[b], copy));
    }
    GK_CUDA(cudaEventRecord(c->ev1, c->stream));
    unsigned long long h[4];
    GK_CUDA(cudaMemcpyAsync(h, cnt, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(copy));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    float ms = 0.f;
    GK_CUDA(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    if (report) {
      report->N = nt;
      report->m = mesh->m;
      report->n = mesh->n;
      report->predicted_calls = predicted(nt, mesh->m, mesh->n);
      report->actual_calls = 3ull * mesh->m * mesh->n * (row_end - row_begin) * (nt - 1);
      report->fallback_calls = h[0] + h[1];
      report->wall_time_s = ms * 1e-3;
      report->evaluations = gk::path_counts_evaluations(path) ? h[3] : report->actual_calls;
      report->path = path;
    }
    raise_fill_errors(h);
  } catch (...) {
    cleanup();
    throw;
  }
  cleanup();
}

}  // namespace

gk_status gk_fill_rows_host(gk_ctx* c, const gk_mesh* mesh, gk_mode mode, const gk_table* t,
                            gk_kind kind, double k_re, double k_im, size_t row_begin,
                            size_t row_end, gk_c128* z_host, size_t ldz,
                            const gk_fill_options* opts, gk_fill_report* report) {
  return guarded([&] {
    check_ctx(c);
    need(mesh != nullptr, GK_ERR_INVALID_ARGUMENT, "null mesh");
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    use_device(c);
    fill_rows_to_host(c, mesh, mode, t, kind, k_re, k_im, row_begin, row_end, z_host, ldz,
                      opts ? *opts : c->opts, report);
  });
}

gk_status gk_fill_matrix_host(gk_ctx* c, const double* verts, size_t nv, const uint32_t* tris,
                              size_t nt, int m, int n, gk_mode mode,
                              const gk_sampling_config* cfg, const gk_medium* med, gk_kind kind,
                              gk_c128* z_host, gk_fill_report* report) {
  gk_mesh* mesh = nullptr;
  gk_table* table = nullptr;
  gk_status st = guarded([&] {
    check_ctx(c);
    need(med && z_host, GK_ERR_INVALID_ARGUMENT, "null argument");
    need(mode != GK_MODE_TABLE || cfg, GK_ERR_INVALID_ARGUMENT, "TABLE mode needs a config");
    double k_re, k_im;
    wavenumber(*med, k_re, k_im);
    // the mesh's own status (invalid_argument, or runtime_error for a CUDA /
    // out-of-memory failure) is the call's
    const gk_status ms = gk_mesh_create(c, verts, nv, tris, nt, m, n, &mesh);
    if (ms != GK_OK) gk::fail(ms, g_last_error);
    if (mode == GK_MODE_TABLE) {
      gk_sampling_config cc = *cfg;
      if (cc.r_min <= 0.0 || cc.r_max <= 0.0) {
        double lo, hi;
        const gk_status s = gk_distance_range(c, mesh, 0, nt, &lo, &hi);
        if (s != GK_OK) gk::fail(s, g_last_error);
        if (cc.r_min <= 0.0) cc.r_min = lo;
        if (cc.r_max <= 0.0) cc.r_max = hi;
      }
      const gk_status s = gk_table_build(c, &cc, med, 3, &table);
      if (s != GK_OK) gk::fail(s, g_last_error);
    }
    use_device(c);
    fill_rows_to_host(c, mesh, mode, table, kind, k_re, k_im, 0, nt, z_host, nt, c->opts, report);
  });
  gk_table_destroy(table);
  gk_mesh_destroy(mesh);
  return st;
}

gk_status gk_bench_compare(gk_ctx* c, const double* verts, size_t nv, const uint32_t* tris,
                           size_t nt, int m, int n, const gk_medium* med,
                           const gk_sampling_config* cfg, int degree, gk_kind kind, int repeats,
                           gk_bench_report* out) {
  gk_mesh* mesh = nullptr;
  gk_table* table = nullptr;
  gk::DevBuf<gk_c128> za, zi;
  gk_status st = guarded([&] {
    check_ctx(c);
    need(med && cfg && out, GK_ERR_INVALID_ARGUMENT, "null argument");
    need(repeats >= 1, GK_ERR_INVALID_ARGUMENT, "bench_compare: repeats must be >= 1");
    need(kind == GK_KIND_EXP || kind == GK_KIND_GREEN, GK_ERR_INVALID_ARGUMENT, "bad kind");
    double k_re, k_im;
    wavenumber(*med, k_re, k_im);
    auto ok = [](gk_status s) {
      if (s != GK_OK) gk::fail(s, g_last_error);
    };
    ok(gk_mesh_create(c, verts, nv, tris, nt, m, n, &mesh));
    double maxd = 0.0;
    ok(gk_max_vertex_distance(c, mesh, &maxd));
    gk_sampling_config cc = *cfg;
    cc.r_max = maxd * 1.01;  // matfill.hpp:270
    ok(gk_table_build(c, &cc, med, degree, &table));
    use_device(c);
    za.alloc(nt * nt, c->stream);
    zi.alloc(nt * nt, c->stream);
    gk_fill_report ra{}, ri{};
    fill_rows_impl(c, mesh, GK_MODE_DIRECT, nullptr, kind, k_re, k_im, 0, nt, za.p, nullptr, nt,
                   nullptr, &ra);
    fill_rows_impl(c, mesh, GK_MODE_TABLE, table, kind, k_re, k_im, 0, nt, zi.p, nullptr, nt,
                   nullptr, &ri);
    for (int rep = 1; rep < repeats; ++rep) {  // interleaved (matfill.hpp:279-284)
      gk_fill_report r2{}, r3{};
      fill_rows_impl(c, mesh, GK_MODE_DIRECT, nullptr, kind, k_re, k_im, 0, nt, za.p, nullptr,
                     nt, nullptr, &r2);
      ra.wall_time_s = std::min(ra.wall_time_s, r2.wall_time_s);
      fill_rows_impl(c, mesh, GK_MODE_TABLE, table, kind, k_re, k_im, 0, nt, zi.p, nullptr, nt,
                     nullptr, &r3);
      ri.wall_time_s = std::min(ri.wall_time_s, r3.wall_time_s);
    }
    gk_bench_report r{};
    r.fill = ri;
    ok(gk_compare_fills(c, zi.p, za.p, nt, nt, 0, nt, &r.max_rel_re, &r.max_rel_im));
    r.table_build_s = table->info.build_ms * 1e-3;
    r.analytic_time_s = ra.wall_time_s;
    r.interp_time_s = ri.wall_time_s + r.table_build_s;
    r.speedup = r.analytic_time_s / r.interp_time_s;
    *out = r;
  });
  za.reset();
  zi.reset();
  gk_table_destroy(table);
  gk_mesh_destroy(mesh);
  return st;
}

gk_status gk_shared_alloc(gk_ctx* c, size_t bytes, void** dptr, unsigned char* handle) {
  return guarded([&] {
    check_ctx(c);
    need(dptr && handle && bytes > 0, GK_ERR_INVALID_ARGUMENT, "gk_shared_alloc: bad argument");
    use_device(c);
    void* p = nullptr;
    GK_CUDA(cudaMalloc(&p, bytes));  // IPC needs a plain cudaMalloc allocation
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
      cudaFree(p);
      gk::fail(GK_ERR_RUNTIME, std::string("cudaIpcGetMemHandle: ") + cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == GK_IPC_HANDLE_BYTES, "IPC handle size");
    std::memcpy(handle, &h, sizeof(h));
    *dptr = p;
  });
}

gk_status gk_shared_free(gk_ctx* c, void* dptr) {
  return guarded([&] {
    check_ctx(c);
    if (!dptr) return;
    use_device(c);
    GK_CUDA(cudaDeviceSynchronize());
    GK_CUDA(cudaFree(dptr));
  });
}

gk_status gk_ipc_open(gk_ctx* c, const unsigned char* handle, void** dptr) {
  return guarded([&] {
    check_ctx(c);
    need(handle && dptr, GK_ERR_INVALID_ARGUMENT, "gk_ipc_open: bad argument");
    use_device(c);
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, sizeof(h));
    void* p = nullptr;
    GK_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    *dptr = p;
  });
}

gk_status gk_ipc_close(gk_ctx* c, void* dptr) {
  return guarded([&] {
    check_ctx(c);
    if (!dptr) return;
    use_device(c);
    GK_CUDA(cudaStreamSynchronize(c->stream));
    GK_CUDA(cudaIpcCloseMemHandle(dptr));
  });
}

gk_status gk_predicted_calls(uint64_t N, uint64_t m, uint64_t n, uint64_t* out) {
  return guarded([&] {
    need(out != nullptr, GK_ERR_INVALID_ARGUMENT, "null output");
    *out = predicted(N, m, n);
  });
}

gk_status gk_sphere_mesh(double radius, int subdivisions, double* verts, size_t* nv,
                         uint32_t* tris, size_t* nt) {
  return guarded([&] {
    need(nv && nt, GK_ERR_INVALID_ARGUMENT, "null counts");
    std::vector<double> v;
    std::vector<uint32_t> t;
    gk::sphere_mesh(radius, subdivisions, v, t);
    gk::validate_mesh(v.data(), v.size() / 3, t.data(), t.size() / 3);
    *nv = v.size() / 3;
    *nt = t.size() / 3;
    if (verts) std::memcpy(verts, v.data(), v.size() * sizeof(double));
    if (tris) std::memcpy(tris, t.data(), t.size() * sizeof(uint32_t));
  });
}

gk_status gk_plate_mesh(double side, int cells, double* verts, size_t* nv, uint32_t* tris,
                        size_t* nt) {
  return guarded([&] {
    need(nv && nt, GK_ERR_INVALID_ARGUMENT, "null counts");
    std::vector<double> v;
    std::vector<uint32_t> t;
    gk::plate_mesh(side, cells, v, t);
    *nv = v.size() / 3;
    *nt = t.size() / 3;
    if (verts) std::memcpy(verts, v.data(), v.size() * sizeof(double));
    if (tris) std::memcpy(tris, t.data(), t.size() * sizeof(uint32_t));
  });
}

gk_status gk_jitter(double* verts, size_t nv, uint64_t seed, double amp) {
  return guarded([&] {
    need(nv == 0 || verts, GK_ERR_INVALID_ARGUMENT, "null vertices");
    gk::jitter(verts, nv, seed, amp);
  });
}

gk_status gk_bench_fp64_peak(gk_ctx* c, double* tflops) {
  return guarded([&] {
    check_ctx(c);
    need(tflops != nullptr, GK_ERR_INVALID_ARGUMENT, "null output");
    use_device(c);
    *tflops = gk::run_fp64_peak(c);
  });
}

gk_status gk_device_info(gk_ctx* c, int* sm_count, int* clock_khz, int* major, int* minor) {
  return guarded([&] {
    check_ctx(c);
    cudaDeviceProp p{};
    GK_CUDA(cudaGetDeviceProperties(&p, c->device));
    if (sm_count) *sm_count = p.multiProcessorCount;
    int clk = 0;
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, c->device);
    if (clock_khz) *clock_khz = clk;
    if (major) *major = p.major;
    if (minor) *minor = p.minor;
  });
}

}  // extern "C"
