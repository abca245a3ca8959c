// gk_sharded_fill -- the multi-GPU fill driven from C++ only (no Python, no
// torch): one process, one host thread per GPU, NCCL communicators made by
// gk_comm_init_all (ncclCommInitAll's pattern).  Each rank takes the
// reference's row chunk (matfill.hpp:206-221, gk_rows_of), and gk_fill_sharded
// runs K1 + the 16-byte NCCL all-reduce + the table build (TABLE) + the fill
// of its rows; --gather collects Z on rank 0 (gk_gather_rows).  Timing: CUDA
// events per rank around the step, max over ranks (the bench convention).
//
// usage: gk_sharded_fill [--gpus N] [--level L] [--m M] [--n N] [--lambda X]
//                        [--mode direct|table] [--S S] [--reps R] [--gather 0|1]
//                        [--check 0|1]
// --check compares the gathered matrix with a one-GPU gk_fill_rows bit for bit
// (meshes up to icosphere level 4).  Prints one JSON line.
#include <cuda_runtime.h>

#include <algorithm>
#include <barrier>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "gk/gk.h"

#define OK(call)                                                                          \
  do {                                                                                    \
    const gk_status s_ = (call);                                                          \
    if (s_ != GK_OK) {                                                                    \
      std::fprintf(stderr, "%s failed (%d): %s\n", #call, static_cast<int>(s_), gk_last_error()); \
      std::exit(1);                                                                       \
    }                                                                                     \
  } while (0)
#define CU(call)                                                                      \
  do {                                                                                \
    const cudaError_t e_ = (call);                                                    \
    if (e_ != cudaSuccess) {                                                          \
      std::fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));        \
      std::exit(1);                                                                   \
    }                                                                                 \
  } while (0)

int main(int argc, char** argv) {
  int gpus = 1, level = 5, m = 6, n = 4, reps = 3, gather = 0, check = 0, S = 10000;
  double lambda0 = 0.3;
  gk_mode mode = GK_MODE_DIRECT;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string a = argv[i], v = argv[i + 1];
    if (a == "--gpus") gpus = std::atoi(v.c_str());
    else if (a == "--level") level = std::atoi(v.c_str());
    else if (a == "--m") m = std::atoi(v.c_str());
    else if (a == "--n") n = std::atoi(v.c_str());
    else if (a == "--lambda") lambda0 = std::atof(v.c_str());
    else if (a == "--mode") mode = v == "table" ? GK_MODE_TABLE : GK_MODE_DIRECT;
    else if (a == "--S") S = std::atoi(v.c_str());
    else if (a == "--reps") reps = std::atoi(v.c_str());
    else if (a == "--gather") gather = std::atoi(v.c_str());
    else if (a == "--check") check = std::atoi(v.c_str());
    else {
      std::fprintf(stderr, "unknown option %s\n", a.c_str());
      return 2;
    }
  }
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (gpus < 1 || gpus > ndev) {
    std::fprintf(stderr, "--gpus %d: %d device(s) visible\n", gpus, ndev);
    return 2;
  }
  if (check) gather = 1;

  // the bench workload: icosphere + seeded jitter (host-only entry points)
  size_t nv = 0, nt = 0;
  OK(gk_sphere_mesh(1.0, level, nullptr, &nv, nullptr, &nt));
  std::vector<double> verts(3 * nv);
  std::vector<uint32_t> tris(3 * nt);
  OK(gk_sphere_mesh(1.0, level, verts.data(), &nv, tris.data(), &nt));
  OK(gk_jitter(verts.data(), nv, 1901, 1e-3));
  const uint64_t N = nt;
  const gk_medium med{lambda0, 1.0, 1.0, 0.0};
  gk_sampling_config cfg{0.0, 0.0, S, 2, 2.0, 0.5, 1};  // r_min/r_max <= 0: the global K1 range

  std::vector<gk_ctx*> ctx(gpus);
  for (int r = 0; r < gpus; ++r) OK(gk_ctx_create(r, &ctx[r]));
  std::vector<gk_comm*> comm(gpus);
  OK(gk_comm_init_all(ctx.data(), gpus, comm.data()));

  std::vector<double> ms(gpus, 0.0), lo(gpus), hi(gpus);
  std::vector<uint64_t> evals(gpus, 0), calls(gpus, 0);
  std::vector<int> nranks_seen(gpus, 0);
  gk_c128* zfull = nullptr;
  std::barrier sync(gpus);
  auto rank_main = [&](int r) {
    CU(cudaSetDevice(r));
    int nr = 0, rk = 0;
    OK(gk_comm_info(comm[r], &nr, &rk));
    // the rank's work runs on this stream; the timing events go on it too
    cudaStream_t st;
    CU(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    OK(gk_ctx_set_stream(ctx[r], st));
    nranks_seen[r] = nr;
    gk_mesh* mesh = nullptr;
    OK(gk_mesh_create(ctx[r], verts.data(), nv, tris.data(), nt, m, n, &mesh));
    uint64_t rb = 0, re = 0;
    OK(gk_rows_of(N, gpus, r, &rb, &re));
    gk_c128* z = nullptr;
    CU(cudaMalloc(&z, std::max<uint64_t>(re - rb, 1) * N * sizeof(gk_c128)));
    if (r == 0 && gather) CU(cudaMalloc(&zfull, N * N * sizeof(gk_c128)));
    gk_fill_report rep{};
    double rng[2] = {0.0, 0.0};
    OK(gk_fill_sharded(ctx[r], comm[r], mesh, mode, &cfg, &med, GK_KIND_GREEN, z, N, nullptr,
                       &rep, rng));  // warm-up
    double best = 1e30;
    for (int i = 0; i < reps; ++i) {
      OK(gk_ctx_synchronize(ctx[r]));
      sync.arrive_and_wait();
      cudaEvent_t e0, e1;
      CU(cudaEventCreate(&e0));
      CU(cudaEventCreate(&e1));
      CU(cudaEventRecord(e0, st));
      OK(gk_fill_sharded(ctx[r], comm[r], mesh, mode, &cfg, &med, GK_KIND_GREEN, z, N, nullptr,
                         &rep, rng));
      CU(cudaEventRecord(e1, st));
      CU(cudaEventSynchronize(e1));
      float t = 0.f;
      CU(cudaEventElapsedTime(&t, e0, e1));
      best = std::min(best, static_cast<double>(t));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    }
    ms[r] = best;
    evals[r] = rep.evaluations;
    calls[r] = rep.actual_calls;
    lo[r] = rng[0];
    hi[r] = rng[1];
    sync.arrive_and_wait();
    if (gather) OK(gk_gather_rows(ctx[r], comm[r], z, N, 0, r == 0 ? zfull : nullptr));
    sync.arrive_and_wait();
    CU(cudaFree(z));
    OK(gk_mesh_destroy(mesh));
    OK(gk_ctx_use_own_stream(ctx[r]));
    CU(cudaStreamDestroy(st));
  };
  std::vector<std::thread> th;
  for (int r = 0; r < gpus; ++r) th.emplace_back(rank_main, r);
  for (auto& t : th) t.join();

  bool same_range = true, checked = false, equal = true;
  for (int r = 1; r < gpus; ++r) same_range = same_range && lo[r] == lo[0] && hi[r] == hi[0];
  if (check) {  // the one-GPU fill of the whole matrix, bit for bit
    checked = true;
    CU(cudaSetDevice(0));
    gk_mesh* mesh = nullptr;
    OK(gk_mesh_create(ctx[0], verts.data(), nv, tris.data(), nt, m, n, &mesh));
    gk_c128* z1 = nullptr;
    CU(cudaMalloc(&z1, N * N * sizeof(gk_c128)));
    double k_re = 0.0, k_im = 0.0;
    OK(gk_wavenumber(&med, &k_re, &k_im));
    gk_table* table = nullptr;
    if (mode == GK_MODE_TABLE) {
      gk_sampling_config c1 = cfg;
      OK(gk_distance_range(ctx[0], mesh, 0, N, &c1.r_min, &c1.r_max));
      OK(gk_table_build(ctx[0], &c1, &med, 3, &table));
    }
    gk_fill_report rep{};
    OK(gk_fill_rows(ctx[0], mesh, mode, table, GK_KIND_GREEN, k_re, k_im, 0, N, z1, N, nullptr,
                    &rep));
    std::vector<gk_c128> a(N * N), b(N * N);
    CU(cudaMemcpy(a.data(), z1, N * N * sizeof(gk_c128), cudaMemcpyDeviceToHost));
    CU(cudaMemcpy(b.data(), zfull, N * N * sizeof(gk_c128), cudaMemcpyDeviceToHost));
    equal = std::memcmp(a.data(), b.data(), N * N * sizeof(gk_c128)) == 0;
    CU(cudaFree(z1));
    gk_table_destroy(table);
    gk_mesh_destroy(mesh);
  }
  if (zfull) {
    CU(cudaSetDevice(0));
    CU(cudaFree(zfull));
  }
  double mx = 0.0;
  uint64_t tot_calls = 0, tot_evals = 0;
  bool nranks_ok = true;
  for (int r = 0; r < gpus; ++r) {
    mx = std::max(mx, ms[r]);
    tot_calls += calls[r];
    tot_evals += evals[r];
    nranks_ok = nranks_ok && nranks_seen[r] == gpus;
  }
  std::printf(
      "{\"tool\": \"gk_sharded_fill\", \"n_gpus\": %d, \"N\": %llu, \"mode\": \"%s\", "
      "\"fill_ms_max_over_ranks\": %.4f, \"evals_per_s\": %.6e, \"actual_calls\": %llu, "
      "\"evaluations\": %llu, \"nccl_nranks_ok\": %s, \"same_table_range_on_every_rank\": %s, "
      "\"r_min\": %.17g, \"r_max\": %.17g, \"gathered\": %s, \"bitwise_equal_to_one_gpu\": %s}\n",
      gpus, static_cast<unsigned long long>(N), mode == GK_MODE_TABLE ? "table" : "direct", mx,
      static_cast<double>(tot_calls) / (mx * 1e-3), static_cast<unsigned long long>(tot_calls),
      static_cast<unsigned long long>(tot_evals), nranks_ok ? "true" : "false",
      same_range ? "true" : "false", lo[0], hi[0], gather ? "true" : "false",
      checked ? (equal ? "true" : "false") : "null");
  for (int r = 0; r < gpus; ++r) OK(gk_comm_destroy(comm[r]));
  for (int r = 0; r < gpus; ++r) OK(gk_ctx_destroy(ctx[r]));
  return (checked && !equal) || !nranks_ok || !same_range ? 1 : 0;
}
