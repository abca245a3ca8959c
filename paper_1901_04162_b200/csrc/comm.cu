// comm.cu -- the multi-GPU fill behind the C ABI: row blocks, one 16-byte
// NCCL all-reduce, and the optional gather of Z.
//
// The reference parallelises fill_matrix over std::threads that each take a
// contiguous chunk of observation rows, chunk = ceil(N / threads)
// (matfill.hpp:206-221); entries are independent, so the result does not
// depend on the split.  Here one rank per GPU takes the same chunk:
//
//   1. K1 over the rank's own rows (launch_range_device),
//   2. ONE ncclAllReduce(MIN) of the 16 bytes {min d^2, -max d^2} on the
//      device -- the global pair-distance range,
//   3. every rank builds the identical table from it (the device build is
//      deterministic: same inputs, same code, same GPU model),
//   4. every rank fills its rows -- no data-path collective,
//   5. optionally the row blocks are gathered to one rank (grouped
//      ncclSend / ncclRecv straight into the root's row slices).
//
// Host code is C++ throughout; torch.distributed is not needed (the Python
// layer ships the 128-byte ncclUniqueId over whatever transport it has).
//
// NCCL is bound at first use (dlopen), not linked: a process that already
// has an NCCL loaded (PyTorch bundles its own, newer one) must keep using it
// -- a DT_NEEDED on the system libnccl.so.2 would claim the soname first and
// break `import torch` after libgk.  Order: the libnccl.so.2 already in the
// process, else the dynamic loader's default (the system NCCL).
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "gk_internal.h"

namespace {

struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*);
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int);
  ncclResult_t (*CommDestroy)(ncclComm_t);
  ncclResult_t (*CommCount)(const ncclComm_t, int*);
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*);
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t);
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t);
  ncclResult_t (*GroupStart)();
  ncclResult_t (*GroupEnd)();
  const char* (*GetErrorString)(ncclResult_t);
};

const Nccl& nccl() {
  static Nccl api{};
  static std::string err;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW);
    if (!h) {
      const char* e = dlerror();
      err = std::string("NCCL not available: ") + (e ? e : "dlopen(libnccl.so.2) failed");
      return;
    }
    bool ok = true;
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) {
        ok = false;
        err = std::string("NCCL symbol missing: ") + name;
      }
    };
    sym(api.GetUniqueId, "ncclGetUniqueId");
    sym(api.CommInitRank, "ncclCommInitRank");
    sym(api.CommDestroy, "ncclCommDestroy");
    sym(api.CommCount, "ncclCommCount");
    sym(api.CommUserRank, "ncclCommUserRank");
    sym(api.AllReduce, "ncclAllReduce");
    sym(api.Send, "ncclSend");
    sym(api.Recv, "ncclRecv");
    sym(api.GroupStart, "ncclGroupStart");
    sym(api.GroupEnd, "ncclGroupEnd");
    sym(api.GetErrorString, "ncclGetErrorString");
    if (!ok) api = Nccl{};
  });
  if (!api.GetUniqueId) gk::fail(GK_ERR_RUNTIME, err);
  return api;
}

}  // namespace

struct gk_comm {
  gk_ctx* ctx = nullptr;
  ncclComm_t nccl = nullptr;
  int nranks = 0, rank = 0;
  gk::DevBuf<double> range;  // the 16 bytes the range all-reduce moves
};

namespace {

void nccl_ok(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    gk::fail(r == ncclInvalidArgument || r == ncclInvalidUsage ? GK_ERR_INVALID_ARGUMENT
                                                               : GK_ERR_RUNTIME,
             std::string(what) + ": " + nccl().GetErrorString(r));
}

void rows_of(uint64_t N, int nranks, int rank, uint64_t& b, uint64_t& e) {
  // matfill.hpp:211-215: chunk = ceil(N / threads), worker w takes
  // [w chunk, min(N, (w + 1) chunk))
  const uint64_t chunk = (N + static_cast<uint64_t>(nranks) - 1) / static_cast<uint64_t>(nranks);
  b = std::min<uint64_t>(N, static_cast<uint64_t>(rank) * chunk);
  e = std::min<uint64_t>(N, b + chunk);
}

void check_comm(const gk_ctx* c, const gk_comm* m) {
  gk::need(c != nullptr && m != nullptr, GK_ERR_INVALID_ARGUMENT, "null gk_ctx / gk_comm");
  gk::need(m->ctx == c, GK_ERR_INVALID_ARGUMENT,
           "gk_comm: the communicator belongs to another context (device)");
}

}  // namespace

extern "C" {

gk_status gk_rows_of(uint64_t N, int nranks, int rank, uint64_t* row_begin, uint64_t* row_end) {
  return gk::guarded([&] {
    gk::need(row_begin && row_end, GK_ERR_INVALID_ARGUMENT, "null output");
    gk::need(nranks >= 1 && rank >= 0 && rank < nranks, GK_ERR_INVALID_ARGUMENT,
             "gk_rows_of: need 0 <= rank < nranks");
    rows_of(N, nranks, rank, *row_begin, *row_end);
  });
}

gk_status gk_comm_unique_id(unsigned char id[GK_COMM_ID_BYTES]) {
  return gk::guarded([&] {
    gk::need(id != nullptr, GK_ERR_INVALID_ARGUMENT, "null id");
    static_assert(sizeof(ncclUniqueId) == GK_COMM_ID_BYTES, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    nccl_ok(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

gk_status gk_comm_init(gk_ctx* c, const unsigned char id[GK_COMM_ID_BYTES], int nranks, int rank,
                       gk_comm** out) {
  return gk::guarded([&] {
    gk::need(c && id && out, GK_ERR_INVALID_ARGUMENT, "null argument");
    gk::need(nranks >= 1 && rank >= 0 && rank < nranks, GK_ERR_INVALID_ARGUMENT,
             "gk_comm_init: need 0 <= rank < nranks");
    GK_CUDA(cudaSetDevice(c->device));
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto* m = new gk_comm();
    try {
      m->ctx = c;
      m->nranks = nranks;
      m->rank = rank;
      nccl_ok(nccl().CommInitRank(&m->nccl, nranks, u, rank), "ncclCommInitRank");
      m->range.alloc(2, c->stream);
    } catch (...) {
      if (m->nccl) nccl().CommDestroy(m->nccl);
      delete m;
      throw;
    }
    *out = m;
  });
}

gk_status gk_comm_init_all(gk_ctx* const* ctxs, int n, gk_comm** comms) {
  return gk::guarded([&] {
    gk::need(ctxs && comms && n >= 1, GK_ERR_INVALID_ARGUMENT, "gk_comm_init_all: bad arguments");
    for (int i = 0; i < n; ++i) {
      gk::need(ctxs[i] != nullptr, GK_ERR_INVALID_ARGUMENT, "gk_comm_init_all: null context");
      for (int j = 0; j < i; ++j)
        gk::need(ctxs[j]->device != ctxs[i]->device, GK_ERR_INVALID_ARGUMENT,
                 "gk_comm_init_all: one context per device");
      comms[i] = nullptr;
    }
    // ncclCommInitAll's pattern: one unique id, every rank initialised inside
    // one group from this thread
    ncclUniqueId u;
    nccl_ok(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::vector<gk_comm*> made(static_cast<size_t>(n), nullptr);
    try {
      for (int i = 0; i < n; ++i) {
        made[i] = new gk_comm();
        made[i]->ctx = ctxs[i];
        made[i]->nranks = n;
        made[i]->rank = i;
      }
      nccl_ok(nccl().GroupStart(), "ncclGroupStart");
      for (int i = 0; i < n; ++i) {
        GK_CUDA(cudaSetDevice(ctxs[i]->device));
        nccl_ok(nccl().CommInitRank(&made[i]->nccl, n, u, i), "ncclCommInitRank");
      }
      nccl_ok(nccl().GroupEnd(), "ncclGroupEnd");
      for (int i = 0; i < n; ++i) {
        GK_CUDA(cudaSetDevice(ctxs[i]->device));
        made[i]->range.alloc(2, ctxs[i]->stream);
      }
    } catch (...) {
      for (gk_comm* m : made)
        if (m) {
          if (m->nccl) nccl().CommDestroy(m->nccl);
          delete m;
        }
      throw;
    }
    for (int i = 0; i < n; ++i) comms[i] = made[i];
  });
}

gk_status gk_comm_destroy(gk_comm* m) {
  return gk::guarded([&] {
    if (!m) return;
    cudaSetDevice(m->ctx->device);
    cudaStreamSynchronize(m->ctx->stream);
    m->range.reset();
    if (m->nccl) nccl().CommDestroy(m->nccl);
    delete m;
  });
}

gk_status gk_comm_info(const gk_comm* m, int* nranks, int* rank) {
  return gk::guarded([&] {
    gk::need(m && nranks && rank, GK_ERR_INVALID_ARGUMENT, "null argument");
    int n = 0, r = 0;
    nccl_ok(nccl().CommCount(m->nccl, &n), "ncclCommCount");
    nccl_ok(nccl().CommUserRank(m->nccl, &r), "ncclCommUserRank");
    *nranks = n;
    *rank = r;
  });
}

gk_status gk_distance_range_global(gk_ctx* c, gk_comm* m, const gk_mesh* mesh, double* r_min,
                                   double* r_max) {
  return gk::guarded([&] {
    check_comm(c, m);
    gk::need(mesh && r_min && r_max, GK_ERR_INVALID_ARGUMENT, "null argument");
    gk::need(mesh->N >= 2, GK_ERR_INVALID_ARGUMENT,
             "gk_distance_range: need at least two triangles");
    GK_CUDA(cudaSetDevice(c->device));
    uint64_t b, e;
    rows_of(mesh->N, m->nranks, m->rank, b, e);
    gk::launch_range_device(c, mesh, b, e, m->range.p);
    nccl_ok(nccl().AllReduce(m->range.p, m->range.p, 2, ncclDouble, ncclMin, m->nccl, c->stream),
            "ncclAllReduce");
    double h[2];
    GK_CUDA(cudaMemcpyAsync(h, m->range.p, sizeof(h), cudaMemcpyDeviceToHost, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
    // gk_distance_range's widening (every radius the fill computes lies inside)
    *r_min = std::sqrt(h[0]) * (1.0 - 0x1p-49);
    *r_max = std::sqrt(-h[1]) * (1.0 + 0x1p-49);
  });
}

gk_status gk_fill_sharded(gk_ctx* c, gk_comm* m, const gk_mesh* mesh, gk_mode mode,
                          const gk_sampling_config* cfg, const gk_medium* medium, gk_kind kind,
                          gk_c128* z_rows, size_t ldz, const gk_fill_options* opts,
                          gk_fill_report* report, double* r_range) {
  return gk::guarded([&] {
    check_comm(c, m);
    gk::need(mesh && medium, GK_ERR_INVALID_ARGUMENT, "null argument");
    gk::need(mode != GK_MODE_TABLE || cfg, GK_ERR_INVALID_ARGUMENT, "TABLE mode needs a config");
    uint64_t b, e;
    rows_of(mesh->N, m->nranks, m->rank, b, e);
    double k_re = 0.0, k_im = 0.0;
    gk::ok(gk_wavenumber(medium, &k_re, &k_im));
    gk_table* table = nullptr;
    struct Guard {
      gk_table*& t;
      ~Guard() { gk_table_destroy(t); }
    } guard{table};
    if (mode == GK_MODE_TABLE) {
      gk_sampling_config cc = *cfg;
      if (cc.r_min <= 0.0 || cc.r_max <= 0.0) {  // the global K1 range (one all-reduce)
        double lo = 0.0, hi = 0.0;
        gk::ok(gk_distance_range_global(c, m, mesh, &lo, &hi));
        if (cc.r_min <= 0.0) cc.r_min = lo;
        if (cc.r_max <= 0.0) cc.r_max = hi;
      }
      if (r_range) {
        r_range[0] = cc.r_min;
        r_range[1] = cc.r_max;
      }
      gk::ok(gk_table_build(c, &cc, medium, 3, &table));
    }
    gk::ok(gk_fill_rows(c, mesh, mode, table, kind, k_re, k_im, b, e, z_rows, ldz, opts, report));
  });
}

gk_status gk_gather_rows(gk_ctx* c, gk_comm* m, const gk_c128* z_rows, uint64_t N, int root,
                         gk_c128* z_full) {
  return gk::guarded([&] {
    check_comm(c, m);
    gk::need(root >= 0 && root < m->nranks, GK_ERR_INVALID_ARGUMENT, "gk_gather_rows: bad root");
    gk::need(m->rank != root || z_full != nullptr, GK_ERR_INVALID_ARGUMENT,
             "gk_gather_rows: the root needs z_full");
    GK_CUDA(cudaSetDevice(c->device));
    uint64_t b, e;
    rows_of(N, m->nranks, m->rank, b, e);
    gk::need(e == b || z_rows != nullptr, GK_ERR_INVALID_ARGUMENT, "gk_gather_rows: null z_rows");
    // complex128 rows move as pairs of doubles; every block lands in its row
    // slice of the root's matrix (no staging copy)
    nccl_ok(nccl().GroupStart(), "ncclGroupStart");
    if (m->rank == root) {
      for (int r = 0; r < m->nranks; ++r) {
        uint64_t rb, re;
        rows_of(N, m->nranks, r, rb, re);
        if (r == root || re == rb) continue;
        nccl_ok(nccl().Recv(z_full + rb * N, 2 * (re - rb) * N, ncclDouble, r, m->nccl, c->stream),
                "ncclRecv");
      }
    } else if (e > b) {
      nccl_ok(nccl().Send(z_rows, 2 * (e - b) * N, ncclDouble, root, m->nccl, c->stream),
              "ncclSend");
    }
    nccl_ok(nccl().GroupEnd(), "ncclGroupEnd");
    if (m->rank == root && e > b && z_full + b * N != z_rows)
      GK_CUDA(cudaMemcpyAsync(z_full + b * N, z_rows, (e - b) * N * sizeof(gk_c128),
                              cudaMemcpyDeviceToDevice, c->stream));
    GK_CUDA(cudaStreamSynchronize(c->stream));
  });
}

}  // extern "C"
