// Ablation harness for the K4 direct-fill inner loop (standalone; not part
// of libgk).  Same tiling/prefetch as csrc/fill.cu::direct_kernel on synthetic
// points; each variant removes one ingredient so its cost can be attributed.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1901_04162_b200/csrc \
//        -o scripts/direct_variants scripts/direct_variants.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gk/gk.h"
#include "gk_device.cuh"

using namespace gk;

constexpr int kRows = 8, kThreads = 256, CPT = 32;

enum Var { BASE = 0, NO_LDS = 1, NO_MUFU = 2, OUTER_REG = 3, NO_GLOAD = 4, NO_STORE = 5, ALL_CONST = 6 };

template <int MO, int VAR, int MINB>
__global__ void __launch_bounds__(kThreads, MINB) kvar(const double4* outer, const double4* inner,
                                                         size_t N, int ipt, size_t rows,
                                                         double2* z, const double2* phase,
                                                         double K1) {
  extern __shared__ double2 tab[];
  __shared__ double so[kRows][MO][4];
  for (int i = threadIdx.x; i < kPhaseM; i += blockDim.x) tab[i] = phase[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ncb_total = (N + 32 * CPT - 1) / (32 * CPT);
  const size_t ntiles = ((rows + kRows - 1) / kRows) * ncb_total;
  double (*my)[4] = so[warp];
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t tr = tile / ncb_total, tc = tile - tr * ncb_total;
    const size_t p = tr * kRows + warp;
    if (p >= rows) continue;
    double rx[MO], ry[MO], rz[MO], rw[MO];
    __syncwarp();
    if (lane < MO) {
      const double4 P = outer[p * MO + lane];
      my[lane][0] = P.x; my[lane][1] = P.y; my[lane][2] = P.z; my[lane][3] = P.w;
    }
    __syncwarp();
    if (VAR == OUTER_REG)
      for (int o = 0; o < MO; ++o) { rx[o] = my[o][0]; ry[o] = my[o][1]; rz[o] = my[o][2]; rw[o] = my[o][3]; }
    const size_t q0 = tc * 32 * CPT;
    const int ncb = CPT;
    const int iters = ncb * ipt;
    double2 nxy, nzw;
    auto load = [&](int cb, int i) {
      const size_t q = q0 + 32 * cb + lane < N ? q0 + 32 * cb + lane : N - 1;
      if (VAR == NO_GLOAD || VAR == ALL_CONST) {
        nxy = make_double2(0.3 + 1e-3 * i + 1e-5 * lane, -0.2 + 1e-4 * cb);
        nzw = make_double2(0.1 * i, 0.01);
      } else {
        const double2* ptr = reinterpret_cast<const double2*>(inner + static_cast<size_t>(i) * N + q);
        nxy = __ldg(ptr);
        nzw = __ldg(ptr + 1);
      }
    };
    load(0, 0);
    double2 acc[MO];
    for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
    int cbn = 0, ni = 0;
    for (int it = 0; it < iters; ++it) {
      const double2 pxy = nxy, pzw = nzw;
      const int cbc = cbn;
      if (++ni == ipt) { ni = 0; ++cbn; }
      if (it + 1 < iters) load(cbn, ni);
#pragma unroll
      for (int o = 0; o < MO; ++o) {
        double ox, oy, oz;
        if (VAR == OUTER_REG) { ox = rx[o]; oy = ry[o]; oz = rz[o]; }
        else { const double2 a = *reinterpret_cast<const double2*>(&my[o][0]); ox = a.x; oy = a.y; oz = my[o][2]; }
        const double d2 = dist2(ox, oy, oz, pxy.x, pxy.y, pzw.x);
        double y;
        if (VAR == NO_MUFU || VAR == ALL_CONST) {
          const double y0 = __dmul_rn(d2, 0.75);
          const double e = __fma_rn(-d2, __dmul_rn(y0, y0), 1.0);
          y = __fma_rn(__dmul_rn(y0, e), __fma_rn(0.375, e, 0.5), y0);
        } else {
          y = rsqrt_fast(d2);
        }
        const double r = __dmul_rn(d2, y);
        double2 cs;
        if (VAR == NO_LDS || VAR == ALL_CONST) {
          constexpr double C = 2.0 * kPi / kPhaseM;
          const double t = __fma_rn(r, K1, kMagicRint);
          const double nf = t - kMagicRint;
          const double f = __fma_rn(r, K1, -nf);
          const double g = __dmul_rn(f, f);
          const double v = __dmul_rn(g, __fma_rn(C * C * C * C / 24.0, g, -C * C / 2.0));
          const double s = __dmul_rn(f, __fma_rn(-C * C * C / 6.0, g, C));
          const double2 T = make_double2(0.6, 0.8 + 1e-9 * __double2loint(t));
          cs = make_double2(__fma_rn(-T.y, s, __fma_rn(T.x, v, T.x)), __fma_rn(T.x, s, __fma_rn(T.y, v, T.y)));
        } else {
          cs = cis_phase(r, K1, tab);
        }
        const double wgt = __dmul_rn(pzw.y, y);
        acc[o].x = __fma_rn(wgt, cs.x, acc[o].x);
        acc[o].y = __fma_rn(-wgt, cs.y, acc[o].y);
      }
      if (ni == 0) {
        double2 res = make_double2(0.0, 0.0);
        for (int o = 0; o < MO; ++o) {
          const double wo = VAR == OUTER_REG ? rw[o] : my[o][3];
          res.x = __fma_rn(wo, acc[o].x, res.x);
          res.y = __fma_rn(wo, acc[o].y, res.y);
          acc[o] = make_double2(0.0, 0.0);
        }
        const size_t q = q0 + 32 * cbc + lane;
        if (VAR == NO_STORE || VAR == ALL_CONST) {
          if (res.x == 1234.5) z[0] = res;
        } else if (q < N) {
          __stcs(z + (p * N + q), res);
        }
      }
    }
  }
}


// v4: IPT compile-time, i-loop fully unrolled with register prefetch;
// OREG: outer points in registers (else broadcast LDS from shared memory)
template <int MO, int IPT, bool OREG, int MINB, int WARPS = 8>
__global__ void __launch_bounds__(32 * WARPS, MINB) kv4(const double4* outer, const double4* inner,
                                                       size_t N, size_t rows, double2* z,
                                                       const double2* phase, double K1) {
  extern __shared__ double2 tab[];
  __shared__ double so[WARPS][MO][4];
  for (int i = threadIdx.x; i < kPhaseM; i += blockDim.x) tab[i] = phase[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t ncb_total = (N + 32 * CPT - 1) / (32 * CPT);
  const size_t ntiles = ((rows + WARPS - 1) / WARPS) * ncb_total;
  double (*my)[4] = so[warp];
  for (size_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const size_t tr = tile / ncb_total, tc = tile - tr * ncb_total;
    const size_t p = tr * WARPS + warp;
    if (p >= rows) continue;
    double ox[MO], oy[MO], oz[MO];
    __syncwarp();
    if (lane < MO) {
      const double4 P = outer[p * MO + lane];
      my[lane][0] = P.x; my[lane][1] = P.y; my[lane][2] = P.z; my[lane][3] = P.w;
    }
    __syncwarp();
    if (OREG)
#pragma unroll
      for (int o = 0; o < MO; ++o) { ox[o] = my[o][0]; oy[o] = my[o][1]; oz[o] = my[o][2]; }
    const size_t q0 = tc * 32 * CPT;
    int nblk = static_cast<int>((N - q0 + 31) / 32);
    if (nblk > CPT) nblk = CPT;
    const double4* colp = inner + q0 + lane;      // column block 0, i = 0
    const double4* last = inner + (N - 1);
    double2 cxy, czw;
    {
      const double2* ptr = reinterpret_cast<const double2*>(colp <= last ? colp : last);
      cxy = __ldg(ptr); czw = __ldg(ptr + 1);
    }
    for (int cb = 0; cb < nblk; ++cb) {
      const double4* cp = colp <= last ? colp : last;
      double2 acc[MO];
#pragma unroll
      for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < IPT; ++i) {
        const double2 pxy = cxy, pzw = czw;
        // prefetch the next inner point (next i, or i = 0 of the next column block)
        const double4* np = (i + 1 < IPT) ? cp + (i + 1) * N : (colp + 32 <= last ? colp + 32 : last);
        const double2* nptr = reinterpret_cast<const double2*>(np);
        cxy = __ldg(nptr);
        czw = __ldg(nptr + 1);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          double oxv, oyv, ozv;
          if (OREG) { oxv = ox[o]; oyv = oy[o]; ozv = oz[o]; }
          else { const double2 a = *reinterpret_cast<const double2*>(&my[o][0]); oxv = a.x; oyv = a.y; ozv = my[o][2]; }
          const double d2 = dist2(oxv, oyv, ozv, pxy.x, pxy.y, pzw.x);
          const double y = rsqrt_fast(d2);
          const double r = __dmul_rn(d2, y);
          const double2 cs = cis_phase(r, K1, tab);
          const double wgt = __dmul_rn(pzw.y, y);
          acc[o].x = __fma_rn(wgt, cs.x, acc[o].x);
          acc[o].y = __fma_rn(-wgt, cs.y, acc[o].y);
        }
      }
      double2 res = make_double2(0.0, 0.0);
#pragma unroll
      for (int o = 0; o < MO; ++o) {
        const double wo = my[o][3];
        res.x = __fma_rn(wo, acc[o].x, res.x);
        res.y = __fma_rn(wo, acc[o].y, res.y);
      }
      const size_t q = q0 + 32 * cb + lane;
      if (q < N) __stcs(z + (p * N + q), res);
      colp += 32;
    }
  }
}

template <bool OREG, int MINB, int WARPS = 8>
float run4(const double4* o, const double4* in, size_t N, size_t rows, double2* z, const double2* ph,
           double K1, int sm) {
  auto k = kv4<6, 12, OREG, MINB, WARPS>;
  const size_t smem = kPhaseM * sizeof(double2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, 32 * WARPS, smem);
  const int grid = sm * per;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, 32 * WARPS, smem>>>(o, in, N, rows, z, ph, K1);
  cudaEventRecord(a);
  k<<<grid, 32 * WARPS, smem>>>(o, in, N, rows, z, ph, K1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, k);
  const double evals = double(rows) * N * 72;
  std::printf("v4 oreg %d minb %d warps %2d: %7.3f ms  %.3e evals/s  regs %d  occ %d  local %zu  %s\n", OREG, MINB,
              WARPS, ms, evals / (ms * 1e-3), at.numRegs, per, at.localSizeBytes,
              cudaGetErrorString(cudaGetLastError()));
  return ms;
}

template <int VAR, int MINB>
float run(const double4* o, const double4* in, size_t N, size_t rows, double2* z, const double2* ph,
          double K1, int sm) {
  auto k = kvar<6, VAR, MINB>;
  const size_t smem = kPhaseM * sizeof(double2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k, kThreads, smem);
  const int grid = sm * per;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<grid, kThreads, smem>>>(o, in, N, 12, rows, z, ph, K1);
  cudaEventRecord(a);
  k<<<grid, kThreads, smem>>>(o, in, N, 12, rows, z, ph, K1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, k);
  const double evals = double(rows) * N * 72;
  std::printf("var %d minb %d: %7.3f ms  %.3e evals/s  regs %d  occ %d  local %zu  %s\n", VAR, MINB, ms,
              evals / (ms * 1e-3), at.numRegs, per, at.localSizeBytes,
              cudaGetErrorString(cudaGetLastError()));
  return ms;
}

int main() {
  const size_t N = 32768, rows = 2048;
  std::vector<double4> ho(rows * 6), hi(12 * N);
  srand(1);
  auto rnd = [] { return rand() / (double)RAND_MAX; };
  for (auto& v : ho) v = make_double4(rnd() - 0.5, rnd() - 0.5, rnd() - 0.5, rnd());
  for (auto& v : hi) v = make_double4(rnd() - 0.5, rnd() - 0.5, rnd() - 0.5, rnd());
  double4 *o, *in;
  double2 *z, *ph;
  cudaMalloc(&o, ho.size() * 32);
  cudaMalloc(&in, hi.size() * 32);
  cudaMalloc(&z, rows * N * 16);
  cudaMalloc(&ph, kPhaseM * 16);
  cudaMemcpy(o, ho.data(), ho.size() * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(in, hi.data(), hi.size() * 32, cudaMemcpyHostToDevice);
  std::vector<double2> hp(kPhaseM);
  for (int i = 0; i < kPhaseM; ++i) hp[i] = make_double2(cos(2 * kPi * i / kPhaseM), sin(2 * kPi * i / kPhaseM));
  cudaMemcpy(ph, hp.data(), kPhaseM * 16, cudaMemcpyHostToDevice);
  int sm;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const double K1 = 2 * kPi / 0.15 * kPhaseM / (2 * kPi);
  run<BASE, 2>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 1, 8>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 2, 4>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 3, 4>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 1, 12>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 1, 16>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 1, 6>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 1, 4>(o, in, N, rows, z, ph, K1, sm);
  run4<true, 2, 6>(o, in, N, rows, z, ph, K1, sm);
  if (getenv("V4ONLY")) return 0;
  run<NO_LDS, 2>(o, in, N, rows, z, ph, K1, sm);
  run<NO_MUFU, 2>(o, in, N, rows, z, ph, K1, sm);
  run<OUTER_REG, 2>(o, in, N, rows, z, ph, K1, sm);
  run<NO_GLOAD, 2>(o, in, N, rows, z, ph, K1, sm);
  run<NO_STORE, 2>(o, in, N, rows, z, ph, K1, sm);
  run<ALL_CONST, 2>(o, in, N, rows, z, ph, K1, sm);
  run<BASE, 1>(o, in, N, rows, z, ph, K1, sm);
  run<ALL_CONST, 1>(o, in, N, rows, z, ph, K1, sm);
  return 0;
}
