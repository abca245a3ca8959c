// Harness for the far path of the shared-edge direct fill (direct_edge_kernel,
// csrc/fill_kernels.cuh): standalone, synthetic blocks of 11 x 32 edge slots x
// 4 points, 12 rows per tile, the 128 KB phase table and the per-warp edge
// sums in shared memory as in the product kernel.  It compares the product's
// difference form (25.5 FP64 operations per term) with the expanded distance
//   |o - P|^2 / w^2 = |a|^2 s + B + a.q,   a = o - c,  q = -2 (P - c) s,
//   B = |P - c|^2 s,  s = 1 / w^2   (22.7 operations, rsqrt gives w / r)
// in several loop structures (DESIGN.md §5 "K4f").
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1901_04162_b200/csrc \
//        -I include -o scripts/far_variants scripts/far_variants.cu
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "gk/gk.h"
#include "gk_device.cuh"

using namespace gk;

constexpr int MO = 6, NPE = 4, NCH = 11, W = 12;
constexpr int kSlots = NCH * 32;

enum Form {
  DIFF = 0,       // product: difference form + tan rotation
  EXP_REG = 1,    // expanded, a[] in registers, one point ahead in registers
  EXP_SMEM = 2,   // expanded, a[] re-read from shared memory per term (broadcast)
  EXP_SPLIT = 3,  // expanded, two lanes per edge: 3 outer points each
  EXP_NOPF = 4,   // expanded, a[] in registers, no register prefetch
  DIFF_SPLIT = 5, // difference form, two lanes per edge
  DIFF_PF2 = 6,   // difference form, two points ahead in registers
  DIFF_PLANAR = 7, // difference form, the points as two double2 planes (512 B runs per warp load)
};

__device__ __forceinline__ void tan_accumulate(double rphase, double K, double base, const double2* tab,
                                               double2& acc) {
  double c, sn, v;
  cis_phase_tan(rphase, K, tab, c, sn, v);
  const double wk = __fma_rn(base, v, base);
  acc.x = __fma_rn(wk, c, acc.x);
  acc.y = __fma_rn(-wk, sn, acc.y);
}

__device__ __forceinline__ void term_diff(double ox, double oy, double oz, double2 pxy, double2 pzw,
                                          double K1, const double2* tab, double2& acc) {
  const double d2 = dist2(ox, oy, oz, pxy.x, pxy.y, pzw.x);
  const double y = rsqrt_fast(d2);
  const double r = __dmul_rn(d2, y);
  tan_accumulate(r, K1, __dmul_rn(pzw.y, y), tab, acc);
}

__device__ __forceinline__ void term_exp(double ax, double ay, double az, double aA, double2 q01,
                                         double2 q23, double s, double wK, const double2* tab,
                                         double2& acc) {
  const double d2 = __fma_rn(ax, q01.x, __fma_rn(ay, q01.y, __fma_rn(az, q23.x, __fma_rn(aA, s, q23.y))));
  const double y = rsqrt_fast(d2);
  const double rs = __dmul_rn(d2, y);
  tan_accumulate(rs, wK, y, tab, acc);
}

__device__ __forceinline__ double lds_f64(const double* p) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(smem_u32(p)));
  return v;
}

struct Args {
  const double4* outer;   // [rows][MO] (x, y, z, w)
  const double4* ep;      // [nblk][NCH][NPE][32]
  const double2* epf;     // [nblk][NCH][NPE][3][32]
  const double2* ep2;     // [nblk][NCH][NPE][2][32]: (x, y) plane, (z, w) plane
  const double4* centre;  // [nblk]
  const double2* phase;
  double2* z;             // [rows][nblk * kSlots]
  size_t nblk, ntiles;
  double K1;
};

template <int FORM>
__global__ void __launch_bounds__(32 * W, 1) kfar(const Args A) {
  extern __shared__ double2 tab[];
  __shared__ double sw[W][MO];
  __shared__ double sa[W][MO][4];
  for (int i = threadIdx.x; i < kPhaseSlots; i += blockDim.x) tab[i] = A.phase[i];
  __syncthreads();
  double2* const sE = tab + kPhaseSlots;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const myE = sE + warp * kSlots;
  for (size_t tile = blockIdx.x; tile < A.ntiles; tile += gridDim.x) {
    const size_t tr = tile / A.nblk, b = tile - tr * A.nblk;
    const size_t p = tr * W + warp;
    double ox[MO], oy[MO], oz[MO], aA[MO];
    const double4 cb = A.centre[b];
#pragma unroll
    for (int o = 0; o < MO; ++o) {
      const double4 P = A.outer[p * MO + o];
      ox[o] = P.x; oy[o] = P.y; oz[o] = P.z;
      if (lane == 0) sw[warp][o] = P.w;
      if constexpr (FORM != DIFF && FORM != DIFF_SPLIT && FORM != DIFF_PF2 && FORM != DIFF_PLANAR) {
        ox[o] -= cb.x; oy[o] -= cb.y; oz[o] -= cb.z;
        aA[o] = __fma_rn(oz[o], oz[o], __fma_rn(oy[o], oy[o], __dmul_rn(ox[o], ox[o])));
        if (lane == 0) { sa[warp][o][0] = ox[o]; sa[warp][o][1] = oy[o]; sa[warp][o][2] = oz[o]; sa[warp][o][3] = aA[o]; }
      }
    }
    __syncwarp();
    if constexpr (FORM == DIFF) {
      const double4* ep = A.ep + b * NCH * NPE * 32 + lane;
      double2 cxy = __ldg(reinterpret_cast<const double2*>(ep)), czw = __ldg(reinterpret_cast<const double2*>(ep) + 1);
      for (int c = 0; c < NCH; ++c) {
        double2 acc[MO];
#pragma unroll
        for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < NPE; ++g) {
          const double2 pxy = cxy, pzw = czw;
          const double4* np = ep + (g + 1 < NPE ? (c * NPE + g + 1) * 32 : (c + 1 < NCH ? (c + 1) * NPE * 32 : 0));
          cxy = __ldg(reinterpret_cast<const double2*>(np));
          czw = __ldg(reinterpret_cast<const double2*>(np) + 1);
#pragma unroll
          for (int o = 0; o < MO; ++o) term_diff(ox[o], oy[o], oz[o], pxy, pzw, A.K1, tab, acc[o]);
        }
        double2 e = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          e.x = __fma_rn(sw[warp][o], acc[o].x, e.x);
          e.y = __fma_rn(sw[warp][o], acc[o].y, e.y);
        }
        myE[c * 32 + lane] = e;
      }
    } else if constexpr (FORM == DIFF_PLANAR) {
      const double2* ep = A.ep2 + b * NCH * NPE * 64 + lane;
      double2 cxy = __ldg(ep), czw = __ldg(ep + 32);
      for (int c = 0; c < NCH; ++c) {
        double2 acc[MO];
#pragma unroll
        for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < NPE; ++g) {
          const double2 pxy = cxy, pzw = czw;
          const double2* np = ep + (g + 1 < NPE ? (c * NPE + g + 1) * 64 : (c + 1 < NCH ? (c + 1) * NPE * 64 : 0));
          cxy = __ldg(np);
          czw = __ldg(np + 32);
#pragma unroll
          for (int o = 0; o < MO; ++o) term_diff(ox[o], oy[o], oz[o], pxy, pzw, A.K1, tab, acc[o]);
        }
        double2 e = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          e.x = __fma_rn(sw[warp][o], acc[o].x, e.x);
          e.y = __fma_rn(sw[warp][o], acc[o].y, e.y);
        }
        myE[c * 32 + lane] = e;
      }
    } else if constexpr (FORM == DIFF_PF2) {
      const double4* ep = A.ep + b * NCH * NPE * 32 + lane;
      constexpr int NP = NCH * NPE;
      double2 cxy = __ldg(reinterpret_cast<const double2*>(ep)), czw = __ldg(reinterpret_cast<const double2*>(ep) + 1);
      double2 dxy = __ldg(reinterpret_cast<const double2*>(ep + 32)), dzw = __ldg(reinterpret_cast<const double2*>(ep + 32) + 1);
      for (int c = 0; c < NCH; ++c) {
        double2 acc[MO];
#pragma unroll
        for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < NPE; ++g) {
          const double2 pxy = cxy, pzw = czw;
          cxy = dxy; czw = dzw;
          const int nx = c * NPE + g + 2;
          const double4* np = ep + (nx < NP ? nx : 0) * 32;
          dxy = __ldg(reinterpret_cast<const double2*>(np));
          dzw = __ldg(reinterpret_cast<const double2*>(np) + 1);
#pragma unroll
          for (int o = 0; o < MO; ++o) term_diff(ox[o], oy[o], oz[o], pxy, pzw, A.K1, tab, acc[o]);
        }
        double2 e = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          e.x = __fma_rn(sw[warp][o], acc[o].x, e.x);
          e.y = __fma_rn(sw[warp][o], acc[o].y, e.y);
        }
        myE[c * 32 + lane] = e;
      }
    } else if constexpr (FORM == EXP_REG || FORM == EXP_NOPF || FORM == EXP_SMEM) {
      const double2* fp = A.epf + b * NCH * NPE * 96 + lane;
      double2 c01, c23, csw;
      if constexpr (FORM == EXP_REG) { c01 = __ldg(fp); c23 = __ldg(fp + 32); csw = __ldg(fp + 64); }
      for (int c = 0; c < NCH; ++c) {
        double2 acc[MO];
#pragma unroll
        for (int o = 0; o < MO; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < NPE; ++g) {
          double2 q01, q23, sw_;
          if constexpr (FORM == EXP_REG) {
            q01 = c01; q23 = c23; sw_ = csw;
            const double2* np = fp + (g + 1 < NPE ? (c * NPE + g + 1) * 96 : (c + 1 < NCH ? (c + 1) * NPE * 96 : 0));
            c01 = __ldg(np); c23 = __ldg(np + 32); csw = __ldg(np + 64);
          } else {
            const double2* np = fp + (c * NPE + g) * 96;
            q01 = __ldg(np); q23 = __ldg(np + 32); sw_ = __ldg(np + 64);
          }
          const double wK = __dmul_rn(sw_.y, A.K1);
#pragma unroll
          for (int o = 0; o < MO; ++o) {
            if constexpr (FORM == EXP_SMEM) {
              const double* a = sa[warp][o];
              term_exp(lds_f64(a), lds_f64(a + 1), lds_f64(a + 2), lds_f64(a + 3), q01, q23, sw_.x, wK, tab, acc[o]);
            } else {
              term_exp(ox[o], oy[o], oz[o], aA[o], q01, q23, sw_.x, wK, tab, acc[o]);
            }
          }
        }
        double2 e = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < MO; ++o) {
          e.x = __fma_rn(sw[warp][o], acc[o].x, e.x);
          e.y = __fma_rn(sw[warp][o], acc[o].y, e.y);
        }
        myE[c * 32 + lane] = e;
      }
    } else {  // two lanes per edge: lane & 15 = edge of the half chunk, lane >> 4 = outer-point half
      constexpr int H = MO / 2;
      const int half = lane >> 4, el = lane & 15;
      double hx[H], hy[H], hz[H], hA[H], hw[H];
#pragma unroll
      for (int o = 0; o < H; ++o) {  // this lane's three outer points
        hx[o] = half ? ox[o + H] : ox[o];
        hy[o] = half ? oy[o + H] : oy[o];
        hz[o] = half ? oz[o + H] : oz[o];
        hA[o] = half ? aA[o + H] : aA[o];
        hw[o] = sw[warp][o + half * H];
      }
      for (int hc = 0; hc < 2 * NCH; ++hc) {
        const int c = hc >> 1, slot = ((hc & 1) << 4) + el;
        double2 acc[H];
#pragma unroll
        for (int o = 0; o < H; ++o) acc[o] = make_double2(0.0, 0.0);
#pragma unroll
        for (int g = 0; g < NPE; ++g) {
          if constexpr (FORM == EXP_SPLIT) {
            const double2* np = A.epf + b * NCH * NPE * 96 + (c * NPE + g) * 96 + slot;
            const double2 q01 = __ldg(np), q23 = __ldg(np + 32), sw_ = __ldg(np + 64);
            const double wK = __dmul_rn(sw_.y, A.K1);
#pragma unroll
            for (int o = 0; o < H; ++o) term_exp(hx[o], hy[o], hz[o], hA[o], q01, q23, sw_.x, wK, tab, acc[o]);
          } else {
            const double4* np = A.ep + b * NCH * NPE * 32 + (c * NPE + g) * 32 + slot;
            const double2 pxy = __ldg(reinterpret_cast<const double2*>(np)), pzw = __ldg(reinterpret_cast<const double2*>(np) + 1);
#pragma unroll
            for (int o = 0; o < H; ++o) term_diff(hx[o], hy[o], hz[o], pxy, pzw, A.K1, tab, acc[o]);
          }
        }
        double2 e = make_double2(0.0, 0.0);
#pragma unroll
        for (int o = 0; o < H; ++o) {
          e.x = __fma_rn(hw[o], acc[o].x, e.x);
          e.y = __fma_rn(hw[o], acc[o].y, e.y);
        }
        e.x += __shfl_xor_sync(0xffffffffu, e.x, 16);
        e.y += __shfl_xor_sync(0xffffffffu, e.y, 16);
        if (!half) myE[c * 32 + slot] = e;
      }
    }
    __syncwarp();
    double2* zr = A.z + (p * A.nblk + b) * kSlots;
    for (int j = lane; j < kSlots; j += 32) __stcs(zr + j, myE[j]);
    __syncwarp();
  }
}

template <int FORM>
void run(const char* name, Args A, int sm, std::vector<double2>* out) {
  auto k = kfar<FORM>;
  const size_t smem = (kPhaseSlots + W * kSlots) * sizeof(double2);
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  k<<<sm, 32 * W, smem>>>(A);
  float best = 1e9f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k<<<sm, 32 * W, smem>>>(A);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, k);
  const double evals = double(A.ntiles) * W * kSlots * NPE * MO;
  const size_t nz = (A.ntiles / A.nblk) * W * A.nblk * kSlots;
  std::vector<double2> h(nz);
  cudaMemcpy(h.data(), A.z, nz * 16, cudaMemcpyDeviceToHost);
  double dmax = 0.0, zmax = 0.0;
  if (out->empty()) *out = h;
  for (size_t i = 0; i < nz; ++i) {
    const double dx = h[i].x - (*out)[i].x, dy = h[i].y - (*out)[i].y;
    dmax = fmax(dmax, sqrt(dx * dx + dy * dy));
    zmax = fmax(zmax, sqrt((*out)[i].x * (*out)[i].x + (*out)[i].y * (*out)[i].y));
  }
  std::printf("%-44s %7.3f ms  %.3e evals/s  regs %3d  local %zu  max|dE|/max|E| %.1e  %s\n", name, best,
              evals / (best * 1e-3), at.numRegs, (size_t)at.localSizeBytes, dmax / zmax,
              cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sm;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  const size_t nblk = 381, rowgroups = 24;  // 24 x 381 tiles of 12 rows x 352 slots
  const size_t rows = rowgroups * W, ntiles = rowgroups * nblk;
  srand(1901);
  auto rnd = [] { return rand() / (double)RAND_MAX; };
  // blocks: centres on the unit sphere, points within 0.15 of the centre,
  // weights ~ edge length x Gauss weight; rows: outer points on a sphere of
  // radius 3 around the origin (every tile is far: |a| >= 2 >> 3 x 0.15)
  std::vector<double4> hc(nblk), hep(nblk * NCH * NPE * 32), ho(rows * MO);
  std::vector<double2> hepf(nblk * NCH * NPE * 96), hep2(nblk * NCH * NPE * 64);
  for (size_t b = 0; b < nblk; ++b) {
    double x = rnd() - 0.5, y = rnd() - 0.5, z = rnd() - 0.5;
    const double n = sqrt(x * x + y * y + z * z);
    hc[b] = make_double4(x / n, y / n, z / n, 0.15);
    for (int i = 0; i < NCH * NPE * 32; ++i) {
      const double px = hc[b].x + 0.17 * (rnd() - 0.5), py = hc[b].y + 0.17 * (rnd() - 0.5),
                   pz = hc[b].z + 0.17 * (rnd() - 0.5), w = 2e-3 + 3e-3 * rnd();
      hep[b * NCH * NPE * 32 + i] = make_double4(px, py, pz, w);
      hep2[b * NCH * NPE * 64 + static_cast<size_t>(i / 32) * 64 + (i & 31)] = make_double2(px, py);
      hep2[b * NCH * NPE * 64 + static_cast<size_t>(i / 32) * 64 + 32 + (i & 31)] = make_double2(pz, w);
      const double s = 1.0 / (w * w), dx = px - hc[b].x, dy = py - hc[b].y, dz = pz - hc[b].z;
      const size_t at = b * NCH * NPE * 96 + static_cast<size_t>(i / 32) * 96 + (i & 31);
      hepf[at] = make_double2(-2.0 * dx * s, -2.0 * dy * s);
      hepf[at + 32] = make_double2(-2.0 * dz * s, (dx * dx + dy * dy + dz * dz) * s);
      hepf[at + 64] = make_double2(s, w);
    }
  }
  for (auto& v : ho) {
    double x = rnd() - 0.5, y = rnd() - 0.5, z = rnd() - 0.5;
    const double n = sqrt(x * x + y * y + z * z) / 3.0;
    v = make_double4(x / n, y / n, z / n, 1e-4 * (1.0 + rnd()));
  }
  Args A{};
  double4 *o, *ep, *ce;
  double2 *epf, *ep2, *ph, *z;
  cudaMalloc(&o, ho.size() * 32);
  cudaMalloc(&ep, hep.size() * 32);
  cudaMalloc(&epf, hepf.size() * 16);
  cudaMalloc(&ep2, hep2.size() * 16);
  cudaMemcpy(ep2, hep2.data(), hep2.size() * 16, cudaMemcpyHostToDevice);
  cudaMalloc(&ce, hc.size() * 32);
  cudaMalloc(&ph, kPhaseSlots * 16);
  cudaMalloc(&z, rows * nblk * kSlots * 16);
  cudaMemcpy(o, ho.data(), ho.size() * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(ep, hep.data(), hep.size() * 32, cudaMemcpyHostToDevice);
  cudaMemcpy(epf, hepf.data(), hepf.size() * 16, cudaMemcpyHostToDevice);
  cudaMemcpy(ce, hc.data(), hc.size() * 32, cudaMemcpyHostToDevice);
  std::vector<double2> hp(kPhaseSlots);  // slot i holds angle index i >> kPhaseCopyLog2
  for (int i = 0; i < kPhaseSlots; ++i) {
    const int n = i >> kPhaseCopyLog2;
    hp[i] = make_double2(cos(2 * kPi * n / kPhaseM), sin(2 * kPi * n / kPhaseM));
  }
  cudaMemcpy(ph, hp.data(), kPhaseSlots * 16, cudaMemcpyHostToDevice);
  std::printf("phase table: %d angles x %d copies\n", kPhaseM, 1 << kPhaseCopyLog2);
  A.outer = o; A.ep = ep; A.epf = epf; A.ep2 = ep2; A.centre = ce; A.phase = ph; A.z = z;
  A.nblk = nblk; A.ntiles = ntiles;
  A.K1 = 2 * kPi / 0.15 * kPhaseM / (2 * kPi);
  std::vector<double2> ref;
  run<DIFF>("difference form (product)", A, sm, &ref);
  run<EXP_REG>("expanded, a[] in registers, prefetch", A, sm, &ref);
  run<EXP_NOPF>("expanded, a[] in registers, no prefetch", A, sm, &ref);
  run<EXP_SMEM>("expanded, a[] from shared memory", A, sm, &ref);
  run<EXP_SPLIT>("expanded, two lanes per edge", A, sm, &ref);
  run<DIFF_SPLIT>("difference form, two lanes per edge", A, sm, &ref);
  run<DIFF_PF2>("difference form, two points ahead", A, sm, &ref);
  run<DIFF_PLANAR>("difference form, planar points", A, sm, &ref);
  return 0;
}
