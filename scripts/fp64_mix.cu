// FP64 issue-ceiling microbenchmarks on B200 (standalone; not part of libgk).
//   A: DFMA chains with constant operands (gk_bench_fp64_peak style)
//   B: DFMA chains with 3 distinct register operands
//   C: the fill's mix per "eval": 16 DFMA + 8 DMUL + 3 DADD, register operands
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_mix fp64_mix.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int K = 8;

__global__ void __launch_bounds__(256) kA(double* sink, int iters, double b, double c) {
  double a[K];
  for (int k = 0; k < K; ++k) a[k] = 1.0 + 1e-9 * (threadIdx.x + k);
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = __fma_rn(a[k], b, c);
  double s = 0;
  for (int k = 0; k < K; ++k) s += a[k];
  if (s == 1234.5) sink[0] = s;
}

__global__ void __launch_bounds__(256) kB(double* sink, int iters, const double* in) {
  double a[K], b[K], c[K];
  for (int k = 0; k < K; ++k) {
    a[k] = in[threadIdx.x % 32 + k];
    b[k] = in[threadIdx.x % 32 + k + 8] * 1e-9 + 0.9999999;
    c[k] = in[threadIdx.x % 32 + k + 16] * 1e-12;
  }
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int u = 0; u < 16; ++u)
#pragma unroll
      for (int k = 0; k < K; ++k) a[k] = __fma_rn(a[k], b[(k + u) % K], c[(k + 3 * u) % K]);
  double s = 0;
  for (int k = 0; k < K; ++k) s += a[k];
  if (s == 1234.5) sink[0] = s;
}

// 27 FP64 ops shaped like one direct eval, 6 independent "evals" per iteration
__global__ void __launch_bounds__(256, 2) kC(double* sink, int iters, const double* in) {
  double x[6], acc[6];
  for (int k = 0; k < 6; ++k) { x[k] = in[threadIdx.x % 32 + k] * 1e-3 + 0.5; acc[k] = 0; }
  double px = in[1], py = in[2], pz = in[3], w = in[4];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double dx = x[o] - px, dy = x[(o + 1) % 6] - py, dz = x[(o + 2) % 6] - pz;   // 3 DADD
      double d2 = __fma_rn(dz, dz, __fma_rn(dy, dy, __dmul_rn(dx, dx)));          // 3
      double y = d2 * 0.7;                                                         // 1
      double e = __fma_rn(-d2, __dmul_rn(y, y), 1.0);                              // 2
      double ye = __dmul_rn(y, e);                                                 // 1
      y = __fma_rn(ye, __fma_rn(0.375, e, 0.5), y);                                // 2
      double r = __dmul_rn(d2, y);                                                 // 1
      double t = __fma_rn(r, 13.7, 6755399441055744.0);                            // 1
      double nf = t - 6755399441055744.0;                                          // 1
      double f = __fma_rn(r, 13.7, -nf);                                           // 1
      double g = __dmul_rn(f, f);                                                  // 1
      double v = __dmul_rn(g, __fma_rn(1e-9, g, -1e-6));                           // 2
      double s = __dmul_rn(f, __fma_rn(-1e-10, g, 1.5e-3));                        // 2
      double c = __fma_rn(-y, s, __fma_rn(x[o], v, x[o]));                         // 2
      double sn = __fma_rn(x[o], s, __fma_rn(y, v, y));                            // 2
      double wg = __dmul_rn(w, y);                                                 // 1
      acc[o] = __fma_rn(wg, c, acc[o]);                                            // 1
      acc[(o + 3) % 6] = __fma_rn(-wg, sn, acc[(o + 3) % 6]);                      // 1
    }
    px += 1e-12; py -= 1e-12;
  }
  double s = 0;
  for (int k = 0; k < 6; ++k) s += acc[k];
  if (s == 1234.5) sink[0] = s;
}

// 22 FP64 ops shaped like one term of the expanded far path (far_term): the
// squared distance as a chain of four 3-register FMAs, the folded weight, the
// tan-form rotation; 6 independent "evals" per iteration
template <int TPB, int MINB>
__global__ void __launch_bounds__(TPB, MINB) kD(double* sink, int iters, const double* in) {
  double ax[6], ay[6], az[6], aA[6], ex[6], ey[6];
  for (int k = 0; k < 6; ++k) {
    ax[k] = in[threadIdx.x % 32 + k] * 1e-3 + 0.5;
    ay[k] = in[threadIdx.x % 32 + k + 6] * 1e-3 + 0.4;
    az[k] = in[threadIdx.x % 32 + k + 12] * 1e-3 + 0.3;
    aA[k] = ax[k] * ax[k] + ay[k] * ay[k] + az[k] * az[k];
    ex[k] = ey[k] = 0;
  }
  double qx = in[1], qy = in[2], qz = in[3], B = in[4], s = in[5], wK = in[6], tx = in[7], ty = in[8];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double d2 = __fma_rn(ax[o], qx, __fma_rn(ay[o], qy, __fma_rn(az[o], qz, __fma_rn(aA[o], s, B))));  // 4
      double y = d2 * 0.7;                                                         // 1 (stands for MUFU)
      double e = __fma_rn(-d2, __dmul_rn(y, y), 1.0);                              // 2
      double ye = __dmul_rn(y, e);                                                 // 1
      y = __fma_rn(ye, __fma_rn(0.375, e, 0.5), y);                                // 2
      double r = __dmul_rn(d2, y);                                                 // 1
      double t = __fma_rn(r, wK, 6755399441055744.0);                              // 1
      double nf = t - 6755399441055744.0;                                          // 1
      double f = __fma_rn(r, wK, -nf);                                             // 1
      double g = __dmul_rn(f, f);                                                  // 1
      double tau = __dmul_rn(f, __fma_rn(1e-10, g, 1.5e-3));                       // 2
      double v = __dmul_rn(g, -1e-6);                                              // 1
      double wk = __fma_rn(y, v, y);                                               // 1
      double c = __fma_rn(-tau, ty, tx);                                           // 1
      double sn = __fma_rn(tau, tx, ty);                                           // 1
      ex[o] = __fma_rn(wk, c, ex[o]);                                              // 1
      ey[o] = __fma_rn(-wk, sn, ey[o]);                                            // 1
    }
    qx += 1e-12; qy -= 1e-12; tx += 1e-13; ty -= 1e-13;
  }
  double r = 0;
  for (int k = 0; k < 6; ++k) r += ex[k] + ey[k];
  if (r == 1234.5) sink[0] = r;
}

// kC's mix (the difference form) in the same shape as kD: per-o coordinates
// and two accumulators per o
template <int TPB, bool TAN, int MINB>
__global__ void __launch_bounds__(TPB, MINB) kE(double* sink, int iters, const double* in) {
  double ox[6], oy[6], oz[6], ex[6], ey[6];
  for (int k = 0; k < 6; ++k) {
    ox[k] = in[threadIdx.x % 32 + k] * 1e-3 + 0.5;
    oy[k] = in[threadIdx.x % 32 + k + 6] * 1e-3 + 0.4;
    oz[k] = in[threadIdx.x % 32 + k + 12] * 1e-3 + 0.3;
    ex[k] = ey[k] = 0;
  }
  double px = in[1], py = in[2], pz = in[3], w = in[4], K1 = in[6], tx = in[7], ty = in[8];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      double dx = ox[o] - px, dy = oy[o] - py, dz = oz[o] - pz;                    // 3
      double d2 = __fma_rn(dz, dz, __fma_rn(dy, dy, __dmul_rn(dx, dx)));          // 3
      double y = d2 * 0.7;
      double e = __fma_rn(-d2, __dmul_rn(y, y), 1.0);
      double ye = __dmul_rn(y, e);
      y = __fma_rn(ye, __fma_rn(0.375, e, 0.5), y);
      double r = __dmul_rn(d2, y);
      double t = __fma_rn(r, K1, 6755399441055744.0);
      double nf = t - 6755399441055744.0;
      double f = __fma_rn(r, K1, -nf);
      double g = __dmul_rn(f, f);
      if (TAN) {
        double tau = __dmul_rn(f, __fma_rn(1e-10, g, 1.5e-3));
        double v = __dmul_rn(g, -1e-6);
        double b = __dmul_rn(w, y);
        double wk = __fma_rn(b, v, b);
        double c = __fma_rn(-tau, ty, tx);
        double sn = __fma_rn(tau, tx, ty);
        ex[o] = __fma_rn(wk, c, ex[o]);
        ey[o] = __fma_rn(-wk, sn, ey[o]);
      } else {
        double v = __dmul_rn(g, -1e-6);
        double sd = __dmul_rn(f, __fma_rn(-1e-10, g, 1.5e-3));
        double c = __fma_rn(-ty, sd, __fma_rn(tx, v, tx));
        double sn = __fma_rn(tx, sd, __fma_rn(ty, v, ty));
        double wg = __dmul_rn(w, y);
        ex[o] = __fma_rn(wg, c, ex[o]);
        ey[o] = __fma_rn(-wg, sn, ey[o]);
      }
    }
    px += 1e-12; py -= 1e-12; tx += 1e-13; ty -= 1e-13;
  }
  double r = 0;
  for (int k = 0; k < 6; ++k) r += ex[k] + ey[k];
  if (r == 1234.5) sink[0] = r;
}

// kE's difference-form term with features of kC switched in one at a time
// (F bit 0: K1 immediate; 1: the three coordinates taken from one array of 6;
// 2: 6 accumulators instead of 12; 3: the table entry = (x[o], y) instead of
// two loop-invariant registers): which of them costs kE its 15 % against kC
template <int F>
__global__ void __launch_bounds__(384, 1) kF(double* sink, int iters, const double* in) {
  double ox[6], oy[6], oz[6], ex[6], ey[6];
  for (int k = 0; k < 6; ++k) {
    ox[k] = in[threadIdx.x % 32 + k] * 1e-3 + 0.5;
    oy[k] = in[threadIdx.x % 32 + k + 6] * 1e-3 + 0.4;
    oz[k] = in[threadIdx.x % 32 + k + 12] * 1e-3 + 0.3;
    ex[k] = ey[k] = 0;
  }
  double px = in[1], py = in[2], pz = in[3], w = in[4], K1r = in[6], tx = in[7], ty = in[8];
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int o = 0; o < 6; ++o) {
      const double cx = ox[o], cy = (F & 2) ? ox[(o + 1) % 6] : oy[o], cz = (F & 2) ? ox[(o + 2) % 6] : oz[o];
      double dx = cx - px, dy = cy - py, dz = cz - pz;
      double d2 = __fma_rn(dz, dz, __fma_rn(dy, dy, __dmul_rn(dx, dx)));
      double y = d2 * 0.7;
      double e = __fma_rn(-d2, __dmul_rn(y, y), 1.0);
      double ye = __dmul_rn(y, e);
      y = __fma_rn(ye, __fma_rn(0.375, e, 0.5), y);
      double r = __dmul_rn(d2, y);
      const double K1 = (F & 1) ? 13.7 : K1r;
      double t = __fma_rn(r, K1, 6755399441055744.0);
      double nf = t - 6755399441055744.0;
      double f = __fma_rn(r, K1, -nf);
      double g = __dmul_rn(f, f);
      double v = __dmul_rn(g, -1e-6);
      double sd = __dmul_rn(f, __fma_rn(-1e-10, g, 1.5e-3));
      const double Tx = (F & 8) ? cx : tx, Ty = (F & 8) ? y : ty;
      double c = __fma_rn(-Ty, sd, __fma_rn(Tx, v, Tx));
      double sn = __fma_rn(Tx, sd, __fma_rn(Ty, v, Ty));
      double wg = __dmul_rn(w, y);
      if (F & 4) {
        ex[o] = __fma_rn(wg, c, ex[o]);
        ex[(o + 3) % 6] = __fma_rn(-wg, sn, ex[(o + 3) % 6]);
      } else {
        ex[o] = __fma_rn(wg, c, ex[o]);
        ey[o] = __fma_rn(-wg, sn, ey[o]);
      }
    }
    px += 1e-12; py -= 1e-12; tx += 1e-13; ty -= 1e-13;
  }
  double r = 0;
  for (int k = 0; k < 6; ++k) r += ex[k] + ey[k];
  if (r == 1234.5) sink[0] = r;
}

int main() {
  double *sink, *in;
  cudaMalloc(&sink, 8);
  cudaMalloc(&in, 64 * 8);
  double h[64];
  for (int i = 0; i < 64; ++i) h[i] = 0.1 + 0.01 * i;
  cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int tpb = 256;
  auto run = [&](const char* name, auto launch, double ops_per_thread_iter, int blocks_per_sm, int iters) {
    launch(sm * blocks_per_sm, iters / 4);
    cudaEventRecord(e0);
    launch(sm * blocks_per_sm, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double lane_ops = double(sm) * blocks_per_sm * tpb * double(iters) * ops_per_thread_iter;
    std::printf("%s: %.2f ms, %.1f FP64 lane-ops/clk/SM @ 1.965 GHz (%.1f%% of 64)\n", name, ms,
                lane_ops / (ms * 1e-3) / sm / 1.965e9, 100.0 * lane_ops / (ms * 1e-3) / sm / 1.965e9 / 64);
  };
  for (int bps : {2, 4, 8}) {
    char nm[64];
    std::snprintf(nm, 64, "A const-operand DFMA  (%d CTA/SM)", bps);
    run(nm, [&](int g, int it) { kA<<<g, 256>>>(sink, it, 0.9999999, 1e-7); }, 16.0 * K, bps, 2048);
    std::snprintf(nm, 64, "B 3-register DFMA     (%d CTA/SM)", bps);
    run(nm, [&](int g, int it) { kB<<<g, 256>>>(sink, it, in); }, 16.0 * K, bps, 2048);
  }
  run("C fill-shaped mix 27 ops (2 CTA/SM)", [&](int g, int it) { kC<<<g, 256>>>(sink, it, in); }, 6 * 27.0 + 2, 2, 8192);
  // evaluations per second per SM matter, not lane-ops: the line also gives
  // cycles per warp-eval per SMSP = 4 * 32 * ops / (lane-ops/clk/SM)
  tpb = 384;
  run("E difference form 26 ops, 12 warps, <= 80 regs ", [&](int g, int it) { kE<384, false, 2><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("E' difference + tan 25 ops, 12 warps, <= 80   ", [&](int g, int it) { kE<384, true, 2><<<g, 384>>>(sink, it, in); }, 6 * 25.0, 1, 8192);
  run("D expanded 22 ops, 12 warps, <= 80 regs       ", [&](int g, int it) { kD<384, 2><<<g, 384>>>(sink, it, in); }, 6 * 22.0, 1, 8192);
  run("E  difference 26 ops, 12 warps, <= 168 regs  ", [&](int g, int it) { kE<384, false, 1><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("E' difference + tan 25 ops, <= 168 regs      ", [&](int g, int it) { kE<384, true, 1><<<g, 384>>>(sink, it, in); }, 6 * 25.0, 1, 8192);
  run("D  expanded 22 ops, <= 168 regs              ", [&](int g, int it) { kD<384, 1><<<g, 384>>>(sink, it, in); }, 6 * 22.0, 1, 8192);
  run("F0 = E                                       ", [&](int g, int it) { kF<0><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("F1 K1 immediate                              ", [&](int g, int it) { kF<1><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("F2 shared coordinates                        ", [&](int g, int it) { kF<2><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("F4 6 accumulators                            ", [&](int g, int it) { kF<4><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("F8 table entry from live registers           ", [&](int g, int it) { kF<8><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  run("F15 all (= C's shape)                        ", [&](int g, int it) { kF<15><<<g, 384>>>(sink, it, in); }, 6 * 26.0, 1, 8192);
  tpb = 256;
  run("E difference form 26 ops, 24 warps (3 CTA/SM)", [&](int g, int it) { kE<256, false, 3><<<g, 256>>>(sink, it, in); }, 6 * 26.0, 3, 8192);
  run("E' difference + tan 25 ops, 24 warps        ", [&](int g, int it) { kE<256, true, 3><<<g, 256>>>(sink, it, in); }, 6 * 25.0, 3, 8192);
  run("D expanded 22 ops, 24 warps (3 CTA/SM)       ", [&](int g, int it) { kD<256, 3><<<g, 256>>>(sink, it, in); }, 6 * 22.0, 3, 8192);
  cudaDeviceSynchronize();
  std::printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
