// Accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of one
// quadratic / one cubic Newton step, vs a correctly-rounded reference.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>
__global__ void k(const double* x, double* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d2 = x[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d2));
  double e = fma(-d2, y * y, 1.0);
  double q = fma(y * e, 0.5, y);                       // quadratic
  double c = fma(y * e, fma(0.375, e, 0.5), y);        // cubic
  double ref = 1.0 / sqrt(d2);                         // correctly rounded sqrt + div
  out[4 * i] = y; out[4 * i + 1] = q; out[4 * i + 2] = c; out[4 * i + 3] = ref;
}
int main() {
  const int n = 1 << 22;
  double *x, *o;
  cudaMallocManaged(&x, n * 8);
  cudaMallocManaged(&o, 4 * n * 8);
  unsigned long long s = 1901;
  for (int i = 0; i < n; ++i) {
    s = s * 6364136223846793005ULL + 1442695040888963407ULL;
    double u = (s >> 11) * 0x1.0p-53;
    x[i] = pow(10.0, -7.0 + 7.7 * u);  // r^2 in [1e-7, 5]
  }
  k<<<(n + 255) / 256, 256>>>(x, o, n);
  cudaDeviceSynchronize();
  double w[3] = {0, 0, 0};
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < 3; ++j) {
      double rel = fabs(o[4 * i + j] - o[4 * i + 3]) / o[4 * i + 3];
      if (rel > w[j]) w[j] = rel;
    }
  printf("max rel err: seed %.3e (2^%.1f)  quadratic %.3e (%.2f ulp)  cubic %.3e (%.2f ulp)\n", w[0],
         log2(w[0]), w[1], w[1] / 0x1.0p-53, w[2], w[2] / 0x1.0p-53);
  return 0;
}
