#include <cstdio>
__global__ void k(double* out, double a, int n) {
  double acc = a, b = a * 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) { acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b); acc = __dadd_rn(acc, b); }
  long long t1 = clock64();
  out[0] = acc; out[1] = (double)(t1 - t0) / (4.0 * n);
}
int main() { double* d; cudaMalloc(&d, 16); k<<<1,1>>>(d, 1.0, 100000); double h[2]; cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost); printf("dadd latency %.2f cycles\n", h[1]); }
