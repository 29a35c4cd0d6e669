#include <cstdio>
__global__ void k(double* out, double a, double b, int which, long long* cyc) {
  double x = a;
  long long t0 = clock64();
  if (which == 0) for (int i = 0; i < 1024; ++i) x = __dadd_rn(x, b);
  if (which == 1) for (int i = 0; i < 1024; ++i) x = __ddiv_rn(x, b);
  if (which == 2) for (int i = 0; i < 1024; ++i) x = __dsqrt_rn(x + b);
  if (which == 3) for (int i = 0; i < 1024; ++i) x = __dmul_rn(x, b);
  if (which == 4) for (int i = 0; i < 1024; ++i) x = __fma_rn(x, b, a);
  if (which == 5) { float y = (float)a; for (int i = 0; i < 1024; ++i) y = __fadd_rn(y, (float)b); x = y; }
  long long t1 = clock64();
  out[0] = x; cyc[which] = t1 - t0;
}
int main() {
  double* o; long long* c; cudaMalloc(&o, 8); cudaMalloc(&c, 64);
  const char* nm[] = {"DADD", "DDIV", "DSQRT(+DADD)", "DMUL", "DFMA", "FADD"};
  for (int w = 0; w < 6; ++w) {
    k<<<1,1>>>(o, 1.5, 1.0000001, w, c); cudaDeviceSynchronize();
    k<<<1,1>>>(o, 1.5, 1.0000001, w, c); cudaDeviceSynchronize();
    long long h[8]; cudaMemcpy(h, c, 64, cudaMemcpyDeviceToHost);
    printf("%s latency %.1f cycles\n", nm[w], h[w] / 1024.0);
  }
}
