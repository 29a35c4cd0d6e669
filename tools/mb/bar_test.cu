// Microbenchmark: cycles per __syncthreads for a few CTA shapes, empty and
// after a short divergent FP64 phase (the LLT panel's column loop pattern).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_bar(int iters, int work, long long* out, double* sink) {
  __shared__ double sm[1024];
  const int t = threadIdx.x;
  sm[t] = t;
  __syncthreads();
  double acc = 0.0;
  const long long t0 = clock64();
  for (int i = 0; i < iters; ++i) {
    if (work && (t >> 1) > (i & 63)) {  // divergent, like the panel rows r > c
      for (int w = 0; w < work; ++w) acc = __dadd_rn(acc, __dmul_rn(sm[(t + w) & 1023], 1.0000001));
      sm[t] = acc;
    }
    __syncthreads();
  }
  const long long t1 = clock64();
  if (t == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 12345.0) sink[0] = acc;
}
int main() {
  long long* d; double* sink;
  cudaMalloc(&d, 1024 * sizeof(long long));
  cudaMalloc(&sink, 8);
  const int threads[] = {32, 64, 160, 256, 512};
  for (int th : threads)
    for (int work : {0, 1, 8}) {
      for (int rep = 0; rep < 2; ++rep) k_bar<<<1, th>>>(4096, work, d, sink);
      long long h;
      cudaMemcpy(&h, d, sizeof(h), cudaMemcpyDeviceToHost);
      printf("threads %4d work %d: %.1f cycles per iteration\n", th, work, h / 4096.0);
    }
  return 0;
}
