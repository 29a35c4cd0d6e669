// Prototype: D[128 x N] = A[128 x K] * B[N x K]^T, bf16 in, fp32 accumulate in
// TMEM, one CTA, operands K-major in shared memory (SWIZZLE_NONE canonical
// layout: 8-row x 16-byte core matrices, LBO = next core matrix along K,
// SBO = next along M/N), tcgen05.mma issued by one thread.
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdint>
#include <cmath>
#include <vector>

constexpr int M = 128, N = 128, K = 64;
constexpr int KC = K / 8;  // core matrices along K

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((addr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version (sm100)
  // base offset 0, lbo mode 0, layout type 0 (SWIZZLE_NONE)
  return d;
}
// bf16 x bf16 -> f32, K-major A and B
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
  return (1u << 4)            // c_format F32
       | (1u << 7)            // a_format BF16
       | (1u << 10)           // b_format BF16
       | ((uint32_t)(n >> 3) << 17)
       | ((uint32_t)(m >> 4) << 24);
}

template <int REPS>
__global__ void k_test(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D) {
  __shared__ __align__(128) __nv_bfloat16 sa[M * K];
  __shared__ __align__(128) __nv_bfloat16 sb[N * K];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  // canonical layout: element (r, k) at core (r/8, k/8) -> byte ((r/8)*KC + k/8)*128 + (r%8)*16 + (k%8)*2
  for (int e = t; e < M * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    sa[(((r >> 3) * KC + (k >> 3)) * 64) + (r & 7) * 8 + (k & 7)] = A[e];
  }
  for (int e = t; e < N * K; e += blockDim.x) {
    const int r = e / K, k = e % K;
    sb[(((r >> 3) * KC + (k >> 3)) * 64) + (r & 7) * 8 + (k & 7)] = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  long long t0 = clock64();
  if (t == 0) {
    const uint32_t lbo = 128, sbo = KC * 128;
    for (int rep = 0; rep < REPS; ++rep)
    for (int s = 0; s < K / 16; ++s) {
      const uint64_t da = sdesc(smem_u32(sa) + s * 256, lbo, sbo);
      const uint64_t db = sdesc(smem_u32(sb) + s * 256, lbo, sbo);
      const uint32_t acc = (s > 0) || (rep > 0 && false);
      asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                   "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n"
                   ::"r"(tmem), "l"(da), "l"(db), "r"(idesc_bf16(M, N)), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n"
                 ::"r"(smem_u32(&mbar)) : "memory");
  }
  // wait for the MMAs (phase 0)
  {
    uint32_t done = 0;
    while (!done) {
      asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                   : "=r"(done) : "r"(smem_u32(&mbar)), "r"(0));
    }
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  if (t == 0) printf("REPS %d x %d MMAs (M=%d N=%d K=16): %lld cycles, %.1f cycles/MMA\n", REPS, K / 16, M, N, clock64() - t0, (double)(clock64() - t0) / (REPS * (K / 16)));
  for (int c0 = 0; c0 < N; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(w * 32) << 16) + c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                   "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
                   "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
                   "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int row = w * 32 + lane;
    for (int j = 0; j < 32; ++j) D[row * N + c0 + j] = __uint_as_float(v[j]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(N));
}

int main() {
  std::vector<__nv_bfloat16> A(M * K), B(N * K);
  std::vector<float> fa(M * K), fb(N * K), D(M * N);
  unsigned s = 1;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 9) & 0xffff) / 32768.0f - 1.0f; };
  for (int i = 0; i < M * K; ++i) { A[i] = __float2bfloat16(rnd()); fa[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < N * K; ++i) { B[i] = __float2bfloat16(rnd()); fb[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB; float* dD;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  k_test<1><<<1, 128>>>(dA, dB, dD);
  cudaDeviceSynchronize();
  k_test<100><<<1, 128>>>(dA, dB, dD);
  cudaDeviceSynchronize();
  k_test<1><<<1, 128>>>(dA, dB, dD);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  double maxerr = 0; int bad = 0;
  for (int i = 0; i < M; ++i) for (int j = 0; j < N; ++j) {
    double ref = 0; for (int k = 0; k < K; ++k) ref += (double)fa[i * K + k] * fb[j * K + k];
    double err = fabs(ref - D[i * N + j]); maxerr = fmax(maxerr, err); bad += err > 1e-3;
  }
  printf("max err %.3e, bad %d of %d; D[0]=%f D[1]=%f\n", maxerr, bad, M * N, D[0], D[1]);
}
