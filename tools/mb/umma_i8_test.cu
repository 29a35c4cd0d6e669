// Prototype for the tensor-core ADC filter: D[128 x N] (s32, TMEM) =
// A[128 x K] (u8, TMEM: row i in lane i, four K-bytes per 32-bit column) *
// B[N x K]^T (u8, shared memory, K-major SWIZZLE_NONE canonical layout:
// 8-row x 16-byte core matrices, LBO = next core matrix along K, SBO = next
// along N), tcgen05.mma.kind::i8 issued by one thread. Checks exactness
// against a host integer GEMM, then times a long chain of MMAs
// (K = KLONG, as the ADC filter's 13-bit split: 2 x 16 x M bytes).
#include <cstdint>
#include <cstdio>
#include <vector>

constexpr int M = 128, K = 128, KLONG = 1536;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | ((uint64_t)1 << 46);
}
// u8 x u8 -> s32, K-major A and B
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4)  // D s32
         | (0u << 7)  // A u8
         | (0u << 10)  // B u8
         | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity), "n"(1000000)
        : "memory");
}

template <int N, int KK, bool A_TMEM>
__global__ void k_test(const uint8_t* A, const uint8_t* B, int* D, int reps, long long* cyc, int commit_every, uint64_t* cbar) {
  extern __shared__ __align__(1024) uint8_t sm[];
  uint8_t* sb = sm;                   // N x KK canonical
  uint8_t* sa = sm + N * KK;          // M x KK canonical (A_TMEM = false)
  __shared__ __align__(8) uint64_t mbar;
  __shared__ __align__(8) uint64_t cbars[4];
  cbar = cbars;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, w = t >> 5, lane = t & 31;
  constexpr int KC = KK / 16;  // core matrices along K
  for (int e = t; e < N * KK; e += blockDim.x) {
    const int r = e / KK, k = e % KK;
    sb[((r >> 3) * KC + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15)] = B[e];
  }
  if (!A_TMEM)
    for (int e = t; e < M * KK; e += blockDim.x) {
      const int r = e / KK, k = e % KK;
      sa[((r >> 3) * KC + (k >> 4)) * 128 + (r & 7) * 16 + (k & 15)] = A[e];
    }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (t == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&cbars[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(&tbase)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = tbase;
  const uint32_t tA = tmem, tD = tmem + 512 - N;  // A: KK / 4 columns
  if (A_TMEM) {
    // lane row = 32 w + lane: its KK bytes -> columns 0 .. KK / 4
    const int row = w * 32 + lane;
    for (int c0 = 0; c0 < KK / 4; c0 += 8) {
      uint32_t v[8];
      for (int j = 0; j < 8; ++j) {
        const uint8_t* p = A + (size_t)row * KK + (c0 + j) * 4;
        v[j] = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
      }
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(
              tA + ((uint32_t)(w * 32) << 16) + c0),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  long long t0 = clock64();
  if (t == 0) {
    const uint32_t lbo = 128, sbo = KC * 128;
    for (int r = 0; r < reps; ++r)
      for (int s = 0; s < KK / 32; ++s) {
        const uint64_t db = sdesc(smem_u32(sb) + s * 256, lbo, sbo);
        const uint32_t acc = (r | s) > 0;
        if (commit_every > 0 && s % commit_every == 0 && (r | s))
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"((uint64_t)(cbar + (s / commit_every) % 4)) : "memory");
        const uint32_t tDr = commit_every < 0 ? tD - (uint32_t)((r & 1) * N) : tD;
        const uint32_t accr = commit_every < 0 ? (s > 0) : acc;
        if (commit_every < 0 && s == 0 && r > 0)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.b64 [%0];\n" ::"l"((uint64_t)(cbar + (r & 3))) : "memory");
        if (A_TMEM)
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tDr),
              "r"(tA + (uint32_t)(s * 8)), "l"(db), "r"(idesc_i8(M, N)), "r"(accr));
        else {
          const uint64_t da = sdesc(smem_u32(sa) + s * 256, lbo, sbo);
          asm volatile(
              "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tD),
              "l"(da), "l"(db), "r"(idesc_i8(M, N)), "r"(acc));
        }
      }
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
            smem_u32(&mbar))
        : "memory");
  }
  __syncwarp();
  mbar_wait(smem_u32(&mbar), 0);
  long long t1 = clock64();
  if (t == 0) *cyc = t1 - t0;
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  for (int c0 = 0; c0 < N; c0 += 16) {
    uint32_t v[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(tD + ((uint32_t)(w * 32) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    const int row = w * 32 + lane;
    for (int j = 0; j < 16; ++j) D[row * N + c0 + j] = (int)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512));
}

template <int N, int KK, bool AT>
int run(int reps, int ce = 0) {
  std::vector<uint8_t> A(M * KK), B(N * KK);
  std::vector<int> D(M * N);
  unsigned s = 7;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return s >> 8; };
  for (auto& v : A) v = rnd() % 128;
  for (auto& v : B) { const unsigned r = rnd() % 20; v = r == 0 ? 64 : r == 1 ? 1 : 0; }
  uint8_t *dA, *dB; int* dD; long long* dc;
  cudaMalloc(&dA, A.size()); cudaMalloc(&dB, B.size()); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = N * KK + (AT ? 0 : M * KK);
  cudaFuncSetAttribute(k_test<N, KK, AT>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_test<N, KK, AT><<<1, 128, smem>>>(dA, dB, dD, reps, dc, ce, nullptr);
  cudaError_t e = cudaDeviceSynchronize();
  long long cyc = 0;
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long ref = 0;
      for (int k = 0; k < KK; ++k) ref += (long)A[i * KK + k] * B[j * KK + k];
      ref *= reps;
      bad += ref != D[i * N + j];
    }
  const double macs = (double)M * N * KK * reps;
  printf("N=%d ce=%d K=%d A_%s reps=%d: %s, mismatches %ld of %d, %lld cycles, %.0f MAC/clk (D[0]=%d)\n", N, ce, KK,
         AT ? "tmem" : "smem", reps, cudaGetErrorString(e), bad, M * N, cyc, macs / cyc, D[0]);
  return bad != 0;
}

int main() {
  int bad = 0;
  bad += run<64, KLONG, true>(64, 0);
  bad += run<64, KLONG, true>(64, -1);
  bad += run<64, KLONG, true>(64, 48);
  return bad;
}
