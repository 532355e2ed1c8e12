// tc_probe3.cu -- kind::f16 MMA with the A operand in TENSOR MEMORY (tcgen05.mma [d], [a], b_desc):
// each thread (row) writes its row of A (bf16 pairs, 2 per 32-bit column) with tcgen05.st, one
// elected thread issues D[128][64] = A[128][64] B^T (B = [64 n][64 k] K-major in shared memory),
// every thread reads its D row back. Checked against a host fp64 reference of the bf16 inputs.
// Also times a chain of such MMAs against the same chain with A in shared memory.
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C >> 3) * 128 + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int C, int ks) {
  return sdesc(base + (uint32_t)ks * 256u, 128u, (uint32_t)(C >> 3) * 128u);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_ss(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t dt, uint32_t at, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(dt),
               "r"(at), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)), "r"(phase));
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}

constexpr int M = 128, N = 64, KD = 64;

// mode 0: A from TMEM, mode 1: A from shared memory; `reps` MMA chains of KD/16 k-steps (timing)
__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* D, int mode, int reps,
                      long long* cycles) {
  __shared__ __align__(128) uint8_t sa[M * KD * 2];
  __shared__ __align__(128) uint8_t sb[N * KD * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, w = t >> 5;
  for (int i = t; i < N * KD; i += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sb + cm_off(i / KD, i % KD, KD)) = B[i];
  for (int i = t; i < M * KD; i += blockDim.x)
    *reinterpret_cast<__nv_bfloat16*>(sa + cm_off(i / KD, i % KD, KD)) = A[i];
  if (t == 0) mbar_init(&bar, 1);
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tslot)),
                 "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tD = tslot, tA = tslot + 128;      // D cols [0,64), A cols [128, 128 + KD/2)
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  // row t of A: KD bf16 = KD/2 packed columns
  for (int c8 = 0; c8 < KD / 16; ++c8) {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) {
      __nv_bfloat162 h;
      h.x = A[t * KD + c8 * 16 + 2 * i];
      h.y = A[t * KD + c8 * 16 + 2 * i + 1];
      r[i] = *reinterpret_cast<uint32_t*>(&h);
    }
    st8(tA + lane_off + c8 * 8, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t id = idesc_bf16(M, N, 0, 0);
  long long t0 = clock64();
  uint32_t phase = 0;
  for (int rep = 0; rep < reps; ++rep) {
    if (t == 0) {
      for (int ks = 0; ks < KD / 16; ++ks) {
        if (mode == 0) mma_ts(tD, tA + ks * 8, desc_kmajor(smem_u32(sb), KD, ks), id, ks > 0);
        else mma_ss(tD, desc_kmajor(smem_u32(sa), KD, ks), desc_kmajor(smem_u32(sb), KD, ks), id, ks > 0);
      }
      commit(&bar);
    }
    mbar_wait(&bar, phase);
    phase ^= 1;
  }
  long long t1 = clock64();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c8 = 0; c8 < N / 8; ++c8) {
    float v[8];
    ld8(tD + lane_off + c8 * 8, v);
    for (int i = 0; i < 8; ++i) D[t * N + c8 * 8 + i] = v[i];
  }
  if (t == 0) *cycles = t1 - t0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tslot), "r"(256));
}

int main() {
  std::vector<__nv_bfloat16> A(M * KD), B(N * KD);
  std::vector<float> Af(M * KD), Bf(N * KD);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; };
  for (int i = 0; i < M * KD; ++i) { A[i] = __float2bfloat16(rnd()); Af[i] = __bfloat162float(A[i]); }
  for (int i = 0; i < N * KD; ++i) { B[i] = __float2bfloat16(rnd()); Bf[i] = __bfloat162float(B[i]); }
  __nv_bfloat16 *dA, *dB;
  float* dD;
  long long* dc;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dc, 8);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  std::vector<float> D(M * N);
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(dD, 0, M * N * 4);
    probe<<<1, 128>>>(dA, dB, dD, mode, 1, dc);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("mode %d: CUDA error %s\n", mode, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, M * N * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) {
        double ref = 0;
        for (int k = 0; k < KD; ++k) ref += (double)Af[m * KD + k] * Bf[n * KD + k];
        maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
        maxref = fmax(maxref, fabs(ref));
      }
    long long cyc = 0;
    probe<<<1, 128>>>(dA, dB, dD, mode, 1000, dc);
    cudaDeviceSynchronize();
    cudaMemcpy(&cyc, dc, 8, cudaMemcpyDeviceToHost);
    printf("A from %s: max |err| %.3e (max |ref| %.3e) %s; %.1f cycles per 4-MMA chain (commit + wait)\n",
           mode == 0 ? "TMEM" : "SMEM", maxerr, maxref, maxerr <= 1e-5 * maxref ? "OK" : "MISMATCH", cyc / 1000.0);
  }
  return 0;
}
