// tc_probe4.cu -- layout of tcgen05.ld.16x32bx2 (two threads per TMEM lane) against an M = 64
// accumulator, for the two-network view-dependent kernels (lp_tcv2_kernels.cuh):
//  (1) TMEM filled with value(lane, col) = lane * 1000 + col by 32x32b stores; each warp q loads
//      16x32bx2.x8 at lane 32q, column 0, half-split offset 32: expected thread t -> lane 32q + t%16,
//      columns (t/16)*32 + 0..7.
//  (3) the same load at lane 32q + 16 (upper half of the warp's quarter): expected thread t ->
//      lane 32q + 16 + t%16 (two threads per row of an M = 128 accumulator in one warp).
//  (2) D[64][64] = A[64][32] B^T (M = 64, kind::f16, A K-major, B K-major) read back with
//      16x32bx2.x32 (split 32): expected thread t of warp q -> row 16q + t%16, columns (t/16)*32 + 0..31.
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
// 16x32bx2.x8, half-split offset 32 columns
__device__ __forceinline__ void ld16x2_8(uint32_t taddr, uint32_t (&r)[8]) {
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], 32;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

constexpr int M = 64, N = 64, KD = 32;

__global__ void probe(const __nv_bfloat16* A, const __nv_bfloat16* B, uint32_t* L, float* D, uint32_t* L2) {
  __shared__ __align__(128) uint8_t sa[M * KD * 2];
  __shared__ __align__(128) uint8_t sb[N * KD * 2];
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int t = threadIdx.x, w = t >> 5, l = t & 31;
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
  const uint32_t lane_off = (uint32_t)(w * 32) << 16;
  const uint32_t tV = tslot + 128, tD = tslot;
  // (1) value(lane, col) = lane * 1000 + col in columns [128, 192)
  for (int c8 = 0; c8 < 8; ++c8) {
    uint32_t r[8];
    for (int i = 0; i < 8; ++i) r[i] = (uint32_t)(t * 1000 + c8 * 8 + i);
    st8(tV + lane_off + c8 * 8, r);
  }
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
  {
    uint32_t r[8];
    ld16x2_8(tV + lane_off, r);
    for (int i = 0; i < 8; ++i) L[t * 8 + i] = r[i];
    ld16x2_8(tV + lane_off + (16u << 16), r);
    for (int i = 0; i < 8; ++i) L2[t * 8 + i] = r[i];
  }
  // (2) M = 64 MMA
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t id = idesc_bf16(M, N, 0, 0);
    for (int ks = 0; ks < KD / 16; ++ks)
      mma_ss(tD, desc_kmajor(smem_u32(sa), KD, ks), desc_kmajor(smem_u32(sb), KD, ks), id, ks > 0);
    commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  for (int c8 = 0; c8 < 4; ++c8) {
    uint32_t r[8];
    ld16x2_8(tD + lane_off + c8 * 8, r);
    const int row = 16 * w + (l & 15), col0 = (l >> 4) * 32 + c8 * 8;
    for (int i = 0; i < 8; ++i) D[row * N + col0 + i] = __uint_as_float(r[i]);
  }
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
  uint32_t *dL, *dL2;
  cudaMalloc(&dA, A.size() * 2); cudaMalloc(&dB, B.size() * 2); cudaMalloc(&dD, M * N * 4); cudaMalloc(&dL, 128 * 8 * 4);
  cudaMalloc(&dL2, 128 * 8 * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0xFF, M * N * 4);
  probe<<<1, 128>>>(dA, dB, dL, dD, dL2);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); return 1; }
  std::vector<uint32_t> L(128 * 8);
  std::vector<float> D(M * N);
  cudaMemcpy(L.data(), dL, L.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int t = 0; t < 128; ++t)
    for (int i = 0; i < 8; ++i) {
      const int w = t / 32, l = t % 32;
      const uint32_t want = (uint32_t)((32 * w + (l & 15)) * 1000 + (l >> 4) * 32 + i);
      if (L[t * 8 + i] != want) ++bad;
    }
  printf("(1) 16x32bx2 layout: %s (%d mismatches); warp 0 thread 0: %u %u, thread 1: %u, thread 16: %u, thread 17: %u\n",
         bad ? "UNEXPECTED" : "thread t -> lane t%16, columns (t/16)*split + i", bad, L[0], L[1], L[8], L[16 * 8],
         L[17 * 8]);
  std::vector<uint32_t> L2(128 * 8);
  cudaMemcpy(L2.data(), dL2, L2.size() * 4, cudaMemcpyDeviceToHost);
  bad = 0;
  for (int t = 0; t < 128; ++t)
    for (int i = 0; i < 8; ++i) {
      const int w = t / 32, l = t % 32;
      const uint32_t want = (uint32_t)((32 * w + 16 + (l & 15)) * 1000 + (l >> 4) * 32 + i);
      if (L2[t * 8 + i] != want) ++bad;
    }
  printf("(3) 16x32bx2 at lane offset 16: %s (%d mismatches); warp 0 thread 0: %u, thread 16: %u\n",
         bad ? "UNEXPECTED" : "thread t -> lane 16 + t%16", bad, L2[0], L2[16 * 8]);
  double maxerr = 0, maxref = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double ref = 0;
      for (int k = 0; k < KD; ++k) ref += (double)Af[m * KD + k] * Bf[n * KD + k];
      maxerr = fmax(maxerr, fabs(ref - D[m * N + n]));
      maxref = fmax(maxref, fabs(ref));
    }
  printf("(2) M=64 MMA read with 16x32bx2 (row 16q + t%%16, cols (t/16)*32 + i): max |err| %.3e (max |ref| %.3e) %s\n",
         maxerr, maxref, maxerr <= 1e-5 * maxref ? "OK" : "MISMATCH");
  return 0;
}
