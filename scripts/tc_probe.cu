// tc_probe.cu -- standalone probe of the tcgen05 pieces used by the tensor-core
// kernels: TMEM alloc, SWIZZLE_NONE K-major / MN-major smem descriptors over the
// "[r/8][c/4][r%8][c%4]" core-matrix layout, kind::tf32 MMA (M=128 and M=64),
// commit -> mbarrier, tcgen05.ld 32x32b. Prints max errors vs a CPU reference.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 scripts/tc_probe.cu -o /tmp/tc_probe
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// byte offset of element (r, c) of a [R][C] matrix in the core-matrix layout
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C >> 2) * 128 + (c >> 2) * 128 + (r & 7) * 16 + (c & 3) * 4);
}

// 128B-swizzled layout of X[R][C] (R = rows, e.g. samples; C = cols, e.g. features):
// 1 KB atoms of 8 rows x 32 cols (128 B per row), atom (r/8, c/32) at ((r/8)*(C/32) + c/32) KB,
// 16-B chunk index XORed with the row index inside the atom (Swizzle<3,4,3>).
__host__ __device__ __forceinline__ uint32_t sw_off(int r, int c, int C) {
  return (uint32_t)(((r >> 3) * (C >> 5) + (c >> 5)) * 1024 + (r & 7) * 128 + ((((c & 31) >> 2) ^ (r & 7)) << 4) +
                    (c & 3) * 4);
}
__device__ __forceinline__ uint64_t sdesc_sw128(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version = 1 (sm_100)
  return d;              // base_offset 0, lbo_mode 0, layout SWIZZLE_NONE (0)
}

__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N, int a_mn, int b_mn) {
  return (1u << 4)            // D = F32
       | (2u << 7)            // A = TF32
       | (2u << 10)           // B = TF32
       | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16)
       | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const float (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
      "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(__float_as_uint(v[0])), "r"(__float_as_uint(v[1])), "r"(__float_as_uint(v[2])), "r"(__float_as_uint(v[3])),
      "r"(__float_as_uint(v[4])), "r"(__float_as_uint(v[5])), "r"(__float_as_uint(v[6])), "r"(__float_as_uint(v[7])),
      "r"(__float_as_uint(v[8])), "r"(__float_as_uint(v[9])), "r"(__float_as_uint(v[10])), "r"(__float_as_uint(v[11])),
      "r"(__float_as_uint(v[12])), "r"(__float_as_uint(v[13])), "r"(__float_as_uint(v[14])), "r"(__float_as_uint(v[15])),
      "r"(__float_as_uint(v[16])), "r"(__float_as_uint(v[17])), "r"(__float_as_uint(v[18])), "r"(__float_as_uint(v[19])),
      "r"(__float_as_uint(v[20])), "r"(__float_as_uint(v[21])), "r"(__float_as_uint(v[22])), "r"(__float_as_uint(v[23])),
      "r"(__float_as_uint(v[24])), "r"(__float_as_uint(v[25])), "r"(__float_as_uint(v[26])), "r"(__float_as_uint(v[27])),
      "r"(__float_as_uint(v[28])), "r"(__float_as_uint(v[29])), "r"(__float_as_uint(v[30])), "r"(__float_as_uint(v[31])));
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// T1: A [128][32] K-major, B [64][32] K-major: D1 = A B^T [128][64]          -> cols 0..63
// T2: A2 [128 s][128 m], B2 [128 s][32 n]: D = A2^T B2 [128][32], MN-major    -> cols 128.. (v0), 160.. (v1)
// T3: A3 [64][32] K-major, B3 [32][32] K-major: D = A3 B3^T [64][32], M = 64   -> cols 192..223
__global__ void probe(const float* A, const float* B, const float* A2, const float* B2, const float* A3,
                      const float* B3, float* D1, float* Draw) {
  extern __shared__ __align__(1024) uint8_t dsm[];
  uint8_t* sA = dsm;
  uint8_t* sB = sA + 128 * 32 * 4;
  uint8_t* sA2 = sB + 64 * 32 * 4;
  uint8_t* sB2 = sA2 + 128 * 128 * 4;
  uint8_t* sA3 = sB2 + 128 * 32 * 4;
  uint8_t* sB3 = sA3 + 64 * 32 * 4;
  uint8_t* sw_base = (uint8_t*)(((uintptr_t)(sB3 + 32 * 32 * 4) + 1023) & ~(uintptr_t)1023);
  uint8_t* sA4 = sw_base;                 // A2 data, swizzled [128 s][128 m]
  uint8_t* sB4 = sA4 + 128 * 128 * 4;     // B2 data, swizzled [128 s][32 n]
  uint8_t* sA5 = sB4 + 128 * 32 * 4;      // A data (T1), swizzled [128][32]
  uint8_t* sB5 = sA5 + 128 * 32 * 4;      // B data (T1), swizzled [64][32]
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sA + cm_off(r, c, 32)) = A[i]; }
  for (int i = t; i < 64 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sB + cm_off(r, c, 32)) = B[i]; }
  for (int i = t; i < 128 * 128; i += 128) { int r = i / 128, c = i % 128; *(float*)(sA2 + cm_off(r, c, 128)) = A2[i]; }
  for (int i = t; i < 128 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sB2 + cm_off(r, c, 32)) = B2[i]; }
  for (int i = t; i < 64 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sA3 + cm_off(r, c, 32)) = A3[i]; }
  for (int i = t; i < 32 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sB3 + cm_off(r, c, 32)) = B3[i]; }
  for (int i = t; i < 128 * 128; i += 128) { int r = i / 128, c = i % 128; *(float*)(sA4 + sw_off(r, c, 128)) = A2[i]; }
  for (int i = t; i < 128 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sB4 + sw_off(r, c, 32)) = B2[i]; }
  for (int i = t; i < 128 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sA5 + sw_off(r, c, 32)) = A[i]; }
  for (int i = t; i < 64 * 32; i += 128) { int r = i / 32, c = i % 32; *(float*)(sB5 + sw_off(r, c, 32)) = B[i]; }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
  {
    float z[32];
    for (int i = 0; i < 32; ++i) z[i] = -7.0f;
    for (int c = 128; c < 512; c += 32) tmem_st32(tm + lane_base + c, z);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (t == 0) {
    const uint32_t id1 = idesc_tf32(128, 64, 0, 0);
    for (int s = 0; s < 4; ++s) {
      uint64_t da = sdesc(smem_u32(sA) + s * 256, 128, 1024);
      uint64_t db = sdesc(smem_u32(sB) + s * 256, 128, 1024);
      mma_tf32(tm + 0, da, db, id1, s > 0);
    }
    const uint32_t id2 = idesc_tf32(128, 32, 1, 1);
    for (int v = 0; v < 2; ++v)
      for (int s = 0; s < 16; ++s) {
        const uint32_t ka = (128 / 4) * 128, kb = (32 / 4) * 128;
        uint64_t da = v == 0 ? sdesc(smem_u32(sA2) + s * ka, ka, 128) : sdesc(smem_u32(sA2) + s * ka, 128, ka);
        uint64_t db = v == 0 ? sdesc(smem_u32(sB2) + s * kb, kb, 128) : sdesc(smem_u32(sB2) + s * kb, 128, kb);
        mma_tf32(tm + 128 + 32 * v, da, db, id2, s > 0);
      }
    const uint32_t id3 = idesc_tf32(64, 32, 0, 0);
    for (int s = 0; s < 4; ++s) {
      uint64_t da = sdesc(smem_u32(sA3) + s * 256, 128, 1024);
      uint64_t db = sdesc(smem_u32(sB3) + s * 256, 128, 1024);
      mma_tf32(tm + 192, da, db, id3, s > 0);
    }
    // T4: MN-major, 128B swizzle. Per K-step u (8 samples): start = base + u * (C/32) KB;
    // LBO = next 32-wide MN atom (1 KB), SBO = next 8-deep K group ((C/32) KB).
    for (int u = 0; u < 16; ++u) {
      uint64_t da = sdesc_sw128(smem_u32(sA4) + u * 4 * 1024, 1024, 4 * 1024);
      uint64_t db = sdesc_sw128(smem_u32(sB4) + u * 1 * 1024, 1024, 1 * 1024);
      mma_tf32(tm + 224, da, db, idesc_tf32(128, 32, 1, 1), u > 0);
    }
    // T5: K-major, 128B swizzle (T1 problem). K-step t: start = base + (t/4) KB + (t%4)*32 B; SBO = 8-row group stride.
    for (int t4 = 0; t4 < 4; ++t4) {
      uint64_t da = sdesc_sw128(smem_u32(sA5) + t4 * 32, 16, 1024);
      uint64_t db = sdesc_sw128(smem_u32(sB5) + t4 * 32, 16, 1024);
      mma_tf32(tm + 256, da, db, idesc_tf32(128, 64, 0, 0), t4 > 0);
    }
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[32];
  for (int c0 = 0; c0 < 64; c0 += 32) {
    tmem_ld32(tm + lane_base + c0, v);
    for (int i = 0; i < 32; ++i) D1[t * 64 + c0 + i] = v[i];
  }
  for (int c0 = 128; c0 < 320; c0 += 32) {
    tmem_ld32(tm + lane_base + c0, v);
    for (int i = 0; i < 32; ++i) Draw[t * 192 + (c0 - 128) + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(512));
}

int main() {
  const int nA = 128 * 32, nB = 64 * 32, nA2 = 128 * 128, nB2 = 128 * 32, nA3 = 64 * 32, nB3 = 32 * 32;
  std::vector<float> A(nA), B(nB), A2(nA2), B2(nB2), A3(nA3), B3(nB3);
  uint32_t s = 12345;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return ((s >> 8) & 0xFFFF) / 65536.0f - 0.5f; };
  auto q = [](float x) { return std::round(x * 256.0f) / 256.0f; };
  for (auto* vec : {&A, &B, &A2, &B2, &A3, &B3})
    for (auto& x : *vec) x = q(rnd());
  float *dA, *dB, *dA2, *dB2, *dA3, *dB3, *dD1, *dDraw;
  cudaMalloc(&dA, nA * 4); cudaMalloc(&dB, nB * 4); cudaMalloc(&dA2, nA2 * 4); cudaMalloc(&dB2, nB2 * 4);
  cudaMalloc(&dA3, nA3 * 4); cudaMalloc(&dB3, nB3 * 4);
  cudaMalloc(&dD1, 128 * 64 * 4); cudaMalloc(&dDraw, 128 * 192 * 4);
  cudaMemcpy(dA, A.data(), nA * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), nB * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dA2, A2.data(), nA2 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB2, B2.data(), nB2 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dA3, A3.data(), nA3 * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB3, B3.data(), nB3 * 4, cudaMemcpyHostToDevice);
  const int smem = (nA + nB + nA2 + nB2 + nA3 + nB3) * 4 + 1024 + (128 * 128 + 128 * 32 + 128 * 32 + 64 * 32) * 4;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dA, dB, dA2, dB2, dA3, dB3, dD1, dDraw);
  cudaError_t e = cudaDeviceSynchronize();
  printf("kernel: %s\n", cudaGetErrorString(e));
  std::vector<float> D1(128 * 64), Dr(128 * 192);
  cudaMemcpy(D1.data(), dD1, D1.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(Dr.data(), dDraw, Dr.size() * 4, cudaMemcpyDeviceToHost);
  double e1 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double r = 0;
      for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * B[n * 32 + k];
      e1 = std::fmax(e1, std::fabs(r - D1[m * 64 + n]));
    }
  printf("T1 (M128 N64 K-major) max err %.3g\n", e1);
  for (int v = 0; v < 2; ++v) {
    double e2 = 0;
    for (int m = 0; m < 128; ++m)
      for (int n = 0; n < 32; ++n) {
        double r = 0;
        for (int k = 0; k < 128; ++k) r += (double)A2[k * 128 + m] * B2[k * 32 + n];
        e2 = std::fmax(e2, std::fabs(r - Dr[m * 192 + 32 * v + n]));
      }
    printf("T2 v%d (M128 N32 MN-major, %s) max err %.3g\n", v, v == 0 ? "LBO=k-group SBO=128" : "LBO=128 SBO=k-group", e2);
  }
  for (int m = 0; m < 3; ++m) {
    for (int n = 0; n < 3; ++n) {
      double r = 0;
      for (int k = 0; k < 128; ++k) r += (double)A2[k * 128 + m] * B2[k * 32 + n];
      printf("T2 m%d n%d ref %.5f v0 %.5f v1 %.5f\n", m, n, r, Dr[m * 192 + n], Dr[m * 192 + 32 + n]);
    }
  }
  // T3: M = 64 -> which lanes
  int found = 0;
  for (int m = 0; m < 64; ++m) {
    int lane = -1;
    for (int l = 0; l < 128; ++l) {
      double err = 0;
      for (int n = 0; n < 32; ++n) {
        double r = 0;
        for (int k = 0; k < 32; ++k) r += (double)A3[m * 32 + k] * B3[n * 32 + k];
        err = std::fmax(err, std::fabs(r - Dr[l * 192 + 64 + n]));
      }
      if (err < 1e-5) { lane = l; break; }
    }
    if (lane >= 0) ++found;
    if (m < 3 || (m > 14 && m < 18) || (m > 30 && m < 34) || m > 61) printf("T3 row %d -> lane %d\n", m, lane);
  }
  printf("T3 (M64 K-major) rows found %d/64\n", found);
  double e4 = 0, e5 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double r = 0;
      for (int k = 0; k < 128; ++k) r += (double)A2[k * 128 + m] * B2[k * 32 + n];
      e4 = std::fmax(e4, std::fabs(r - Dr[m * 192 + 96 + n]));
    }
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 64; ++n) {
      double r = 0;
      for (int k = 0; k < 32; ++k) r += (double)A[m * 32 + k] * B[n * 32 + k];
      e5 = std::fmax(e5, std::fabs(r - Dr[m * 192 + 128 + n]));
    }
  printf("T4 (M128 N32 MN-major SW128) max err %.3g   T5 (M128 N64 K-major SW128) max err %.3g\n", e4, e5);
  return 0;
}
