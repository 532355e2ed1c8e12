// tc_probe2.cu -- kind::f16 (bf16 inputs, fp32 accumulate) with K-major and MN-major
// operands over the sample-major core-matrix layout, SWIZZLE_NONE and SWIZZLE_128B.
#include <cstdint>
#include <cstdio>
#include <cmath>
#include <vector>
#include <cuda_runtime.h>
#include <cuda_bf16.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// bf16 element (r, c) of X[R][C] (2-byte elements): core matrices 8 rows x 16 B (8 elements)
__host__ __device__ __forceinline__ uint32_t cm_off(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C >> 3) * 128 + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}
// 128B swizzle: atoms of 8 rows x 64 elements (128 B/row), atom (r/8, c/64)
__host__ __device__ __forceinline__ uint32_t sw_off(int r, int c, int C) {
  return (uint32_t)(((r >> 3) * (C >> 6) + (c >> 6)) * 1024 + (r & 7) * 128 + ((((c & 63) >> 3) ^ (r & 7)) << 4) +
                    (c & 7) * 2);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo, uint32_t layout) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)layout << 61;
  return d;
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t dt, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
               "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dt),
               "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(n));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile("{\n\t.reg .pred P1;\n\tLAB_WAIT:\n\t"
               "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
               "@P1 bra DONE;\n\tbra LAB_WAIT;\n\tDONE:\n\t}" ::"r"(smem_u32(bar)), "r"(phase));
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
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// X: [128 s][64 f] ; Y: [128 s][32 n]
// Tk: D[128 s][32 n] = X_first32? no: K-major test D = X Wt: X [128][64] (K=64), W [32][64] -> D [128][32]
// Tm: D[64 f][32 n] = X^T Y (K = s = 128), MN-major both
__global__ void probe(const __nv_bfloat16* X, const __nv_bfloat16* W, const __nv_bfloat16* Y, float* out) {
  extern __shared__ uint8_t dsm[];
  uint8_t* base = (uint8_t*)(((uintptr_t)dsm + 1023) & ~(uintptr_t)1023);
  uint8_t* xN = base;                 // X, SWIZZLE_NONE  (16 KB)
  uint8_t* wN = xN + 128 * 64 * 2;    // W, NONE          (4 KB)
  uint8_t* yN = wN + 32 * 64 * 2;     // Y, NONE          (8 KB)
  uint8_t* xS = yN + 128 * 32 * 2;    // X, SW128
  uint8_t* wS = xS + 128 * 64 * 2;    // W, SW128 (C=64)
  uint8_t* yS = wS + 32 * 64 * 2;     // Y, SW128 -> C=32 < 64: use a padded C=64 atom row
  __shared__ uint64_t bar;
  __shared__ uint32_t tbase;
  const int t = threadIdx.x, warp = t >> 5;
  for (int i = t; i < 128 * 64; i += 128) {
    int r = i / 64, c = i % 64;
    *(__nv_bfloat16*)(xN + cm_off(r, c, 64)) = X[i];
    *(__nv_bfloat16*)(xS + sw_off(r, c, 64)) = X[i];
  }
  for (int i = t; i < 32 * 64; i += 128) {
    int r = i / 64, c = i % 64;
    *(__nv_bfloat16*)(wN + cm_off(r, c, 64)) = W[i];
    *(__nv_bfloat16*)(wS + sw_off(r, c, 64)) = W[i];
  }
  for (int i = t; i < 128 * 32; i += 128) {
    int r = i / 32, c = i % 32;
    *(__nv_bfloat16*)(yN + cm_off(r, c, 32)) = Y[i];
  }
  for (int i = t; i < 128 * 64; i += 128) {   // Y padded to 64 cols for the swizzled atom
    int r = i / 64, c = i % 64;
    *(__nv_bfloat16*)(yS + sw_off(r, c, 64)) = c < 32 ? Y[r * 32 + c] : __float2bfloat16(0.0f);
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tbase)), "r"(256));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) mbar_init(&bar, 1);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tm = tbase;
  if (t == 0) {
    // K-major NONE: D0 [128][32] = X W^T, 4 K-steps of 16 (2 chunks of 8 elems each)
    for (int k = 0; k < 4; ++k)
      mma_f16(tm + 0, sdesc(smem_u32(xN) + k * 256, 128, 8 * 128, 0), sdesc(smem_u32(wN) + k * 256, 128, 8 * 128, 0),
              idesc_bf16(128, 32, 0, 0), k > 0);
    // K-major SW128: K-step k: start + k*32 B; SBO = 1 KB (8-row group, C=64 -> 1 atom per row group)
    for (int k = 0; k < 4; ++k)
      mma_f16(tm + 32, sdesc(smem_u32(xS) + k * 32, 16, 1024, 2), sdesc(smem_u32(wS) + k * 32, 16, 1024, 2),
              idesc_bf16(128, 32, 0, 0), k > 0);
    // MN-major NONE: D [64 f][32 n] = X^T Y; K-step u = 16 samples = 2 row groups
    //   X view: MN = f (groups of 8 elems = 16 B, stride 128 B), K = s (8-row groups stride (64/8)*128 B)
    for (int u = 0; u < 8; ++u)
      mma_f16(tm + 64, sdesc(smem_u32(xN) + u * 2 * 8 * 128, 8 * 128, 128, 0),
              sdesc(smem_u32(yN) + u * 2 * 4 * 128, 4 * 128, 128, 0), idesc_bf16(64, 32, 1, 1), u > 0);
    for (int u = 0; u < 8; ++u)   // same with LBO/SBO swapped
      mma_f16(tm + 96, sdesc(smem_u32(xN) + u * 2 * 8 * 128, 128, 8 * 128, 0),
              sdesc(smem_u32(yN) + u * 2 * 4 * 128, 128, 4 * 128, 0), idesc_bf16(64, 32, 1, 1), u > 0);
    // MN-major SW128: K-step u = 16 samples = 2 atoms along K (8 rows each): SBO = K-atom stride (1 KB),
    //   LBO = MN-atom stride (64 elems); X has 1 atom per 8-row group (C=64), so MN atoms: only one (64 = M).
    for (int u = 0; u < 8; ++u)
      mma_f16(tm + 128, sdesc(smem_u32(xS) + u * 2 * 1024, 1024, 1024, 2),
              sdesc(smem_u32(yS) + u * 2 * 1024, 1024, 1024, 2), idesc_bf16(64, 32, 1, 1), u > 0);
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  float v[32];
  for (int c0 = 0; c0 < 160; c0 += 32) {
    tmem_ld32(tm + ((uint32_t)(warp * 32) << 16) + c0, v);
    for (int i = 0; i < 32; ++i) out[t * 160 + c0 + i] = v[i];
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tm), "r"(256));
}

int main() {
  std::vector<float> X(128 * 64), W(32 * 64), Y(128 * 32);
  uint32_t s = 777;
  auto rnd = [&]() { s = s * 1664525u + 1013904223u; return std::round((((s >> 8) & 0xFFFF) / 65536.0f - 0.5f) * 64) / 64; };
  for (auto* v : {&X, &W, &Y}) for (auto& x : *v) x = rnd();
  std::vector<__nv_bfloat16> Xb(X.size()), Wb(W.size()), Yb(Y.size());
  for (size_t i = 0; i < X.size(); ++i) Xb[i] = __float2bfloat16(X[i]);
  for (size_t i = 0; i < W.size(); ++i) Wb[i] = __float2bfloat16(W[i]);
  for (size_t i = 0; i < Y.size(); ++i) Yb[i] = __float2bfloat16(Y[i]);
  __nv_bfloat16 *dX, *dW, *dY; float* dO;
  cudaMalloc(&dX, Xb.size() * 2); cudaMalloc(&dW, Wb.size() * 2); cudaMalloc(&dY, Yb.size() * 2); cudaMalloc(&dO, 128 * 160 * 4);
  cudaMemcpy(dX, Xb.data(), Xb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dW, Wb.data(), Wb.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dY, Yb.data(), Yb.size() * 2, cudaMemcpyHostToDevice);
  int smem = 1024 + (128 * 64 + 32 * 64 + 128 * 32 + 128 * 64 + 32 * 64 + 128 * 64) * 2;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  probe<<<1, 128, smem>>>(dX, dW, dY, dO);
  printf("kernel: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  std::vector<float> O(128 * 160);
  cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  double e0 = 0, e1 = 0;
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < 32; ++n) {
      double r = 0;
      for (int k = 0; k < 64; ++k) r += (double)X[m * 64 + k] * W[n * 64 + k];
      e0 = std::fmax(e0, std::fabs(r - O[m * 160 + n]));
      e1 = std::fmax(e1, std::fabs(r - O[m * 160 + 32 + n]));
    }
  printf("K-major NONE err %.3g   K-major SW128 err %.3g\n", e0, e1);
  const char* names[3] = {"MN NONE (LBO=k,SBO=mn)", "MN NONE (LBO=mn,SBO=k)", "MN SW128"};
  for (int v = 0; v < 3; ++v) {
    double e = 0;
    for (int f = 0; f < 64; ++f) {
      int lane = (f / 16) * 32 + f % 16;   // M = 64 row -> TMEM lane
      for (int n = 0; n < 32; ++n) {
        double r = 0;
        for (int k = 0; k < 128; ++k) r += (double)X[k * 64 + f] * Y[k * 32 + n];
        e = std::fmax(e, std::fabs(r - O[lane * 160 + 64 + 32 * v + n]));
      }
    }
    printf("%s err %.3g (sample %f)\n", names[v], e, O[0 * 160 + 64 + 32 * v]);
  }
  return 0;
}
