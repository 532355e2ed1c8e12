// lp_tc.cuh -- sm_100a tensor-core (tcgen05 / TMEM) building blocks for the fused
// ray march: TMEM allocation, UMMA shared-memory descriptors, kind::f16 MMA with
// fp32 accumulation, commit -> mbarrier, TMEM loads, and exact fp32 -> bf16
// piece splitting.
//
// Precision: every contraction runs on bf16 "pieces" of the fp32 operands,
// x = x0 + x1 + x2 (x_i = bf16 round-to-nearest of the remaining residual; three
// 8-bit pieces hold all 24 significand bits exactly), products accumulated in
// fp32 in TMEM. Dropping the piece products below 2^-16 (2 pieces) or 2^-24
// (3 pieces) relative leaves an fp32-class (3 pieces) or 1.5e-5-class
// (2 pieces) contraction -- DESIGN.md "Tensor-core precision".
//
// Shared-memory layout (one for every operand tile): a row-major matrix X[R][C]
// of bf16 is stored as 8x8 "core matrices" (8 rows x 16 bytes, contiguous),
//   byte(r, c) = (r/8)*(C/8)*128 + (c/8)*128 + (r%8)*16 + (c%8)*2   (SWIZZLE_NONE).
// The same bytes are a K-major UMMA operand with K along c (LBO = 128 B between
// K chunks, SBO = (C/8)*128 B between 8-row groups) and an MN-major operand
// with MN along c and K along r (LBO = (C/8)*128 B between 8-row K groups,
// SBO = 128 B between 8-column MN groups). Probed on B200 (scripts/tc_probe2.cu):
// kind::f16 accepts both views; kind::tf32 silently returns zeros for MN-major,
// hence bf16 pieces.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace lp {
namespace tc {

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__host__ __device__ constexpr uint32_t cm_off(int r, int c, int C) {
  return (uint32_t)((r >> 3) * (C >> 3) * 128 + (c >> 3) * 128 + (r & 7) * 16 + (c & 7) * 2);
}

// UMMA shared-memory matrix descriptor (SWIZZLE_NONE, sm_100 version field = 1)
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;
  return d;
}
// K-major view of X[R][C] (K along c), K-step ks covers columns [16ks, 16ks+16)
__device__ __forceinline__ uint64_t desc_kmajor(uint32_t base, int C, int ks) {
  return sdesc(base + (uint32_t)ks * 256u, 128u, (uint32_t)(C >> 3) * 128u);
}
// MN-major view of X[R][C] (MN along c, K along r), K-step ks covers rows [16ks, 16ks+16)
__device__ __forceinline__ uint64_t desc_mnmajor(uint32_t base, int C, int ks) {
  return sdesc(base + (uint32_t)ks * 2u * (uint32_t)(C >> 3) * 128u, (uint32_t)(C >> 3) * 128u, 128u);
}

// Precomputed descriptors: the K-major / MN-major view of a tile at `base`, moved by a byte
// offset with one add (the start-address field holds addr >> 4 in its low 14 bits, and
// shared-memory offsets stay below 256 KB, so the add never carries out of the field).
// K-step ks: +ks * 256 B (K-major), +ks * 2 (C / 8) * 128 B (MN-major).
__device__ __forceinline__ uint64_t kdesc0(uint32_t base, int C) { return sdesc(base, 128u, (uint32_t)(C >> 3) * 128u); }
__device__ __forceinline__ uint64_t mdesc0(uint32_t base, int C) { return sdesc(base, (uint32_t)(C >> 3) * 128u, 128u); }
__device__ __forceinline__ uint64_t dplus(uint64_t d, uint32_t bytes) { return d + (uint64_t)(bytes >> 4); }

// Instruction descriptor: kind::f16, A/B = BF16, D = F32.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, int a_mn, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)a_mn << 15) | ((uint32_t)b_mn << 16) |
         ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_bf16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// Same with the A operand in tensor memory (M = 128 lanes = rows, bf16 K pairs packed per
// 32-bit column: K-step ks of 16 elements = 8 columns); probed: scripts/tc_probe3.cu.
__device__ __forceinline__ void mma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                            uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst_smem)),
               "r"(ncols)
               : "memory");
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}

__device__ __forceinline__ void fence_before_sync() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_after_sync() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
// generic-proxy smem writes -> visible to the tensor core (async proxy)
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void named_bar(int id, int nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {   // release.cta: prior writes visible to the waiters
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n\t.reg .pred P1;\n\tLP_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
      "@P1 bra LP_DONE_%=;\n\tbra LP_WAIT_%=;\n\tLP_DONE_%=:\n\t}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// TMEM -> registers: lane = row of the warp's 32-lane quarter, N consecutive fp32 columns.
template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[N]);

#define LP_TMEM_LD8(OFF)                                                                                       \
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"                         \
               : "=r"(r[OFF + 0]), "=r"(r[OFF + 1]), "=r"(r[OFF + 2]), "=r"(r[OFF + 3]), "=r"(r[OFF + 4]),     \
                 "=r"(r[OFF + 5]), "=r"(r[OFF + 6]), "=r"(r[OFF + 7])                                           \
               : "r"(taddr + OFF))

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, float (&v)[N]) {
  static_assert(N % 8 == 0, "TMEM load width");
  uint32_t r[N];
#pragma unroll
  for (int i = 0; i < N; i += 8) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[i + 0]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), "=r"(r[i + 5]),
                   "=r"(r[i + 6]), "=r"(r[i + 7])
                 : "r"(taddr + (uint32_t)i));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);
}
#undef LP_TMEM_LD8

// TMEM -> registers for an M = 64 accumulator (row i in lane (i/16)*32 + i%16), two threads
// per row: thread t of the warp reads lane t%16 of the warp's quarter, columns
// [taddr.col + (t/16)*SPLIT, + N). Shape 16x32bx2 (probed: scripts/tc_probe4.cu).
template <int N, int SPLIT>
__device__ __forceinline__ void tmem_ld16x2(uint32_t taddr, float (&v)[N]) {
  static_assert(N % 8 == 0, "TMEM load width");
  uint32_t r[N];
#pragma unroll
  for (int i = 0; i < N; i += 8) {
    asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
                 : "=r"(r[i + 0]), "=r"(r[i + 1]), "=r"(r[i + 2]), "=r"(r[i + 3]), "=r"(r[i + 4]), "=r"(r[i + 5]),
                   "=r"(r[i + 6]), "=r"(r[i + 7])
                 : "r"(taddr + (uint32_t)i), "n"(SPLIT));
  }
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __uint_as_float(r[i]);
}

// registers -> TMEM: lane = row of the warp's 32-lane quarter, N consecutive 32-bit columns.
// The caller issues tmem_wait_st() (or to_tensor_core-style fences) before the MMA reads them.
template <int N>
__device__ __forceinline__ void tmem_st(uint32_t taddr, const uint32_t (&r)[N]) {
  static_assert(N % 8 == 0, "TMEM store width");
#pragma unroll
  for (int i = 0; i < N; i += 8)
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr + (uint32_t)i),
                 "r"(r[i + 0]), "r"(r[i + 1]), "r"(r[i + 2]), "r"(r[i + 3]), "r"(r[i + 4]), "r"(r[i + 5]),
                 "r"(r[i + 6]), "r"(r[i + 7])
                 : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- bf16 pieces
__device__ __forceinline__ uint32_t pack_bf16x2(float a, float b) {
  __nv_bfloat162 h = __floats2bfloat162_rn(a, b);  // .x = a (low half), .y = b
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ float bf16lo_to_f(uint32_t p) { return __uint_as_float(p << 16); }
__device__ __forceinline__ float bf16hi_to_f(uint32_t p) { return __uint_as_float(p & 0xFFFF0000u); }

// Split a pair (a, b) into NP bf16x2 pieces: a = sum_i lo(piece_i), b = sum_i hi(piece_i).
template <int NP>
__device__ __forceinline__ void split_pair(float a, float b, uint32_t (&p)[NP]) {
#pragma unroll
  for (int i = 0; i < NP; ++i) {
    p[i] = pack_bf16x2(a, b);
    a -= bf16lo_to_f(p[i]);
    b -= bf16hi_to_f(p[i]);
  }
}

// Store 8 consecutive values v[0..8) of row r (columns c0..c0+7, c0 % 8 == 0) of an
// X[R][C] tile as NP bf16 pieces (piece i at base + i * piece_stride).
template <int NP>
__device__ __forceinline__ void store8(uint8_t* base, uint32_t piece_stride, int r, int c0, int C, const float* v) {
  uint32_t p0[NP], p1[NP], p2[NP], p3[NP];
  split_pair<NP>(v[0], v[1], p0);
  split_pair<NP>(v[2], v[3], p1);
  split_pair<NP>(v[4], v[5], p2);
  split_pair<NP>(v[6], v[7], p3);
  const uint32_t off = cm_off(r, c0, C);
#pragma unroll
  for (int i = 0; i < NP; ++i)
    *reinterpret_cast<uint4*>(base + i * piece_stride + off) = make_uint4(p0[i], p1[i], p2[i], p3[i]);
}
// 3-piece split of 8 consecutive values: pieces 0 and 1 stored like store8<2>, piece 2
// returned as 4 packed bf16x2 words (for a TMEM-resident copy of the last piece).
__device__ __forceinline__ void store8_split3(uint8_t* base, uint32_t piece_stride, int r, int c0, int C,
                                              const float* v, uint32_t* p2) {
  uint32_t q[4][3];
#pragma unroll
  for (int i = 0; i < 4; ++i) split_pair<3>(v[2 * i], v[2 * i + 1], q[i]);
  const uint32_t off = cm_off(r, c0, C);
#pragma unroll
  for (int i = 0; i < 2; ++i)
    *reinterpret_cast<uint4*>(base + i * piece_stride + off) = make_uint4(q[0][i], q[1][i], q[2][i], q[3][i]);
#pragma unroll
  for (int i = 0; i < 4; ++i) p2[i] = q[i][2];
}
// Same for 4 consecutive values (c0 % 4 == 0): 8-byte stores.
template <int NP>
__device__ __forceinline__ void store4(uint8_t* base, uint32_t piece_stride, int r, int c0, int C, const float* v) {
  uint32_t p0[NP], p1[NP];
  split_pair<NP>(v[0], v[1], p0);
  split_pair<NP>(v[2], v[3], p1);
  const uint32_t off = cm_off(r, c0, C);
#pragma unroll
  for (int i = 0; i < NP; ++i)
    *reinterpret_cast<uint2*>(base + i * piece_stride + off) = make_uint2(p0[i], p1[i]);
}

}  // namespace tc
}  // namespace lp
