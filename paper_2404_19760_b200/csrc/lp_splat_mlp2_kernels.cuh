// lp_splat_mlp2_kernels.cuh -- the Splatter with the paper's 3-layer g_s (Eq. 2, P:272-282;
// "Both the Splatter and Renderer components are equipped with 3-layer MLPs with a width of
// 64"): g_s = [v (32) | h_prior (32) | direnc (6F)] -> 64 -> 64 -> 32 (ReLU, ReLU,
// identity), params packed W0 [64][C_in + K_p + 6F], b0, W1 [64][64], b1, W2 [32][64], b2.
//
// Tiles of 64 rays with M = 64 MMAs, as the renderer's two-network kernels (lp_tcv2_kernels.cuh):
// the three 3-piece weight matrices take 72 KB of shared memory, which leaves no room for the
// 128-row activation tiles of an extra layer. CG column groups of 4 warps, 2 CG threads per ray
// (thread (cg, half) owns hidden units [32 cg + UPT half, + UPT), UPT = 32 / CG), reading the
// M = 64 accumulators with the 16x32bx2 TMEM load. Per step:
//   forward   gather h_prior | Z1 = A W0^T | a1 -> A1 | Z2 = A1 W1^T | a2 -> A1 | V~ = A2 W2^T |
//             v~ + b2 -> fp32 staging, splatted (with the weight pass) by the scatter warps
//   backward  gather h_prior, gather g / theta_weight -> DV | Z1 | a1 -> A1 | Z2 | a2 -> A2 |
//             dA2 = DV W2, [dW2 db2] += DV^T [A2 | 1] | delta2 -> D | dA1 = D2 W1,
//             [dW1 db1] += D2^T [A1 | 1] | delta1 -> D | dA = D1 W0 (v and prior columns),
//             [dW0 db0] += D1^T [A | 1] | dL/dv accumulated per ray, dh_prior staged for the
//             scatter warps
// Precision as in lp_tc.cuh (forward-type products 3 x 3 pieces, gradient-type 2 x 2).
#pragma once

#include "lp_splat_mlp_kernels.cuh"
#include "lp_tcv2_kernels.cuh"

namespace lp {

#ifndef LP_GS2_CG
#define LP_GS2_CG 2
#endif
constexpr int kGs2CG = LP_GS2_CG;
#ifndef LP_GS2_SW
#define LP_GS2_SW 2
#endif
constexpr int kGs2ScatterWarps = LP_GS2_SW;

struct Gs2Layout {
  static constexpr int CG = kGs2CG, UPT = 32 / CG, OPT = 16 / CG, NC = 128 * CG;
  // weights, K-major [out][in], 3 bf16 pieces
  static constexpr uint32_t W0 = 0, W1 = kGsH * kGsKA * 2, W2 = W1 + kGsH * kGsH * 2;
  static constexpr uint32_t W_PIECE = W2 + kGsK * kGsH * 2;
  static constexpr uint32_t FP = 3 * W_PIECE;                         // b0 [64], b1 [64], b2 [32]
  static constexpr uint32_t GRP = (FP + (2 * kGsH + kGsK) * 4 + 127) & ~127u;
  static_assert(CG == 1 || CG == 2, "column groups");
};

// packed parameter offsets
struct Gs2Packed {
  __device__ static int B0(int nin) { return kGsH * nin; }
  __device__ static int W1(int nin) { return B0(nin) + kGsH; }
  __device__ static int B1(int nin) { return W1(nin) + kGsH * kGsH; }
  __device__ static int W2(int nin) { return B1(nin) + kGsH; }
  __device__ static int B2(int nin) { return W2(nin) + kGsK * kGsH; }
};

__device__ __forceinline__ void stage_gs2_weights(uint8_t* smem, const float* __restrict__ g, int E) {
  using L = Gs2Layout;
  const int nin = kGsC + kGsKp + E;
  const int n0 = kGsH * nin, n1 = n0 + kGsH * kGsH, n2 = n1 + kGsK * kGsH;
  for (int i = threadIdx.x; i < n2; i += blockDim.x) {
    uint32_t off;
    float v;
    if (i < n0) {   // [v | prior | direnc] share the A tile's column order
      off = L::W0 + tc::cm_off(i / nin, i % nin, kGsKA);
      v = g[i];
    } else if (i < n1) {
      const int j = i - n0;
      off = L::W1 + tc::cm_off(j / kGsH, j % kGsH, kGsH);
      v = g[Gs2Packed::W1(nin) + j];
    } else {
      const int j = i - n1;
      off = L::W2 + tc::cm_off(j / kGsH, j % kGsH, kGsH);
      v = g[Gs2Packed::W2(nin) + j];
    }
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(smem + pc * L::W_PIECE + off) = b;
      v -= __bfloat162float(b);
    }
  }
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  for (int i = threadIdx.x; i < kGsH; i += blockDim.x) {
    fp[i] = g[Gs2Packed::B0(nin) + i];
    fp[kGsH + i] = g[Gs2Packed::B1(nin) + i];
  }
  for (int i = threadIdx.x; i < kGsK; i += blockDim.x) fp[2 * kGsH + i] = g[Gs2Packed::B2(nin) + i];
}

// this thread's UPT pre-activations (+ bias) -> ReLU mask bits and NP-piece tile stores
template <int NP, int UPT>
__device__ __forceinline__ uint32_t gs2_relu_store(const float (&z)[UPT], const float* b, uint8_t* tile, uint32_t piece,
                                                   int row, int c0, int C) {
  uint32_t mask = 0;
#pragma unroll
  for (int c8 = 0; c8 < UPT / 8; ++c8) {
    float a[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const float zz = z[8 * c8 + u] + b[8 * c8 + u];
      mask |= (zz > 0.0f ? 1u : 0u) << (8 * c8 + u);
      a[u] = fmaxf(zz, 0.0f);
    }
    tc::store8<NP>(tile, piece, row, c0 + 8 * c8, C, a);
  }
  return mask;
}

// ================================================================= forward
template <int KIND>
struct Gs2FwdSmem : Gs2Layout {
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  static constexpr uint32_t A_PIECE = 64 * kGsKA * 2;      // [v | prior | direnc] [64][96]
  static constexpr uint32_t A1_PIECE = 64 * kGsH * 2;      // a1, then a2 [64][64]
  static constexpr uint32_t A = GRP;
  static constexpr uint32_t A1 = A + 3 * A_PIECE;
  static constexpr uint32_t DHS = A1 + 3 * A1_PIECE;        // fp32 v~ rows [64][K + 4]
  static constexpr uint32_t PTAPS = DHS + 64 * (kGsK + 4) * 4;
  static constexpr uint32_t TAPS = PTAPS + 64 * NPL * 16;   // [CG][64][NPL]
  static constexpr uint32_t BAR = (TAPS + CG * 64 * NPL * 16 + 127) & ~127u;   // MMA, staged, drained, tmem slot
  static constexpr uint32_t BYTES = BAR + 32;
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int KIND>
__global__ void __launch_bounds__(128 * kGs2CG + 32 * kGs2ScatterWarps, 1) lp_splat_mlp2_fwd_kernel(const SplatMlpArgs a) {
  using L = Gs2FwdSmem<KIND>;
  constexpr int NPL = L::NPL, KC = kGsKp / 4, CG = L::CG, UPT = L::UPT, OPT = L::OPT, NC = L::NC;
  constexpr int SW = kGs2ScatterWarps;
  static_assert(SW == 1 || SW == 2, "scatter warps");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* At = smem + L::A;
  uint8_t* A1t = smem + L::A1;
  float* dhs = reinterpret_cast<float*>(smem + L::DHS);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  const float* fp = reinterpret_cast<const float*>(smem + L::FP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* bar_st = bar + 1;   // NC compute threads: v~ of the step staged
  uint64_t* bar_dr = bar + 2;   // every lane of the scatter warps: staging read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 24);
  const SplatArgs& s = a.s;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_gs2_weights(smem, a.params, 6 * a.dir_freqs);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, NC);
    tc::mbar_init(bar_dr, 32 * SW);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 256);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int64_t ntiles = (s.M + 63) / 64;

  if (threadIdx.x >= NC) {   // ---- scatter warps: the splat of every staged step (v~ and the weight pass)
    const int sw = (threadIdx.x - NC) >> 5, sl = threadIdx.x & 31;
    float* sth[3] = {s.theta[0], s.theta[1], s.theta[2]};
    float* swt[3] = {s.weight[0], s.weight[1], s.weight[2]};
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int j = 0; j < s.S; ++j) {
        tc::mbar_wait(bar_st, ph);
        ph ^= 1;
        for (int rb = sw; rb < 2; rb += SW)
          coop_scatter<KIND, kGsK>(sth, ptaps, s.dims, dhs, rb * 32, sl, 0, kGsK / 4, swt);
        __syncwarp();
        tc::mbar_arrive(bar_dr);   // every lane: its own reads of the staging precede it
      }
  } else {   // ---- compute warps
    const int gt = threadIdx.x, w = gt >> 5, wq = w & 3, cg = w >> 2, lane = gt & 31, hf = lane >> 4;
    const int rt = 16 * wq + (lane & 15), u0 = 32 * cg + UPT * hf, o0 = OPT * (2 * cg + hf);
    const bool lead = cg == 0 && hf == 0;
    float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + cg * 64 * NPL;
    const uint32_t tZ1 = *tslot, tZ2 = tZ1 + 64, tV = tZ1 + 128;
    const uint32_t tl = (uint32_t)(wq * 32) << 16;
    const uint32_t id64 = tc::idesc_bf16(64, kGsH, 0, 0), id_v = tc::idesc_bf16(64, kGsK, 0, 0);
    const uint32_t w_addr = tc::smem_u32(smem);
    const uint64_t kA = tc::kdesc0(tc::smem_u32(At), kGsKA), kA1 = tc::kdesc0(tc::smem_u32(A1t), kGsH);
    const uint64_t kW0 = tc::kdesc0(w_addr + L::W0, kGsKA), kW1 = tc::kdesc0(w_addr + L::W1, kGsH);
    const uint64_t kW2 = tc::kdesc0(w_addr + L::W2, kGsH);
    const float* prior[3] = {a.prior[0], a.prior[1], a.prior[2]};
    uint32_t phase = 0, dphase = 0;
    bool staged = false;
    const int R = s.S - 1;
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, NC);
    };
    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };
    // one forward-type contraction: D = X Y^T over nks K-steps (3 x 3 pieces, 6 products)
    auto mma6 = [&](uint32_t d, uint64_t x, uint32_t xp, uint64_t y, int nks, uint32_t idesc) {
#pragma unroll
      for (int c = 0; c < 6; ++c)
        for (int ks = 0; ks < nks; ++ks)
          tc::mma_bf16(d, tc::dplus(x, v2pa(c) * xp + ks * 256), tc::dplus(y, v2pb(c) * L::W_PIECE + ks * 256), idesc,
                       (ks | c) != 0);
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 64 + ray_slot<kGsKp>(rt);
      const bool valid = r0 < s.M;
      const int64_t r = valid ? r0 : s.M - 1;
      const RayIn ray = load_ray(s.orig, s.dir, s.tnear, s.tfar, r, R);
      if (lead) {   // the pixel feature v_i: columns [0, 32)
        float v[kGsC];
#pragma unroll
        for (int k4 = 0; k4 < kGsC / 4; ++k4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(s.feat + r * kGsC) + k4);
          v[4 * k4] = t.x, v[4 * k4 + 1] = t.y, v[4 * k4 + 2] = t.z, v[4 * k4 + 3] = t.w;
        }
        store32<3>(At, L::A_PIECE, rt, 0, kGsKA, v);
      }
      if (cg == CG - 1 && hf == 1) write_direnc(At, L::A_PIECE, rt, kGsC + kGsKp, kGsKA, ray.d, a.dir_freqs);
      for (int j = 0; j <= R; ++j) {
        if (hf == 0) {
          double x[3];
          sample_point(ray, j, s.contract, x);
          write_taps<KIND, kGsKp>(taps + rt * NPL, x, s.dims);
          if (!valid) {
#pragma unroll
            for (int p = 0; p < NPL; ++p) taps[rt * NPL + p].x = __int_as_float(-1);
          }
        }
        __syncwarp();
        // h_prior -> columns [32, 64) (byte offset 4 core-matrix columns)
        coop_gather<KIND, kGsKp, kGsKA, 3>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, 16 * wq, lane, nullptr,
                                           nullptr, nullptr, cg * (KC / 2 / CG), (cg + 1) * (KC / 2 / CG));
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma6(tZ1, kA, L::A_PIECE, kW0, kGsKA / 16, id64);
          tc::mma_commit(bar);
        }
        mma_done();
        {
          float z[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + (uint32_t)(32 * cg), z);
          gs2_relu_store<3, UPT>(z, fp + u0, A1t, L::A1_PIECE, rt, u0, kGsH);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma6(tZ2, kA1, L::A1_PIECE, kW1, kGsH / 16, id64);
          tc::mma_commit(bar);
        }
        mma_done();
        {   // a2 over the consumed a1
          float z[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + (uint32_t)(32 * cg), z);
          gs2_relu_store<3, UPT>(z, fp + kGsH + u0, A1t, L::A1_PIECE, rt, u0, kGsH);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma6(tV, kA1, L::A1_PIECE, kW2, kGsH / 16, id_v);
          tc::mma_commit(bar);
        }
        mma_done();
        if (staged) {   // dhs / ptaps still hold the previous step's staging
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        {   // v~ = V~ + b2, this thread's OPT channels -> fp32 staging
          float v[OPT];
          tc::tmem_ld16x2<OPT, OPT>(tV + tl + (uint32_t)(2 * OPT * cg), v);
#pragma unroll
          for (int k4 = 0; k4 < OPT / 4; ++k4) {
            const float* b2 = fp + 2 * kGsH + o0 + 4 * k4;
            *reinterpret_cast<float4*>(dhs + rt * (kGsK + 4) + o0 + 4 * k4) =
                make_float4(v[4 * k4] + b2[0], v[4 * k4 + 1] + b2[1], v[4 * k4 + 2] + b2[2], v[4 * k4 + 3] + b2[3]);
          }
        }
        if (lead) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) ptaps[rt * NPL + p] = taps[rt * NPL + p];
        }
        tc::mbar_arrive(bar_st);
        staged = true;
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, 256);
  }
}

// ================================================================= backward
template <int KIND>
struct Gs2BwdSmem : Gs2Layout {
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  static constexpr int AC = kGsKA + 8;                       // [v | prior | direnc | 1]: ones at 96 (db0)
  static constexpr int HC = kGsH + 8;                        // [a | 1]: ones at 64 (db1, db2)
  static constexpr uint32_t A_PIECE = 64 * AC * 2;
  static constexpr uint32_t H_PIECE = 64 * HC * 2;
  static constexpr uint32_t X_PIECE = 64 * 64 * 2;           // DV [g' | 0], D [delta2, then delta1]
  static constexpr uint32_t A = GRP;
  static constexpr uint32_t A1 = A + 3 * A_PIECE;            // 3 pieces (Z2 reads it)
  static constexpr uint32_t A2 = A1 + 3 * H_PIECE;           // 2 pieces (dW2 only)
  static constexpr uint32_t DV = A2 + 2 * H_PIECE;
  static constexpr uint32_t D = DV + 2 * X_PIECE;
  static constexpr uint32_t DHS = D + 2 * X_PIECE;           // fp32 prior-gradient rows [64][Kp + 4]
  static constexpr uint32_t PTAPS = DHS + 64 * (kGsKp + 4) * 4;
  static constexpr uint32_t TAPS = PTAPS + 64 * NPL * 16;    // [CG][64][NPL]
  static constexpr uint32_t BAR = (TAPS + CG * 64 * NPL * 16 + 127) & ~127u;   // MMA, staged, drained, tmem slot
  static constexpr uint32_t BYTES = BAR + 32;
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

// TMEM: S1 [0, 64) Z1 -> dA1; S2 [64, 128) Z2 -> dA2 -> dA; dW2|db2 [128, 200) (M = 64, rows < 32 real);
// dW1|db1 [200, 272); dW0|db0 [272, 376)
template <int KIND>
__global__ void __launch_bounds__(128 * kGs2CG + 32 * kGs2ScatterWarps, 1) lp_splat_mlp2_bwd_kernel(const SplatMlpArgs a) {
  using L = Gs2BwdSmem<KIND>;
  constexpr int NPL = L::NPL, KC = kGsKp / 4, CG = L::CG, UPT = L::UPT, NC = L::NC, AC = L::AC, HC = L::HC;
  constexpr int SW = kGs2ScatterWarps;
  static_assert(SW == 1 || SW == 2, "scatter warps");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* At = smem + L::A;
  uint8_t* A1t = smem + L::A1;
  uint8_t* A2t = smem + L::A2;
  uint8_t* DVt = smem + L::DV;
  uint8_t* Dt = smem + L::D;
  float* dhs = reinterpret_cast<float*>(smem + L::DHS);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  const float* fp = reinterpret_cast<const float*>(smem + L::FP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* bar_st = bar + 1;
  uint64_t* bar_dr = bar + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 24);
  const SplatArgs& s = a.s;
  const int E = 6 * a.dir_freqs, nin = kGsC + kGsKp + E;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_gs2_weights(smem, a.params, E);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, NC);
    tc::mbar_init(bar_dr, 32 * SW);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 512);
  if (threadIdx.x < 64) {   // ones columns (piece 0, never overwritten): A[:, 96] -> db0, A1/A2[:, 64] -> db1, db2
    *reinterpret_cast<__nv_bfloat16*>(At + tc::cm_off(threadIdx.x, kGsKA, AC)) = __float2bfloat16_rn(1.0f);
    *reinterpret_cast<__nv_bfloat16*>(A1t + tc::cm_off(threadIdx.x, kGsH, HC)) = __float2bfloat16_rn(1.0f);
    *reinterpret_cast<__nv_bfloat16*>(A2t + tc::cm_off(threadIdx.x, kGsH, HC)) = __float2bfloat16_rn(1.0f);
  }
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int64_t ntiles = (s.M + 63) / 64;

  if (threadIdx.x >= NC) {   // ---- scatter warps: the prior-gradient reductions of every staged step
    const int sw = (threadIdx.x - NC) >> 5, sl = threadIdx.x & 31;
    float* sgp[3] = {a.gprior[0], a.gprior[1], a.gprior[2]};
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int q = 0; q < s.S; ++q) {
        tc::mbar_wait(bar_st, ph);
        ph ^= 1;
        for (int rb = sw; rb < 2; rb += SW) coop_scatter<KIND, kGsKp>(sgp, ptaps, s.dims, dhs, rb * 32, sl);
        __syncwarp();
        tc::mbar_arrive(bar_dr);
      }
  } else {   // ---- compute warps
    const int gt = threadIdx.x, w = gt >> 5, wq = w & 3, cg = w >> 2, lane = gt & 31, hf = lane >> 4;
    const int rt = 16 * wq + (lane & 15), u0 = 32 * cg + UPT * hf;
    const bool lead = cg == 0 && hf == 0;
    const bool vthread = u0 < kGsC;   // this thread's dA columns: dL/dv (else the prior gradient)
    float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + cg * 64 * NPL;
    const uint32_t tb = *tslot;
    const uint32_t tS1 = tb, tS2 = tb + 64, tW2 = tb + 128, tW1 = tb + 200, tW0 = tb + 272;
    const uint32_t tl = (uint32_t)(wq * 32) << 16, tc0 = (uint32_t)(32 * cg);
    const uint32_t id64 = tc::idesc_bf16(64, kGsH, 0, 0);      // Z1, Z2
    const uint32_t id_da = tc::idesc_bf16(64, kGsH, 0, 1);     // dA2, dA1, dA (B MN-major)
    const uint32_t id_wh = tc::idesc_bf16(64, HC, 1, 1);       // dW2 | db2, dW1 | db1
    const uint32_t id_w0 = tc::idesc_bf16(64, AC, 1, 1);       // dW0 | db0
    const uint32_t a_addr = tc::smem_u32(At), a1_addr = tc::smem_u32(A1t), a2_addr = tc::smem_u32(A2t);
    const uint32_t dv_addr = tc::smem_u32(DVt), d_addr = tc::smem_u32(Dt), w_addr = tc::smem_u32(smem);
    const uint64_t kA = tc::kdesc0(a_addr, AC), kA1 = tc::kdesc0(a1_addr, HC);
    const uint64_t kDV = tc::kdesc0(dv_addr, 64), kD = tc::kdesc0(d_addr, 64);
    const uint64_t mA = tc::mdesc0(a_addr, AC), mA1 = tc::mdesc0(a1_addr, HC), mA2 = tc::mdesc0(a2_addr, HC);
    const uint64_t mDV = tc::mdesc0(dv_addr, 64), mD = tc::mdesc0(d_addr, 64);
    const uint64_t kW0 = tc::kdesc0(w_addr + L::W0, kGsKA), kW1 = tc::kdesc0(w_addr + L::W1, kGsH);
    const uint64_t mW0 = tc::mdesc0(w_addr + L::W0, kGsKA), mW1 = tc::mdesc0(w_addr + L::W1, kGsH);
    const uint64_t mW2 = tc::mdesc0(w_addr + L::W2, kGsH);
    constexpr uint32_t MSA = 2 * (AC / 8) * 128, MSH = 2 * (HC / 8) * 128, MSX = 2 * (64 / 8) * 128;
    constexpr uint32_t MSW0 = 2 * (kGsKA / 8) * 128, MSWH = 2 * (kGsH / 8) * 128;
    const float* prior[3] = {a.prior[0], a.prior[1], a.prior[2]};
    const float* gout[3] = {s.gout[0], s.gout[1], s.gout[2]};
    const float* wgt[3] = {s.weight[0], s.weight[1], s.weight[2]};
    uint32_t phase = 0, wacc = 0, dphase = 0;
    bool staged = false;
    const int R = s.S - 1;
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, NC);
    };
    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };
    // gradient-type products: D (+)= X Y over nks K-steps, 2 x 2 pieces (3 products)
    auto mma3 = [&](uint32_t d, uint64_t x, uint32_t xp, uint32_t xks, uint64_t y, uint32_t yp, uint32_t yks, int nks,
                    uint32_t idesc, uint32_t acc) {
#pragma unroll
      for (int c = 0; c < 3; ++c)
        for (int ks = 0; ks < nks; ++ks)
          tc::mma_bf16(d, tc::dplus(x, v2qa(c) * xp + ks * xks), tc::dplus(y, v2qb(c) * yp + ks * yks), idesc,
                       acc | (uint32_t)((ks | c) != 0));
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 64 + ray_slot<kGsKp>(rt);
      const bool valid = r0 < s.M;
      const int64_t r = valid ? r0 : s.M - 1;
      const RayIn ray = load_ray(s.orig, s.dir, s.tnear, s.tfar, r, R);
      if (lead) {
        float v[kGsC];
#pragma unroll
        for (int k4 = 0; k4 < kGsC / 4; ++k4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(s.feat + r * kGsC) + k4);
          v[4 * k4] = t.x, v[4 * k4 + 1] = t.y, v[4 * k4 + 2] = t.z, v[4 * k4 + 3] = t.w;
        }
        store32<3>(At, L::A_PIECE, rt, 0, AC, v);
      }
      if (cg == CG - 1 && hf == 1) write_direnc(At, L::A_PIECE, rt, kGsC + kGsKp, AC, ray.d, a.dir_freqs);
      float gv[UPT];   // dL/dv_i columns [u0, u0 + UPT) of this ray (v threads)
#pragma unroll
      for (int k = 0; k < UPT; ++k) gv[k] = 0.0f;
      for (int q = R; q >= 0; --q) {
        if (hf == 0) {
          double x[3];
          sample_point(ray, q, s.contract, x);
          write_taps<KIND, kGsKp>(taps + rt * NPL, x, s.dims);
          if (!valid) {
#pragma unroll
            for (int p = 0; p < NPL; ++p) taps[rt * NPL + p].x = __int_as_float(-1);
          }
        }
        __syncwarp();
        const int it0 = cg * (KC / 2 / CG), it1 = it0 + KC / 2 / CG;
        coop_gather<KIND, kGsKp, AC, 3>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, 16 * wq, lane, nullptr, nullptr,
                                        nullptr, it0, it1);
        coop_gather_gnorm<KIND, kGsK>(gout, wgt, taps, s.dims, DVt, L::X_PIECE, 64, 16 * wq, lane, it0, it1);
        to_tensor_core();
        if (gt == 0) {   // Z1 = A W0^T
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < 6; ++c)
            for (int ks = 0; ks < kGsKA / 16; ++ks)
              tc::mma_bf16(tS1, tc::dplus(kA, v2pa(c) * L::A_PIECE + ks * 256),
                           tc::dplus(kW0, v2pb(c) * L::W_PIECE + ks * 256), id64, (ks | c) != 0);
          tc::mma_commit(bar);
        }
        mma_done();
        uint32_t mask1, mask2;
        {
          float z[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tS1 + tl + tc0, z);
          mask1 = gs2_relu_store<3, UPT>(z, fp + u0, A1t, L::H_PIECE, rt, u0, HC);
        }
        to_tensor_core();
        if (gt == 0) {   // Z2 = A1 W1^T
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < 6; ++c)
            for (int ks = 0; ks < kGsH / 16; ++ks)
              tc::mma_bf16(tS2, tc::dplus(kA1, v2pa(c) * L::H_PIECE + ks * 256),
                           tc::dplus(kW1, v2pb(c) * L::W_PIECE + ks * 256), id64, (ks | c) != 0);
          tc::mma_commit(bar);
        }
        mma_done();
        {
          float z[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tS2 + tl + tc0, z);
          mask2 = gs2_relu_store<2, UPT>(z, fp + kGsH + u0, A2t, L::H_PIECE, rt, u0, HC);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA2 = DV W2  (B = W2 [K][H] viewed MN-major: MN = hidden, K = channels)
          mma3(tS2, kDV, L::X_PIECE, 256, mW2, L::W_PIECE, MSWH, kGsK / 16, id_da, 0);
          // [dW2 | db2] += DV^T [A2 | 1]   (M = 64 over the DV columns: rows >= 32 are zero)
          mma3(tW2, mDV, L::X_PIECE, MSX, mA2, L::H_PIECE, MSH, 4, id_wh, wacc);
          tc::mma_commit(bar);
        }
        mma_done();
        {   // delta2 = ReLU'(z2) dA2 -> D
          float d[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tS2 + tl + tc0, d);
#pragma unroll
          for (int c8 = 0; c8 < UPT / 8; ++c8) {
            float d8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d8[u] = (mask2 >> (8 * c8 + u)) & 1u ? d[8 * c8 + u] : 0.0f;
            tc::store8<2>(Dt, L::X_PIECE, rt, u0 + 8 * c8, 64, d8);
          }
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma3(tS1, kD, L::X_PIECE, 256, mW1, L::W_PIECE, MSWH, kGsH / 16, id_da, 0);   // dA1 = D2 W1
          mma3(tW1, mD, L::X_PIECE, MSX, mA1, L::H_PIECE, MSH, 4, id_wh, wacc);      // [dW1 | db1] += D2^T [A1 | 1]
          tc::mma_commit(bar);
        }
        mma_done();
        {   // delta1 = ReLU'(z1) dA1 -> D (over delta2, consumed)
          float d[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tS1 + tl + tc0, d);
#pragma unroll
          for (int c8 = 0; c8 < UPT / 8; ++c8) {
            float d8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d8[u] = (mask1 >> (8 * c8 + u)) & 1u ? d[8 * c8 + u] : 0.0f;
            tc::store8<2>(Dt, L::X_PIECE, rt, u0 + 8 * c8, 64, d8);
          }
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA = D1 W0 over the v and prior columns (B = W0 [H][KA] MN-major, N = 64)
          mma3(tS2, kD, L::X_PIECE, 256, mW0, L::W_PIECE, MSW0, kGsH / 16, id_da, 0);
          mma3(tW0, mD, L::X_PIECE, MSX, mA, L::A_PIECE, MSA, 4, id_w0, wacc);           // [dW0 | db0] += D1^T [A | 1]
          tc::mma_commit(bar);
        }
        wacc = 1;
        mma_done();
        if (staged) {   // dhs / ptaps still hold the previous step's staging
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        {
          float d[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tS2 + tl + tc0, d);
          if (vthread) {
#pragma unroll
            for (int k = 0; k < UPT; ++k) gv[k] += d[k];
          } else {   // prior-gradient rows -> fp32 staging
#pragma unroll
            for (int k4 = 0; k4 < UPT / 4; ++k4)
              *reinterpret_cast<float4*>(dhs + rt * (kGsKp + 4) + (u0 - kGsC) + 4 * k4) =
                  make_float4(d[4 * k4], d[4 * k4 + 1], d[4 * k4 + 2], d[4 * k4 + 3]);
          }
        }
        if (lead) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) ptaps[rt * NPL + p] = taps[rt * NPL + p];
        }
        tc::mbar_arrive(bar_st);
        staged = true;
      }
      if (vthread && valid) {
#pragma unroll
        for (int k4 = 0; k4 < UPT / 4; ++k4)
          reinterpret_cast<float4*>(s.gfeat + r * kGsC + u0)[k4] =
              make_float4(gv[4 * k4], gv[4 * k4 + 1], gv[4 * k4 + 2], gv[4 * k4 + 3]);
      }
    }

    // ---- flush: M = 64 accumulators, row i in TMEM lane (i/16)*32 + i%16; the CG warps of a
    // lane quarter split the 8-column chunks
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    const int row = 16 * wq + (lane & 15);
    const bool row_ok = had_tiles && lane < 16;
#pragma unroll 1
    for (int c0 = 8 * cg; c0 < AC; c0 += 8 * CG) {   // dW0 | db0: hidden unit `row` against [v | prior | direnc | 1]
      float wv[8];
      tc::tmem_ld<8>(tW0 + tl + (uint32_t)c0, wv);
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = c0 + i;
          if (c < nin) atomicAdd(a.gparams + row * nin + c, wv[i]);
          else if (c == kGsKA) atomicAdd(a.gparams + Gs2Packed::B0(nin) + row, wv[i]);
        }
      }
    }
#pragma unroll 1
    for (int c0 = 8 * cg; c0 < HC; c0 += 8 * CG) {   // dW1 | db1 (hidden unit rows), dW2 | db2 (channel rows < 32)
      float w1[8], w2[8];
      tc::tmem_ld<8>(tW1 + tl + (uint32_t)c0, w1);
      tc::tmem_ld<8>(tW2 + tl + (uint32_t)c0, w2);
      if (row_ok) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int c = c0 + i;
          if (c < kGsH) {
            atomicAdd(a.gparams + Gs2Packed::W1(nin) + row * kGsH + c, w1[i]);
            if (row < kGsK) atomicAdd(a.gparams + Gs2Packed::W2(nin) + row * kGsH + c, w2[i]);
          } else if (c == kGsH) {
            atomicAdd(a.gparams + Gs2Packed::B1(nin) + row, w1[i]);
            if (row < kGsK) atomicAdd(a.gparams + Gs2Packed::B2(nin) + row, w2[i]);
          }
        }
      }
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, 512);
  }
}

}  // namespace lp
