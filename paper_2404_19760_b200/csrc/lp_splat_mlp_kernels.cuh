// lp_splat_mlp_kernels.cuh -- the Splatter with its MLP g_s (Eq. 2):
//   v~_ij = g_s(v_i, h_prior(x_ij), direnc(d_i)),  theta += sum_ij w(x_ij) v~_ij,
//   theta_weight += sum_ij w(x_ij) (the second pass, MLPs off),
// with g_s: [v (32) | h_prior (32) | direnc (6F <= 32)] -> 64 (ReLU) -> 32 on tcgen05
// (reading R30). A group of 128 rays marches like the renderer, two
// threads per ray (256 threads, one group per CTA):
//   forward   gather h_prior (+ splat of step j-1's v~ and weights) | Z = A W0^T |
//             a1 -> A1 | V~ = A1 W1^T | v~ -> fp32 staging (splatted by the next step's gather)
//   backward  gather h_prior (+ scatter of step j+1's prior gradient) | gather
//             g / theta_weight -> DV | Z recompute | a1 -> A1 | dA1 = DV W1,
//             dW1|db1 += DV^T [A1|1] | delta1 -> D1 | dA = D1 W0 (v and prior columns),
//             dW0|db0 += D1^T [A|1] | dv accumulated per ray, dh_prior staged.
// The per-ray columns (v_i, direnc(d_i)) are written into the A tile once per ray.
#pragma once

#include "lp_splat_kernels.cuh"
#include "lp_tc2_kernels.cuh"
#include "lp_tcv_kernels.cuh"

namespace lp {

constexpr int kGsC = 32;                              // pixel feature channels C_in
constexpr int kGsKp = 32;                             // prior grid channels
constexpr int kGsH = 64;                              // g_s hidden width
constexpr int kGsK = 32;                              // target channels (g_s output)
constexpr int kGsKA = kGsC + kGsKp + kDirEP;          // 96 A-tile input columns

struct SplatMlpArgs {
  SplatArgs s;             // geometry, rays, theta / theta_weight (fwd), gout / theta_weight (bwd), gfeat
  const float* prior[3];   // theta^ [..][kGsKp]
  float* gprior[3];        // bwd: accumulated
  const float* params;     // W0 [H][C + Kp + E], b0 [H], W1 [K][H], b1 [K]
  float* gparams;          // bwd: accumulated
  int dir_freqs;
  int n_hidden;            // 1, or 2 (the paper's 3-layer g_s: lp_splat_mlp2_kernels.cuh)
};

struct GsLayout {          // shared by both kernels
  static constexpr int NPL3 = 3;
  static constexpr uint32_t W0_PIECE = kGsH * kGsKA * 2;
  static constexpr uint32_t W1_PIECE = kGsK * kGsH * 2;
  static constexpr uint32_t W0P = 0;
  static constexpr uint32_t W1P = W0P + 3 * W0_PIECE;
  static constexpr uint32_t FP = W1P + 3 * W1_PIECE;          // b0 [H], b1 [K]
  static constexpr uint32_t GRP = (FP + (kGsH + kGsK) * 4 + 127) & ~127u;
};

__device__ __forceinline__ void stage_gs_weights(uint8_t* smem, const float* __restrict__ g, int E) {
  using L = GsLayout;
  const int nin = kGsC + kGsKp + E;
  for (int i = threadIdx.x; i < kGsH * nin + kGsK * kGsH; i += blockDim.x) {
    int r, c, C;
    uint32_t base, piece;
    float v;
    if (i < kGsH * nin) {
      r = i / nin;
      const int cc = i % nin;
      c = cc;                                   // [v | prior | direnc] share the A tile's column order
      C = kGsKA;
      base = L::W0P;
      piece = L::W0_PIECE;
      v = g[i];
    } else {
      const int j = i - kGsH * nin;
      r = j / kGsH, c = j % kGsH;
      C = kGsH;
      base = L::W1P;
      piece = L::W1_PIECE;
      v = g[kGsH * nin + kGsH + j];
    }
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(smem + base + pc * piece + tc::cm_off(r, c, C)) = b;
      v -= __bfloat162float(b);
    }
  }
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  for (int i = threadIdx.x; i < kGsH; i += blockDim.x) fp[i] = g[kGsH * nin + i];
  for (int i = threadIdx.x; i < kGsK; i += blockDim.x) fp[kGsH + i] = g[kGsH * nin + kGsH + kGsK * kGsH + i];
}

// 32 consecutive values of row r into tile columns [c0, c0 + 32) as NP pieces
template <int NP>
__device__ __forceinline__ void store32(uint8_t* t, uint32_t piece, int r, int c0, int C, const float* v) {
#pragma unroll
  for (int c8 = 0; c8 < 4; ++c8) tc::store8<NP>(t, piece, r, c0 + 8 * c8, C, v + 8 * c8);
}

// ================================================================= forward
template <int KIND>
struct GsFwdSmem : GsLayout {
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  static constexpr uint32_t A_PIECE = 128 * kGsKA * 2;
  static constexpr uint32_t A1_PIECE = 128 * kGsH * 2;
  static constexpr uint32_t A = GRP;
  static constexpr uint32_t A1 = A + kTc2Pieces * A_PIECE;      // activation operands: kTc2Pieces bf16 pieces
  static constexpr uint32_t DHS = A1 + kTc2Pieces * A1_PIECE;           // fp32 v~ rows [128][K + 4]
  static constexpr uint32_t PTAPS = DHS + 128 * (kGsK + 4) * 4;
  static constexpr uint32_t TAPS = PTAPS + 128 * NPL * 16;     // [2 halves][128][NPL]
  static constexpr uint32_t BAR = (TAPS + 2 * 128 * NPL * 16 + 127) & ~127u;   // MMA, tmem slot, staged, drained
  static constexpr uint32_t BYTES = BAR + 32;
};

// dedicated warps issue each staged step's splat reductions (v~ and the weight pass),
// as the renderer backward's scatter warps do (lp_tc_kernels.cuh)
#ifndef LP_SPLAT_SW
#define LP_SPLAT_SW 4
#endif
#ifndef LP_SPLAT_SW_VOXEL   // voxel grids (8 corner lines per sample): 2 measured better (s1g 5.62 -> 5.92 M rays/s)
#define LP_SPLAT_SW_VOXEL 2
#endif
template <int KIND>
constexpr int splat_scatter_warps() { return KIND == 1 ? LP_SPLAT_SW_VOXEL : LP_SPLAT_SW; }

template <int KIND>
__global__ void __launch_bounds__(256 + 32 * splat_scatter_warps<KIND>(), 1) lp_splat_mlp_fwd_kernel(const SplatMlpArgs a) {
  using L = GsFwdSmem<KIND>;
  constexpr int NPL = L::NPL, KC = kGsKp / 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* At = smem + L::A;
  uint8_t* A1t = smem + L::A1;
  float* dhs = reinterpret_cast<float*>(smem + L::DHS);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  const float* fp = reinterpret_cast<const float*>(smem + L::FP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8);
  uint64_t* bar_st = reinterpret_cast<uint64_t*>(smem + L::BAR + 16);   // 256 compute threads
  uint64_t* bar_dr = reinterpret_cast<uint64_t*>(smem + L::BAR + 24);   // the scatter warps
  constexpr int SW = splat_scatter_warps<KIND>();
  static_assert(SW == 0 || 4 % SW == 0, "scatter warps");
  const int gt = threadIdx.x, hf = gt >> 7, rt = gt & 127, wq = (gt >> 5) & 3, lane = gt & 31;
  float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + hf * 128 * NPL;
  const SplatArgs& s = a.s;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_gs_weights(smem, a.params, 6 * a.dir_freqs);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, 256);
    tc::mbar_init(bar_dr, SW > 0 ? 32 * SW : 1);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 128);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (SW > 0) {
    if (threadIdx.x >= 256) {   // ---- scatter warps: the splat of every staged step
      const int sw = (threadIdx.x - 256) / 32, sl = threadIdx.x & 31;
      float* sth[3] = {s.theta[0], s.theta[1], s.theta[2]};
      float* swt[3] = {s.weight[0], s.weight[1], s.weight[2]};
      uint32_t ph = 0;
      const int64_t nt = (s.M + 127) / 128;
      for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x)
        for (int j = 0; j < s.S; ++j) {
          tc::mbar_wait(bar_st, ph);
          ph ^= 1;
          for (int rb = sw; rb < 4; rb += SW) coop_scatter<KIND, kGsK>(sth, ptaps, s.dims, dhs, rb * 32, sl, 0, kGsK / 4, swt);
          __syncwarp();
          tc::mbar_arrive(bar_dr);   // every lane: its own reads of the staging precede it
        }
    }
  }
  if (SW == 0 || threadIdx.x < 256) {   // ---- compute warps
    const uint32_t tZ = *tslot, tV = *tslot + 64;
    const uint32_t tq = (uint32_t)(wq * 32) << 16;
    const int it0 = hf * (KC / 2), it1 = it0 + KC / 2;
    const uint32_t a_addr = tc::smem_u32(At), a1_addr = tc::smem_u32(A1t);
    const uint32_t w0_addr = tc::smem_u32(smem + L::W0P), w1_addr = tc::smem_u32(smem + L::W1P);
    const uint32_t id_z = tc::idesc_bf16(128, kGsH, 0, 0), id_v = tc::idesc_bf16(128, kGsK, 0, 0);
    const float* prior[3] = {a.prior[0], a.prior[1], a.prior[2]};
    float* theta[3] = {s.theta[0], s.theta[1], s.theta[2]};
    float* weight[3] = {s.weight[0], s.weight[1], s.weight[2]};
    uint32_t phase = 0, dphase = 0;
    bool pending = false, staged = false;
    const int R = s.S - 1;
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, 256);
    };
    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };

    const int64_t ntiles = (s.M + 127) / 128;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<kGsKp>(rt);
      const bool valid = r0 < s.M;
      const int64_t r = valid ? r0 : s.M - 1;
      const RayIn ray = load_ray(s.orig, s.dir, s.tnear, s.tfar, r, R);
      if (hf == 0) {   // the pixel feature v_i: columns [0, 32)
        float v[kGsC];
#pragma unroll
        for (int k4 = 0; k4 < kGsC / 4; ++k4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(s.feat + r * kGsC) + k4);
          v[4 * k4] = t.x, v[4 * k4 + 1] = t.y, v[4 * k4 + 2] = t.z, v[4 * k4 + 3] = t.w;
        }
        store32<kTc2Pieces>(At, L::A_PIECE, rt, 0, kGsKA, v);
      } else {         // direnc(d_i): columns [64, 96)
        write_direnc(At, L::A_PIECE, rt, kGsC + kGsKp, kGsKA, ray.d, a.dir_freqs);
      }
      for (int j = 0; j <= R; ++j) {
        double x[3];
        sample_point(ray, j, s.contract, x);
        write_taps<KIND, kGsKp>(taps + rt * NPL, x, s.dims);
        if (!valid) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) taps[rt * NPL + p].x = __int_as_float(-1);
        }
        __syncwarp();
        // h_prior -> columns [32, 64) (byte offset 4 core-matrix columns), fused with step j-1's splat
        if (SW == 0 && pending)
          coop_gather<KIND, kGsKp, kGsKA, kTc2Pieces, true>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, wq * 32, lane, theta,
                                                   ptaps, dhs, it0, it1, weight);
        else
          coop_gather<KIND, kGsKp, kGsKA, kTc2Pieces>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, wq * 32, lane, nullptr,
                                             nullptr, nullptr, it0, it1);
        pending = false;
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma_split6(tZ, a_addr, L::A_PIECE, kGsKA, w0_addr, L::W0_PIECE, kGsKA, kGsKA / 16, id_z);
          tc::mma_commit(bar);
        }
        mma_done();
        {   // a1 = relu(z + b0), this half's 32 hidden units
          float z[32];
          tc::tmem_ld<32>(tZ + tq + (uint32_t)(hf * 32), z);
#pragma unroll
          for (int i = 0; i < 32; ++i) z[i] = fmaxf(z[i] + fp[hf * 32 + i], 0.0f);
          store32<kTc2Pieces>(A1t, L::A1_PIECE, rt, hf * 32, kGsH, z);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma_split6(tV, a1_addr, L::A1_PIECE, kGsH, w1_addr, L::W1_PIECE, kGsH, kGsH / 16, id_v);
          tc::mma_commit(bar);
        }
        mma_done();
        if (SW > 0 && staged) {   // dhs / ptaps still hold the previous step's staging
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        {   // v~ = V~ + b1 (this half's 16 channels) -> fp32 staging
          float v[16];
          tc::tmem_ld<16>(tV + tq + (uint32_t)(hf * 16), v);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4)
            *reinterpret_cast<float4*>(dhs + rt * (kGsK + 4) + hf * 16 + 4 * k4) =
                make_float4(v[4 * k4] + fp[kGsH + hf * 16 + 4 * k4], v[4 * k4 + 1] + fp[kGsH + hf * 16 + 4 * k4 + 1],
                            v[4 * k4 + 2] + fp[kGsH + hf * 16 + 4 * k4 + 2], v[4 * k4 + 3] + fp[kGsH + hf * 16 + 4 * k4 + 3]);
        }
        if (hf == 0) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) ptaps[rt * NPL + p] = taps[rt * NPL + p];
        }
        pending = true;
        if constexpr (SW > 0) {
          tc::mbar_arrive(bar_st);
          staged = true;
        }
        tc::fence_before_sync();
        tc::named_bar(1, 256);
      }
    }
    if (SW == 0 && pending) coop_scatter<KIND, kGsK>(theta, ptaps, s.dims, dhs, wq * 32, lane, it0, it1, weight);
  }   // compute warps
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, 128);
  }
}

// ================================================================= backward
// Warp-cooperative gather of g' = grad_out / theta_weight at the samples' corners
// (the renderer's gather with a per-corner 1/theta_weight) into DV columns [0, 32).
template <int KIND, int K>
__device__ __forceinline__ void coop_gather_gnorm(const float* const* gout, const float* const* wgt,
                                                  const float4* taps, const GridDims& g, uint8_t* DV, uint32_t piece,
                                                  int C, int row0, int lane, int it0, int it1) {
  constexpr int KC = K / 4, RPI = 32 / KC, NPL = KIND == 0 ? 3 : 1;
  const int ch = lane % KC, sub = lane / KC;
  for (int it = it0; it < it1; ++it) {
    const int row = row0 + it * RPI + sub;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int p = 0; p < NPL; ++p) {
      const float4 rec = taps[row * NPL + p];
      Corners<KIND, K> c;
      record_corners<KIND, K>(rec, p, g, c);   // weights 0 for an invalid record
      float4 v[Corners<KIND, K>::N];
      float wc[Corners<KIND, K>::N];
#pragma unroll
      for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
        v[cc] = __ldg(reinterpret_cast<const float4*>(gout[p] + c.off[cc]) + ch);
        wc[cc] = __ldg(wgt[p] + c.off[cc] / K);
      }
#pragma unroll
      for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
        const float sc = wc[cc] > 0.0f ? c.w[cc] / wc[cc] : 0.0f;
        acc[0] = fmaf(sc, v[cc].x, acc[0]);
        acc[1] = fmaf(sc, v[cc].y, acc[1]);
        acc[2] = fmaf(sc, v[cc].z, acc[2]);
        acc[3] = fmaf(sc, v[cc].w, acc[3]);
      }
    }
    tc::store4<2>(DV, piece, row, 4 * ch, C, acc);
  }
}

template <int KIND>
struct GsBwdSmem : GsLayout {
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  static constexpr int AC = kGsKA + 8;                          // + ones column (db0)
  static constexpr int A1C = kGsH + 8;                          // + ones column (db1)
  static constexpr uint32_t A_PIECE = 128 * AC * 2;
  static constexpr uint32_t A1_PIECE = 128 * A1C * 2;
  static constexpr uint32_t X_PIECE = 128 * 64 * 2;             // DV, then D1, then dh staging
  static constexpr uint32_t A = GRP;
  static constexpr uint32_t A1 = A + kTc2Pieces * A_PIECE;
  static constexpr uint32_t X = A1 + 2 * A1_PIECE;
  static constexpr uint32_t PTAPS = X + 128 * (kGsKp + 4) * 4;  // inside X, after the fp32 staging
  static constexpr uint32_t TAPS = X + 2 * X_PIECE;
  static constexpr uint32_t BAR = (TAPS + 2 * 128 * NPL * 16 + 127) & ~127u;   // MMA, tmem slot, staged, drained
  static constexpr uint32_t BYTES = BAR + 32;
  static_assert(128 * (kGsKp + 4) * 4 + 128 * NPL * 16 <= 2 * X_PIECE, "staging fits X");
};

// scatter warps of the g_s backward (the prior-gradient reductions); the staging lives in
// X, which the next step's g/theta_weight gather overwrites, so they drain it during the
// next step's taps and prior gather
#ifndef LP_SPLAT_BWD_SW
#define LP_SPLAT_BWD_SW 4
#endif
#ifndef LP_SPLAT_BWD_SW_VOXEL   // voxel grids: 2 (s1g bwd 123.7 -> 118.0 ms)
#define LP_SPLAT_BWD_SW_VOXEL 2
#endif
template <int KIND>
constexpr int splat_bwd_scatter_warps() { return KIND == 1 ? LP_SPLAT_BWD_SW_VOXEL : LP_SPLAT_BWD_SW; }

// TMEM: S0 [0,64) Z -> dA1 -> dA; dW1|db1 [64,136) (M = 64, rows < 32 real); dW0|db0 [136,240)
template <int KIND>
__global__ void __launch_bounds__(256 + 32 * splat_bwd_scatter_warps<KIND>(), 1) lp_splat_mlp_bwd_kernel(const SplatMlpArgs a) {
  using L = GsBwdSmem<KIND>;
  constexpr int NPL = L::NPL, KC = kGsKp / 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* At = smem + L::A;
  uint8_t* A1t = smem + L::A1;
  uint8_t* Xt = smem + L::X;
  float* dhs = reinterpret_cast<float*>(smem + L::X);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  const float* fp = reinterpret_cast<const float*>(smem + L::FP);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8);
  uint64_t* bar_st = reinterpret_cast<uint64_t*>(smem + L::BAR + 16);   // 256 compute threads
  uint64_t* bar_dr = reinterpret_cast<uint64_t*>(smem + L::BAR + 24);   // the scatter warps
  constexpr int SW = splat_bwd_scatter_warps<KIND>();
  static_assert(SW == 0 || 4 % SW == 0, "scatter warps");
  const int gt = threadIdx.x, hf = gt >> 7, rt = gt & 127, wq = (gt >> 5) & 3, lane = gt & 31;
  float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + hf * 128 * NPL;
  const SplatArgs& s = a.s;
  const int E = 6 * a.dir_freqs, nin = kGsC + kGsKp + E;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_gs_weights(smem, a.params, E);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, 256);
    tc::mbar_init(bar_dr, SW > 0 ? 32 * SW : 1);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, 256);
  if (threadIdx.x >= 256) {
  } else if (hf == 0) {
    *reinterpret_cast<__nv_bfloat16*>(At + tc::cm_off(rt, kGsKA, L::AC)) = __float2bfloat16_rn(1.0f);
  } else {
    *reinterpret_cast<__nv_bfloat16*>(A1t + tc::cm_off(rt, kGsH, L::A1C)) = __float2bfloat16_rn(1.0f);
  }
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (SW > 0) {
    if (threadIdx.x >= 256) {   // ---- scatter warps: prior-gradient reductions of every staged step
      const int sw = (threadIdx.x - 256) / 32, sl = threadIdx.x & 31;
      float* sgp[3] = {a.gprior[0], a.gprior[1], a.gprior[2]};
      uint32_t ph = 0;
      const int64_t nt = (s.M + 127) / 128;
      for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x)
        for (int q = 0; q < s.S; ++q) {
          tc::mbar_wait(bar_st, ph);
          ph ^= 1;
          for (int rb = sw; rb < 4; rb += SW) coop_scatter<KIND, kGsKp>(sgp, ptaps, s.dims, dhs, rb * 32, sl);
          __syncwarp();
          tc::mbar_arrive(bar_dr);   // every lane: its own reads of the staging precede it
        }
    }
  }
  if (SW == 0 || threadIdx.x < 256) {   // ---- compute warps
    const uint32_t tS = *tslot, tW1 = *tslot + 64, tW0 = *tslot + 136;
    const uint32_t tq = (uint32_t)(wq * 32) << 16;
    const int it0 = hf * (KC / 2), it1 = it0 + KC / 2;
    const uint32_t a_addr = tc::smem_u32(At), a1_addr = tc::smem_u32(A1t), x_addr = tc::smem_u32(Xt);
    const uint32_t w0_addr = tc::smem_u32(smem + L::W0P), w1_addr = tc::smem_u32(smem + L::W1P);
    const uint32_t id_z = tc::idesc_bf16(128, kGsH, 0, 0);
    const uint32_t id_da1 = tc::idesc_bf16(128, kGsH, 0, 1);
    const uint32_t id_w1 = tc::idesc_bf16(64, L::A1C, 1, 1);
    const uint32_t id_da = tc::idesc_bf16(128, kGsC + kGsKp, 0, 1);
    const uint32_t id_w0 = tc::idesc_bf16(64, L::AC, 1, 1);
    constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
    const float* prior[3] = {a.prior[0], a.prior[1], a.prior[2]};
    float* gprior[3] = {a.gprior[0], a.gprior[1], a.gprior[2]};
    const float* gout[3] = {s.gout[0], s.gout[1], s.gout[2]};
    const float* wgt[3] = {s.weight[0], s.weight[1], s.weight[2]};
    uint32_t phase = 0, wacc1 = 0, wacc0 = 0;
    bool pending = false;
    uint32_t dphase = 0;
    const int R = s.S - 1;
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, 256);
    };
    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };

    const int64_t ntiles = (s.M + 127) / 128;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<kGsKp>(rt);
      const bool valid = r0 < s.M;
      const int64_t r = valid ? r0 : s.M - 1;
      const RayIn ray = load_ray(s.orig, s.dir, s.tnear, s.tfar, r, R);
      if (hf == 0) {
        float v[kGsC];
#pragma unroll
        for (int k4 = 0; k4 < kGsC / 4; ++k4) {
          const float4 t = __ldg(reinterpret_cast<const float4*>(s.feat + r * kGsC) + k4);
          v[4 * k4] = t.x, v[4 * k4 + 1] = t.y, v[4 * k4 + 2] = t.z, v[4 * k4 + 3] = t.w;
        }
        store32<kTc2Pieces>(At, L::A_PIECE, rt, 0, L::AC, v);
      } else {
        write_direnc(At, L::A_PIECE, rt, kGsC + kGsKp, L::AC, ray.d, a.dir_freqs);
      }
      float gv[kGsC];   // dL/dv_i of this ray (half 0)
#pragma unroll
      for (int k = 0; k < kGsC; ++k) gv[k] = 0.0f;
      for (int q = R; q >= 0; --q) {
        double x[3];
        sample_point(ray, q, s.contract, x);
        write_taps<KIND, kGsKp>(taps + rt * NPL, x, s.dims);
        if (!valid) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) taps[rt * NPL + p].x = __int_as_float(-1);
        }
        __syncwarp();
        if (SW == 0 && pending)   // h_prior, fused with the prior-gradient scatter of step q+1
          coop_gather<KIND, kGsKp, L::AC, kTc2Pieces, true>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, wq * 32, lane, gprior,
                                                   ptaps, dhs, it0, it1);
        else
          coop_gather<KIND, kGsKp, L::AC, kTc2Pieces>(prior, taps, s.dims, At + 4 * 128, L::A_PIECE, wq * 32, lane, nullptr,
                                             nullptr, nullptr, it0, it1);
        if (SW > 0 && pending) {   // the scatter warps have read the staging in X before DV overwrites it
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        pending = false;
        tc::named_bar(1, 256);   // the staging in X has been read by every warp before DV overwrites it
        coop_gather_gnorm<KIND, kGsK>(gout, wgt, taps, s.dims, Xt, L::X_PIECE, 64, wq * 32, lane, it0, it1);
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          mma_split6(tS, a_addr, L::A_PIECE, L::AC, w0_addr, L::W0_PIECE, kGsKA, kGsKA / 16, id_z);
          tc::mma_commit(bar);
        }
        mma_done();
        uint32_t mask = 0;
        {
          float z[32];
          tc::tmem_ld<32>(tS + tq + (uint32_t)(hf * 32), z);
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            const float zz = z[i] + fp[hf * 32 + i];
            mask |= (zz > 0.0f ? 1u : 0u) << i;
            z[i] = fmaxf(zz, 0.0f);
          }
          store32<2>(A1t, L::A1_PIECE, rt, hf * 32, L::A1C, z);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA1 = DV W1   (B = W1 [K][H] viewed MN-major: MN = hidden, K = channels)
#pragma unroll
          for (int ks = 0; ks < kGsK / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tS, tc::desc_kmajor(x_addr + QA[c] * L::X_PIECE, 64, ks),
                           tc::desc_mnmajor(w1_addr + QB[c] * L::W1_PIECE, kGsH, ks), id_da1, (ks | c) != 0);
          // dW1 | db1 += DV^T [A1 | 1]   (M = 64: rows >= 32 unused)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW1, tc::desc_mnmajor(x_addr + QA[c] * L::X_PIECE, 64, ks),
                           tc::desc_mnmajor(a1_addr + QB[c] * L::A1_PIECE, L::A1C, ks), id_w1, wacc1);
              wacc1 = 1;
            }
          tc::mma_commit(bar);
        }
        mma_done();
        {   // delta1 = ReLU'(z) dA1 -> D1 (over the consumed DV)
          float d[32];
          tc::tmem_ld<32>(tS + tq + (uint32_t)(hf * 32), d);
#pragma unroll
          for (int i = 0; i < 32; ++i) d[i] = (mask >> i) & 1u ? d[i] : 0.0f;
          store32<2>(Xt, L::X_PIECE, rt, hf * 32, 64, d);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA = D1 W0 over the v and prior columns (B = W0 [H][KA] MN-major, N = 64)
#pragma unroll
          for (int ks = 0; ks < kGsH / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tS, tc::desc_kmajor(x_addr + QA[c] * L::X_PIECE, 64, ks),
                           tc::desc_mnmajor(w0_addr + QB[c] * L::W0_PIECE, kGsKA, ks), id_da, (ks | c) != 0);
          // dW0 | db0 += D1^T [A | 1]
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW0, tc::desc_mnmajor(x_addr + QA[c] * L::X_PIECE, 64, ks),
                           tc::desc_mnmajor(a_addr + QB[c] * L::A_PIECE, L::AC, ks), id_w0, wacc0);
              wacc0 = 1;
            }
          tc::mma_commit(bar);
        }
        mma_done();
        {
          float d[32];
          tc::tmem_ld<32>(tS + tq + (uint32_t)(hf * 32), d);
          if (hf == 0) {        // dL/dv_i += dA[:, 0:32]
#pragma unroll
            for (int k = 0; k < kGsC; ++k) gv[k] += d[k];
          } else {              // prior gradient rows -> fp32 staging (scattered by the next step's gather)
#pragma unroll
            for (int k4 = 0; k4 < kGsKp / 4; ++k4)
              *reinterpret_cast<float4*>(dhs + rt * (kGsKp + 4) + 4 * k4) =
                  make_float4(d[4 * k4], d[4 * k4 + 1], d[4 * k4 + 2], d[4 * k4 + 3]);
          }
        }
        if (hf == 1) {
#pragma unroll
          for (int p = 0; p < NPL; ++p) ptaps[rt * NPL + p] = taps[rt * NPL + p];
        }
        pending = true;
        if constexpr (SW > 0) tc::mbar_arrive(bar_st);
        tc::fence_before_sync();
        tc::named_bar(1, 256);
      }
      if (hf == 0 && valid) {
#pragma unroll
        for (int k4 = 0; k4 < kGsC / 4; ++k4)
          reinterpret_cast<float4*>(s.gfeat + r * kGsC)[k4] =
              make_float4(gv[4 * k4], gv[4 * k4 + 1], gv[4 * k4 + 2], gv[4 * k4 + 3]);
      }
    }
    if (SW == 0 && pending) coop_scatter<KIND, kGsKp>(gprior, ptaps, s.dims, dhs, wq * 32, lane, it0, it1);

    // flush: M = 64 accumulators, row i in TMEM lane (i/16)*32 + i%16
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    const int row = 16 * wq + lane;
    const int oW1 = kGsH * nin + kGsH;
    if (hf == 0) {
      float w[L::AC];
      tc::tmem_ld<L::AC>(tW0 + tq, w);
      if (had_tiles && lane < 16) {
        for (int c = 0; c < nin; ++c) atomicAdd(a.gparams + row * nin + c, w[c]);
        atomicAdd(a.gparams + kGsH * nin + row, w[kGsKA]);   // ones column: db0
      }
    } else {
      float w[L::A1C];
      tc::tmem_ld<L::A1C>(tW1 + tq, w);
      if (had_tiles && lane < 16 && row < kGsK) {
#pragma unroll
        for (int c = 0; c < kGsH; ++c) atomicAdd(a.gparams + oW1 + row * kGsH + c, w[c]);
        atomicAdd(a.gparams + oW1 + kGsK * kGsH + row, w[kGsH]);   // ones column: db1
      }
    }
  }   // compute warps
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, 256);
  }
}

}  // namespace lp
