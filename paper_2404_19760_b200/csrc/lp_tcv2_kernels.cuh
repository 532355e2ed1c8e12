// lp_tcv2_kernels.cuh -- tensor-core ray march for the paper's own renderer field:
// sigma = g_sigma(h) and c = g_v(h, direnc(d)) (reading R29), each network a
// "3-layer MLP with a width of 64": g_sigma K -> 64 -> 64 -> 1, g_v K + E -> 64 -> 64 -> 3.
// K1tcv2 (forward, Eq. 1) and K2tcv2 (backward, Eq. 3 with reverse marching).
//
// Tiles of 64 rays (M = 64 MMAs). Both networks are carried at once: 128 hidden units per
// layer and sample, which at 128 rays per tile would not fit in shared memory next to the
// 84 KB of 3-piece weights. Two threads per ray, in the same warp: thread (half, r) of warp
// q owns ray slot 16q + r and hidden units [32 half, 32 half + 32) of BOTH networks; it
// reads its accumulator columns with the 16x32bx2 TMEM load (lane = ray, column half =
// thread half; scripts/tc_probe4.cu), and the halves add their partial output-layer sums
// with one warp shuffle, so both hold the same per-ray EA state.
// Per step (a group = 4 warps, one elected thread issues every MMA):
//   forward   gather H | Z1 = [H | E] W0'^T | a1 -> A1 (over H) | Z2 = A1 W1'^T | a2, o, heads, EA
//   backward  gather H | Z1 | a1 -> A1 | Z2 | a2, o, heads, Eq. 3, delta2 -> D, dL/do -> A1 |
//             dA1 = D2 W1', dW1 (+ db1) += D2^T [A1 | 1] | delta1 -> D, a2 -> A1 |
//             dH = D1 W0'_h, dW0 (+ db0) += D1^T [H | E | 1], dWo += A2^T DOUT | dH -> fp32
//             staging, reduced into grad theta by 2 scatter warps during the next step
// W0' = [[W_s0, 0], [W_vh, W_ve]] (the direction encoding E is a per-ray constant in spare
// tile columns, written once per ray) and W1' = diag(W_s1, W_v1) (two N = 64 products).
// The weight-gradient contractions run with M = 128 over both networks' units; their
// off-diagonal blocks (sigma units x g_v inputs and vice versa) are discarded at the flush.
// Precision as in lp_tc.cuh: Z1, Z2 on 3 x 3 bf16 pieces (fp32-class), gradient-type
// contractions on 2 pieces.
#pragma once

#include "lp_tcv_kernels.cuh"

namespace lp {

struct Tcv2Params {  // fp32 copies used on CUDA cores (unit index u < 64 within its network)
  static constexpr int BS0 = 0, BV0 = 64, BS1 = 128, BV1 = 192;
  static constexpr int WS2 = 256;        // [64] g_sigma output weights
  static constexpr int WV2T = 320;       // [64][4] g_v output weights transposed (col 3 unused)
  static constexpr int BO = 576;         // [4] = (b_s2, b_v2[0..2])
  static constexpr int N = 580;
};

// Packed parameters (oracle split_nets order): g_sigma W0[64][K] b0 W1[64][64] b1 W2[1][64] b2,
// then g_v W0[64][K+E] b0 W1[64][64] b1 W2[3][64] b2.
template <int K>
struct Vd3Packed {
  __host__ __device__ static constexpr int WS0() { return 0; }
  __host__ __device__ static constexpr int BS0() { return 64 * K; }
  __host__ __device__ static constexpr int WS1() { return 64 * K + 64; }
  __host__ __device__ static constexpr int BS1() { return WS1() + 64 * 64; }
  __host__ __device__ static constexpr int WS2() { return BS1() + 64; }
  __host__ __device__ static constexpr int BS2() { return WS2() + 64; }
  __host__ __device__ static constexpr int WV0() { return BS2() + 1; }
  __device__ static int BV0(int E) { return WV0() + 64 * (K + E); }
  __device__ static int WV1(int E) { return BV0(E) + 64; }
  __device__ static int BV1(int E) { return WV1(E) + 64 * 64; }
  __device__ static int WV2(int E) { return BV1(E) + 64; }
  __device__ static int BV2(int E) { return WV2(E) + 3 * 64; }
};

template <int KIND, int K>
struct Tcv2Shape {
  static_assert(K == 32, "view-dependent 3-layer kernels: K = 32");
  static constexpr int KP = 32, EP = kDirEP, HID = 64, ROWS = 64;
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  // weights, K-major [out][in], 3 bf16 pieces: W_s0 [64][KP], W_v0 [64][KP + EP] (h | direnc
  // columns), W_s1 [64][64], W_v1 [64][64]
  static constexpr uint32_t W0S = 0, W0V = 64 * KP * 2, W1S = W0V + 64 * (KP + EP) * 2, W1V = W1S + 64 * 64 * 2;
  static constexpr uint32_t W_PIECE = W1V + 64 * 64 * 2;
  static constexpr uint32_t FP = 3 * W_PIECE;
  static constexpr uint32_t GRP = (FP + Tcv2Params::N * 4 + 127) & ~127u;
  static constexpr uint32_t TAPS = ROWS * NPL * 16;
};

template <int K>
__device__ __forceinline__ void stage_tcv2_weights(uint8_t* wp, float* fp, const float* __restrict__ g, int E) {
  using T = Tcv2Shape<0, K>;
  using P = Vd3Packed<K>;
  using F = Tcv2Params;
  constexpr int KP = T::KP, KV = T::KP + T::EP;
  const int KE = K + E;
  const int n0 = 64 * K, n1 = n0 + 64 * KE, n2 = n1 + 64 * 64, n3 = n2 + 64 * 64;
  for (int i = threadIdx.x; i < n3; i += blockDim.x) {
    uint32_t off;
    float v;
    if (i < n0) {
      const int r = i / K, c = i % K;
      off = T::W0S + tc::cm_off(r, c, KP);
      v = g[P::WS0() + i];
    } else if (i < n1) {
      const int j = i - n0, r = j / KE, cc = j % KE;
      off = T::W0V + tc::cm_off(r, cc < K ? cc : KP + (cc - K), KV);
      v = g[P::WV0() + j];
    } else if (i < n2) {
      const int j = i - n1;
      off = T::W1S + tc::cm_off(j / 64, j % 64, 64);
      v = g[P::WS1() + j];
    } else {
      const int j = i - n2;
      off = T::W1V + tc::cm_off(j / 64, j % 64, 64);
      v = g[P::WV1(E) + j];
    }
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(wp + pc * T::W_PIECE + off) = b;
      v -= __bfloat162float(b);
    }
  }
  for (int i = threadIdx.x; i < 64; i += blockDim.x) {
    fp[F::BS0 + i] = g[P::BS0() + i];
    fp[F::BV0 + i] = g[P::BV0(E) + i];
    fp[F::BS1 + i] = g[P::BS1() + i];
    fp[F::BV1 + i] = g[P::BV1(E) + i];
    fp[F::WS2 + i] = g[P::WS2() + i];
#pragma unroll
    for (int c = 0; c < 3; ++c) fp[F::WV2T + 4 * i + c] = g[P::WV2(E) + c * 64 + i];
    fp[F::WV2T + 4 * i + 3] = 0.0f;
  }
  if (threadIdx.x == 0) {
    fp[F::BO + 0] = g[P::BS2()];
#pragma unroll
    for (int c = 0; c < 3; ++c) fp[F::BO + 1 + c] = g[P::BV2(E) + c];
  }
}

// piece products of a 3-piece x 3-piece contraction (forward-type, fp32-class) and of a
// 2-piece x 2-piece one (gradient-type)
__host__ __device__ constexpr uint32_t v2pa(int c) { return c == 2 || c == 4 ? 1u : c == 5 ? 2u : 0u; }   // 0 0 1 0 1 2
__host__ __device__ constexpr uint32_t v2pb(int c) { return c == 1 || c == 4 ? 1u : c == 3 ? 2u : 0u; }   // 0 1 0 2 1 0
__host__ __device__ constexpr uint32_t v2qa(int c) { return c == 2 ? 1u : 0u; }                           // 0 0 1
__host__ __device__ constexpr uint32_t v2qb(int c) { return c == 1 ? 1u : 0u; }                           // 0 1 0

// The second-layer epilogue shared by both kernels: a2 = relu(z2 + b1) of this thread's UPT
// units of both networks (from unit u0), and the partial output layer summed over the two
// halves of the warp (shuffle). Leaves a2 in zs (g_sigma units) / zv (g_v units); returns
// the partial (sigma logit, 3 colour logits) without the output bias.
template <int UPT>
__device__ __forceinline__ float4 tcv2_out_partial(const float* fp, int u0, float (&zs)[UPT], float (&zv)[UPT]) {
  using F = Tcv2Params;
  const float* bs1 = fp + F::BS1 + u0;
  const float* bv1 = fp + F::BV1 + u0;
  const float* ws2 = fp + F::WS2 + u0;
  const float4* wv2 = reinterpret_cast<const float4*>(fp + F::WV2T) + u0;
  float s = 0.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f;
#pragma unroll
  for (int i = 0; i < UPT; ++i) {
    zs[i] = fmaxf(zs[i] + bs1[i], 0.0f);
    s = fmaf(ws2[i], zs[i], s);
    zv[i] = fmaxf(zv[i] + bv1[i], 0.0f);
    const float4 w = wv2[i];
    c0 = fmaf(w.x, zv[i], c0);
    c1 = fmaf(w.y, zv[i], c1);
    c2 = fmaf(w.z, zv[i], c2);
  }
  s += __shfl_xor_sync(0xffffffffu, s, 16);
  c0 += __shfl_xor_sync(0xffffffffu, c0, 16);
  c1 += __shfl_xor_sync(0xffffffffu, c1, 16);
  c2 += __shfl_xor_sync(0xffffffffu, c2, 16);
  return make_float4(s, c0, c1, c2);
}

// ================================================================= K1tcv2 forward
// G groups of 64 rays per CTA; each group has CG column groups of 4 warps (2 CG threads per
// ray, UPT = 32 / CG units of each network per thread), as in the backward.
#ifndef LP_FWDV2_CG
#define LP_FWDV2_CG 1
#endif
constexpr int kFwdv2CG = LP_FWDV2_CG;

template <int KIND, int K, int G>
struct FwdTcv2Smem : Tcv2Shape<KIND, K> {
  using T = Tcv2Shape<KIND, K>;
  static constexpr int CG = kFwdv2CG;
  static constexpr uint32_t H_PIECE = T::ROWS * T::KP * 2;   // H tile [64][KP]
  static constexpr uint32_t A_PIECE = T::ROWS * 128 * 2;     // A1 tile [64][128] (over H)
  static constexpr uint32_t E_PIECE = T::ROWS * T::EP * 2;   // direnc tile [64][EP]
  static constexpr uint32_t X = 0;
  static constexpr uint32_t E = X + 3 * A_PIECE;
  static constexpr uint32_t TAPS = E + 3 * E_PIECE;          // [CG][64][NPL]
  static constexpr uint32_t XO = TAPS + CG * T::TAPS;        // [CG][64] float4
  static constexpr uint32_t GSIZE = (XO + CG * 64 * 16 + 127) & ~127u;
  static constexpr uint32_t BAR = T::GRP + G * GSIZE;
  static constexpr uint32_t BYTES = BAR + 8 * G + 16;
  static constexpr uint32_t TMEM_COLS = G * 256 <= 256 ? 256 : 512;
  static_assert(CG == 1 || CG == 2, "column groups");
  static_assert(1 + G + 4 * G <= 16, "named barriers");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int KIND, int K, int G>
__global__ void __launch_bounds__(128 * kFwdv2CG * G, 1) lp_fwd_tcv2_kernel(const KernelArgs a) {
  using L = FwdTcv2Smem<KIND, K, G>;
  using F = Tcv2Params;
  constexpr int KP = L::KP, EP = L::EP, NPL = L::NPL, KC = K / 4, CG = L::CG, UPT = 32 / CG, NG = 128 * CG;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* wp = smem;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8 * G);
  const int g = threadIdx.x / NG, gt = threadIdx.x % NG, w = gt >> 5, wq = w & 3, cg = w >> 2, lane = gt & 31;
  const int hf = lane >> 4, rt = 16 * wq + (lane & 15), u0 = 32 * cg + UPT * hf;
  const bool lead = cg == 0 && hf == 0;
  uint8_t* gsm = smem + L::GRP + g * L::GSIZE;
  uint8_t* X = gsm + L::X;
  uint8_t* Et = gsm + L::E;
  float4* taps = reinterpret_cast<float4*>(gsm + L::TAPS) + cg * 64 * NPL;
  float4* xo = reinterpret_cast<float4*>(gsm + L::XO);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tcv2_weights<K>(wp, fp, a.params, 6 * a.dir_freqs);
  if (threadIdx.x < G) tc::mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tZ1 = *tslot + (uint32_t)(g * 256), tZ2 = tZ1 + 128;
  const uint32_t tl = ((uint32_t)(wq * 32) << 16) + (uint32_t)(32 * cg);

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
  const uint32_t id64 = tc::idesc_bf16(64, 64, 0, 0);
  const uint32_t x_addr = tc::smem_u32(X), e_addr = tc::smem_u32(Et), w_addr = tc::smem_u32(wp);
  const uint64_t kH = tc::kdesc0(x_addr, KP), kE = tc::kdesc0(e_addr, EP), kA = tc::kdesc0(x_addr, 128);
  const uint64_t kW0S = tc::kdesc0(w_addr + L::W0S, KP), kW0V = tc::kdesc0(w_addr + L::W0V, KP + EP);
  const uint64_t kW1S = tc::kdesc0(w_addr + L::W1S, 64), kW1V = tc::kdesc0(w_addr + L::W1V, 64);
  const float* bs0 = fp + F::BS0 + u0;
  const float* bv0 = fp + F::BV0 + u0;
  uint32_t phase = 0;

  const int64_t ntiles = (a.M + 63) / 64;
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < ntiles; tile += (int64_t)gridDim.x * G) {
    const int64_t r0 = tile * 64 + ray_slot<K>(rt);
    const bool valid = r0 < a.M;
    const int64_t r = valid ? r0 : a.M - 1;
    const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
    if (cg == CG - 1 && hf == 1) write_direnc(Et, L::E_PIECE, rt, 0, EP, ray.d, a.dir_freqs);   // once per ray
    float tau = 0.0f, tau_e = 0.0f, dep = 0.0f;
    float v[kC] = {0.0f, 0.0f, 0.0f};
    for (int j = 0; j <= R; ++j) {
      if (hf == 0) {
        double x[3];
        sample_point(ray, j, a.contract, x);                                 // F2
        write_taps<KIND, K>(taps + rt * NPL, x, a.dims);                     // F3 (cells)
      }
      __syncwarp();
      coop_gather<KIND, K, KP, 3>(planes, taps, a.dims, X, L::H_PIECE, 16 * wq, lane, nullptr, nullptr, nullptr,
                                  cg * (KC / 2 / CG), (cg + 1) * (KC / 2 / CG));   // F3 (gather)
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1 + g, NG);
      if (gt == 0) {   // F4: Z1 = [H | E] W0'^T (g_sigma: the h columns only)
        tc::fence_after_sync();
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const uint32_t pa = v2pa(c) * L::H_PIECE, pw = v2pb(c) * L::W_PIECE;
#pragma unroll
          for (int ks = 0; ks < KP / 16; ++ks) {
            tc::mma_bf16(tZ1, tc::dplus(kH, pa + ks * 256), tc::dplus(kW0S, pw + ks * 256), id64, (ks | c) != 0);
            tc::mma_bf16(tZ1 + 64, tc::dplus(kH, pa + ks * 256), tc::dplus(kW0V, pw + ks * 256), id64, (ks | c) != 0);
          }
#pragma unroll
          for (int ks = 0; ks < EP / 16; ++ks)
            tc::mma_bf16(tZ1 + 64, tc::dplus(kE, v2pa(c) * L::E_PIECE + ks * 256),
                         tc::dplus(kW0V, pw + (KP / 16 + ks) * 256), id64, 1);
        }
        tc::mma_commit(&bars[g]);
      }
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      tc::fence_after_sync();
      {   // a1 = relu(z1 + b0) of this thread's units -> A1 tile (over the consumed H tile)
        float zs[UPT], zv[UPT];
        tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl, zs);
        tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + 64, zv);
#pragma unroll
        for (int c8 = 0; c8 < UPT / 8; ++c8) {
          float as[8], av[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            as[u] = fmaxf(zs[8 * c8 + u] + bs0[8 * c8 + u], 0.0f);
            av[u] = fmaxf(zv[8 * c8 + u] + bv0[8 * c8 + u], 0.0f);
          }
          tc::store8<3>(X, L::A_PIECE, rt, u0 + 8 * c8, 128, as);
          tc::store8<3>(X, L::A_PIECE, rt, 64 + u0 + 8 * c8, 128, av);
        }
      }
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1 + g, NG);
      if (gt == 0) {   // Z2 = A1 W1'^T: A1_s W_s1^T | A1_v W_v1^T
        tc::fence_after_sync();
#pragma unroll
        for (int c = 0; c < 6; ++c) {
          const uint32_t pa = v2pa(c) * L::A_PIECE, pw = v2pb(c) * L::W_PIECE;
#pragma unroll
          for (int ks = 0; ks < 4; ++ks) {
            tc::mma_bf16(tZ2, tc::dplus(kA, pa + ks * 256), tc::dplus(kW1S, pw + ks * 256), id64, (ks | c) != 0);
            tc::mma_bf16(tZ2 + 64, tc::dplus(kA, pa + (4 + ks) * 256), tc::dplus(kW1V, pw + ks * 256), id64,
                         (ks | c) != 0);
          }
        }
        tc::mma_commit(&bars[g]);
      }
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      tc::fence_after_sync();
      float o[kOut];
      {
        float zs[UPT], zv[UPT];
        tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl, zs);
        tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + 64, zv);
        float4 part = tcv2_out_partial<UPT>(fp, u0, zs, zv);
        if constexpr (CG == 2) {   // the other warp of the pair holds the other half of the units
          xo[cg * 64 + rt] = part;
          tc::named_bar(1 + G + 4 * g + wq, 64);
          const float4 p0 = xo[rt], p1 = xo[64 + rt];
          part = make_float4(p0.x + p1.x, p0.y + p1.y, p0.z + p1.z, p0.w + p1.w);
        }
        o[0] = fp[F::BO + 0] + part.x;
        o[1] = fp[F::BO + 1] + part.y;
        o[2] = fp[F::BO + 2] + part.z;
        o[3] = fp[F::BO + 3] + part.w;
      }
      const float ds = (float)ray.delta * softplus_f(o[0]);                // F5
      if (j > 0) {                                                         // F6
        const float w_ = expf(-(tau + tau_e)) * (-expm1f(-ds));
#pragma unroll
        for (int c = 0; c < kC; ++c) v[c] = fmaf(w_, sigmoid_f(o[1 + c]), v[c]);
        dep = fmaf(w_, (float)ray_t(ray, j), dep);
      }
      two_sum_add(tau, tau_e, ds);
    }
    if (valid && lead) {                                                   // F7
      const float tauR = tau + tau_e;
      const float TR = expf(-tauR);
#pragma unroll
      for (int c = 0; c < kC; ++c) a.out[3 * r + c] = fmaf(TR, bg[c], v[c]);
      a.tau[r] = tauR;
      if (a.depth) a.depth[r] = dep;
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

// ================================================================= K2tcv2 backward
// CG column groups: 2 CG threads per ray. Warps w and w + 4 (CG = 2) read the same TMEM lanes
// (rows) and split the hidden units: thread (cg, half) of a ray owns units
// [32 cg + half UPT, + UPT), UPT = 32 / CG, of both networks; the four partial output-layer
// sums meet by shuffle (halves) and through shared memory between the warp pair.
#ifndef LP_BWDV2_CG
#define LP_BWDV2_CG 2
#endif
constexpr int kBwdv2CG = LP_BWDV2_CG;

template <int KIND, int K>
struct BwdTcv2Smem : Tcv2Shape<KIND, K> {
  using T = Tcv2Shape<KIND, K>;
  static constexpr int CG = kBwdv2CG;
  static constexpr int XC = T::KP + T::EP + 16;   // [H | E | 1 | 0]: ones column at KP + EP (db0)
  static constexpr int AC = 144;                  // [A1_s | A1_v | 1 | 0 | DOUT | 0]: ones at 128, dL/do at 136
  static constexpr uint32_t X_PIECE = T::ROWS * XC * 2;
  static constexpr uint32_t A_PIECE = T::ROWS * AC * 2;
  static constexpr uint32_t D_PIECE = T::ROWS * 128 * 2;   // [D_s | D_v] (delta2, then delta1)
  static constexpr uint32_t X = T::GRP;
  static constexpr uint32_t A = X + 3 * X_PIECE;
  static constexpr uint32_t D = A + 3 * A_PIECE;
  static constexpr uint32_t DHS = D + 2 * D_PIECE;          // fp32 dH rows [64][K + 4]
  static constexpr uint32_t TAPS = DHS + T::ROWS * (K + 4) * 4;   // [CG][64][NPL] (one copy per column group)
  static constexpr uint32_t PTAPS = TAPS + CG * T::TAPS;
  static constexpr uint32_t XO = PTAPS + T::TAPS;           // [CG][64] float4 partial outputs
  static constexpr uint32_t BAR = (XO + CG * 64 * 16 + 127) & ~127u;   // MMA, staged, drained, tmem slot
  static constexpr uint32_t BYTES = BAR + 40;   // + the split-commit mbarrier at BAR + 32
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(CG == 1 || CG == 2, "column groups");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

#ifndef LP_BWDV2_SW
#define LP_BWDV2_SW 2
#endif
#ifndef LP_TCV2_SPLIT   // commit dA1 / dH ahead of the weight-gradient MMAs of their round
#define LP_TCV2_SPLIT 0
#endif
constexpr int kBwdv2ScatterWarps = LP_BWDV2_SW;

// TMEM: Z1 [0, 128) (then dA1), Z2 [128, 256) (then dH), dW1 [256, 400), dWo [400, 416), dW0 [416, 496)
template <int KIND, int K>
__global__ void __launch_bounds__(128 * kBwdv2CG + 32 * kBwdv2ScatterWarps, 1) lp_bwd_tcv2_kernel(const KernelArgs a) {
  using L = BwdTcv2Smem<KIND, K>;
  using F = Tcv2Params;
  using P = Vd3Packed<K>;
  constexpr int KP = L::KP, EP = L::EP, XC = L::XC, AC = L::AC, NPL = L::NPL, KC = K / 4;
  constexpr int SW = kBwdv2ScatterWarps, CG = L::CG, UPT = 32 / CG, NC = 128 * CG;
  static_assert(SW == 1 || SW == 2, "scatter warps");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* wp = smem;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint8_t* Xt = smem + L::X;
  uint8_t* At = smem + L::A;
  uint8_t* Dt = smem + L::D;
  float* dhs = reinterpret_cast<float*>(smem + L::DHS);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  float4* xo = reinterpret_cast<float4*>(smem + L::XO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* bar_st = bar + 1;   // NC compute threads: dH of the step staged
  uint64_t* bar_dr = bar + 2;   // every lane of the scatter warps: staging read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 24);
  const int E = 6 * a.dir_freqs;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tcv2_weights<K>(wp, fp, a.params, E);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, NC);
    tc::mbar_init(bar_dr, 32 * SW);
    tc::mbar_init(bar + 4, 1);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  if (threadIdx.x < 64) {   // ones columns (piece 0; never overwritten): X[:, KP + EP] -> db0, A1[:, 128] -> db1
    *reinterpret_cast<__nv_bfloat16*>(Xt + tc::cm_off(threadIdx.x, KP + EP, XC)) = __float2bfloat16_rn(1.0f);
    *reinterpret_cast<__nv_bfloat16*>(At + tc::cm_off(threadIdx.x, 128, AC)) = __float2bfloat16_rn(1.0f);
  }
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 63) / 64;

  if (threadIdx.x >= NC) {   // ---- scatter warps: B6 of every staged step
    const int sw = (threadIdx.x - NC) >> 5, sl = threadIdx.x & 31;
    float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    uint32_t ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int q = 0; q < a.S; ++q) {
        tc::mbar_wait(bar_st, ph);
        ph ^= 1;
        for (int rb = sw; rb < 2; rb += SW) coop_scatter<KIND, K>(sgpl, ptaps, a.dims, dhs, rb * 32, sl);
        __syncwarp();
        tc::mbar_arrive(bar_dr);   // every lane: its own reads of the staging precede it
      }
  } else {   // ---- compute warps: 64 rays, 2 CG threads per ray
    const int gt = threadIdx.x, w = gt >> 5, wq = w & 3, cg = w >> 2, lane = gt & 31, hf = lane >> 4;
    const int rt = 16 * wq + (lane & 15), u0 = 32 * cg + UPT * hf;   // ray slot, first owned unit
    const bool lead = cg == 0 && hf == 0;                            // one thread per ray
    float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + cg * 64 * NPL;
    const uint32_t tbase = *tslot;
    const uint32_t tZ1 = tbase, tZ2 = tbase + 128, tW1 = tbase + 256, tWo = tbase + 400, tW0 = tbase + 416;
    const uint32_t tl = (uint32_t)(wq * 32) << 16, tc0 = (uint32_t)(32 * cg);
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id64 = tc::idesc_bf16(64, 64, 0, 0);       // Z1, Z2 (K-major x K-major)
    const uint32_t id_da = tc::idesc_bf16(64, 64, 0, 1);      // dA1 (B MN-major)
    const uint32_t id_dh = tc::idesc_bf16(64, KP, 0, 1);      // dH
    const uint32_t id_w1 = tc::idesc_bf16(128, AC, 1, 1);     // dW1 | db1 (+ discarded columns)
    const uint32_t id_w0 = tc::idesc_bf16(128, XC, 1, 1);     // dW0 | db0
    const uint32_t id_wo = tc::idesc_bf16(128, 16, 1, 1);     // dWo
    const uint32_t x_addr = tc::smem_u32(Xt), a_addr = tc::smem_u32(At), d_addr = tc::smem_u32(Dt);
    const uint32_t w_addr = tc::smem_u32(wp);
    const uint64_t kX = tc::kdesc0(x_addr, XC), kA = tc::kdesc0(a_addr, AC), kD = tc::kdesc0(d_addr, 128);
    const uint64_t mX = tc::mdesc0(x_addr, XC), mA = tc::mdesc0(a_addr, AC), mD = tc::mdesc0(d_addr, 128);
    const uint64_t mDO = tc::mdesc0(a_addr + (128 / 8) * 128, AC);   // [1 | 0 | DOUT | 0] columns of the A1 tile
    const uint64_t kW0S = tc::kdesc0(w_addr + L::W0S, KP), kW0V = tc::kdesc0(w_addr + L::W0V, KP + EP);
    const uint64_t kW1S = tc::kdesc0(w_addr + L::W1S, 64), kW1V = tc::kdesc0(w_addr + L::W1V, 64);
    const uint64_t mW0S = tc::mdesc0(w_addr + L::W0S, KP), mW0V = tc::mdesc0(w_addr + L::W0V, KP + EP);
    const uint64_t mW1S = tc::mdesc0(w_addr + L::W1S, 64), mW1V = tc::mdesc0(w_addr + L::W1V, 64);
    // MN-major K-step (16 rows) bytes of each tile
    constexpr uint32_t MSX = 2 * (XC / 8) * 128, MSA = 2 * (AC / 8) * 128, MSD = 2 * (128 / 8) * 128;
    constexpr uint32_t MSW0S = 2 * (KP / 8) * 128, MSW0V = 2 * ((KP + EP) / 8) * 128, MSW1 = 2 * (64 / 8) * 128;
    const float* bs0 = fp + F::BS0 + u0;
    const float* bv0 = fp + F::BV0 + u0;
    const float* bs1 = fp + F::BS1 + u0;
    const float* bv1 = fp + F::BV1 + u0;
    const float* ws2 = fp + F::WS2 + u0;
    const float4* wv2 = reinterpret_cast<const float4*>(fp + F::WV2T) + u0;
    uint32_t phase = 0, phase2 = 0, wacc1 = 0, wacc0 = 0, dphase = 0;
    uint64_t* bar2 = bar + 4;   // the gradient-input half of a split MMA round (LP_TCV2_SPLIT)
    auto grad_inputs_done = [&]() {
      if constexpr (LP_TCV2_SPLIT) {
        tc::mbar_wait(bar2, phase2);
        phase2 ^= 1;
        tc::fence_after_sync();
      } else {
        tc::mbar_wait(bar, phase);
        phase ^= 1;
        tc::fence_after_sync();
      }
    };
    bool staged = false;
    float dbo[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};

    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, NC);
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 64 + ray_slot<K>(rt);
      const bool valid = r0 < a.M;
      const int64_t r = valid ? r0 : a.M - 1;   // tail rows march a real ray with zero upstream
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
      if (cg == CG - 1 && hf == 1) write_direnc(Xt, L::X_PIECE, rt, KP, XC, ray.d, a.dir_freqs);   // once per ray
      float p[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) p[c] = valid ? __ldg(a.grad_out + 3 * r + c) : 0.0f;
      const float gtau = (valid && a.grad_tau) ? __ldg(a.grad_tau + r) : 0.0f;
      const float gdep = (valid && a.grad_depth) ? __ldg(a.grad_depth + r) : 0.0f;
      const float tauR = __ldg(a.tau + r);
      float pbg = 0.0f;
#pragma unroll
      for (int c = 0; c < kC; ++c) pbg = fmaf(p[c], bg[c], pbg);
      float G_ = expf(-tauR) * pbg;      // B1
      float U = 0.0f, Ue = 0.0f;

      for (int q = R; q >= 0; --q) {
        // ---- B2: recompute the sample (taps + cooperative gather; the CG warps of a row
        // block split its iterations, each with its own copy of the taps)
        if (hf == 0) {
          double x[3];
          sample_point(ray, q, a.contract, x);
          write_taps<KIND, K>(taps + rt * NPL, x, a.dims);
        }
        __syncwarp();
        coop_gather<KIND, K, XC, 3>(planes, taps, a.dims, Xt, L::X_PIECE, 16 * wq, lane, nullptr, nullptr, nullptr,
                                    cg * (KC / 2 / CG), (cg + 1) * (KC / 2 / CG));
        to_tensor_core();
        if (gt == 0) {   // Z1 = [H | E] W0'^T
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            const uint32_t pa = v2pa(c) * L::X_PIECE, pw = v2pb(c) * L::W_PIECE;
#pragma unroll
            for (int ks = 0; ks < KP / 16; ++ks)
              tc::mma_bf16(tZ1, tc::dplus(kX, pa + ks * 256), tc::dplus(kW0S, pw + ks * 256), id64, (ks | c) != 0);
#pragma unroll
            for (int ks = 0; ks < (KP + EP) / 16; ++ks)
              tc::mma_bf16(tZ1 + 64, tc::dplus(kX, pa + ks * 256), tc::dplus(kW0V, pw + ks * 256), id64,
                           (ks | c) != 0);
          }
          tc::mma_commit(bar);
        }
        mma_done();
        uint32_t ms1 = 0, mv1 = 0;   // ReLU'(z1) of this thread's units
        {
          float zs[UPT], zv[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + tc0, zs);
          tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + tc0 + 64, zv);
#pragma unroll
          for (int c8 = 0; c8 < UPT / 8; ++c8) {
            float as[8], av[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float a_s = zs[8 * c8 + u] + bs0[8 * c8 + u], a_v = zv[8 * c8 + u] + bv0[8 * c8 + u];
              ms1 |= (a_s > 0.0f ? 1u : 0u) << (8 * c8 + u);
              mv1 |= (a_v > 0.0f ? 1u : 0u) << (8 * c8 + u);
              as[u] = fmaxf(a_s, 0.0f);
              av[u] = fmaxf(a_v, 0.0f);
            }
            tc::store8<3>(At, L::A_PIECE, rt, u0 + 8 * c8, AC, as);
            tc::store8<3>(At, L::A_PIECE, rt, 64 + u0 + 8 * c8, AC, av);
          }
        }
        to_tensor_core();
        if (gt == 0) {   // Z2 = A1 W1'^T
          tc::fence_after_sync();
#pragma unroll
          for (int c = 0; c < 6; ++c) {
            const uint32_t pa = v2pa(c) * L::A_PIECE, pw = v2pb(c) * L::W_PIECE;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              tc::mma_bf16(tZ2, tc::dplus(kA, pa + ks * 256), tc::dplus(kW1S, pw + ks * 256), id64, (ks | c) != 0);
              tc::mma_bf16(tZ2 + 64, tc::dplus(kA, pa + (4 + ks) * 256), tc::dplus(kW1V, pw + ks * 256), id64,
                           (ks | c) != 0);
            }
          }
          tc::mma_commit(bar);
        }
        mma_done();
        float o[kOut];
        uint32_t ms2 = 0, mv2 = 0;   // ReLU'(z2)
        {
          float zs[UPT], zv[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + tc0, zs);
          tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + tc0 + 64, zv);
#pragma unroll
          for (int i = 0; i < UPT; ++i) {
            ms2 |= (zs[i] + bs1[i] > 0.0f ? 1u : 0u) << i;
            mv2 |= (zv[i] + bv1[i] > 0.0f ? 1u : 0u) << i;
          }
          float4 part = tcv2_out_partial<UPT>(fp, u0, zs, zv);
          if constexpr (CG == 2) {   // the other warp of the pair holds the other half of the units
            xo[cg * 64 + rt] = part;
            tc::named_bar(2 + wq, 64);
            const float4 p0 = xo[rt], p1 = xo[64 + rt];
            part = make_float4(p0.x + p1.x, p0.y + p1.y, p0.z + p1.z, p0.w + p1.w);
          }
          o[0] = fp[F::BO + 0] + part.x;
          o[1] = fp[F::BO + 1] + part.y;
          o[2] = fp[F::BO + 2] + part.z;
          o[3] = fp[F::BO + 3] + part.w;
        }
        const float s_sig = sigmoid_f(o[0]);
        const float ds = (float)ray.delta * softplus_f(o[0]);
        float col[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) col[c] = sigmoid_f(o[1 + c]);
        // ---- B3: Eq. 3, log-domain reverse update (R12); every thread of the ray holds the same state
        const float tau_q = (tauR - U) - Ue;
        two_sum_add(U, Ue, ds);
        const float tau_qm1 = (tauR - U) - Ue;
        float aq = 0.0f;
#pragma unroll
        for (int c = 0; c < kC; ++c) aq = fmaf(p[c], col[c], aq);
        aq = fmaf(gdep, (float)ray_t(ray, q), aq);
        const float wq_ = q > 0 ? expf(-tau_qm1) * (-expm1f(-ds)) : 0.0f;
        const float Tq_aq = q > 0 ? expf(-tau_q) * aq : 0.0f;
        const float dsig = (float)ray.delta * (gtau - (G_ - Tq_aq));
        G_ = fmaf(wq_, aq, G_);
        // ---- B4: head VJP
        float dout[8];
        dout[0] = dsig * s_sig;
#pragma unroll
        for (int c = 0; c < kC; ++c) dout[1 + c] = wq_ * p[c] * col[c] * (1.0f - col[c]);
#pragma unroll
        for (int c = 4; c < 8; ++c) dout[c] = 0.0f;
        // ---- B5: delta2 -> D tile, dL/do -> A1 tile columns [136, 144)
        if (lead) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(At, L::A_PIECE, rt, 136, AC, dout);
        }
#pragma unroll
        for (int c8 = 0; c8 < UPT / 8; ++c8) {
          float ds8[8], dv8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = 8 * c8 + u;
            const float4 w4 = wv2[i];
            float sv = w4.x * dout[1];
            sv = fmaf(w4.y, dout[2], sv);
            sv = fmaf(w4.z, dout[3], sv);
            ds8[u] = (ms2 >> i) & 1u ? ws2[i] * dout[0] : 0.0f;
            dv8[u] = (mv2 >> i) & 1u ? sv : 0.0f;
          }
          tc::store8<2>(Dt, L::D_PIECE, rt, u0 + 8 * c8, 128, ds8);
          tc::store8<2>(Dt, L::D_PIECE, rt, 64 + u0 + 8 * c8, 128, dv8);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA1 = D2 W1'  (B = W1 [out][in] viewed MN-major: MN = in, K = out)
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const uint32_t pa = v2qa(c) * L::D_PIECE, pw = v2qb(c) * L::W_PIECE;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              tc::mma_bf16(tZ1, tc::dplus(kD, pa + ks * 256), tc::dplus(mW1S, pw + ks * MSW1), id_da, (ks | c) != 0);
              tc::mma_bf16(tZ1 + 64, tc::dplus(kD, pa + (4 + ks) * 256), tc::dplus(mW1V, pw + ks * MSW1), id_da,
                           (ks | c) != 0);
            }
          }
          if constexpr (LP_TCV2_SPLIT) tc::mma_commit(bar2);   // dA1 complete
          // [dW1 | db1 | .] += D2^T [A1 | 1 | DOUT]  (M = 128 units, K = the 64 samples of this step)
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              tc::mma_bf16(tW1, tc::dplus(mD, v2qa(c) * L::D_PIECE + ks * MSD),
                           tc::dplus(mA, v2qb(c) * L::A_PIECE + ks * MSA), id_w1, wacc1);
              wacc1 = 1;
            }
          tc::mma_commit(bar);
        }
        grad_inputs_done();
        {   // delta1 = ReLU'(z1) dA1 -> D (over delta2, consumed); a2 -> A1 columns [0, 128) (consumed)
          float da_s[UPT], da_v[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + tc0, da_s);
          tc::tmem_ld16x2<UPT, UPT>(tZ1 + tl + tc0 + 64, da_v);
          if constexpr (LP_TCV2_SPLIT) mma_done();   // dW1 has read D2 and A1
#pragma unroll
          for (int c8 = 0; c8 < UPT / 8; ++c8) {
            float ds8[8], dv8[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = 8 * c8 + u;
              ds8[u] = (ms1 >> i) & 1u ? da_s[i] : 0.0f;
              dv8[u] = (mv1 >> i) & 1u ? da_v[i] : 0.0f;
            }
            tc::store8<2>(Dt, L::D_PIECE, rt, u0 + 8 * c8, 128, ds8);
            tc::store8<2>(Dt, L::D_PIECE, rt, 64 + u0 + 8 * c8, 128, dv8);
          }
          float zs[UPT], zv[UPT];
          tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + tc0, zs);
          tc::tmem_ld16x2<UPT, UPT>(tZ2 + tl + tc0 + 64, zv);
#pragma unroll
          for (int c8 = 0; c8 < UPT / 8; ++c8) {
            float as[8], av[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              as[u] = fmaxf(zs[8 * c8 + u] + bs1[8 * c8 + u], 0.0f);
              av[u] = fmaxf(zv[8 * c8 + u] + bv1[8 * c8 + u], 0.0f);
            }
            tc::store8<2>(At, L::A_PIECE, rt, u0 + 8 * c8, AC, as);
            tc::store8<2>(At, L::A_PIECE, rt, 64 + u0 + 8 * c8, AC, av);
          }
        }
        to_tensor_core();   // (its tcgen05 fence orders the Z2 reads above before the dH MMA into those columns)
        if (gt == 0) {
          tc::fence_after_sync();
          // dH = D1_s W_s0 + D1_v W_v0[:, h columns]
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            const uint32_t pa = v2qa(c) * L::D_PIECE, pw = v2qb(c) * L::W_PIECE;
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_bf16(tZ2, tc::dplus(kD, pa + ks * 256), tc::dplus(mW0S, pw + ks * MSW0S), id_dh, (ks | c) != 0);
#pragma unroll
            for (int ks = 0; ks < 4; ++ks)
              tc::mma_bf16(tZ2, tc::dplus(kD, pa + (4 + ks) * 256), tc::dplus(mW0V, pw + ks * MSW0V), id_dh, 1);
          }
          if constexpr (LP_TCV2_SPLIT) tc::mma_commit(bar2);   // dH complete
          // [dW0 | db0] += D1^T [H | E | 1 | 0];  dWo^T += A2^T [1 | 0 | DOUT | 0]
#pragma unroll
          for (int c = 0; c < 3; ++c)
#pragma unroll
            for (int ks = 0; ks < 4; ++ks) {
              const uint32_t qa = v2qa(c), qb = v2qb(c);
              tc::mma_bf16(tW0, tc::dplus(mD, qa * L::D_PIECE + ks * MSD), tc::dplus(mX, qb * L::X_PIECE + ks * MSX),
                           id_w0, wacc0);
              tc::mma_bf16(tWo, tc::dplus(mA, qa * L::A_PIECE + ks * MSA), tc::dplus(mDO, qb * L::A_PIECE + ks * MSA),
                           id_wo, wacc0);
              wacc0 = 1;
            }
          tc::mma_commit(bar);
        }
        grad_inputs_done();
        // ---- B6: dH rows -> fp32 staging for the scatter warps
        if (staged) {   // the staging still holds the previous step
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        {
          constexpr int DHC = 32 / (2 * CG);   // channels of dH per thread
          float dh[DHC];
          tc::tmem_ld16x2<DHC, DHC>(tZ2 + tl + (uint32_t)(2 * DHC * cg), dh);
          if constexpr (LP_TCV2_SPLIT) mma_done();   // dW0 and dWo have read D1, X and A2 (the next step's writes)
#pragma unroll
          for (int k4 = 0; k4 < DHC / 4; ++k4)
            *reinterpret_cast<float4*>(dhs + rt * (K + 4) + 2 * DHC * cg + DHC * hf + 4 * k4) =
                make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        if (lead) {
#pragma unroll
          for (int pp = 0; pp < NPL; ++pp) ptaps[rt * NPL + pp] = taps[rt * NPL + pp];
        }
        tc::mbar_arrive(bar_st);
        staged = true;
      }
    }

    // ---- B7: flush the weight-gradient accumulators (M = 128: row u = TMEM lane u; the CG warps of
    // a lane quarter split the columns) and the bias sums
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    const int u = 32 * wq + lane;          // hidden unit: g_sigma u < 64, g_v u - 64
    const bool sig = u < 64;
    const int uu = sig ? u : u - 64;
    const int KE = K + E;
#pragma unroll 1
    for (int c0 = 16 * cg; c0 < AC; c0 += 16 * CG) {   // dW1, db1 (row u against A1 columns)
      float wv[16];
      tc::tmem_ld<16>(tW1 + tl + (uint32_t)c0, wv);
      if (!had_tiles) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = c0 + i;
        if (c < 128) {
          if (sig && c < 64) atomicAdd(a.gparams + P::WS1() + uu * 64 + c, wv[i]);
          if (!sig && c >= 64) atomicAdd(a.gparams + P::WV1(E) + uu * 64 + (c - 64), wv[i]);
        } else if (c == 128) {
          atomicAdd(a.gparams + (sig ? P::BS1() : P::BV1(E)) + uu, wv[i]);
        }
      }
    }
#pragma unroll 1
    for (int c0 = 16 * cg; c0 < XC; c0 += 16 * CG) {   // dW0, db0 (row u against [H | E | 1])
      float wv[16];
      tc::tmem_ld<16>(tW0 + tl + (uint32_t)c0, wv);
      if (!had_tiles) continue;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int c = c0 + i;
        if (c < K) {
          atomicAdd(a.gparams + (sig ? P::WS0() + uu * K : P::WV0() + uu * KE) + c, wv[i]);
        } else if (c >= KP && c < KP + E) {
          if (!sig) atomicAdd(a.gparams + P::WV0() + uu * KE + K + (c - KP), wv[i]);
        } else if (c == KP + EP) {
          atomicAdd(a.gparams + (sig ? P::BS0() : P::BV0(E)) + uu, wv[i]);
        }
      }
    }
    if (cg == 0) {   // dWo (row u against the DOUT columns 8..11 of [1 | 0 | DOUT | 0])
      float wv[16];
      tc::tmem_ld<16>(tWo + tl, wv);
      if (had_tiles) {
        if (sig) {
          atomicAdd(a.gparams + P::WS2() + uu, wv[8]);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) atomicAdd(a.gparams + P::WV2(E) + c * 64 + uu, wv[9 + c]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < kOut; ++i) {
      float sum = dbo[i];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, off);
      dbo[i] = sum;
    }
    if (lane == 0 && cg == 0 && had_tiles) {
      atomicAdd(a.gparams + P::BS2(), dbo[0]);
#pragma unroll
      for (int c = 0; c < 3; ++c) atomicAdd(a.gparams + P::BV2(E) + c, dbo[1 + c]);
    }
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

}  // namespace lp
