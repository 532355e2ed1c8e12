// lp_tcv_kernels.cuh -- tensor-core ray march for view-dependent fields
// (SURVEY 8(f) row 1): sigma = g_sigma(h), c = g_v(h, direnc(d)) (
// DESIGN.md reading R29), each network K(+E) -> HID -> 1 (resp. C).
//
// The two first layers run as ONE block-structured contraction on the tensor
// core: the A tile is [h | direnc(d)] (the direction encoding is a per-ray
// constant written into spare columns of the tile once per ray, so it costs no
// per-sample work) and the B operand is W' = [[W_s0, 0], [W_vh, W_ve]] with 2 HID
// output units, Z = [H | E] W'^T. Two threads per ray: thread (half, row) owns
// the g_sigma units (half 0) or the g_v units (half 1) of its ray's sample, so
// each epilogue touches HID units, the same as the one-network kernels.
//   forward   gather H | Z | a, density logit (half 0) / colour logits (half 1), exchange, EA
//   backward  gather H (+ scatter of step q+1) | Z | a, o, heads, Eq. 3, delta -> D' |
//             dH = D' W'_h, dW' += D'^T [H | E | 1] | a -> A' (over D'), dWo^T += A'^T DOUT |
//             dH -> fp32 staging (scattered by the next step's gather)
#pragma once

#include "lp_tc_kernels.cuh"

namespace lp {

constexpr int kDirEP = 32;   // direnc columns in the A tile (E = 6F <= 32)

template <int HID>
struct TcvParams {  // fp32 copies used on CUDA cores
  static constexpr int BS0 = 0;               // [HID] g_sigma hidden bias
  static constexpr int WS1 = HID;             // [HID] g_sigma output weights
  static constexpr int BV0 = 2 * HID;         // [HID] g_v hidden bias
  static constexpr int WV1T = 3 * HID;        // [HID][4] g_v output weights (transposed, col 3 unused)
  static constexpr int BO = 7 * HID;          // [4] = (b_s1, b_v1[0..2])
  static constexpr int N = round4(BO + 4);
};

// Packed parameters (oracle split_nets order): W_s0[HID][K], b_s0, W_s1[1][HID], b_s1,
// W_v0[HID][K+E], b_v0, W_v1[3][HID], b_v1.
template <int K, int HID>
struct VdPacked {
  __host__ __device__ static constexpr int WS0() { return 0; }
  __host__ __device__ static constexpr int BS0() { return HID * K; }
  __host__ __device__ static constexpr int WS1() { return HID * K + HID; }
  __host__ __device__ static constexpr int BS1() { return HID * K + 2 * HID; }
  __host__ __device__ static constexpr int WV0() { return HID * K + 2 * HID + 1; }
  __device__ static int BV0(int E) { return WV0() + HID * (K + E); }
  __device__ static int WV1(int E) { return BV0(E) + HID; }
  __device__ static int BV1(int E) { return WV1(E) + 3 * HID; }
};

template <int KIND, int K, int HID>
struct TcvShape {
  static constexpr int KP = K < 16 ? 16 : K;      // h columns
  static constexpr int KV = KP + kDirEP;          // [h | e] columns = MMA K of Z
  static constexpr int N2 = 2 * HID;              // hidden units of both networks
  static constexpr int MP = N2 < 64 ? 64 : N2;    // D' / A' tile columns (M of the weight-gradient MMAs)
  static constexpr int HCB = KV + 16;             // backward A tile: [h | e | 1 | dout]
  static constexpr int NPL = KIND == 0 ? 3 : 1;
  static constexpr uint32_t W_PIECE = N2 * KV * 2;
  static constexpr uint32_t XF_PIECE = 128 * KV * 2;
  static constexpr uint32_t XB_PIECE = 128 * HCB * 2;
  static constexpr uint32_t D_PIECE = 128 * MP * 2;
  static constexpr uint32_t TAPS = 128 * NPL * 16;
  static constexpr uint32_t WP = 0;
  static constexpr uint32_t FP = WP + 3 * W_PIECE;
  static constexpr uint32_t GRP = (FP + TcvParams<HID>::N * 4 + 127) & ~127u;
  static_assert(N2 <= 128 && HID % 16 == 0, "hidden width");
  static_assert(K % 4 == 0 && K <= 32 && (K / 4) % 2 == 0, "channels");
};

// W' = [[W_s0, 0], [W_vh, W_ve]] as 3 bf16 pieces [2 HID][KV] (K-major), fp32 head params.
template <int K, int HID>
__device__ __forceinline__ void stage_tcv_weights(uint8_t* wp, float* fp, const float* __restrict__ g, int E) {
  using T = TcvShape<0, K, HID>;
  using P = VdPacked<K, HID>;
  using F = TcvParams<HID>;
  const int KE = K + E;
  for (int i = threadIdx.x; i < HID * K + HID * KE; i += blockDim.x) {
    int r, c;
    float v;
    if (i < HID * K) {
      r = i / K, c = i % K;
      v = g[P::WS0() + i];
    } else {
      const int j = i - HID * K;
      const int rr = j / KE, cc = j % KE;
      r = HID + rr;
      c = cc < K ? cc : T::KP + (cc - K);
      v = g[P::WV0() + j];
    }
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(wp + pc * T::W_PIECE + tc::cm_off(r, c, T::KV)) = b;
      v -= __bfloat162float(b);
    }
  }
  for (int i = threadIdx.x; i < HID; i += blockDim.x) {
    fp[F::BS0 + i] = g[P::BS0() + i];
    fp[F::WS1 + i] = g[P::WS1() + i];
    fp[F::BV0 + i] = g[P::BV0(E) + i];
#pragma unroll
    for (int c = 0; c < 3; ++c) fp[F::WV1T + 4 * i + c] = g[P::WV1(E) + c * HID + i];
    fp[F::WV1T + 4 * i + 3] = 0.0f;
  }
  if (threadIdx.x == 0) {
    fp[F::BO + 0] = g[P::BS1()];
#pragma unroll
    for (int c = 0; c < 3; ++c) fp[F::BO + 1 + c] = g[P::BV1(E) + c];
  }
}

// direnc(d) of this thread's ray into columns [KP, KP + E) of row `row` of an A tile
// (3 bf16 pieces): per axis k, per frequency 2^i, (sin(pi 2^i d_k), cos(pi 2^i d_k)).
#ifndef LP_TCV_PIECES
#define LP_TCV_PIECES 3
#endif
// bf16 pieces of the [h | direnc(d)] operand of Z = [H | E] W'^T (the weights keep 3):
// 3 = fp32-class (default); 2 = 16 significant bits, 5 products (experiment, c4v +9%)
constexpr int kTcvPieces = LP_TCV_PIECES;
// unpaired H-tile stores in the cooperative gather for K1tcv / K2tcv (paired: c4v 10.70 -> 9.59 M rays/s)
constexpr bool kTcvPair = false;

__device__ __forceinline__ void write_direnc(uint8_t* tile, uint32_t piece, int row, int col0, int C, const float d[3],
                                             int F) {
  float e[kDirEP];
#pragma unroll
  for (int i = 0; i < kDirEP; ++i) e[i] = 0.0f;
#pragma unroll
  for (int k = 0; k < 3; ++k)
    for (int i = 0; i < F; ++i) {
      double s, c;
      sincospi(ldexp((double)d[k], i), &s, &c);
      e[2 * (k * F + i)] = (float)s;
      e[2 * (k * F + i) + 1] = (float)c;
    }
#pragma unroll
  for (int c8 = 0; c8 < kDirEP / 8; ++c8) tc::store8<kTcvPieces>(tile, piece, row, col0 + 8 * c8, C, e + 8 * c8);
}

// ================================================================= K1tcv forward
template <int KIND, int K, int HID, int G>
struct FwdTcvSmem : TcvShape<KIND, K, HID> {
  using T = TcvShape<KIND, K, HID>;
  static constexpr uint32_t X = 0;                       // [h | e] tile, kTcvPieces pieces
  static constexpr uint32_t TAPS = X + kTcvPieces * T::XF_PIECE;  // [2 halves][128][NPL]
  static constexpr uint32_t XO = TAPS + 2 * T::TAPS;     // [2 halves][128] float4
  static constexpr uint32_t GSIZE = (XO + 2 * 128 * 16 + 127) & ~127u;
  static constexpr uint32_t BAR = T::GRP + G * GSIZE;
  static constexpr uint32_t BYTES = BAR + 8 * G + 16;
  static constexpr uint32_t TCOLS = T::N2 < 32 ? 32 : T::N2;
  static constexpr uint32_t TMEM_COLS = G * TCOLS <= 32 ? 32 : G * TCOLS <= 64 ? 64 : G * TCOLS <= 128 ? 128
                                      : G * TCOLS <= 256 ? 256 : 512;
};

template <int KIND, int K, int HID, int G>
__global__ void __launch_bounds__(256 * G, 1) lp_fwd_tcv_kernel(const KernelArgs a) {
  using L = FwdTcvSmem<KIND, K, HID, G>;
  using F = TcvParams<HID>;
  constexpr int KP = L::KP, KV = L::KV, NPL = L::NPL, KC = K / 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* wp = smem + L::WP;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8 * G);
  const int g = threadIdx.x >> 8, gt = threadIdx.x & 255, hf = gt >> 7, rt = gt & 127;
  const int wq = (gt >> 5) & 3, lane = gt & 31;
  uint8_t* gsm = smem + L::GRP + g * L::GSIZE;
  uint8_t* X = gsm + L::X;
  float4* taps = reinterpret_cast<float4*>(gsm + L::TAPS) + hf * 128 * NPL;
  float4* xo = reinterpret_cast<float4*>(gsm + L::XO);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tcv_weights<K, HID>(wp, fp, a.params, 6 * a.dir_freqs);
  if (threadIdx.x < G) tc::mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tZ = *tslot + (uint32_t)(g * L::TCOLS);
  const uint32_t tl = ((uint32_t)(wq * 32) << 16) + (uint32_t)(hf * HID);
  const int it0 = hf * (KC / 2), it1 = it0 + KC / 2;

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
  const uint32_t idesc = tc::idesc_bf16(128, L::N2, 0, 0);
  const uint32_t x_addr = tc::smem_u32(X), w_addr = tc::smem_u32(wp);
  const float* b0 = fp + (hf == 0 ? F::BS0 : F::BV0);
  uint32_t phase = 0;

  const int64_t ntiles = (a.M + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < ntiles; tile += (int64_t)gridDim.x * G) {
    const int64_t r0 = tile * 128 + ray_slot<K>(rt);
    const bool valid = r0 < a.M;
    const int64_t r = valid ? r0 : a.M - 1;
    const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
    if (hf == 1) write_direnc(X, L::XF_PIECE, rt, KP, KV, ray.d, a.dir_freqs);   // once per ray
    float tau = 0.0f, tau_e = 0.0f, dep = 0.0f;
    float v[kC] = {0.0f, 0.0f, 0.0f};
    for (int j = 0; j <= R; ++j) {
      double x[3];
      sample_point(ray, j, a.contract, x);                                 // F2
      write_taps<KIND, K>(taps + rt * NPL, x, a.dims);                     // F3 (cells)
      __syncwarp();
      coop_gather<KIND, K, KV, kTcvPieces, false, kTcvPair, 1>(planes, taps, a.dims, X, L::XF_PIECE, wq * 32, lane, nullptr, nullptr, nullptr,
                                  it0, it1);                               // F3 (gather)
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1 + g, 256);
      if (gt == 0) {                                                       // F4: Z = [H | E] W'^T
        tc::fence_after_sync();
        constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
        constexpr int NPROD = kTcvPieces == 3 ? 6 : 5;
        uint32_t acc = 0;
#pragma unroll
        for (int ks = 0; ks < KV / 16; ++ks)
#pragma unroll
          for (int c = 0; c < NPROD; ++c) {
            tc::mma_bf16(tZ, tc::desc_kmajor(x_addr + PA[c] * L::XF_PIECE, KV, ks),
                         tc::desc_kmajor(w_addr + PB[c] * L::W_PIECE, KV, ks), idesc, acc);
            acc = 1;
          }
        tc::mma_commit(&bars[g]);
      }
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      tc::fence_after_sync();
      {
        float z[HID];
        tc::tmem_ld<HID>(tZ + tl, z);
        float4 part = make_float4(0.f, 0.f, 0.f, 0.f);
        if (hf == 0) {            // g_sigma: density logit
#pragma unroll
          for (int i = 0; i < HID; ++i) part.x = fmaf(fp[F::WS1 + i], fmaxf(z[i] + b0[i], 0.0f), part.x);
        } else {                  // g_v: colour logits
#pragma unroll
          for (int i = 0; i < HID; ++i) {
            const float av = fmaxf(z[i] + b0[i], 0.0f);
            const float4 w = reinterpret_cast<const float4*>(fp + F::WV1T)[i];
            part.y = fmaf(w.x, av, part.y);
            part.z = fmaf(w.y, av, part.z);
            part.w = fmaf(w.z, av, part.w);
          }
        }
        xo[hf * 128 + rt] = part;
      }
      xo_exchange_barrier(1 + g, 256, 1 + G + 4 * g + wq);
      float o[kOut];
      {
        const float4 p0 = xo[rt], p1 = xo[128 + rt];
        o[0] = fp[F::BO + 0] + p0.x;
        o[1] = fp[F::BO + 1] + p1.y;
        o[2] = fp[F::BO + 2] + p1.z;
        o[3] = fp[F::BO + 3] + p1.w;
      }
      const float ds = (float)ray.delta * softplus_f(o[0]);               // F5
      if (j > 0) {                                                         // F6
        const float w = expf(-(tau + tau_e)) * (-expm1f(-ds));
#pragma unroll
        for (int c = 0; c < kC; ++c) v[c] = fmaf(w, sigmoid_f(o[1 + c]), v[c]);
        dep = fmaf(w, (float)ray_t(ray, j), dep);
      }
      two_sum_add(tau, tau_e, ds);
    }
    if (valid && hf == 0) {                                                // F7
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

// ================================================================= K2tcv backward
template <int KIND, int K, int HID>
struct BwdTcvSmem : TcvShape<KIND, K, HID> {
  using T = TcvShape<KIND, K, HID>;
  static constexpr uint32_t H = T::GRP;                      // [h | e | 1 | dout], 3 pieces
  static constexpr uint32_t D = H + kTcvPieces * T::XB_PIECE;  // D' then A', 2 pieces [128][MP]
  static constexpr uint32_t DHS = D + 2 * T::D_PIECE;        // fp32 dH rows [128][K + 4]
  static constexpr uint32_t PTAPS = DHS + 128 * (K + 4) * 4; // previous step's tap records
  static constexpr uint32_t TAPS = PTAPS + T::TAPS;          // [2 halves][128][NPL]
  static constexpr uint32_t XO = TAPS + 2 * T::TAPS;         // [2 halves][128] float4
  static constexpr uint32_t BAR = (XO + 2 * 128 * 16 + 127) & ~127u;   // MMA, tmem slot, staged, drained
  static constexpr uint32_t BYTES = BAR + 32;
  static constexpr uint32_t TMEM_COLS = 256;
};

// dedicated warps for the grid-gradient reductions of each staged step (as in K2tc)
#ifndef LP_BWDV_SW
#define LP_BWDV_SW 4
#endif
constexpr int kBwdvScatterWarps = LP_BWDV_SW;

// TMEM: Z [0, 2 HID) (then free), dH [128, 128 + KP), dW' [160, 160 + KV + 8), dWo [240, 248)
template <int KIND, int K, int HID>
__global__ void __launch_bounds__(256 + 32 * kBwdvScatterWarps, 1) lp_bwd_tcv_kernel(const KernelArgs a) {
  using L = BwdTcvSmem<KIND, K, HID>;
  using F = TcvParams<HID>;
  using P = VdPacked<K, HID>;
  constexpr int KP = L::KP, KV = L::KV, HCB = L::HCB, MP = L::MP, NPL = L::NPL, KC = K / 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* wp = smem + L::WP;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint8_t* Ht = smem + L::H;
  uint8_t* Dt = smem + L::D;
  float* dhs = reinterpret_cast<float*>(smem + L::DHS);
  float4* ptaps = reinterpret_cast<float4*>(smem + L::PTAPS);
  float4* xo = reinterpret_cast<float4*>(smem + L::XO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8);
  uint64_t* bar_st = reinterpret_cast<uint64_t*>(smem + L::BAR + 16);   // 256 compute threads
  uint64_t* bar_dr = reinterpret_cast<uint64_t*>(smem + L::BAR + 24);   // the scatter warps
  constexpr int SW = kBwdvScatterWarps;
  static_assert(SW == 0 || 4 % SW == 0, "scatter warps");
  const int gt = threadIdx.x, hf = gt >> 7, rt = gt & 127, wq = (gt >> 5) & 3, lane = gt & 31;
  float4* taps = reinterpret_cast<float4*>(smem + L::TAPS) + hf * 128 * NPL;
  const int E = 6 * a.dir_freqs;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tcv_weights<K, HID>(wp, fp, a.params, E);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar_st, 256);
    tc::mbar_init(bar_dr, SW > 0 ? 32 * SW : 1);
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  if (hf == 0) *reinterpret_cast<__nv_bfloat16*>(Ht + tc::cm_off(rt, KV, HCB)) = __float2bfloat16_rn(1.0f);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (SW > 0) {
    if (threadIdx.x >= 256) {   // ---- scatter warps: B6 of every staged step
      const int sw = (threadIdx.x - 256) / 32, sl = threadIdx.x & 31;
      float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
      uint32_t ph = 0;
      const int64_t nt = (a.M + 127) / 128;
      for (int64_t tile = blockIdx.x; tile < nt; tile += gridDim.x)
        for (int q = 0; q < a.S; ++q) {
          tc::mbar_wait(bar_st, ph);
          ph ^= 1;
          for (int rb = sw; rb < 4; rb += SW) coop_scatter<KIND, K>(sgpl, ptaps, a.dims, dhs, rb * 32, sl);
          __syncwarp();
          tc::mbar_arrive(bar_dr);   // every lane: its own reads of the staging precede it
        }
    }
  }
  if (SW == 0 || threadIdx.x < 256) {   // ---- compute warps
    const uint32_t tbase = *tslot;
    const uint32_t tZ = tbase, tDH = tbase + 128, tW = tbase + 160, tWo = tbase + 240;
    const uint32_t tq = (uint32_t)(wq * 32) << 16;
    const int it0 = hf * (KC / 2), it1 = it0 + KC / 2;

    const int R = a.S - 1;
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    float* gplanes[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id_z = tc::idesc_bf16(128, L::N2, 0, 0);
    const uint32_t id_dh = tc::idesc_bf16(128, KP, 0, 1);
    const uint32_t id_w = tc::idesc_bf16(MP, KV + 8, 1, 1);
    const uint32_t id_wo = tc::idesc_bf16(MP, 8, 1, 1);
    const uint32_t h_addr = tc::smem_u32(Ht), d_addr = tc::smem_u32(Dt), w_addr = tc::smem_u32(wp);
    constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
    uint32_t phase = 0, wacc = 0, wacc_o = 0;
    bool pending = false;
    uint32_t dphase = 0;
    bool staged = false;   // a step is staged for the scatter warps
    float dbo[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float* b0 = fp + (hf == 0 ? F::BS0 : F::BV0);

    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };
    auto to_tensor_core = [&]() {
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, 256);
    };

    const int64_t ntiles = (a.M + 127) / 128;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<K>(rt);
      const bool valid = r0 < a.M;
      const int64_t r = valid ? r0 : a.M - 1;
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
      if (hf == 1) write_direnc(Ht, L::XB_PIECE, rt, KP, HCB, ray.d, a.dir_freqs);
      float p[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) p[c] = valid ? __ldg(a.grad_out + 3 * r + c) : 0.0f;
      const float gtau = (valid && a.grad_tau) ? __ldg(a.grad_tau + r) : 0.0f;
      const float gdep = (valid && a.grad_depth) ? __ldg(a.grad_depth + r) : 0.0f;
      const float tauR = __ldg(a.tau + r);
      float pbg = 0.0f;
#pragma unroll
      for (int c = 0; c < kC; ++c) pbg = fmaf(p[c], bg[c], pbg);
      float G_ = expf(-tauR) * pbg;
      float U = 0.0f, Ue = 0.0f;

      for (int q = R; q >= 0; --q) {
        double x[3];
        sample_point(ray, q, a.contract, x);
        write_taps<KIND, K>(taps + rt * NPL, x, a.dims);
        __syncwarp();
        if (SW == 0 && pending)
          coop_gather<KIND, K, HCB, kTcvPieces, true, false, 1>(planes, taps, a.dims, Ht, L::XB_PIECE, wq * 32, lane, gplanes, ptaps, dhs,
                                             it0, it1);
        else
          coop_gather<KIND, K, HCB, kTcvPieces, false, kTcvPair, 1>(planes, taps, a.dims, Ht, L::XB_PIECE, wq * 32, lane, nullptr, nullptr, nullptr,
                                       it0, it1);
        pending = false;
        to_tensor_core();
        if (gt == 0) {                   // Z = [H | E] W'^T
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
          constexpr int NPROD = kTcvPieces == 3 ? 6 : 5;
          uint32_t acc = 0;
#pragma unroll
          for (int ks = 0; ks < KV / 16; ++ks)
#pragma unroll
            for (int c = 0; c < NPROD; ++c) {
              tc::mma_bf16(tZ, tc::desc_kmajor(h_addr + PA[c] * L::XB_PIECE, HCB, ks),
                           tc::desc_kmajor(w_addr + PB[c] * L::W_PIECE, KV, ks), id_z, acc);
              acc = 1;
            }
          tc::mma_commit(bar);
        }
        mma_done();
        float av[HID];                   // this half's activations (g_sigma or g_v units)
        {
          tc::tmem_ld<HID>(tZ + tq + (uint32_t)(hf * HID), av);
          float4 part = make_float4(0.f, 0.f, 0.f, 0.f);
          if (hf == 0) {
#pragma unroll
            for (int i = 0; i < HID; ++i) {
              av[i] = fmaxf(av[i] + b0[i], 0.0f);
              part.x = fmaf(fp[F::WS1 + i], av[i], part.x);
            }
          } else {
#pragma unroll
            for (int i = 0; i < HID; ++i) {
              av[i] = fmaxf(av[i] + b0[i], 0.0f);
              const float4 w = reinterpret_cast<const float4*>(fp + F::WV1T)[i];
              part.y = fmaf(w.x, av[i], part.y);
              part.z = fmaf(w.y, av[i], part.z);
              part.w = fmaf(w.z, av[i], part.w);
            }
          }
          xo[hf * 128 + rt] = part;
        }
        xo_exchange_barrier(1, 256, 2 + wq);
        float o[kOut];
        {
          const float4 p0 = xo[rt], p1 = xo[128 + rt];
          o[0] = fp[F::BO + 0] + p0.x;
          o[1] = fp[F::BO + 1] + p1.y;
          o[2] = fp[F::BO + 2] + p1.z;
          o[3] = fp[F::BO + 3] + p1.w;
        }
        const float s_sig = sigmoid_f(o[0]);
        const float ds = (float)ray.delta * softplus_f(o[0]);
        float col[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) col[c] = sigmoid_f(o[1 + c]);
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
        float dout[8];
        dout[0] = dsig * s_sig;
#pragma unroll
        for (int c = 0; c < kC; ++c) dout[1 + c] = wq_ * p[c] * col[c] * (1.0f - col[c]);
#pragma unroll
        for (int c = 4; c < 8; ++c) dout[c] = 0.0f;
        if (hf == 0) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(Ht, L::XB_PIECE, rt, KV + 8, HCB, dout);
        }
        // delta of this half's units -> D' columns [hf*HID, hf*HID + HID)
#pragma unroll
        for (int c8 = 0; c8 < HID / 8; ++c8) {
          float d8[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int i = 8 * c8 + u;
            float s;
            if (hf == 0) {
              s = fp[F::WS1 + i] * dout[0];
            } else {
              const float4 w = reinterpret_cast<const float4*>(fp + F::WV1T)[i];
              s = w.x * dout[1];
              s = fmaf(w.y, dout[2], s);
              s = fmaf(w.z, dout[3], s);
            }
            d8[u] = av[i] > 0.0f ? s : 0.0f;
          }
          tc::store8<2>(Dt, L::D_PIECE, rt, hf * HID + 8 * c8, MP, d8);
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dH = D' W'_h  (B = W' [2 HID][KV] viewed MN-major over its first KP columns)
#pragma unroll
          for (int ks = 0; ks < L::N2 / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tDH, tc::desc_kmajor(d_addr + QA[c] * L::D_PIECE, MP, ks),
                           tc::desc_mnmajor(w_addr + QB[c] * L::W_PIECE, KV, ks), id_dh, (ks | c) != 0);
          // dW' (+ b0 via the ones column) += D'^T [H | E | 1]
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW, tc::desc_mnmajor(d_addr + QA[c] * L::D_PIECE, MP, ks),
                           tc::desc_mnmajor(h_addr + QB[c] * L::XB_PIECE, HCB, ks), id_w, wacc);
              wacc = 1;
            }
          tc::mma_commit(bar);
        }
        mma_done();
        // activations -> A' over the consumed D' tile; dWo^T += A'^T DOUT (completes in
        // issue order before the next step's Z MMA commit, no wait here)
#pragma unroll
        for (int c8 = 0; c8 < HID / 8; ++c8) tc::store8<2>(Dt, L::D_PIECE, rt, hf * HID + 8 * c8, MP, av + 8 * c8);
        if (SW > 0 && staged) {   // dhs / ptaps still hold the previous step's staging
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
        }
        {
          constexpr int HK = KP / 2;
          float dh[HK];
          tc::tmem_ld<HK>(tDH + tq + (uint32_t)(hf * HK), dh);
#pragma unroll
          for (int k4 = 0; k4 < HK / 4; ++k4)
            if (hf * HK + 4 * k4 < K)
              *reinterpret_cast<float4*>(dhs + rt * (K + 4) + hf * HK + 4 * k4) =
                  make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        if (hf == 0) {
#pragma unroll
          for (int pp = 0; pp < NPL; ++pp) ptaps[rt * NPL + pp] = taps[rt * NPL + pp];
        }
        pending = true;
        if constexpr (SW > 0) {
          tc::mbar_arrive(bar_st);
          staged = true;
        }
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          const uint32_t do_addr = h_addr + (uint32_t)((KV + 8) / 8) * 128u;   // DOUT columns of the H tile
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tWo, tc::desc_mnmajor(d_addr + QA[c] * L::D_PIECE, MP, ks),
                           tc::desc_mnmajor(do_addr + QB[c] * L::XB_PIECE, HCB, ks), id_wo, wacc_o);
              wacc_o = 1;
            }
        }
      }
    }
    if (SW == 0 && pending) coop_scatter<KIND, K>(gplanes, ptaps, a.dims, dhs, wq * 32, lane, it0, it1);
    if (gt == 0) tc::mma_commit(bar);   // drain the last dWo MMAs
    if (blockIdx.x < ntiles) mma_done();

    // ---- flush: M = MP accumulators (row i in TMEM lane i for MP = 128; (i/16)*32 + i%16 for 64)
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    const int row = MP == 128 ? 32 * wq + lane : 16 * wq + lane;
    const bool row_ok = MP == 128 ? true : lane < 16;
    if (hf == 0) {
      float wrow[KV + 8];
      tc::tmem_ld<KV + 8>(tW + tq, wrow);
      if (had_tiles && row_ok && row < 2 * HID) {
        if (row < HID) {   // g_sigma hidden unit
#pragma unroll
          for (int c = 0; c < K; ++c) atomicAdd(a.gparams + P::WS0() + row * K + c, wrow[c]);
          atomicAdd(a.gparams + P::BS0() + row, wrow[KV]);
        } else {           // g_v hidden unit: h columns then direnc columns
          const int u = row - HID;
          for (int c = 0; c < K; ++c) atomicAdd(a.gparams + P::WV0() + u * (K + E) + c, wrow[c]);
          for (int c = 0; c < E; ++c) atomicAdd(a.gparams + P::WV0() + u * (K + E) + K + c, wrow[KP + c]);
          atomicAdd(a.gparams + P::BV0(E) + u, wrow[KV]);
        }
      }
#pragma unroll
      for (int i = 0; i < kOut; ++i) {
        float s = dbo[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        dbo[i] = s;
      }
      if (lane == 0 && had_tiles) {
        atomicAdd(a.gparams + P::BS1(), dbo[0]);
#pragma unroll
        for (int c = 0; c < 3; ++c) atomicAdd(a.gparams + P::BV1(E) + c, dbo[1 + c]);
      }
    } else {
      float orow[8];
      tc::tmem_ld<8>(tWo + tq, orow);
      if (had_tiles && row_ok && row < 2 * HID) {
        if (row < HID) {
          atomicAdd(a.gparams + P::WS1() + row, orow[0]);
        } else {
#pragma unroll
          for (int c = 0; c < 3; ++c) atomicAdd(a.gparams + P::WV1(E) + c * HID + (row - HID), orow[1 + c]);
        }
      }
    }
  }   // compute warps
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

}  // namespace lp
