// lp_tc2_kernels.cuh -- tensor-core (tcgen05) ray march for two-hidden-layer MLPs
// (the paper's own field MLP: 3 linear layers of width 64): K1tc2 (forward,
// Eq. 1) and K2tc2 (backward, Eq. 3).
//
// Same tile scheme as lp_tc_kernels.cuh (a group owns 128 rays, marched step by
// step; the cooperative gather fills a bf16-piece H tile; one elected thread
// issues tcgen05.mma into TMEM), with two threads per ray: the group has 256
// threads, thread (half, row) handles hidden units [half*HID/2, (half+1)*HID/2)
// of its ray's sample in every epilogue, so the per-thread dependency chains are
// half as long and twice as many warps hide the gather/MMA latencies. The two
// halves exchange the 4 partial output-layer sums through shared memory and
// then both hold the (identical) per-ray EA state. Per step:
//   forward   gather H | Z1 = H W0^T | a1 -> A1 tile | Z2 = A1 W1^T | a2, o, heads, EA
//   backward  (producer warps: taps + gather H of the next step) | Z1 | a1 -> A1 | Z2 | a2, o,
//             heads, Eq. 3, [delta2 | a2] -> D tile, dL/do -> A1 tile |
//             dA1 = D2 W1, [dW1 db1 . ; . . dWo^T] += [D2 | A2]^T [A1 | 1 | DO] | delta1 -> D1 |
//             dH = D1 W0, dW0|db0 += D1^T [H|1] | dH -> fp32 staging over the consumed H tile
//             (reduced by the scatter warps during the next step)
// Precision as in lp_tc.cuh: forward-type contractions (Z1, Z2) on 3 bf16 pieces
// with 6 piece products (fp32-class), gradient contractions on 2 pieces with 3
// products.
#pragma once

#include "lp_tc_kernels.cuh"

namespace lp {

template <int HID>
struct Tc2Params {  // fp32 copies used on CUDA cores
  static constexpr int B0 = 0;                // [HID]
  static constexpr int B1 = HID;              // [HID]
  static constexpr int WOT = 2 * HID;         // [HID][4]
  static constexpr int BO = WOT + 4 * HID;    // [4]
  static constexpr int N = round4(BO + 4);
};

template <int KIND, int K, int HID>
struct Tc2Shape : TcShape<KIND, K, HID> {
  using S = TcShape<KIND, K, HID>;
  static constexpr int HH = HID / 2;                           // hidden units per half-thread
  static constexpr int HC1 = HID + 16;                         // A1 tile columns (+ ones, dL/do: bwd)
  static constexpr uint32_t W1_PIECE = HID * HID * 2;
  static constexpr uint32_t W0P = 0;                           // W0 [HID][KP], 3 pieces
  static constexpr uint32_t W1P = W0P + 3 * S::W0_PIECE;       // W1 [HID][HID], 3 pieces
  static constexpr uint32_t FP = W1P + 3 * W1_PIECE;
  static constexpr uint32_t GRP = (FP + Tc2Params<HID>::N * 4 + 127) & ~127u;
  static_assert(HID == 64, "two-hidden-layer tensor-core kernels: hidden width 64");
  static_assert(K / 4 >= 2, "the two halves split the cooperative gather");
};

template <int K, int HID, int KP>
__device__ __forceinline__ void stage_tc2_weights(uint8_t* w0p, uint8_t* w1p, float* fp, const float* __restrict__ g) {
  using P = PackedParams<K, HID, 2>;
  using F = Tc2Params<HID>;
  for (int i = threadIdx.x; i < HID * K + HID * HID; i += blockDim.x) {
    const bool l0 = i < HID * K;
    const int j = l0 ? i : i - HID * K;
    const int C = l0 ? K : HID, CP = l0 ? KP : HID;
    const int r = j / C, c = j % C;
    float v = g[(l0 ? P::W0 : P::W1) + j];
    uint8_t* base = l0 ? w0p : w1p;
    const uint32_t ps = (uint32_t)(HID * CP * 2);
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(base + pc * ps + tc::cm_off(r, c, CP)) = b;
      v -= __bfloat162float(b);
    }
  }
  for (int i = threadIdx.x; i < HID; i += blockDim.x) {
    fp[F::B0 + i] = g[P::B0 + i];
    fp[F::B1 + i] = g[P::B1 + i];
  }
  for (int i = threadIdx.x; i < 4 * HID; i += blockDim.x) {
    const int r = i / HID, c = i % HID;
    fp[F::WOT + c * 4 + r] = g[P::WO + i];
  }
  if (threadIdx.x < 4) fp[F::BO + threadIdx.x] = g[P::BO + threadIdx.x];
}

#ifndef LP_TC2_PIECES
#define LP_TC2_PIECES 3
#endif
// bf16 pieces of the activation operands (h, a1) of the forward-type contractions in
// K1tc2 / K2tc2 (the weights keep 3). 3: fp32-class (default); 2: 16 significant bits,
// 5 products -- c4p +6%, but more ReLU decisions flip against the oracle (experiment).
constexpr int kTc2Pieces = LP_TC2_PIECES;

// piece products of a kTc2Pieces-piece x 3-piece K-major contraction (forward-type):
// 6 for 3 x 3 (fp32-class), 5 for 2 x 3
__device__ __forceinline__ void mma_split6(uint32_t d, uint32_t a, uint32_t a_piece, int CA, uint32_t b,
                                           uint32_t b_piece, int CB, int nks, uint32_t idesc) {
  constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
  constexpr int NPROD = kTc2Pieces == 3 ? 6 : 5;
  uint32_t acc = 0;
  for (int ks = 0; ks < nks; ++ks)
#pragma unroll
    for (int c = 0; c < NPROD; ++c) {
      tc::mma_bf16(d, tc::desc_kmajor(a + PA[c] * a_piece, CA, ks), tc::desc_kmajor(b + PB[c] * b_piece, CB, ks),
                   idesc, acc);
      acc = 1;
    }
}

// ================================================================= K1tc2 forward
#ifndef LP_FWD2_UNROLL   // cooperative-gather iterations in flight in K1tc2
#define LP_FWD2_UNROLL 2
#endif
template <int KIND, int K, int HID, int G>
struct Fwd2Smem : Tc2Shape<KIND, K, HID> {
  using T = Tc2Shape<KIND, K, HID>;
  static constexpr uint32_t A_PIECE = 128 * HID * 2;
  static constexpr uint32_t X = 0;   // H tile (kTc2Pieces x H_PIECE), overlaid by the A1 tile
  static constexpr uint32_t XSZ = kTc2Pieces * (T::H_PIECE > A_PIECE ? T::H_PIECE : A_PIECE);
  static constexpr uint32_t TAPS = X + XSZ;            // [2 halves][128][NPL]
  static constexpr uint32_t XO = TAPS + 2 * T::TAPS;   // [2 halves][128] float4 partial outputs
  static constexpr uint32_t GSIZE = (XO + 2 * 128 * 16 + 127) & ~127u;
  static constexpr uint32_t BAR = T::GRP + G * GSIZE;
  static constexpr uint32_t BYTES = BAR + 8 * G + 16;
  static constexpr uint32_t TMEM_COLS = G * 128 <= 128 ? 128 : G * 128 <= 256 ? 256 : 512;
};

template <int KIND, int K, int HID, int G>
__global__ void __launch_bounds__(256 * G, 1) lp_fwd_tc2_kernel(const KernelArgs a) {
  using L = Fwd2Smem<KIND, K, HID, G>;
  using F = Tc2Params<HID>;
  constexpr int HH = L::HH, KP = L::KP, NPL = L::NPL, KC = K / 4;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  uint8_t* w1p = smem + L::W1P;
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
  stage_tc2_weights<K, HID, KP>(w0p, w1p, fp, a.params);
  if (threadIdx.x < G) tc::mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tZ1 = *tslot + (uint32_t)(g * 128), tZ2 = tZ1 + 64;
  const uint32_t tl = ((uint32_t)(wq * 32) << 16) + (uint32_t)(hf * HH);
  const int it0 = hf * (KC / 2), it1 = hf ? KC : KC / 2;

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
  const uint32_t idesc = tc::idesc_bf16(128, HID, 0, 0);
  const uint32_t x_addr = tc::smem_u32(X), w0_addr = tc::smem_u32(w0p), w1_addr = tc::smem_u32(w1p);
  uint32_t phase = 0;
  const float* b0 = fp + F::B0 + hf * HH;
  const float* b1 = fp + F::B1 + hf * HH;
  const float4* wot = reinterpret_cast<const float4*>(fp + F::WOT) + hf * HH;

  const int64_t ntiles = (a.M + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < ntiles; tile += (int64_t)gridDim.x * G) {
    const int64_t r0 = tile * 128 + ray_slot<K>(rt);
    const bool valid = r0 < a.M;
    const int64_t r = valid ? r0 : a.M - 1;
    const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
    float tau = 0.0f, tau_e = 0.0f;
    float v[kC] = {0.0f, 0.0f, 0.0f};
    float dep = 0.0f;
    for (int j = 0; j <= R; ++j) {
      double x[3];
      sample_point(ray, j, a.contract, x);                                                // F2
      write_taps<KIND, K>(taps + rt * NPL, x, a.dims);                     // F3 (cells)
      __syncwarp();
      coop_gather<KIND, K, KP, kTc2Pieces, false, true, LP_FWD2_UNROLL>(planes, taps, a.dims, X, L::H_PIECE, wq * 32, lane,
                                                                        nullptr, nullptr, nullptr,
                                  it0, it1);                               // F3 (gather)
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1 + g, 256);
      if (gt == 0) {                                                       // F4: Z1 = H W0^T
        tc::fence_after_sync();
        mma_split6(tZ1, x_addr, L::H_PIECE, KP, w0_addr, L::W0_PIECE, KP, KP / 16, idesc);
        tc::mma_commit(&bars[g]);
      }
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      tc::fence_after_sync();
      {                                                                    // a1 = relu(z1 + b0) -> A1 tile
        float z[HH];
        tc::tmem_ld<HH>(tZ1 + tl, z);
#pragma unroll
        for (int c = 0; c < HH / 8; ++c) {
          float a1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) a1[u] = fmaxf(z[8 * c + u] + b0[8 * c + u], 0.0f);
          tc::store8<kTc2Pieces>(X, L::A_PIECE, rt, hf * HH + 8 * c, HID, a1);
        }
      }
      tc::fence_before_sync();
      tc::fence_async_smem();
      tc::named_bar(1 + g, 256);
      if (gt == 0) {                                                       // Z2 = A1 W1^T
        tc::fence_after_sync();
        mma_split6(tZ2, x_addr, L::A_PIECE, HID, w1_addr, L::W1_PIECE, HID, HID / 16, idesc);
        tc::mma_commit(&bars[g]);
      }
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      tc::fence_after_sync();
      {                                                                    // a2, partial output layer
        float z[HH];
        tc::tmem_ld<HH>(tZ2 + tl, z);
        float4 part = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
        for (int i = 0; i < HH; ++i) {
          const float a2 = fmaxf(z[i] + b1[i], 0.0f);
          const float4 w = wot[i];
          part.x = fmaf(w.x, a2, part.x);
          part.y = fmaf(w.y, a2, part.y);
          part.z = fmaf(w.z, a2, part.z);
          part.w = fmaf(w.w, a2, part.w);
        }
        xo[hf * 128 + rt] = part;
      }
      xo_exchange_barrier(1 + g, 256, 1 + G + 4 * g + wq);
      const float4 p0 = xo[rt], p1 = xo[128 + rt];
      float o[kOut];
      o[0] = fp[F::BO + 0] + p0.x + p1.x;
      o[1] = fp[F::BO + 1] + p0.y + p1.y;
      o[2] = fp[F::BO + 2] + p0.z + p1.z;
      o[3] = fp[F::BO + 3] + p0.w + p1.w;
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

// ================================================================= K2tc2 backward
// kBwd2ScatterWarps dedicated warps issue each staged step's grid-gradient reductions.
#ifndef LP_BWD2_SW
#define LP_BWD2_SW 4
#endif
constexpr int kBwd2ScatterWarps = LP_BWD2_SW;

#ifndef LP_PT_ROLES   // phase timers per role of lp_bwd_tc2p_kernel: 1 compute, 2 producers, 4 scatter
#define LP_PT_ROLES 7
#endif
#define LP_PT_ROLE(bit, x) \
  if constexpr ((LP_PT_ROLES & (bit)) != 0) { x; }
#ifndef LP_PHASES
// Without the debug timers the compute role still reads the clock at its phase boundaries and
// accumulates the deltas (kept alive by a store that is never taken). Measured, not derived:
// ptxas schedules the epilogues around these reads better -- c4p backward 509 -> 472 ms, cu
// 196 -> 190 ms; bare clock reads without the arithmetic give 486 ms, compiler-only barriers
// (asm volatile("" ::: "memory")) 508 ms.
#define LP_PTC_DECL unsigned long long lpk_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long lpk_t = clock64();
#define LP_PTC(i) { long long now_ = clock64(); lpk_acc[i] += (unsigned long long)(now_ - lpk_t); lpk_t = now_; }
#define LP_PTC_KEEP_FLUSH if (a.M < 0) for (int i_ = 0; i_ < 8; ++i_) a.tau[i_] = (float)lpk_acc[i_];
#else
#define LP_PTC_DECL
#define LP_PTC(i) LP_PT_ROLE(1, LP_PT(i))
#define LP_PTC_KEEP_FLUSH
#endif
#define LP_PTP(i) LP_PT_ROLE(2, LP_PT(i))
#define LP_PTS(i) LP_PT_ROLE(4, LP_PT(i))
#define LP_PTC_FLUSH(k) LP_PT_ROLE(1, LP_PT_FLUSH(k))
#define LP_PTP_FLUSH(k) LP_PT_ROLE(2, LP_PT_FLUSH(k))
#define LP_PTS_FLUSH(k) LP_PT_ROLE(4, LP_PT_FLUSH(k))

// ================================================================= K2tc2 backward, warp-specialised
// The recompute's taps + cooperative gather (B2/F3) run outside the compute warps' chain:
// four producer warps march one step ahead into a second H tile (double buffer, full/empty mbarriers), so the gather overlaps the compute
// warps' four serial MMA rounds and epilogues (the phase timers of the single-role kernel:
// gather + taps 35% of the compute warps' time, MMA waits 38%, epilogues 26%). The shared
// memory this needs comes from the A1 tile: its third bf16 piece feeds only Z2 = A1 W1^T
// (one of the six piece products), so it lives in tensor memory and that product reads its
// A operand from TMEM (tcgen05.mma [d], [a_tmem], b_desc); the gradient-type dW1 contraction
// reads pieces 0 and 1 from shared memory as before. Warps: 8 compute (2 per ray), 4
// producers (one 32-row block each, all K/4 gather iterations), SW scatter warps.
#ifndef LP_TC2P_UNROLL
#define LP_TC2P_UNROLL 2
#endif
#ifndef LP_TC2P_PAIR   // paired H-tile stores in the producers' gather
#define LP_TC2P_PAIR 1
#endif
#ifndef LP_TC2P_SPLIT   // commit the gradient-input MMAs (dA1, dH) ahead of the weight-gradient ones
#define LP_TC2P_SPLIT 1
#endif
template <int KIND, int K, int HID>
struct Bwd2pSmem : Tc2Shape<KIND, K, HID> {
  using T = Tc2Shape<KIND, K, HID>;
  static constexpr int HCP = T::KP + 8;                       // [H | 1] (ones column at KP -> db0)
  static constexpr uint32_t HP_PIECE = 128 * HCP * 2;
  static constexpr uint32_t A1_PIECE = 128 * T::HC1 * 2;      // [A1 | 1 | DO]
  static constexpr uint32_t DP = 128 * 2 * HID * 2;           // [D2 | A2] piece
  static constexpr uint32_t H = T::GRP;                       // 2 buffers x 3 pieces
  static constexpr uint32_t A1 = H + 2 * 3 * HP_PIECE;        // 2 pieces (piece 2 of the A1 units: TMEM)
  static constexpr uint32_t D = A1 + 2 * A1_PIECE;            // [D2 | A2] x 2, then D1, then fp32 dH
  static constexpr uint32_t TAPS = D + 2 * DP;                // 2 buffers [128][NPL]
  static constexpr uint32_t XO = TAPS + 2 * T::TAPS;          // [2 halves][128] float4
  static constexpr uint32_t BAR = (XO + 2 * 128 * 16 + 127) & ~127u;
  // mbarriers: MMA, staged[2], full[2], empty[2]; then the TMEM slot
  static constexpr uint32_t BYTES = BAR + 8 * 8 + 16;
  static constexpr uint32_t TMEM_COLS = 512;
  static_assert(2 * HP_PIECE >= 128 * (K + 4) * 4, "dH staging fits pieces 0-1 of an H buffer");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int KIND, int K, int HID>
__global__ void __launch_bounds__(256 + 128 + 32 * kBwd2ScatterWarps, 1) lp_bwd_tc2p_kernel(const KernelArgs a) {
  using L = Bwd2pSmem<KIND, K, HID>;
  using F = Tc2Params<HID>;
  using P = PackedParams<K, HID, 2>;
  constexpr int HH = L::HH, KP = L::KP, HCP = L::HCP, HC1 = L::HC1, NPL = L::NPL;
  constexpr int SW = kBwd2ScatterWarps;
  static_assert(SW > 0 && 4 % SW == 0, "scatter warps");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  uint8_t* w1p = smem + L::W1P;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint8_t* A1t = smem + L::A1;
  uint8_t* Dt = smem + L::D;
  float4* xo = reinterpret_cast<float4*>(smem + L::XO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  // Buffer b = step & 1 holds, in turn: the producers' taps and H tile of the step (full[b]),
  // read by Z1 and dW0; then the step's fp32 dH rows, written over H pieces 0-1 once those
  // MMAs are done (staged[b]); the scatter warps reduce them with the step's taps and free
  // the buffer (empty[b]). The compute warps never wait for the scatter: it has the whole
  // next step to drain, and only the producers, two steps later, wait for it.
  uint64_t* staged = bar + 1;    // [2] 256 compute threads: dH of the step staged in H[b]
  uint64_t* full = bar + 3;      // [2] 128 producer threads: H / taps buffer written
  uint64_t* empty = bar + 5;     // [2] every lane of the SW scatter warps: staging + taps read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 64);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tc2_weights<K, HID, KP>(w0p, w1p, fp, a.params);
  uint64_t* bar2 = bar + 7;      // the gradient-input half of a split MMA round (LP_TC2P_SPLIT)
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar2, 1);
    for (int b = 0; b < 2; ++b) {
      tc::mbar_init(&staged[b], 256);
      tc::mbar_init(&full[b], 128);
      tc::mbar_init(&empty[b], 32 * SW);
    }
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  // ones columns (piece 0 only; never overwritten): H[b][:, KP] -> db0, A1[:, HID] -> db1
  if (threadIdx.x < 128) {
    for (int b = 0; b < 2; ++b)
      *reinterpret_cast<__nv_bfloat16*>(smem + L::H + b * 3 * L::HP_PIECE + tc::cm_off(threadIdx.x, KP, HCP)) =
          __float2bfloat16_rn(1.0f);
    *reinterpret_cast<__nv_bfloat16*>(A1t + tc::cm_off(threadIdx.x, HID, HC1)) = __float2bfloat16_rn(1.0f);
  }
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 127) / 128;
  LP_PT_DECL
  LP_PTC_DECL

  if (threadIdx.x >= 384) {   // ---- scatter warps: B6 of every staged step
    const int sw = (threadIdx.x - 384) / 32, sl = threadIdx.x & 31;
    float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    uint32_t n = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int q = 0; q < a.S; ++q, ++n) {
        const int b = n & 1;
        tc::mbar_wait(&staged[b], (n >> 1) & 1);
        LP_PTS(2)
        const float4* staps = reinterpret_cast<const float4*>(smem + L::TAPS + b * L::T::TAPS);
        const float* dhs = reinterpret_cast<const float*>(smem + L::H + b * 3 * L::HP_PIECE);
        for (int rb = sw; rb < 4; rb += SW) coop_scatter<KIND, K>(sgpl, staps, a.dims, dhs, rb * 32, sl);
        __syncwarp();
        tc::mbar_arrive(&empty[b]);   // every lane: its own reads of the staging / taps precede it
        LP_PTS(3)
      }
    LP_PTS_FLUSH(0)
  } else if (threadIdx.x >= 256) {   // ---- producers: taps + cooperative gather, one step ahead
    const int pw = (threadIdx.x - 256) >> 5, lane = threadIdx.x & 31, row = pw * 32 + lane;
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    uint32_t n = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<K>(row);
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r0 < a.M ? r0 : a.M - 1, R);
      for (int q = R; q >= 0; --q, ++n) {
        const int b = n & 1;
        float4* taps = reinterpret_cast<float4*>(smem + L::TAPS + b * L::T::TAPS);
        uint8_t* Hb = smem + L::H + b * 3 * L::HP_PIECE;
        tc::mbar_wait(&empty[b], ((n >> 1) & 1) ^ 1);
        LP_PTP(0)
        {   // the staging of step n - 2 overwrote pieces 0-1: restore this row's columns [KP, KP + 8)
          const uint32_t off = tc::cm_off(row, KP, HCP);
          *reinterpret_cast<uint4*>(Hb + off) = make_uint4(0x3F80u, 0u, 0u, 0u);   // bf16 1.0, then zeros
          *reinterpret_cast<uint4*>(Hb + L::HP_PIECE + off) = make_uint4(0u, 0u, 0u, 0u);
        }
        double x[3];
        sample_point(ray, q, a.contract, x);
        write_taps<KIND, K>(taps + row * NPL, x, a.dims);
        __syncwarp();
        coop_gather<KIND, K, HCP, 3, false, LP_TC2P_PAIR != 0, LP_TC2P_UNROLL>(planes, taps, a.dims, Hb, L::HP_PIECE, pw * 32, lane);
        tc::fence_async_smem();
        tc::mbar_arrive(&full[b]);
        LP_PTP(1)
      }
    }
    LP_PTP_FLUSH(0)
  } else {   // ---- compute warps
    const int gt = threadIdx.x, hf = gt >> 7, rt = gt & 127, wq = (gt >> 5) & 3;
    const uint32_t tbase = *tslot;
    const uint32_t tS0 = tbase, tS1 = tbase + 64, tW1 = tbase + 128, tW0 = tbase + 208, tA2 = tbase + 256;
    const uint32_t tq = (uint32_t)(wq * 32) << 16;
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id_z = tc::idesc_bf16(128, HID, 0, 0);
    const uint32_t id_da1 = tc::idesc_bf16(128, HID, 0, 1);
    const uint32_t id_dh = tc::idesc_bf16(128, KP, 0, 1);
    const uint32_t id_w1 = tc::idesc_bf16(128, HC1, 1, 1);
    const uint32_t id_w0 = tc::idesc_bf16(64, KP + 8, 1, 1);
    const uint32_t h_addr = tc::smem_u32(smem + L::H), a1_addr = tc::smem_u32(A1t), d_addr = tc::smem_u32(Dt);
    const uint32_t w0_addr = tc::smem_u32(w0p), w1_addr = tc::smem_u32(w1p);
    constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
    // base descriptors (the issuing thread adds compile-time piece / K-step offsets)
    const uint64_t kH = tc::kdesc0(h_addr, HCP), kW0 = tc::kdesc0(w0_addr, KP), kA1 = tc::kdesc0(a1_addr, HC1);
    const uint64_t kW1 = tc::kdesc0(w1_addr, HID), kD = tc::kdesc0(d_addr, 2 * HID);
    const uint64_t mW1 = tc::mdesc0(w1_addr, HID), mD = tc::mdesc0(d_addr, 2 * HID), mA1 = tc::mdesc0(a1_addr, HC1);
    const uint64_t mW0 = tc::mdesc0(w0_addr, KP), mH = tc::mdesc0(h_addr, HCP);
    constexpr uint32_t MSD = 2 * (2 * HID / 8) * 128, MSA1 = 2 * (HC1 / 8) * 128, MSW1 = 2 * (HID / 8) * 128;
    constexpr uint32_t MSW0 = 2 * (KP / 8) * 128, MSH = 2 * (HCP / 8) * 128;   // MN-major K-step bytes
    uint32_t phase = 0, phase2 = 0, wacc = 0, wacc0 = 0, n = 0;
    float dbo[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float* b0 = fp + F::B0 + hf * HH;
    const float* b1 = fp + F::B1 + hf * HH;
    const float4* wot = reinterpret_cast<const float4*>(fp + F::WOT) + hf * HH;

    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
      phase ^= 1;
      tc::fence_after_sync();
    };
    auto to_tensor_core = [&]() {   // this thread's smem / TMEM writes -> the MMA issuer
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1, 256);
    };

    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<K>(rt);
      const bool valid = r0 < a.M;
      const int64_t r = valid ? r0 : a.M - 1;   // tail rows march a real ray with zero upstream
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
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

      for (int q = R; q >= 0; --q, ++n) {
        const int b = n & 1;
        const uint64_t kHb = tc::dplus(kH, (uint32_t)(b * 3) * L::HP_PIECE);
        const uint64_t mHb = tc::dplus(mH, (uint32_t)(b * 3) * L::HP_PIECE);
        // ---- B2: Z1 = H W0^T on the producers' H tile of this step
        if (gt == 0) {
          tc::mbar_wait(&full[b], (n >> 1) & 1);
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
          for (int ks = 0; ks < KP / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 6; ++c)
              tc::mma_bf16(tS0, tc::dplus(kHb, PA[c] * L::HP_PIECE + ks * 256), tc::dplus(kW0, PB[c] * L::W0_PIECE + ks * 256),
                           id_z, (ks | c) != 0);
          tc::mma_commit(bar);
        }
        mma_done();
        LP_PTC(2)
        uint32_t mask1 = 0;   // ReLU'(z1) of this half's hidden units
        {
          float z[HH];
          uint32_t p2[HH / 2];
          tc::tmem_ld<HH>(tS0 + tq + hf * HH, z);
#pragma unroll
          for (int c = 0; c < HH / 8; ++c) {
            float a1[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const float zz = z[8 * c + u] + b0[8 * c + u];
              mask1 |= (zz > 0.0f ? 1u : 0u) << (8 * c + u);
              a1[u] = fmaxf(zz, 0.0f);
            }
            tc::store8_split3(A1t, L::A1_PIECE, rt, hf * HH + 8 * c, HC1, a1, p2 + 4 * c);
          }
          tc::tmem_st<HH / 2>(tA2 + tq + (uint32_t)(hf * HH / 2), p2);   // piece 2 of a1 -> TMEM
          tc::tmem_wait_st();
        }
        LP_PTC(3)
        to_tensor_core();
        if (gt == 0) {   // Z2 = A1 W1^T: pieces 0, 1 of A1 from shared memory, piece 2 from TMEM
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 6; ++c) {
              const uint64_t bd = tc::dplus(kW1, PB[c] * L::W1_PIECE + ks * 256);
              if (PA[c] < 2)
                tc::mma_bf16(tS1, tc::dplus(kA1, PA[c] * L::A1_PIECE + ks * 256), bd, id_z, (ks | c) != 0);
              else
                tc::mma_bf16_ts(tS1, tA2 + (uint32_t)(ks * 8), bd, id_z, 1);
            }
          tc::mma_commit(bar);
        }
        mma_done();
        LP_PTC(4)
        float a2[HH];
        {
          tc::tmem_ld<HH>(tS1 + tq + hf * HH, a2);
          float4 part = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < HH; ++i) {
            a2[i] = fmaxf(a2[i] + b1[i], 0.0f);
            const float4 w = wot[i];
            part.x = fmaf(w.x, a2[i], part.x);
            part.y = fmaf(w.y, a2[i], part.y);
            part.z = fmaf(w.z, a2[i], part.z);
            part.w = fmaf(w.w, a2[i], part.w);
          }
          xo[hf * 128 + rt] = part;
        }
        xo_exchange_barrier(1, 256, 2 + wq);
        float o[kOut];
        {
          const float4 p0 = xo[rt], p1 = xo[128 + rt];
          o[0] = fp[F::BO + 0] + p0.x + p1.x;
          o[1] = fp[F::BO + 1] + p0.y + p1.y;
          o[2] = fp[F::BO + 2] + p0.z + p1.z;
          o[3] = fp[F::BO + 3] + p0.w + p1.w;
        }
        const float s_sig = sigmoid_f(o[0]);
        const float ds = (float)ray.delta * softplus_f(o[0]);
        float col[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) col[c] = sigmoid_f(o[1 + c]);
        // ---- B3: Eq. 3, log-domain reverse update (R12); both halves hold the same state
        const float tau_q = (tauR - U) - Ue;
        two_sum_add(U, Ue, ds);
        const float tau_qm1 = (tauR - U) - Ue;
        float aq = 0.0f;
#pragma unroll
        for (int c = 0; c < kC; ++c) aq = fmaf(p[c], col[c], aq);
        aq = fmaf(gdep, (float)ray_t(ray, q), aq);   // depth channel: "colour" t_q, no MLP gradient
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
        // ---- B5: delta2 = ReLU'(z2) (Wo^T dout) -> D2, a2 -> A2, dout -> A1 tile columns [HID+8, HID+16)
        if (hf == 0) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(A1t, L::A1_PIECE, rt, HID + 8, HC1, dout);
        }
#pragma unroll
        for (int c = 0; c < HH / 8; ++c) {
          float d2[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w = wot[8 * c + u];
            float s = w.x * dout[0];
            s = fmaf(w.y, dout[1], s);
            s = fmaf(w.z, dout[2], s);
            s = fmaf(w.w, dout[3], s);
            d2[u] = a2[8 * c + u] > 0.0f ? s : 0.0f;
          }
          tc::store8<2>(Dt, L::DP, rt, hf * HH + 8 * c, 2 * HID, d2);
          tc::store8<2>(Dt, L::DP, rt, HID + hf * HH + 8 * c, 2 * HID, a2 + 8 * c);
        }
        LP_PTC(3)
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dA1 = D2 W1   (B = W1 [out][in] viewed MN-major: MN = in, K = out)
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tS0, tc::dplus(kD, QA[c] * L::DP + ks * 256), tc::dplus(mW1, QB[c] * L::W1_PIECE + ks * MSW1),
                           id_da1, (ks | c) != 0);
          if constexpr (LP_TC2P_SPLIT) tc::mma_commit(bar2);   // dA1 complete
          // [dW1 db1 . ; . . dWo^T] += [D2 | A2]^T [A1 | 1 | DOUT]   (K = the 128 samples of this step)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW1, tc::dplus(mD, QA[c] * L::DP + ks * MSD), tc::dplus(mA1, QB[c] * L::A1_PIECE + ks * MSA1),
                           id_w1, wacc);
              wacc = 1;
            }
          tc::mma_commit(bar);
        }
        if constexpr (LP_TC2P_SPLIT) {   // dA1 first: its TMEM loads overlap the dW1 MMAs
          tc::mbar_wait(bar2, phase2);
          phase2 ^= 1;
          tc::fence_after_sync();
        } else {
          mma_done();
        }
        LP_PTC(4)
        {   // delta1 = ReLU'(z1) dA1 -> D1 (over D2, consumed)
          float da[HH];
          tc::tmem_ld<HH>(tS0 + tq + hf * HH, da);
          if constexpr (LP_TC2P_SPLIT) mma_done();   // dW1 has read D2
#pragma unroll
          for (int c = 0; c < HH / 8; ++c) {
            float d1[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) d1[u] = (mask1 >> (8 * c + u)) & 1u ? da[8 * c + u] : 0.0f;
            tc::store8<2>(Dt, L::DP, rt, hf * HH + 8 * c, 2 * HID, d1);
          }
        }
        LP_PTC(3)
        to_tensor_core();
        if (gt == 0) {
          tc::fence_after_sync();
          // dH = D1 W0 ; dW0|db0 += D1^T [H|1]
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tS1, tc::dplus(kD, QA[c] * L::DP + ks * 256), tc::dplus(mW0, QB[c] * L::W0_PIECE + ks * MSW0),
                           id_dh, (ks | c) != 0);
          if constexpr (LP_TC2P_SPLIT) tc::mma_commit(bar2);   // dH complete
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW0, tc::dplus(mD, QA[c] * L::DP + ks * MSD), tc::dplus(mHb, QB[c] * L::HP_PIECE + ks * MSH),
                           id_w0, wacc0);
              wacc0 = 1;
            }
          tc::mma_commit(bar);
        }
        if constexpr (LP_TC2P_SPLIT) {   // dH first: its TMEM loads overlap the dW0 MMAs
          tc::mbar_wait(bar2, phase2);
          phase2 ^= 1;
          tc::fence_after_sync();
        } else {
          mma_done();
        }
        LP_PTC(4)
        // ---- B6: this half's dH channels -> fp32 staging over H[b] (Z1, dW0 are done with it)
        {
          float* dhs_b = reinterpret_cast<float*>(smem + L::H + b * 3 * L::HP_PIECE);
          constexpr int HK = KP / 2;
          float dh[HK];
          tc::tmem_ld<HK>(tS1 + tq + hf * HK, dh);
          if constexpr (LP_TC2P_SPLIT) mma_done();   // dW0 has read H[b]
#pragma unroll
          for (int k4 = 0; k4 < HK / 4; ++k4)
            if (hf * HK + 4 * k4 < K)
              *reinterpret_cast<float4*>(dhs_b + rt * (K + 4) + hf * HK + 4 * k4) =
                  make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        tc::mbar_arrive(&staged[b]);
        tc::fence_before_sync();
        tc::named_bar(1, 256);
        LP_PTC(3)
      }
    }
    LP_PTC_FLUSH(1)
    LP_PTC_KEEP_FLUSH

    // ---- B7: flush the gradient partials (TMEM accumulators + register bias sums)
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    const int lane = gt & 31;
    if (hf == 0) {
      // M = 64 accumulator: row i lives in TMEM lane (i/16)*32 + i%16
      const int row = 16 * wq + lane;
      float w0row[KP + 8];
      tc::tmem_ld<KP + 8>(tW0 + tq, w0row);
      if (had_tiles && lane < 16) {
#pragma unroll
        for (int c = 0; c < K; ++c) atomicAdd(a.gparams + P::W0 + row * K + c, w0row[c]);
        atomicAdd(a.gparams + P::B0 + row, w0row[KP]);   // ones column: db0
      }
#pragma unroll
      for (int i = 0; i < kOut; ++i) {
        float s = dbo[i];
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        dbo[i] = s;
      }
      if (lane == 0 && had_tiles) {
#pragma unroll
        for (int i = 0; i < kOut; ++i) atomicAdd(a.gparams + P::BO + i, dbo[i]);
      }
    } else {
      // M = 128 accumulator: row i in TMEM lane i; rows < HID: D2 units (dW1, db1), rows >= HID: A2 units (dWo^T)
      const int row = 32 * wq + lane;
      float w1row[HC1];
      tc::tmem_ld<HC1>(tW1 + tq, w1row);
      if (had_tiles && row < HID) {
#pragma unroll
        for (int c = 0; c < HID; ++c) atomicAdd(a.gparams + P::W1 + row * HID + c, w1row[c]);
        atomicAdd(a.gparams + P::B1 + row, w1row[HID]);   // ones column: db1
      }
      if (had_tiles && row >= HID) {
#pragma unroll
        for (int rr = 0; rr < kOut; ++rr) atomicAdd(a.gparams + P::WO + rr * HID + (row - HID), w1row[HID + 8 + rr]);
      }
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
