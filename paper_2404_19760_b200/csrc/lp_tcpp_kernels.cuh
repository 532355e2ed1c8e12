// lp_tcpp_kernels.cuh -- K2tc backward for K = 32 with two ping-pong halves (lp_bwd_tcpp_kernel).
//
// The producer design of lp_bwd_tcp_kernel (4 producer warps gather one step ahead into a
// ring of [H | 1 | DO] buffers, 4 scatter warps reduce the staged dH, 8 compute warps run the
// MLP and Eq. 3), with the 128-ray tile split into two halves of 64 rays that each run their
// own M = 64 MMA rounds under their own mbarrier and named barrier: while one half waits for
// its tensor-core round, the other runs its epilogue. Thread mapping of a half (4 warps, one
// per TMEM lane quarter): the two threads of a ray sit in one warp and read their hidden-unit
// halves of the M = 64 accumulator with the 16x32bx2 TMEM load (scripts/tc_probe4.cu), so
// the output-layer partials meet by shuffle. The weight-gradient accumulator [dW0 db0 . ; .
// dWo^T] (M = 128 over [D1 | A1]) is shared: each half adds its 64 samples (K = 64), the
// tensor pipe serialises the two halves' contributions.
// Buffers are half-major: half h's 64 rows of the three bf16 pieces are one contiguous
// block, so a half stages its fp32 dH rows over its own block once its Z and dW MMAs are done.
#pragma once

#include "lp_tc_kernels.cuh"

namespace lp {

#ifndef LP_BWDPP_SW
#define LP_BWDPP_SW 4
#endif
constexpr int kBwdppScatterWarps = LP_BWDPP_SW;

template <int KIND, int K, int HID>
struct BwdTcppSmem {
  using S = TcShape<KIND, K, HID>;
  static constexpr int NB = kBwdpBuffers;
  static constexpr int HC = S::HC;
  static constexpr uint32_t HH_PIECE = 64 * HC * 2;                           // one half's rows, one piece
  static constexpr uint32_t HHALF = 3 * HH_PIECE;                             // one half, 3 pieces
  static constexpr uint32_t HBUF = 2 * HHALF;
  static constexpr uint32_t W0P = 0;
  static constexpr uint32_t FP = W0P + 3 * S::W0_PIECE;
  static constexpr uint32_t H = (FP + TcParams<K, HID>::N * 4 + 127) & ~127u;   // NB buffers
  static constexpr uint32_t DA = H + NB * HBUF;                                  // [D1 | A1], 2 pieces
  static constexpr uint32_t TAPS = DA + 2 * S::DA_PIECE;                         // NB buffers [128][NPL]
  static constexpr uint32_t BAR = (TAPS + NB * S::TAPS + 127) & ~127u;
  // mbarriers: MMA[2 halves], staged[NB], full[NB], empty[NB]; then the TMEM slot
  static constexpr uint32_t SLOT = 8 * (2 + 3 * NB);
  static constexpr uint32_t BYTES = BAR + SLOT + 16;
  static constexpr uint32_t TMEM_COLS = 256;
  static_assert(2 * HH_PIECE >= 64 * (K + 4) * 4, "a half's dH staging fits its pieces 0-1");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

template <int KIND, int K, int HID>
__global__ void __launch_bounds__(256 + 128 + 32 * kBwdppScatterWarps, 1) lp_bwd_tcpp_kernel(const KernelArgs a) {
  using L = BwdTcppSmem<KIND, K, HID>;
  using S = TcShape<KIND, K, HID>;
  using F = TcParams<K, HID>;
  using P = PackedParams<K, HID, 1>;
  constexpr int HH = HID / 2, KP = S::KP, HC = S::HC, HP = S::HP, NPL = S::NPL;
  constexpr int SW = kBwdppScatterWarps, NB = L::NB;
  static_assert(SW > 0 && 4 % SW == 0, "scatter warps");
  static_assert(K == 32 && HID == 64, "K2tcpp: K = 32, one hidden layer of 64");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint8_t* DAt = smem + L::DA;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);   // [2] one MMA barrier per half
  uint64_t* staged = bar + 2;          // [NB] 256 compute threads: dH of the step staged in H[b]
  uint64_t* full = bar + 2 + NB;       // [NB] 128 producer threads: H / taps buffer written
  uint64_t* empty = bar + 2 + 2 * NB;  // [NB] every lane of the scatter warps: staging + taps read
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + L::SLOT);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tc_weights<K, HID, KP>(w0p, fp, a.params);
  if (threadIdx.x == 0) {
    tc::mbar_init(&bar[0], 1);
    tc::mbar_init(&bar[1], 1);
    for (int b = 0; b < NB; ++b) {
      tc::mbar_init(&staged[b], 256);
      tc::mbar_init(&full[b], 128);
      tc::mbar_init(&empty[b], 32 * SW);
    }
  }
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tbase = *tslot;
  const uint32_t tW = tbase + 192;   // [dW0 | db0 | . ; . | dWo^T] accumulator (M = 128, N = HC)
  if (threadIdx.x < 128) {           // zero it: both halves then always accumulate
    const uint32_t z[8] = {0u, 0u, 0u, 0u, 0u, 0u, 0u, 0u};
#pragma unroll
    for (int c = 0; c < HC; c += 8) tc::tmem_st<8>(tW + ((uint32_t)((threadIdx.x >> 5) * 32) << 16) + c, z);
    tc::tmem_wait_st();
  }
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 127) / 128;

  if (threadIdx.x >= 384) {   // ---- scatter warps: B6 of every staged step, one 32-row block each
    const int sw = (threadIdx.x - 384) / 32, sl = threadIdx.x & 31;
    float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    uint32_t b = 0, ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int q = 0; q < a.S; ++q) {
        tc::mbar_wait(&staged[b], ph);
        for (int rb = sw; rb < 4; rb += SW) {   // 32-row block rb of half rb / 2
          const float4* staps = reinterpret_cast<const float4*>(smem + L::TAPS + b * S::TAPS) + (rb >> 1) * 64 * NPL;
          const float* dhs = reinterpret_cast<const float*>(smem + L::H + b * L::HBUF + (rb >> 1) * L::HHALF);
          coop_scatter<KIND, K>(sgpl, staps, a.dims, dhs, (rb & 1) * 32, sl);
        }
        __syncwarp();
        tc::mbar_arrive(&empty[b]);   // every lane: its own reads of the staging / taps precede it
        if (++b == NB) b = 0, ph ^= 1;
      }
  } else if (threadIdx.x >= 256) {   // ---- producers: taps + cooperative gather, ahead of the compute warps
    const int pw = (threadIdx.x - 256) >> 5, lane = threadIdx.x & 31, row = pw * 32 + lane, h = pw >> 1;
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    uint32_t b = 0, ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<K>(row);
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r0 < a.M ? r0 : a.M - 1, R);
      for (int q = R; q >= 0; --q) {
        float4* taps = reinterpret_cast<float4*>(smem + L::TAPS + b * S::TAPS);
        uint8_t* Hh = smem + L::H + b * L::HBUF + h * L::HHALF;   // this warp's half
        const int lr = row & 63;
        tc::mbar_wait(&empty[b], ph ^ 1);
        {   // the staging of step n - NB overwrote pieces 0-1 of the half: restore this row's ones column block
          const uint32_t off = tc::cm_off(lr, KP, HC);
          *reinterpret_cast<uint4*>(Hh + off) = make_uint4(0x3F80u, 0u, 0u, 0u);   // bf16 1.0, then zeros
          *reinterpret_cast<uint4*>(Hh + L::HH_PIECE + off) = make_uint4(0u, 0u, 0u, 0u);
        }
        double x[3];
        sample_point(ray, q, a.contract, x);
        write_taps<KIND, K>(taps + row * NPL, x, a.dims);
        __syncwarp();
        coop_gather<KIND, K, HC, kBwdHPieces>(planes, taps + h * 64 * NPL, a.dims, Hh, L::HH_PIECE, (pw & 1) * 32, lane);
        tc::fence_async_smem();
        tc::mbar_arrive(&full[b]);
        if (++b == NB) b = 0, ph ^= 1;
      }
    }
  } else {   // ---- compute warps: half h = warps 4h..4h+3, 64 rays, two threads per ray in one warp
    const int gt = threadIdx.x, w = gt >> 5, h = w >> 2, wq = w & 3, lane = gt & 31, hf = lane >> 4;
    const int rl = 16 * wq + (lane & 15), rt = 64 * h + rl;   // row in the half / in the tile
    const bool issuer = (gt & 127) == 0;
    const uint32_t tZ = tbase + (uint32_t)(64 * h), tDH = tbase + 128 + (uint32_t)(32 * h);
    const uint32_t tl = (uint32_t)(wq * 32) << 16;
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id_z = tc::idesc_bf16(64, HID, 0, 0);
    const uint32_t id_dh = tc::idesc_bf16(64, KP, 0, 1);
    const uint32_t id_w = tc::idesc_bf16(128, HC, 1, 1);
    const uint32_t h_addr = tc::smem_u32(smem + L::H) + (uint32_t)h * L::HHALF, w_addr = tc::smem_u32(w0p);
    const uint32_t da_addr = tc::smem_u32(DAt);
    const uint64_t kH = tc::kdesc0(h_addr, HC), kW0 = tc::kdesc0(w_addr, KP);
    const uint64_t kDA = tc::kdesc0(da_addr + (uint32_t)h * (64 / 8) * (2 * HP / 8) * 128, 2 * HP);   // this half's rows
    const uint64_t mW0 = tc::mdesc0(w_addr, KP), mDA = tc::mdesc0(da_addr, 2 * HP), mH = tc::mdesc0(h_addr, HC);
    constexpr uint32_t MSDA = 2 * (2 * HP / 8) * 128, MSW0 = 2 * (KP / 8) * 128, MSH = 2 * (HC / 8) * 128;
    constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
    uint32_t phase = 0, b = 0, bph = 0;
    float dbo[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float* b0 = fp + F::B0 + hf * HH;
    const float4* wot = reinterpret_cast<const float4*>(fp + F::WOT) + hf * HH;

    auto mma_done = [&]() {
      tc::mbar_wait(&bar[h], phase);
      phase ^= 1;
      tc::fence_after_sync();
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

      for (int q = R; q >= 0; --q) {
        uint8_t* Hh = smem + L::H + b * L::HBUF + (uint32_t)h * L::HHALF;
        const uint64_t kHb = tc::dplus(kH, (uint32_t)b * L::HBUF);
        const uint64_t mHb = tc::dplus(mH, (uint32_t)b * L::HBUF);
        // ---- B2: Z = H W0^T on the producers' H rows of this half
        if (issuer) {
          tc::mbar_wait(&full[b], bph);
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
#pragma unroll
          for (int ks = 0; ks < KP / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 6; ++c)
              tc::mma_bf16(tZ, tc::dplus(kHb, PA[c] * L::HH_PIECE + ks * 256),
                           tc::dplus(kW0, PB[c] * S::W0_PIECE + ks * 256), id_z, (ks | c) != 0);
          tc::mma_commit(&bar[h]);
        }
        mma_done();
        uint32_t mask1 = 0;   // ReLU'(z) of this thread's units
        float o[kOut];
        {   // this thread's units: a1 = relu(z + b0) -> A1 columns, partial output layer, exchange by shuffle
          float a1[HH];
          tc::tmem_ld16x2<HH, HH>(tZ + tl, a1);
          float4 part = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int c = 0; c < HH / 8; ++c) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
              const int i = 8 * c + u;
              const float zz = a1[i] + b0[i];
              mask1 |= (zz > 0.0f ? 1u : 0u) << i;
              a1[i] = fmaxf(zz, 0.0f);
              const float4 w = wot[i];
              part.x = fmaf(w.x, a1[i], part.x);
              part.y = fmaf(w.y, a1[i], part.y);
              part.z = fmaf(w.z, a1[i], part.z);
              part.w = fmaf(w.w, a1[i], part.w);
            }
            tc::store8<2>(DAt, S::DA_PIECE, rt, HP + hf * HH + 8 * c, 2 * HP, a1 + 8 * c);
          }
          part.x += __shfl_xor_sync(0xffffffffu, part.x, 16);
          part.y += __shfl_xor_sync(0xffffffffu, part.y, 16);
          part.z += __shfl_xor_sync(0xffffffffu, part.z, 16);
          part.w += __shfl_xor_sync(0xffffffffu, part.w, 16);
          o[0] = fp[F::BO + 0] + part.x;
          o[1] = fp[F::BO + 1] + part.y;
          o[2] = fp[F::BO + 2] + part.z;
          o[3] = fp[F::BO + 3] + part.w;
        }
        // reload Wo^T for delta1 below instead of keeping 4 x HH weights live across the heads
        asm volatile("" ::: "memory");
        const float s_sig = sigmoid_f(o[0]);
        const float ds = (float)ray.delta * softplus_f(o[0]);
        float col[kC];
#pragma unroll
        for (int c = 0; c < kC; ++c) col[c] = sigmoid_f(o[1 + c]);
        // ---- B3: Eq. 3, log-domain reverse update (R12); both threads of the ray hold the same state
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
        // ---- B5: dL/do -> H columns [KP + 8, KP + 16) of the row; a1 and delta1 -> [D1 | A1]
        if (hf == 0) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(Hh, L::HH_PIECE, rl, KP + 8, HC, dout);
        }
#pragma unroll
        for (int c = 0; c < HH / 8; ++c) {
          float d1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w = wot[8 * c + u];
            float sacc = w.x * dout[0];
            sacc = fmaf(w.y, dout[1], sacc);
            sacc = fmaf(w.z, dout[2], sacc);
            sacc = fmaf(w.w, dout[3], sacc);
            d1[u] = (mask1 >> (8 * c + u)) & 1u ? sacc : 0.0f;
          }
          tc::store8<2>(DAt, S::DA_PIECE, rt, hf * HH + 8 * c, 2 * HP, d1);
        }
        tc::fence_async_smem();
        tc::fence_before_sync();
        tc::named_bar(1 + h, 128);
        if (issuer) {
          tc::fence_after_sync();
          // dH = D1 W0 on this half's rows  (B = W0 viewed MN-major: MN = channel, K = hidden)
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tDH, tc::dplus(kDA, QA[c] * S::DA_PIECE + ks * 256),
                           tc::dplus(mW0, QB[c] * S::W0_PIECE + ks * MSW0), id_dh, (ks | c) != 0);
          // [dW0 | db0 | . ; . | dWo^T] += [D1 | A1]^T [H | 1 | DOUT] over this half's 64 samples
#pragma unroll
          for (int ks = 0; ks < 4; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tW, tc::dplus(mDA, QA[c] * S::DA_PIECE + (4 * h + ks) * MSDA),
                           tc::dplus(mHb, QB[c] * L::HH_PIECE + ks * MSH), id_w, 1);
          tc::mma_commit(&bar[h]);
        }
        mma_done();
        // ---- B6: this thread's 16 dH channels -> fp32 staging over the half's rows of H[b]
        {
          float* dhs = reinterpret_cast<float*>(Hh);
          float dh[16];
          tc::tmem_ld16x2<16, 16>(tDH + tl, dh);
#pragma unroll
          for (int k4 = 0; k4 < 4; ++k4)
            *reinterpret_cast<float4*>(dhs + rl * (K + 4) + 16 * hf + 4 * k4) =
                make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        tc::mbar_arrive(&staged[b]);
        if (++b == NB) b = 0, bph ^= 1;
      }
    }

    // ---- B7: flush the weight-gradient accumulator (M = 128: row i in TMEM lane i; rows [0, HP)
    // D1 units -> dW0, db0 (ones column); rows [HP, 2 HP) A1 units -> dWo^T) and the bias sums.
    // Both halves' MMAs are complete: each half waited for its last commit, and the CTA barrier
    // below orders the other half's wait before this read.
    tc::fence_before_sync();
    tc::named_bar(1 + 2, 256);
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    if (h == 0) {
      float wrow[HC];
      tc::tmem_ld<HC>(tW + tl, wrow);
      const int row = 32 * wq + lane;
      if (had_tiles && row < HID) {
#pragma unroll
        for (int c = 0; c < K; ++c) atomicAdd(a.gparams + P::W0 + row * K + c, wrow[c]);
        atomicAdd(a.gparams + P::B0 + row, wrow[KP]);
      }
      if (had_tiles && row >= HP && row - HP < HID) {
#pragma unroll
        for (int rr = 0; rr < kOut; ++rr) atomicAdd(a.gparams + P::WO + rr * HID + (row - HP), wrow[KP + 8 + rr]);
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
#pragma unroll
      for (int i = 0; i < kOut; ++i) atomicAdd(a.gparams + P::BO + i, dbo[i]);
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
