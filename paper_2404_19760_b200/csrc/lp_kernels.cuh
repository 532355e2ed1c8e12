// lp_kernels.cuh -- K1 (forward) and K2 (backward) fused ray-march kernels,
// one ray per thread, 128 rays per CTA, persistent grid (sm_100a, FP32 FFMA).
//
// K1 implements Eq. 1 with the per-ray state (tau, v) only
// ("each kernel instance is responsible for a single ray ... only
// store the rendered features and accumulated transmittance").
// K2 implements Eq. 3 by marching q = R..0 from the
// cached tau_R, recomputing sampling and MLP. Gradients of the
// MLP weights are reduced per CTA: every step, the 128 rays stage their
// (layer input, layer delta) vectors in shared memory and each thread owns a
// fixed block of dW, contracting it over the 128 staged samples; one atomic
// flush per parameter per CTA at the end. Grid gradients go straight to
// global memory with 16-byte vector reductions (red.global.add.v4.f32).
#pragma once

#include "lp_device.cuh"

namespace lp {

struct KernelArgs {
  const float* grid[3];
  float* ggrid[3];
  GridDims dims;
  const float* params;
  float* gparams;
  const float* orig;
  const float* dir;
  const float* tnear;
  const float* tfar;
  int64_t M;
  int S;
  const float* bg;       // [3] or null
  float* out;            // fwd: [M][3]
  float* tau;            // fwd: out [M]; bwd: in [M]
  const float* grad_out; // bwd: [M][3]
  const float* grad_tau; // bwd: [M] or null
  float* depth;          // fwd: [M] expected depth sum_j w_j t_j, or null
  const float* grad_depth;  // bwd: [M] or null
  Contract contract;     // sample-point contraction (mode 0 = none)
  int dir_freqs;         // F > 0: view-dependent field (lp_tcv_kernels.cuh)
  unsigned long long* dbg;  // debug phase timers (LP_PHASES variant builds only), else null
};

// ---------------------------------------------------------------- MLP pieces (F4)
// out = relu(b + W x) with W given transposed (WT[IN][OUT]); k-outer loop so
// x_k is reused by OUT/4 consecutive LDS.128 + 4 FFMA groups.
template <int IN, int OUT>
__device__ __forceinline__ void dense_relu(const float* WT, const float* b, const float (&x)[IN], float (&y)[OUT]) {
  lds<OUT>(b, y);
#pragma unroll
  for (int k = 0; k < IN; ++k) {
    const float4* w4 = reinterpret_cast<const float4*>(WT + k * OUT);
#pragma unroll
    for (int i4 = 0; i4 < OUT / 4; ++i4) {
      float4 w = w4[i4];
      y[4 * i4 + 0] = fmaf(w.x, x[k], y[4 * i4 + 0]);
      y[4 * i4 + 1] = fmaf(w.y, x[k], y[4 * i4 + 1]);
      y[4 * i4 + 2] = fmaf(w.z, x[k], y[4 * i4 + 2]);
      y[4 * i4 + 3] = fmaf(w.w, x[k], y[4 * i4 + 3]);
    }
  }
#pragma unroll
  for (int i = 0; i < OUT; ++i) y[i] = fmaxf(y[i], 0.0f);
}

// o = bo + Wo a, Wo given as WoT[HID][4]
template <int HID>
__device__ __forceinline__ void dense_out(const float* WoT, const float* bo, const float (&a)[HID], float (&o)[kOut]) {
  lds<kOut>(bo, o);
#pragma unroll
  for (int i = 0; i < HID; ++i) {
    float4 w = reinterpret_cast<const float4*>(WoT)[i];
    o[0] = fmaf(w.x, a[i], o[0]);
    o[1] = fmaf(w.y, a[i], o[1]);
    o[2] = fmaf(w.z, a[i], o[2]);
    o[3] = fmaf(w.w, a[i], o[3]);
  }
}

// Full MLP forward. Returns the last hidden activation in `last` and, for two
// hidden layers, the first in `a1` (backward needs both).
template <int K, int HID, int NH>
__device__ __forceinline__ void mlp_forward(const float* sp, const float (&h)[K], float (&a1)[HID],
                                            float (&last)[HID], float (&o)[kOut]) {
  using Q = SmemParams<K, HID, NH>;
  dense_relu<K, HID>(sp + Q::W0T, sp + Q::B0, h, a1);
  if constexpr (NH == 2) {
    dense_relu<HID, HID>(sp + Q::W1T, sp + Q::B1, a1, last);
  } else {
#pragma unroll
    for (int i = 0; i < HID; ++i) last[i] = a1[i];
  }
  dense_out<HID>(sp + Q::WOT, sp + Q::BO, last, o);
}

// ================================================================= K1 forward
template <int KIND, int K, int HID, int NH>
__global__ void __launch_bounds__(kThreads) lp_fwd_kernel(const KernelArgs a) {
  extern __shared__ float4 smem4[];
  float* sp = reinterpret_cast<float*>(smem4);
  stage_params<K, HID, NH>(sp, a.params);
  __syncthreads();

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;

  for (int64_t r = (int64_t)blockIdx.x * kThreads + threadIdx.x; r < a.M; r += (int64_t)gridDim.x * kThreads) {
    const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
    float tau = 0.0f, tau_e = 0.0f;  // tau_{j-1} as a compensated sum
    float v[kC] = {0.0f, 0.0f, 0.0f};
    float dep = 0.0f;
    for (int j = 0; j <= R; ++j) {
      double x[3];
      sample_point(ray, j, a.contract, x);  // F2
      Taps<KIND> tp;
      compute_taps<KIND, K>(x, a.dims, tp); // F3
      float h[K];
      gather<KIND, K>(planes, tp, h);
      float a1[HID], last[HID], o[kOut];
      mlp_forward<K, HID, NH>(sp, h, a1, last, o);  // F4
      const float ds = (float)ray.delta * softplus_f(o[0]);  // F5: sigma = softplus
      if (j > 0) {
        // F6: w_j = T_{j-1} - T_j = e^{-tau_{j-1}} (-expm1(-Delta sigma_j))  (reading R13)
        const float w = expf(-(tau + tau_e)) * (-expm1f(-ds));
#pragma unroll
        for (int c = 0; c < kC; ++c) v[c] = fmaf(w, sigmoid_f(o[1 + c]), v[c]);
        dep = fmaf(w, (float)ray_t(ray, j), dep);
      }
      two_sum_add(tau, tau_e, ds);
    }
    const float tauR = tau + tau_e;
    const float TR = expf(-tauR);
#pragma unroll
    for (int c = 0; c < kC; ++c) a.out[3 * r + c] = fmaf(TR, bg[c], v[c]);  // F7
    a.tau[r] = tauR;
    if (a.depth) a.depth[r] = dep;
  }
}

// ================================================================= K2 backward
// Shared-memory staging for the per-CTA weight-gradient contraction.
template <int K, int HID, int NH>
struct Stage {
  static constexpr int SH = K + 4;    // padded rows: conflict-free 16-byte row stores
  static constexpr int SA = HID + 4;
  static constexpr int H = 0;                                   // h      [128][SH]
  static constexpr int A1 = H + kThreads * SH;                  // a1     [128][SA]
  static constexpr int A2 = A1 + kThreads * SA;                 // a2     [128][SA] (NH == 2)
  static constexpr int D1 = A2 + (NH == 2 ? kThreads * SA : 0); // delta1 [128][SA]
  static constexpr int D2 = D1 + kThreads * SA;                 // delta2 [128][SA] (NH == 2)
  static constexpr int DO = D2 + (NH == 2 ? kThreads * SA : 0); // dout   [128][4]
  static constexpr int N = DO + kThreads * kOut;
};

template <int K, int HID, int NH>
constexpr size_t bwd_smem_bytes() {
  return sizeof(float) * (SmemParams<K, HID, NH>::N + Stage<K, HID, NH>::N);
}
template <int K, int HID, int NH>
constexpr size_t fwd_smem_bytes() {
  return sizeof(float) * SmemParams<K, HID, NH>::N;
}

template <int KIND, int K, int HID, int NH>
__global__ void __launch_bounds__(kThreads, NH == 1 ? 2 : 1) lp_bwd_kernel(const KernelArgs a) {
  using Q = SmemParams<K, HID, NH>;
  using P = PackedParams<K, HID, NH>;
  using ST = Stage<K, HID, NH>;
  extern __shared__ float4 smem4[];
  float* sp = reinterpret_cast<float*>(smem4);
  float* st = sp + Q::N;
  stage_params<K, HID, NH>(sp, a.params);

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  // dW ownership: thread t holds rows [ib*BR, ib*BR+BR) x cols [kb*BC, kb*BC+BC)
  const int ib = t >> 3, kb = t & 7;
  constexpr int BR0 = HID / 16, BC0 = K / 8;     // dW0: HID x K = 128 blocks
  constexpr int BR1 = HID / 16, BC1 = HID / 8;   // dW1: HID x HID = 128 blocks (NH == 2)
  constexpr int NOI = (HID + 31) / 32;           // output layer: warp = output row, lane = hidden unit(s)
  static_assert(BR0 >= 1 && BC0 >= 1 && 16 * BR0 == HID && 8 * BC0 == K, "ownership");
  float acc0[BR0][BC0], accb0[BR0];
  float acc1[NH == 2 ? BR1 : 1][NH == 2 ? BC1 : 1], accb1[NH == 2 ? BR1 : 1];
  float acco[NOI], accbo = 0.0f;
#pragma unroll
  for (int i = 0; i < BR0; ++i) {
    accb0[i] = 0.0f;
#pragma unroll
    for (int j = 0; j < BC0; ++j) acc0[i][j] = 0.0f;
  }
  if constexpr (NH == 2) {
#pragma unroll
    for (int i = 0; i < BR1; ++i) {
      accb1[i] = 0.0f;
#pragma unroll
      for (int j = 0; j < BC1; ++j) acc1[i][j] = 0.0f;
    }
  }
#pragma unroll
  for (int m = 0; m < NOI; ++m) acco[m] = 0.0f;
  __syncthreads();

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float* gplanes[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;

  const int64_t ntiles = (a.M + kThreads - 1) / kThreads;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t r0 = tile * kThreads + t;
    const bool valid = r0 < a.M;
    const int64_t r = valid ? r0 : a.M - 1;   // tail lanes march a real ray with zero upstream
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
    // B1: G = sum_{j>q} w_j a_j + T_R (p.bg), starts at q = R with the bg term only
    float G = expf(-tauR) * pbg;
    float U = 0.0f, Ue = 0.0f;  // compensated sum_{j>q} Delta sigma_j; tau_q = tau_R - U

    for (int q = R; q >= 0; --q) {
      // ---- B2: recompute sample q (F2-F5)
      double x[3];
      sample_point(ray, q, a.contract, x);
      Taps<KIND> tp;
      compute_taps<KIND, K>(x, a.dims, tp);
      float h[K];
      gather<KIND, K>(planes, tp, h);
      float a1[HID], last[HID], o[kOut];
      mlp_forward<K, HID, NH>(sp, h, a1, last, o);
      const float s_sig = sigmoid_f(o[0]);          // softplus'(o_0)
      const float ds = (float)ray.delta * softplus_f(o[0]);
      float col[kC];
#pragma unroll
      for (int c = 0; c < kC; ++c) col[c] = sigmoid_f(o[1 + c]);

      // ---- B3: Eq. 3 with the log-domain reverse update of P:352 (reading R12)
      const float tau_q = (tauR - U) - Ue;
      two_sum_add(U, Ue, ds);
      const float tau_qm1 = (tauR - U) - Ue;
      float aq = 0.0f;
#pragma unroll
      for (int c = 0; c < kC; ++c) aq = fmaf(p[c], col[c], aq);
      aq = fmaf(gdep, (float)ray_t(ray, q), aq);   // depth channel: "colour" t_q, no MLP gradient
      const float wq = q > 0 ? expf(-tau_qm1) * (-expm1f(-ds)) : 0.0f;
      const float Tq_aq = q > 0 ? expf(-tau_q) * aq : 0.0f;
      const float dsig = (float)ray.delta * (gtau - (G - Tq_aq));
      G = fmaf(wq, aq, G);

      // ---- B4: head VJP -> dL/do
      float dout[kOut];
      dout[0] = dsig * s_sig;
#pragma unroll
      for (int c = 0; c < kC; ++c) dout[1 + c] = wq * p[c] * col[c] * (1.0f - col[c]);

      // ---- stage layer inputs / deltas for the dW contraction
      sts<K>(st + ST::H + t * ST::SH, h);
      sts<HID>(st + ST::A1 + t * ST::SA, a1);
      if constexpr (NH == 2) sts<HID>(st + ST::A2 + t * ST::SA, last);
      sts<kOut>(st + ST::DO + t * kOut, dout);

      // ---- B5: MLP VJP (dx = W^T delta, ReLU mask from the recomputed activation)
      float dl[HID];  // delta of the last hidden layer
#pragma unroll
      for (int i = 0; i < HID; ++i) {
        float4 w = reinterpret_cast<const float4*>(sp + Q::WOT)[i];
        float s = w.x * dout[0];
        s = fmaf(w.y, dout[1], s);
        s = fmaf(w.z, dout[2], s);
        s = fmaf(w.w, dout[3], s);
        dl[i] = last[i] > 0.0f ? s : 0.0f;
      }
      float d1[HID];
      if constexpr (NH == 2) {
        sts<HID>(st + ST::D2 + t * ST::SA, dl);
#pragma unroll
        for (int k = 0; k < HID; ++k) d1[k] = 0.0f;
#pragma unroll
        for (int i = 0; i < HID; ++i) {
          const float4* w4 = reinterpret_cast<const float4*>(sp + Q::W1 + i * HID);
#pragma unroll
          for (int k4 = 0; k4 < HID / 4; ++k4) {
            float4 w = w4[k4];
            d1[4 * k4 + 0] = fmaf(w.x, dl[i], d1[4 * k4 + 0]);
            d1[4 * k4 + 1] = fmaf(w.y, dl[i], d1[4 * k4 + 1]);
            d1[4 * k4 + 2] = fmaf(w.z, dl[i], d1[4 * k4 + 2]);
            d1[4 * k4 + 3] = fmaf(w.w, dl[i], d1[4 * k4 + 3]);
          }
        }
#pragma unroll
        for (int k = 0; k < HID; ++k) d1[k] = a1[k] > 0.0f ? d1[k] : 0.0f;
      } else {
#pragma unroll
        for (int k = 0; k < HID; ++k) d1[k] = dl[k];
      }
      sts<HID>(st + ST::D1 + t * ST::SA, d1);
      float dh[K];
#pragma unroll
      for (int k = 0; k < K; ++k) dh[k] = 0.0f;
#pragma unroll
      for (int i = 0; i < HID; ++i) {
        const float4* w4 = reinterpret_cast<const float4*>(sp + Q::W0 + i * K);
#pragma unroll
        for (int k4 = 0; k4 < K / 4; ++k4) {
          float4 w = w4[k4];
          dh[4 * k4 + 0] = fmaf(w.x, d1[i], dh[4 * k4 + 0]);
          dh[4 * k4 + 1] = fmaf(w.y, d1[i], dh[4 * k4 + 1]);
          dh[4 * k4 + 2] = fmaf(w.z, d1[i], dh[4 * k4 + 2]);
          dh[4 * k4 + 3] = fmaf(w.w, d1[i], dh[4 * k4 + 3]);
        }
      }
      // ---- B6: grid-gradient scatter (transpose of the gather)
      scatter<KIND, K>(gplanes, tp, dh);

      // ---- B5 (dW part): contract the CTA's 128 staged samples into the owned blocks
      __syncthreads();
#pragma unroll 2
      for (int s = 0; s < kThreads; ++s) {
        float dv[BR0], hv[BC0];
        lds<BR0>(st + ST::D1 + s * ST::SA + ib * BR0, dv);
        lds<BC0>(st + ST::H + s * ST::SH + kb * BC0, hv);
#pragma unroll
        for (int i = 0; i < BR0; ++i) {
#pragma unroll
          for (int j = 0; j < BC0; ++j) acc0[i][j] = fmaf(dv[i], hv[j], acc0[i][j]);
        }
        if (kb == 0) {
#pragma unroll
          for (int i = 0; i < BR0; ++i) accb0[i] += dv[i];
        }
        if constexpr (NH == 2) {
          float dv1[BR1], av[BC1];
          lds<BR1>(st + ST::D2 + s * ST::SA + ib * BR1, dv1);
          lds<BC1>(st + ST::A1 + s * ST::SA + kb * BC1, av);
#pragma unroll
          for (int i = 0; i < BR1; ++i) {
#pragma unroll
            for (int j = 0; j < BC1; ++j) acc1[i][j] = fmaf(dv1[i], av[j], acc1[i][j]);
          }
          if (kb == 0) {
#pragma unroll
            for (int i = 0; i < BR1; ++i) accb1[i] += dv1[i];
          }
        }
        const float dor = st[ST::DO + s * kOut + warp];
        const float* alast = st + (NH == 2 ? ST::A2 : ST::A1) + s * ST::SA;
#pragma unroll
        for (int m = 0; m < NOI; ++m) {
          const int i = lane + 32 * m;
          if (i < HID) acco[m] = fmaf(dor, alast[i], acco[m]);
        }
        if (lane == 0) accbo += dor;
      }
      __syncthreads();
    }
  }

  // ---- B7: one flush of the CTA's MLP-gradient partials
#pragma unroll
  for (int i = 0; i < BR0; ++i) {
    const int row = ib * BR0 + i;
#pragma unroll
    for (int j = 0; j < BC0; ++j) atomicAdd(a.gparams + P::W0 + row * K + kb * BC0 + j, acc0[i][j]);
    if (kb == 0) atomicAdd(a.gparams + P::B0 + row, accb0[i]);
  }
  if constexpr (NH == 2) {
#pragma unroll
    for (int i = 0; i < BR1; ++i) {
      const int row = ib * BR1 + i;
#pragma unroll
      for (int j = 0; j < BC1; ++j) atomicAdd(a.gparams + P::W1 + row * HID + kb * BC1 + j, acc1[i][j]);
      if (kb == 0) atomicAdd(a.gparams + P::B1 + row, accb1[i]);
    }
  }
#pragma unroll
  for (int m = 0; m < NOI; ++m) {
    const int i = lane + 32 * m;
    if (i < HID) atomicAdd(a.gparams + P::WO + warp * HID + i, acco[m]);
  }
  if (lane == 0) atomicAdd(a.gparams + P::BO + warp, accbo);
}

}  // namespace lp
