// lp_device.cuh -- device building blocks of the fused ray march (sm_100a).
//
// Sampling h, MLP g, heads (reading R7) and the
// EA bookkeeping shared by the forward (Eq. 1) and backward (Eq. 3) kernels.
// No code here is shared with oracle/ (independent implementation).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lp {

constexpr int kThreads = 128;  // rays per CTA (one ray per thread)
constexpr int kOut = 4;        // 1 + C outputs (sigma logit, 3 colour logits)
constexpr int kC = 3;

__host__ __device__ constexpr int round4(int x) { return (x + 3) & ~3; }

// ---------------------------------------------------------------- parameters
// Packed layout (lp.h): W0[HID][K], b0[HID], (W1[HID][HID], b1[HID]), Wo[4][HID], bo[4].
template <int K, int HID, int NH>
struct PackedParams {
  static constexpr int W0 = 0;
  static constexpr int B0 = W0 + HID * K;
  static constexpr int W1 = B0 + HID;
  static constexpr int B1 = W1 + (NH == 2 ? HID * HID : 0);
  static constexpr int WO = B1 + (NH == 2 ? HID : 0);
  static constexpr int BO = WO + kOut * HID;
  static constexpr int N = BO + kOut;
};

// Shared-memory copy of the parameters. Every matrix is kept twice: row-major
// W[out][in] (backward: dx = W^T delta walks rows with delta_i reused) and
// transposed WT[in][out] (forward: z += WT[k][:] x_k walks rows with x_k
// reused, one LDS.128 per 4 FFMAs, 4..64 independent accumulators). The output
// layer is only needed as WoT[HID][4] (one LDS.128 per hidden unit both ways).
template <int K, int HID, int NH>
struct SmemParams {
  static constexpr int W0 = 0;                         // [HID][K]
  static constexpr int W0T = W0 + HID * K;             // [K][HID]
  static constexpr int B0 = W0T + HID * K;             // [HID]
  static constexpr int W1 = B0 + HID;                  // [HID][HID]  (NH == 2)
  static constexpr int W1T = W1 + (NH == 2 ? HID * HID : 0);
  static constexpr int B1 = W1T + (NH == 2 ? HID * HID : 0);
  static constexpr int WOT = B1 + (NH == 2 ? HID : 0); // [HID][4]
  static constexpr int BO = WOT + HID * kOut;          // [4]
  static constexpr int N = round4(BO + kOut);
};

template <int K, int HID, int NH>
__device__ __forceinline__ void stage_params(float* s, const float* __restrict__ g) {
  using P = PackedParams<K, HID, NH>;
  using Q = SmemParams<K, HID, NH>;
  for (int i = threadIdx.x; i < HID * K; i += blockDim.x) {
    float v = g[P::W0 + i];
    int r = i / K, c = i % K;
    s[Q::W0 + i] = v;
    s[Q::W0T + c * HID + r] = v;
  }
  for (int i = threadIdx.x; i < HID; i += blockDim.x) s[Q::B0 + i] = g[P::B0 + i];
  if constexpr (NH == 2) {
    for (int i = threadIdx.x; i < HID * HID; i += blockDim.x) {
      float v = g[P::W1 + i];
      int r = i / HID, c = i % HID;
      s[Q::W1 + i] = v;
      s[Q::W1T + c * HID + r] = v;
    }
    for (int i = threadIdx.x; i < HID; i += blockDim.x) s[Q::B1 + i] = g[P::B1 + i];
  }
  for (int i = threadIdx.x; i < kOut * HID; i += blockDim.x) {
    int r = i / HID, c = i % HID;
    s[Q::WOT + c * kOut + r] = g[P::WO + i];
  }
  if (threadIdx.x < kOut) s[Q::BO + threadIdx.x] = g[P::BO + threadIdx.x];
}

// ---------------------------------------------------------------- vector smem helpers
template <int N>
__device__ __forceinline__ void lds(const float* p, float (&v)[N]) {
  static_assert(N == 1 || N == 2 || N % 4 == 0, "vector width");
  if constexpr (N == 1) {
    v[0] = p[0];
  } else if constexpr (N == 2) {
    float2 t = *reinterpret_cast<const float2*>(p);
    v[0] = t.x;
    v[1] = t.y;
  } else {
#pragma unroll
    for (int i = 0; i < N / 4; ++i) {
      float4 t = reinterpret_cast<const float4*>(p)[i];
      v[4 * i] = t.x;
      v[4 * i + 1] = t.y;
      v[4 * i + 2] = t.z;
      v[4 * i + 3] = t.w;
    }
  }
}

template <int N>
__device__ __forceinline__ void sts(float* p, const float* v) {
  static_assert(N % 4 == 0, "vector width");
#pragma unroll
  for (int i = 0; i < N / 4; ++i)
    reinterpret_cast<float4*>(p)[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
}

// ---------------------------------------------------------------- sampling h (F3)
// World [-1,1] -> vertex index space [0, N-1] (align-corners, reading R8);
// the upper edge clamps the cell to N-2 with f = 1. Positions and the index
// mapping are evaluated in fp64 (B200 runs FP64 at half the FP32 rate; this is
// ~15 DFMA-class ops per sample against ~10^4 FP32 FMAs), so the cell choice
// and the fractional offset carry no fp32 cancellation from the camera
// distance (|o| ~ 4 while |x| <= 1). Only the weights and everything after
// the gather are fp32.
__device__ __forceinline__ void axis_cell(double x, int N, int& i, float& f) {
  const double u = __dmul_rn(__dmul_rn(__dadd_rn(x, 1.0), 0.5), (double)(N - 1));
  int ii = (int)floor(u);
  ii = ii > N - 2 ? N - 2 : ii;
  ii = ii < 0 ? 0 : ii;
  i = ii;
  f = (float)__dsub_rn(u, (double)ii);
}

// Taps of one sample point: element offsets (floats) of each corner's K-vector
// within its plane / volume, and the interpolation weights.
template <int KIND>
struct Taps {
  static constexpr int NC = KIND == 0 ? 12 : 8;  // triplane: 3 planes x 4 corners; voxel: 8
  int off[NC];
  float w[NC];
  bool inside;
};

struct GridDims {
  int H, W, D;
};

template <int KIND, int K>
__device__ __forceinline__ void compute_taps(const double x[3], const GridDims& g, Taps<KIND>& tp) {
  // a point with any |x_a| > 1 samples zero and scatters nothing (reading R11)
  tp.inside = fabs(x[0]) <= 1.0 && fabs(x[1]) <= 1.0 && fabs(x[2]) <= 1.0;
  int ix, iy, iz;
  float fx, fy, fz;
  axis_cell(x[0], g.H, ix, fx);
  axis_cell(x[1], g.W, iy, fy);
  axis_cell(x[2], g.D, iz, fz);
  if constexpr (KIND == 1) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      int dx = (c >> 2) & 1, dy = (c >> 1) & 1, dz = c & 1;
      tp.off[c] = (((ix + dx) * g.W + (iy + dy)) * g.D + (iz + dz)) * K;
      tp.w[c] = (dx ? fx : 1.0f - fx) * (dy ? fy : 1.0f - fy) * (dz ? fz : 1.0f - fz);
    }
  } else {
    // plane 0: xy [H][W]; plane 1: yz [W][D]; plane 2: zx [D][H]
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      int a = (c >> 1) & 1, b = c & 1;
      tp.off[c] = ((ix + a) * g.W + (iy + b)) * K;
      tp.w[c] = (a ? fx : 1.0f - fx) * (b ? fy : 1.0f - fy);
      tp.off[4 + c] = ((iy + a) * g.D + (iz + b)) * K;
      tp.w[4 + c] = (a ? fy : 1.0f - fy) * (b ? fz : 1.0f - fz);
      tp.off[8 + c] = ((iz + a) * g.H + (ix + b)) * K;
      tp.w[8 + c] = (a ? fz : 1.0f - fz) * (b ? fx : 1.0f - fx);
    }
  }
}

template <int KIND>
__device__ __forceinline__ const float* tap_plane(const float* const* planes, int c) {
  if constexpr (KIND == 1) return planes[0];
  return planes[c >> 2];
}

// h = sum_c w_c theta[c]  (gather with 16-byte read-only loads)
template <int KIND, int K>
__device__ __forceinline__ void gather(const float* const* planes, const Taps<KIND>& tp, float (&h)[K]) {
#pragma unroll
  for (int k = 0; k < K; ++k) h[k] = 0.0f;
  if (!tp.inside) return;
#pragma unroll
  for (int c = 0; c < Taps<KIND>::NC; ++c) {
    const float4* p = reinterpret_cast<const float4*>(tap_plane<KIND>(planes, c) + tp.off[c]);
    const float w = tp.w[c];
#pragma unroll
    for (int k4 = 0; k4 < K / 4; ++k4) {
      float4 v = __ldg(p + k4);
      h[4 * k4 + 0] = fmaf(w, v.x, h[4 * k4 + 0]);
      h[4 * k4 + 1] = fmaf(w, v.y, h[4 * k4 + 1]);
      h[4 * k4 + 2] = fmaf(w, v.z, h[4 * k4 + 2]);
      h[4 * k4 + 3] = fmaf(w, v.w, h[4 * k4 + 3]);
    }
  }
}

// grad_theta[c] += w_c dh  (the scatter is the transpose of the gather; vector reds)
template <int KIND, int K>
__device__ __forceinline__ void scatter(float* const* gplanes, const Taps<KIND>& tp, const float (&dh)[K]) {
  if (!tp.inside) return;
#pragma unroll
  for (int c = 0; c < Taps<KIND>::NC; ++c) {
    float* base = (KIND == 1 ? gplanes[0] : gplanes[c >> 2]) + tp.off[c];
    const float w = tp.w[c];
#pragma unroll
    for (int k4 = 0; k4 < K / 4; ++k4) {
      float4 v = make_float4(w * dh[4 * k4], w * dh[4 * k4 + 1], w * dh[4 * k4 + 2], w * dh[4 * k4 + 3]);
      atomicAdd(reinterpret_cast<float4*>(base) + k4, v);
    }
  }
}

// ---------------------------------------------------------------- heads (F5)
__device__ __forceinline__ float softplus_f(float x) { return fmaxf(x, 0.0f) + log1pf(expf(-fabsf(x))); }
__device__ __forceinline__ float sigmoid_f(float x) { return 1.0f / (1.0f + expf(-x)); }

// Two-sum accumulation (Knuth): s + e represents the running sum exactly up to
// the last rounding; keeps the reverse-reconstructed optical depth consistent
// with the forward's (reading R12).
__device__ __forceinline__ void two_sum_add(float& s, float& e, float a) {
  float t = s + a;
  float bp = t - s;
  float err = (s - (t - bp)) + (a - bp);
  s = t;
  e += err;
}

// ---------------------------------------------------------------- ray setup (F1, F2)
// Delta = max(far - near, 0) / R and x_j = o + (near + j Delta) d in fp64
// (explicitly rounded mul/add, no contraction), from the fp32 inputs.
struct RayIn {
  float o[3], d[3];
  double t0, delta;
};

__device__ __forceinline__ RayIn load_ray(const float* __restrict__ orig, const float* __restrict__ dir,
                                          const float* __restrict__ tn, const float* __restrict__ tf, int64_t r,
                                          int R) {
  RayIn ray;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    ray.o[a] = __ldg(orig + 3 * r + a);
    ray.d[a] = __ldg(dir + 3 * r + a);
  }
  ray.t0 = (double)__ldg(tn + r);
  const double span = __dsub_rn((double)__ldg(tf + r), ray.t0);
  ray.delta = __ddiv_rn(span > 0.0 ? span : 0.0, (double)R);
  return ray;
}

__device__ __forceinline__ double ray_t(const RayIn& ray, int j) {
  return __dadd_rn(ray.t0, __dmul_rn((double)j, ray.delta));
}

__device__ __forceinline__ void ray_point(const RayIn& ray, int j, double x[3]) {
  const double t = ray_t(ray, j);
#pragma unroll
  for (int a = 0; a < 3; ++a) x[a] = __dadd_rn((double)ray.o[a], __dmul_rn(t, (double)ray.d[a]));
}

// ---------------------------------------------------------------- contraction
// Supp. Eq. "contract", mapping an unbounded scene into the grid cube:
//   CC(x) = 0.5 a x                                  if ||x|| <= 1
//   CC(x) = 0.5 ((2 - a)(1 - 1/||x||) + a) x/||x||   otherwise,
// foreground [-1,1] -> [-a/2, a/2]. mode 1: per axis, ||x|| -> |x_k|
// ("convert X, Y, Z axes into contract coordinates independently", the
// paper's choice; reading R25); mode 2: the displayed radial form. Applied to
// the sample point before the hashing h (F2 -> F3); Delta stays the world
// distance. fp64 with explicit rounding, in the oracle's operation order.
struct Contract {
  int mode;   // 0 none, 1 per-axis, 2 radial
  double a;   // scale a in (0, 2]
};

__device__ __forceinline__ void contract_point(double x[3], const Contract& c) {
  if (c.mode == 1) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      const double n = fabs(x[k]);
      if (n <= 1.0) {
        x[k] = __dmul_rn(0.5, __dmul_rn(c.a, x[k]));
      } else {
        const double s = __dadd_rn(__dmul_rn(__dsub_rn(2.0, c.a), __dsub_rn(1.0, __ddiv_rn(1.0, n))), c.a);
        x[k] = __dmul_rn(0.5, __dmul_rn(s, __ddiv_rn(x[k], n)));
      }
    }
  } else if (c.mode == 2) {
    const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x[0], x[0]), __dmul_rn(x[1], x[1])), __dmul_rn(x[2], x[2])));
    if (n <= 1.0) {
#pragma unroll
      for (int k = 0; k < 3; ++k) x[k] = __dmul_rn(0.5, __dmul_rn(c.a, x[k]));
    } else {
      const double s = __dadd_rn(__dmul_rn(__dsub_rn(2.0, c.a), __dsub_rn(1.0, __ddiv_rn(1.0, n))), c.a);
#pragma unroll
      for (int k = 0; k < 3; ++k) x[k] = __dmul_rn(0.5, __dmul_rn(s, __ddiv_rn(x[k], n)));
    }
  }
}

// F2 (+ optional contraction): the point the hashing scheme h samples for step j.
__device__ __forceinline__ void sample_point(const RayIn& ray, int j, const Contract& c, double x[3]) {
  ray_point(ray, j, x);
  if (c.mode != 0) contract_point(x, c);
}

}  // namespace lp
