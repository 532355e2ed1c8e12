// lp_splat_kernels.cuh -- the Lightplane Splatter (Supp. P:735-756),
// the dual of the renderer: each pixel ray i expands into the renderer's R+1
// equispaced points, every point inherits the pixel feature v_i and
// pushes it into theta with the sampling weights of h, and a second
// "pass" with the MLPs off pushes the scalar 1 into theta_weight.
// The normalised result is theta / theta_weight (0 where no weight
// landed, reading R27). The backward mirrors the renderer's forward:
// dL/dv_i = sum_j h_{g / theta_weight}(x_ij), theta_weight cached.
//
// Both kernels use the renderer's warp-cooperative layout: a warp owns 32 rays,
// lane = (ray of a 32/(K/4)-ray subgroup, 4-channel chunk), so one vector
// reduction / load instruction covers whole 128-byte corner lines. The two
// splat passes are fused into one march (the weight reduction is issued by the
// chunk-0 lane of each ray). No MLP (g_s of Eq. 2 is disabled, as in the
// paper's benchmark).
#pragma once

#include "lp_tc_kernels.cuh"

namespace lp {

struct SplatArgs {
  float* theta[3];            // fwd: accumulation targets [cells][K]
  float* weight[3];           // fwd: [cells] (K = 1); bwd: cached theta_weight (read)
  const float* gout[3];       // bwd: dL/d(normalised theta) [cells][K]
  GridDims dims;
  Contract contract;
  const float* orig;
  const float* dir;
  const float* tnear;
  const float* tfar;
  int64_t M;
  int S;
  const float* feat;          // fwd: [M][K]
  float* gfeat;               // bwd: [M][K] (overwritten)
};

constexpr int kSplatThreads = 256;

// Tap records of the warp's 32 rays for step j (invalid rows get offset -1).
template <int KIND, int K>
__device__ __forceinline__ void splat_taps(const SplatArgs& a, int64_t ray, bool valid, const RayIn& rin, int j,
                                           float4* rec) {
  double x[3];
  sample_point(rin, j, a.contract, x);
  write_taps<KIND, K>(rec, x, a.dims);
  if (!valid) {
#pragma unroll
    for (int p = 0; p < (KIND == 0 ? 3 : 1); ++p) rec[p].x = __int_as_float(-1);
  }
}

template <int KIND, int K>
__global__ void __launch_bounds__(kSplatThreads) lp_splat_fwd_kernel(const SplatArgs a) {
  constexpr int KC = K / 4, RPI = 32 / KC, NPL = KIND == 0 ? 3 : 1, WARPS = kSplatThreads / 32;
  __shared__ float4 taps_all[WARPS][32 * NPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ch = lane % KC, sub = lane / KC;
  float4* taps = taps_all[warp];
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 31) / 32;
  for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles; tile += (int64_t)gridDim.x * WARPS) {
    const int64_t r = tile * 32 + lane;
    const bool valid = r < a.M;
    const RayIn rin = load_ray(a.orig, a.dir, a.tnear, a.tfar, valid ? r : a.M - 1, R);
    float4 v[KC];   // this lane's 4-channel chunk of the features of its KC rays
#pragma unroll
    for (int it = 0; it < KC; ++it) {
      const int64_t rr = tile * 32 + it * RPI + sub;
      v[it] = rr < a.M ? __ldg(reinterpret_cast<const float4*>(a.feat + rr * K) + ch) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    for (int j = 0; j <= R; ++j) {
      splat_taps<KIND, K>(a, r, valid, rin, j, taps + lane * NPL);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < KC; ++it) {
        const int row = it * RPI + sub;
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
          const float4 rec = taps[row * NPL + p];
          if (__float_as_int(rec.x) < 0) continue;
          Corners<KIND, K> c;
          record_corners<KIND, K>(rec, p, a.dims, c);
          float* th = a.theta[p] + 4 * ch;
#pragma unroll
          for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
            const float w = c.w[cc];
            atomicAdd(reinterpret_cast<float4*>(th + c.off[cc]), make_float4(w * v[it].x, w * v[it].y, w * v[it].z,
                                                                             w * v[it].w));
          }
          if (ch == 0) {   // pass 2: the scalar 1 into theta_weight
#pragma unroll
            for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) atomicAdd(a.weight[p] + c.off[cc] / K, c.w[cc]);
          }
        }
      }
      __syncwarp();
    }
  }
}

// out = theta / theta_weight per cell, 0 where theta_weight == 0 (reading R27).
// May run in place (out == theta): theta and out are not restrict-qualified and
// theta is read with plain loads; each element is read, then written, by one thread.
template <int K>
__global__ void __launch_bounds__(256) lp_splat_normalize_kernel(const float* theta,
                                                                 const float* __restrict__ weight,
                                                                 float* out, int64_t ncells) {
  constexpr int KC = K / 4;
  const int64_t n = ncells * KC;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float w = __ldg(weight + i / KC);
    const float4 t = reinterpret_cast<const float4*>(theta)[i];
    const float s = w > 0.0f ? 1.0f / w : 0.0f;
    float4 o = make_float4(t.x * s, t.y * s, t.z * s, t.w * s);
    if (!(w > 0.0f)) o = make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4*>(out)[i] = o;
  }
}

template <int KIND, int K>
__global__ void __launch_bounds__(kSplatThreads) lp_splat_bwd_kernel(const SplatArgs a) {
  constexpr int KC = K / 4, RPI = 32 / KC, NPL = KIND == 0 ? 3 : 1, WARPS = kSplatThreads / 32;
  __shared__ float4 taps_all[WARPS][32 * NPL];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int ch = lane % KC, sub = lane / KC;
  float4* taps = taps_all[warp];
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 31) / 32;
  for (int64_t tile = (int64_t)blockIdx.x * WARPS + warp; tile < ntiles; tile += (int64_t)gridDim.x * WARPS) {
    const int64_t r = tile * 32 + lane;
    const bool valid = r < a.M;
    const RayIn rin = load_ray(a.orig, a.dir, a.tnear, a.tfar, valid ? r : a.M - 1, R);
    float4 acc[KC];
#pragma unroll
    for (int it = 0; it < KC; ++it) acc[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    for (int j = 0; j <= R; ++j) {
      splat_taps<KIND, K>(a, r, valid, rin, j, taps + lane * NPL);
      __syncwarp();
#pragma unroll
      for (int it = 0; it < KC; ++it) {
        const int row = it * RPI + sub;
#pragma unroll
        for (int p = 0; p < NPL; ++p) {
          const float4 rec = taps[row * NPL + p];
          if (__float_as_int(rec.x) < 0) continue;
          Corners<KIND, K> c;
          record_corners<KIND, K>(rec, p, a.dims, c);
          float4 g[Corners<KIND, K>::N];
          float wc[Corners<KIND, K>::N];
#pragma unroll
          for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
            g[cc] = __ldg(reinterpret_cast<const float4*>(a.gout[p] + c.off[cc]) + ch);
            wc[cc] = __ldg(a.weight[p] + c.off[cc] / K);
          }
#pragma unroll
          for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
            const float s = wc[cc] > 0.0f ? c.w[cc] / wc[cc] : 0.0f;
            acc[it].x = fmaf(s, g[cc].x, acc[it].x);
            acc[it].y = fmaf(s, g[cc].y, acc[it].y);
            acc[it].z = fmaf(s, g[cc].z, acc[it].z);
            acc[it].w = fmaf(s, g[cc].w, acc[it].w);
          }
        }
      }
      __syncwarp();
    }
#pragma unroll
    for (int it = 0; it < KC; ++it) {
      const int64_t rr = tile * 32 + it * RPI + sub;
      if (rr < a.M) reinterpret_cast<float4*>(a.gfeat + rr * K)[ch] = acc[it];
    }
  }
}

}  // namespace lp
