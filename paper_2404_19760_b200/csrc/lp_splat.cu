// lp_splat.cu -- C ABI of the Splatter (include/lp.h lp_splat_*): validation,
// instance dispatch and persistent launches of lp_splat_kernels.cuh.
#include <cuda_runtime.h>

#include "../../include/lp.h"
#include "lp_internal.h"
#include "lp_splat_mlp_kernels.cuh"
#include "lp_splat_mlp2_kernels.cuh"

namespace {
using namespace lpi;

template <typename KernelT>
lp_status launch_persistent(KernelT kernel, LaunchShape& sh, int threads, int64_t work_blocks, const lp::SplatArgs& a,
                            cudaStream_t s) {
  int grid = 0;
  lp_status st = persistent_grid(kernel, sh, 0, threads, work_blocks, grid);
  if (st != LP_OK || grid == 0) return st;
  kernel<<<grid, threads, 0, s>>>(a);
  return cuda_check(cudaGetLastError(), "splat kernel launch");
}

template <bool FWD, int KIND, int K>
lp_status run(const lp::SplatArgs& a, cudaStream_t s) {
  static LaunchShape sh;
  constexpr int WARPS = lp::kSplatThreads / 32;
  const int64_t blocks = ((a.M + 31) / 32 + WARPS - 1) / WARPS;
  if constexpr (FWD) return launch_persistent(lp::lp_splat_fwd_kernel<KIND, K>, sh, lp::kSplatThreads, blocks, a, s);
  else return launch_persistent(lp::lp_splat_bwd_kernel<KIND, K>, sh, lp::kSplatThreads, blocks, a, s);
}

template <bool FWD>
lp_status dispatch(const lp_grid* g, const lp::SplatArgs& a, cudaStream_t s) {
  const bool tri = g->kind == LP_GRID_TRIPLANE;
  switch (g->K) {
    case 8: return tri ? run<FWD, 0, 8>(a, s) : run<FWD, 1, 8>(a, s);
    case 16: return tri ? run<FWD, 0, 16>(a, s) : run<FWD, 1, 16>(a, s);
    default: return tri ? run<FWD, 0, 32>(a, s) : run<FWD, 1, 32>(a, s);
  }
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int64_t plane_cells(const lp_grid* g, int i) {
  if (g->kind == LP_GRID_VOXEL) return (int64_t)g->H * g->W * g->D;
  return i == 0 ? (int64_t)g->H * g->W : i == 1 ? (int64_t)g->W * g->D : (int64_t)g->D * g->H;
}

lp_status validate(const lp_grid* g, const lp_rays* r) {
  if (!g) return fail(LP_ERR_INVALID_ARG, "null grid descriptor");
  if (g->kind != LP_GRID_TRIPLANE && g->kind != LP_GRID_VOXEL) return fail(LP_ERR_INVALID_ARG, "bad grid kind %d", g->kind);
  if (g->H < 2 || g->W < 2 || g->D < 2) return fail(LP_ERR_INVALID_ARG, "grid dims must be >= 2");
  if (g->K != 8 && g->K != 16 && g->K != 32) return fail(LP_ERR_UNSUPPORTED, "splat: K must be 8, 16 or 32 (got %d)", g->K);
  if (g->contraction < LP_CONTRACT_NONE || g->contraction > LP_CONTRACT_RADIAL)
    return fail(LP_ERR_INVALID_ARG, "bad contraction mode %d", g->contraction);
  if (g->contraction != LP_CONTRACT_NONE && !(g->contract_scale > 0.0f && g->contract_scale < 2.0f))
    return fail(LP_ERR_INVALID_ARG, "contract_scale must be in (0, 2)");
  const int np = g->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < np; ++i)
    if (plane_cells(g, i) * g->K >= (1LL << 31)) return fail(LP_ERR_UNSUPPORTED, "grid plane/volume has >= 2^31 elements");
  if (r) {
    if (r->n_rays < 0) return fail(LP_ERR_INVALID_ARG, "n_rays < 0");
    if (r->n_samples < 2) return fail(LP_ERR_INVALID_ARG, "n_samples must be >= 2");
    if (r->n_rays > 0 && (!r->origins || !r->dirs || !r->t_near || !r->t_far))
      return fail(LP_ERR_INVALID_ARG, "null ray array");
  }
  return LP_OK;
}

template <typename PtrT>
lp_status check_planes(const lp_grid* g, PtrT const* p, const char* name) {
  if (!p) return fail(LP_ERR_INVALID_ARG, "%s is null", name);
  const int np = g->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < np; ++i) {
    if (!p[i]) return fail(LP_ERR_INVALID_ARG, "%s[%d] is null", name, i);
    if (!aligned16(p[i])) return fail(LP_ERR_MISALIGNED, "%s[%d] not 16-byte aligned", name, i);
  }
  return LP_OK;
}

template <typename PtrT>
lp_status check_weights(const lp_grid* g, PtrT const* p, const char* name) {
  if (!p) return fail(LP_ERR_INVALID_ARG, "%s is null", name);
  const int np = g->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < np; ++i)
    if (!p[i]) return fail(LP_ERR_INVALID_ARG, "%s[%d] is null", name, i);
  return LP_OK;
}

lp::SplatArgs make_args(const lp_grid* g, const lp_rays* r) {
  lp::SplatArgs a{};
  a.dims = lp::GridDims{g->H, g->W, g->D};
  a.contract = lp::Contract{g->contraction, (double)g->contract_scale};
  a.orig = r->origins;
  a.dir = r->dirs;
  a.tnear = r->t_near;
  a.tfar = r->t_far;
  a.M = r->n_rays;
  a.S = r->n_samples;
  return a;
}

}  // namespace

extern "C" {

lp_status lp_splat_forward(const lp_grid* grid, const lp_rays* rays, const float* features, float* const theta[3],
                           float* const theta_weight[3], void* stream) {
  lp_status st = validate(grid, rays);
  if (st != LP_OK) return st;
  if (!rays) return fail(LP_ERR_INVALID_ARG, "null rays descriptor");
  if ((st = check_planes(grid, theta, "theta")) != LP_OK) return st;
  if ((st = check_weights(grid, theta_weight, "theta_weight")) != LP_OK) return st;
  if (rays->n_rays > 0 && !features) return fail(LP_ERR_INVALID_ARG, "null features");
  if (rays->n_rays > 0 && !aligned16(features)) return fail(LP_ERR_MISALIGNED, "features not 16-byte aligned");
  lp::SplatArgs a = make_args(grid, rays);
  const int np = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < 3; ++i) {
    a.theta[i] = i < np ? theta[i] : nullptr;
    a.weight[i] = i < np ? theta_weight[i] : nullptr;
  }
  a.feat = features;
  return dispatch<true>(grid, a, static_cast<cudaStream_t>(stream));
}

lp_status lp_splat_normalize(const lp_grid* grid, const float* const theta[3], const float* const theta_weight[3],
                             float* const out[3], void* stream) {
  lp_status st = validate(grid, nullptr);
  if (st != LP_OK) return st;
  if ((st = check_planes(grid, theta, "theta")) != LP_OK) return st;
  if ((st = check_weights(grid, theta_weight, "theta_weight")) != LP_OK) return st;
  if ((st = check_planes(grid, out, "out")) != LP_OK) return st;
  const int np = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (int i = 0; i < np; ++i) {
    const int64_t cells = plane_cells(grid, i);
    const int64_t n4 = cells * grid->K / 4;
    const int blocks = (int)((n4 + 255) / 256 < 148 * 16 ? (n4 + 255) / 256 : 148 * 16);
    if (blocks == 0) continue;
    if (grid->K == 8) lp::lp_splat_normalize_kernel<8><<<blocks, 256, 0, s>>>(theta[i], theta_weight[i], out[i], cells);
    else if (grid->K == 16) lp::lp_splat_normalize_kernel<16><<<blocks, 256, 0, s>>>(theta[i], theta_weight[i], out[i], cells);
    else lp::lp_splat_normalize_kernel<32><<<blocks, 256, 0, s>>>(theta[i], theta_weight[i], out[i], cells);
    if ((st = cuda_check(cudaGetLastError(), "splat normalize launch")) != LP_OK) return st;
  }
  return LP_OK;
}

lp_status lp_splat_backward(const lp_grid* grid, const lp_rays* rays, const float* const grad_out[3],
                            const float* const theta_weight[3], float* grad_features, void* stream) {
  lp_status st = validate(grid, rays);
  if (st != LP_OK) return st;
  if (!rays) return fail(LP_ERR_INVALID_ARG, "null rays descriptor");
  if ((st = check_planes(grid, grad_out, "grad_out")) != LP_OK) return st;
  if ((st = check_weights(grid, theta_weight, "theta_weight")) != LP_OK) return st;
  if (rays->n_rays > 0 && !grad_features) return fail(LP_ERR_INVALID_ARG, "null grad_features");
  if (rays->n_rays > 0 && !aligned16(grad_features)) return fail(LP_ERR_MISALIGNED, "grad_features not 16-byte aligned");
  lp::SplatArgs a = make_args(grid, rays);
  const int np = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < 3; ++i) {
    a.gout[i] = i < np ? grad_out[i] : nullptr;
    a.weight[i] = i < np ? const_cast<float*>(theta_weight[i]) : nullptr;
  }
  a.gfeat = grad_features;
  return dispatch<false>(grid, a, static_cast<cudaStream_t>(stream));
}

}  // extern "C"

namespace {

lp_status validate_gs(const lp_grid* grid, const lp_splat_mlp* gs) {
  if (!gs || !gs->params) return fail(LP_ERR_INVALID_ARG, "null g_s descriptor / params");
  if (gs->n_hidden < 0 || gs->n_hidden > 2) return fail(LP_ERR_UNSUPPORTED, "g_s n_hidden must be 1 or 2 (got %d)", gs->n_hidden);
  if (gs->hidden != lp::kGsH || gs->C_in != lp::kGsC || gs->K_prior != lp::kGsKp || grid->K != lp::kGsK)
    return fail(LP_ERR_UNSUPPORTED, "g_s instance: C_in = K_prior = K = 32, hidden = 64 (got %d, %d, %d, %d)",
                gs->C_in, gs->K_prior, grid->K, gs->hidden);
  if (gs->dir_freqs < 0 || 6 * gs->dir_freqs > lp::kDirEP) return fail(LP_ERR_INVALID_ARG, "dir_freqs must be in [0, 5]");
  return check_planes(grid, gs->prior, "prior");
}

// the paper's 3-layer g_s (two hidden layers): 64-ray tiles (lp_splat_mlp2_kernels.cuh)
template <bool FWD, int KIND>
lp_status run_gs2(const lp::SplatMlpArgs& a, cudaStream_t s) {
  static LaunchShape sh;
  auto kernel = FWD ? lp::lp_splat_mlp2_fwd_kernel<KIND> : lp::lp_splat_mlp2_bwd_kernel<KIND>;
  const size_t smem = FWD ? lp::Gs2FwdSmem<KIND>::BYTES : lp::Gs2BwdSmem<KIND>::BYTES;
  const int threads = 128 * lp::kGs2CG + 32 * lp::kGs2ScatterWarps;
  int grid = 0;
  lp_status st = persistent_grid(kernel, sh, smem, threads, (a.s.M + 63) / 64, grid);
  if (st != LP_OK || grid == 0) return st;
  kernel<<<grid, threads, smem, s>>>(a);
  return cuda_check(cudaGetLastError(), "g_s splat kernel launch");
}

template <bool FWD, int KIND>
lp_status run_gs(const lp::SplatMlpArgs& a, cudaStream_t s) {
  if (a.n_hidden == 2) return run_gs2<FWD, KIND>(a, s);
  static LaunchShape sh;
  auto kernel = FWD ? lp::lp_splat_mlp_fwd_kernel<KIND> : lp::lp_splat_mlp_bwd_kernel<KIND>;
  const size_t smem = FWD ? lp::GsFwdSmem<KIND>::BYTES : lp::GsBwdSmem<KIND>::BYTES;
  const int threads = 256 + 32 * (FWD ? lp::splat_scatter_warps<KIND>() : lp::splat_bwd_scatter_warps<KIND>());
  int grid = 0;
  lp_status st = persistent_grid(kernel, sh, smem, threads, (a.s.M + 127) / 128, grid);
  if (st != LP_OK || grid == 0) return st;
  kernel<<<grid, threads, smem, s>>>(a);
  return cuda_check(cudaGetLastError(), "g_s splat kernel launch");
}

}  // namespace

extern "C" lp_status lp_splat_forward_mlp(const lp_grid* grid, const lp_rays* rays, const float* features,
                                          const lp_splat_mlp* gs, float* const theta[3], float* const theta_weight[3],
                                          void* stream) {
  lp_status st = validate(grid, rays);
  if (st != LP_OK) return st;
  if (!rays) return fail(LP_ERR_INVALID_ARG, "null rays descriptor");
  if ((st = validate_gs(grid, gs)) != LP_OK) return st;
  if ((st = check_planes(grid, theta, "theta")) != LP_OK) return st;
  if ((st = check_weights(grid, theta_weight, "theta_weight")) != LP_OK) return st;
  if (rays->n_rays > 0 && (!features || !aligned16(features))) return fail(LP_ERR_MISALIGNED, "features null or not 16-byte aligned");
  lp::SplatMlpArgs a{};
  a.s = make_args(grid, rays);
  const int np = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < 3; ++i) {
    a.s.theta[i] = i < np ? theta[i] : nullptr;
    a.s.weight[i] = i < np ? theta_weight[i] : nullptr;
    a.prior[i] = i < np ? gs->prior[i] : nullptr;
  }
  a.s.feat = features;
  a.params = gs->params;
  a.dir_freqs = gs->dir_freqs;
  a.n_hidden = gs->n_hidden == 2 ? 2 : 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return grid->kind == LP_GRID_TRIPLANE ? run_gs<true, 0>(a, s) : run_gs<true, 1>(a, s);
}

extern "C" lp_status lp_splat_backward_mlp(const lp_grid* grid, const lp_rays* rays, const float* features,
                                           const lp_splat_mlp* gs, const float* const grad_out[3],
                                           const float* const theta_weight[3], float* grad_features,
                                           float* const grad_prior[3], float* grad_params, void* stream) {
  lp_status st = validate(grid, rays);
  if (st != LP_OK) return st;
  if (!rays) return fail(LP_ERR_INVALID_ARG, "null rays descriptor");
  if ((st = validate_gs(grid, gs)) != LP_OK) return st;
  if ((st = check_planes(grid, grad_out, "grad_out")) != LP_OK) return st;
  if ((st = check_weights(grid, theta_weight, "theta_weight")) != LP_OK) return st;
  if ((st = check_planes(grid, grad_prior, "grad_prior")) != LP_OK) return st;
  if (!grad_params) return fail(LP_ERR_INVALID_ARG, "null grad_params");
  if (rays->n_rays > 0 && (!features || !aligned16(features) || !grad_features || !aligned16(grad_features)))
    return fail(LP_ERR_MISALIGNED, "features / grad_features null or not 16-byte aligned");
  lp::SplatMlpArgs a{};
  a.s = make_args(grid, rays);
  const int np = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < 3; ++i) {
    a.s.gout[i] = i < np ? grad_out[i] : nullptr;
    a.s.weight[i] = i < np ? const_cast<float*>(theta_weight[i]) : nullptr;
    a.prior[i] = i < np ? gs->prior[i] : nullptr;
    a.gprior[i] = i < np ? grad_prior[i] : nullptr;
  }
  a.s.feat = features;
  a.s.gfeat = grad_features;
  a.params = gs->params;
  a.gparams = grad_params;
  a.dir_freqs = gs->dir_freqs;
  a.n_hidden = gs->n_hidden == 2 ? 2 : 1;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  return grid->kind == LP_GRID_TRIPLANE ? run_gs<false, 0>(a, s) : run_gs<false, 1>(a, s);
}


