// lp_abi.cu -- the C ABI of include/lp.h: host-side validation, kernel-instance
// dispatch, persistent launch shapes, and the host-buffer end-to-end entry.
#include <cuda_runtime.h>

#include <atomic>
#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/lp.h"
#include "lp_internal.h"

namespace lpi {

thread_local std::string g_err;
std::atomic<float> g_l2_hit{0.0f};

float l2_hit_ratio() { return g_l2_hit.load(); }

lp_status fail(lp_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

lp_status cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(LP_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return LP_OK;
}

}  // namespace lpi

namespace {
using namespace lpi;

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

struct Inst {
  int kind, K, hid, nh;
};

// Compiled (kind, K, widths) instances.
bool supported(const lp_grid* g, const lp_mlp* m, Inst* inst) {
  const int L = m->n_layers;
  if (L != 2 && L != 3) return false;
  if (m->widths[L] != 4) return false;
  const int K = g->K, hid = m->widths[1];
  if (L == 3 && m->widths[2] != hid) return false;
  const bool ok = (K == 8 && hid == 16 && L == 2) || (K == 16 && hid == 32 && L == 2) ||
                  (K == 32 && hid == 64 && (L == 2 || L == 3));
  if (!ok) return false;
  *inst = Inst{g->kind, K, hid, L - 1};
  return true;
}

lp_status validate(const lp_grid* g, const lp_mlp* m, const lp_rays* r, Inst* inst) {
  if (!g || !m || !r) return fail(LP_ERR_INVALID_ARG, "null grid/mlp/rays descriptor");
  if (g->kind != LP_GRID_TRIPLANE && g->kind != LP_GRID_VOXEL) return fail(LP_ERR_INVALID_ARG, "bad grid kind %d", g->kind);
  if (g->H < 2 || g->W < 2 || g->D < 2) return fail(LP_ERR_INVALID_ARG, "grid dims must be >= 2 (got %d,%d,%d)", g->H, g->W, g->D);
  if (g->K < 1) return fail(LP_ERR_INVALID_ARG, "K must be >= 1");
  if (g->contraction < LP_CONTRACT_NONE || g->contraction > LP_CONTRACT_RADIAL)
    return fail(LP_ERR_INVALID_ARG, "bad contraction mode %d", g->contraction);
  if (g->contraction != LP_CONTRACT_NONE && !(g->contract_scale > 0.0f && g->contract_scale < 2.0f))
    return fail(LP_ERR_INVALID_ARG, "contract_scale must be in (0, 2) (got %g)", (double)g->contract_scale);
  const int nplanes = g->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < nplanes; ++i) {
    if (!g->data[i]) return fail(LP_ERR_INVALID_ARG, "grid data[%d] is null", i);
    if (!aligned16(g->data[i])) return fail(LP_ERR_MISALIGNED, "grid data[%d] not 16-byte aligned", i);
  }
  const int64_t K = g->K;
  const int64_t n0 = g->kind == LP_GRID_VOXEL ? (int64_t)g->H * g->W * g->D * K : (int64_t)g->H * g->W * K;
  const int64_t n1 = (int64_t)g->W * g->D * K, n2 = (int64_t)g->D * g->H * K;
  if (n0 >= (1LL << 31) || (nplanes == 3 && (n1 >= (1LL << 31) || n2 >= (1LL << 31))))
    return fail(LP_ERR_UNSUPPORTED, "grid plane/volume has >= 2^31 elements");
  if (m->n_layers < 1 || m->n_layers > LP_MAX_LAYERS) return fail(LP_ERR_INVALID_ARG, "n_layers %d out of range", m->n_layers);
  if (m->widths[0] != g->K) return fail(LP_ERR_INVALID_ARG, "widths[0]=%d != K=%d", m->widths[0], g->K);
  for (int l = 0; l <= m->n_layers; ++l)
    if (m->widths[l] < 1) return fail(LP_ERR_INVALID_ARG, "widths[%d] < 1", l);
  if (m->widths[m->n_layers] < 2) return fail(LP_ERR_INVALID_ARG, "output width must be 1 + C >= 2");
  if (!m->params) return fail(LP_ERR_INVALID_ARG, "mlp params is null");
  if (r->n_rays < 0) return fail(LP_ERR_INVALID_ARG, "n_rays < 0");
  if (r->n_samples < 2) return fail(LP_ERR_INVALID_ARG, "n_samples must be >= 2 (got %d)", r->n_samples);
  if (r->n_rays > 0 && (!r->origins || !r->dirs || !r->t_near || !r->t_far))
    return fail(LP_ERR_INVALID_ARG, "null ray array");
  if (!supported(g, m, inst))
    return fail(LP_ERR_UNSUPPORTED, "no kernel instance for K=%d widths(n_layers=%d, hidden=%d, out=%d)", g->K,
                m->n_layers, m->widths[1], m->widths[m->n_layers]);
  if (m->dir_freqs < 0 || m->dir_freqs > 5) return fail(LP_ERR_INVALID_ARG, "dir_freqs must be in [0, 5]");
  if (m->dir_freqs > 0 && !((inst->nh == 1 && ((g->K == 8 && m->widths[1] == 16) || (g->K == 32 && m->widths[1] == 64))) ||
                            (inst->nh == 2 && g->K == 32 && m->widths[1] == 64)))
    return fail(LP_ERR_UNSUPPORTED,
                "view-dependent fields: (K, hidden) = (8, 16) or (32, 64) with one hidden layer, or (32, 64) with two");
  if (m->dir_freqs > 0 && getenv("LP_KERNELS") && getenv("LP_KERNELS")[0] == 'f')
    return fail(LP_ERR_UNSUPPORTED, "view-dependent fields have no FFMA kernel");
  return LP_OK;
}

// Smallest address range covering theta, if it fits one access-policy window.
L2Window theta_window(const lp_grid* g) {
  const int nplanes = g->kind == LP_GRID_TRIPLANE ? 3 : 1;
  size_t sz[3] = {(size_t)g->H * g->W * (g->kind == LP_GRID_VOXEL ? (size_t)g->D : 1) * g->K * 4,
                  (size_t)g->W * g->D * g->K * 4, (size_t)g->D * g->H * g->K * 4};
  uintptr_t lo = UINTPTR_MAX, hi = 0;
  for (int i = 0; i < nplanes; ++i) {
    uintptr_t b = reinterpret_cast<uintptr_t>(g->data[i]);
    lo = b < lo ? b : lo;
    hi = b + sz[i] > hi ? b + sz[i] : hi;
  }
  int dev = 0, maxw = 0;
  L2Window w;
  if (cudaGetDevice(&dev) != cudaSuccess ||
      cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, dev) != cudaSuccess)
    return w;
  if (hi - lo <= (uintptr_t)maxw) {
    w.base = reinterpret_cast<const void*>(lo);
    w.bytes = hi - lo;
  }
  return w;
}

template <bool FWD, int KIND>
lp_status dispatch_kind(const Inst& in, const lp::KernelArgs& a, const L2Window& w, cudaStream_t s) {
  if (a.dir_freqs > 0) {
    if (in.nh == 2) return FWD ? run_fwd_vd2<KIND, 32>(a, w, s) : run_bwd_vd2<KIND, 32>(a, w, s);
    if (in.K == 8) return FWD ? run_fwd_vd<KIND, 8, 16>(a, w, s) : run_bwd_vd<KIND, 8, 16>(a, w, s);
    return FWD ? run_fwd_vd<KIND, 32, 64>(a, w, s) : run_bwd_vd<KIND, 32, 64>(a, w, s);
  }
  if (in.K == 8) return FWD ? run_fwd<KIND, 8, 16, 1>(a, w, s) : run_bwd<KIND, 8, 16, 1>(a, w, s);
  if (in.K == 16) return FWD ? run_fwd<KIND, 16, 32, 1>(a, w, s) : run_bwd<KIND, 16, 32, 1>(a, w, s);
  if (in.nh == 1) return FWD ? run_fwd<KIND, 32, 64, 1>(a, w, s) : run_bwd<KIND, 32, 64, 1>(a, w, s);
  return FWD ? run_fwd<KIND, 32, 64, 2>(a, w, s) : run_bwd<KIND, 32, 64, 2>(a, w, s);
}

template <bool FWD>
lp_status dispatch(const Inst& in, const lp_grid* g, const lp::KernelArgs& a, cudaStream_t s) {
  const L2Window w = g_l2_hit.load() > 0.0f ? theta_window(g) : L2Window{};
  return in.kind == LP_GRID_TRIPLANE ? dispatch_kind<FWD, 0>(in, a, w, s) : dispatch_kind<FWD, 1>(in, a, w, s);
}

}  // namespace

namespace lpi {
#ifdef LP_PHASES
unsigned long long* dbg_buffer() {
  static unsigned long long* d = [] {
    unsigned long long* p = nullptr;
    cudaMalloc(&p, sizeof(unsigned long long) * 16);
    cudaMemset(p, 0, sizeof(unsigned long long) * 16);
    return p;
  }();
  return d;
}
#endif
}  // namespace lpi

namespace {

lp::KernelArgs make_args(const lp_grid* g, const lp_mlp* m, const lp_rays* r, const float* bg) {
  lp::KernelArgs a{};
#ifdef LP_PHASES
  a.dbg = lpi::dbg_buffer();
#endif
  for (int i = 0; i < 3; ++i) a.grid[i] = g->data[i];
  if (g->kind == LP_GRID_VOXEL) a.grid[1] = a.grid[2] = nullptr;
  a.dims = lp::GridDims{g->H, g->W, g->D};
  a.params = m->params;
  a.orig = r->origins;
  a.dir = r->dirs;
  a.tnear = r->t_near;
  a.tfar = r->t_far;
  a.M = r->n_rays;
  a.S = r->n_samples;
  a.bg = bg;
  a.contract = lp::Contract{g->contraction, (double)g->contract_scale};
  a.dir_freqs = m->dir_freqs;
  return a;
}

lp_status check_grad_buffers(const lp_grid* grid, float* const grad_data[3], const float* grad_params) {
  if (!grad_data || !grad_params) return fail(LP_ERR_INVALID_ARG, "null gradient buffers");
  const int nplanes = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < nplanes; ++i) {
    if (!grad_data[i]) return fail(LP_ERR_INVALID_ARG, "grad_data[%d] is null", i);
    if (!aligned16(grad_data[i])) return fail(LP_ERR_MISALIGNED, "grad_data[%d] not 16-byte aligned", i);
  }
  return LP_OK;
}

// Copy streams and events of lp_render_fwd_bwd_host, created once per device
// (no device memory); calls serialise on one mutex (each call synchronises anyway).
constexpr int kHostChunks = 4;
struct HostPipe {
  cudaStream_t h2d = nullptr, d2h = nullptr;
  cudaEvent_t ev_start, ev_grad, ev_end, ev_in[kHostChunks], ev_fwd[kHostChunks];
  bool ready = false;
};

std::mutex& host_entry_mutex() {
  static std::mutex m;
  return m;
}

lp_status host_pipe(HostPipe** out) {   // caller holds host_entry_mutex()
  static HostPipe pipes[LaunchShape::kMaxDevices];
  int dev = 0;
  lp_status st = cuda_check(cudaGetDevice(&dev), "cudaGetDevice");
  if (st != LP_OK) return st;
  if (dev < 0 || dev >= LaunchShape::kMaxDevices) return fail(LP_ERR_UNSUPPORTED, "device ordinal %d", dev);
  HostPipe& p = pipes[dev];
  if (!p.ready) {
    const unsigned f = cudaEventDisableTiming;
    cudaError_t e = cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_start, f);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_grad, f);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_end, f);
    for (int i = 0; i < kHostChunks && e == cudaSuccess; ++i) {
      e = cudaEventCreateWithFlags(&p.ev_in[i], f);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&p.ev_fwd[i], f);
    }
    if (e != cudaSuccess) return cuda_check(e, "fwd_bwd_host streams/events");
    p.ready = true;
  }
  *out = &p;
  return LP_OK;
}

}  // namespace

extern "C" {

int lp_abi_version(void) { return LP_ABI_VERSION; }

const char* lp_last_error(void) { return lpi::g_err.c_str(); }

lp_status lp_render_forward(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays, const float* bg, float* out,
                            float* tau_out, float* depth_out, void* stream) {
  Inst in;
  lp_status st = validate(grid, mlp, rays, &in);
  if (st != LP_OK) return st;
  if (rays->n_rays > 0 && (!out || !tau_out)) return fail(LP_ERR_INVALID_ARG, "null out/tau_out");
  lp::KernelArgs a = make_args(grid, mlp, rays, bg);
  a.out = out;
  a.tau = tau_out;
  a.depth = depth_out;
  return dispatch<true>(in, grid, a, static_cast<cudaStream_t>(stream));
}

lp_status lp_render_backward(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays, const float* bg,
                             const float* tau, const float* grad_out, const float* grad_tau,
                             const float* grad_depth, float* const grad_data[3], float* grad_params, void* stream) {
  Inst in;
  lp_status st = validate(grid, mlp, rays, &in);
  if (st != LP_OK) return st;
  if ((st = check_grad_buffers(grid, grad_data, grad_params)) != LP_OK) return st;
  if (rays->n_rays > 0 && (!tau || !grad_out)) return fail(LP_ERR_INVALID_ARG, "null tau/grad_out");
  lp::KernelArgs a = make_args(grid, mlp, rays, bg);
  const int nplanes = grid->kind == LP_GRID_TRIPLANE ? 3 : 1;
  for (int i = 0; i < 3; ++i) a.ggrid[i] = i < nplanes ? grad_data[i] : nullptr;
  a.gparams = grad_params;
  a.tau = const_cast<float*>(tau);
  a.grad_out = grad_out;
  a.grad_tau = grad_tau;
  a.grad_depth = grad_depth;
  return dispatch<false>(in, grid, a, static_cast<cudaStream_t>(stream));
}

size_t lp_fwd_bwd_host_workspace_bytes(int64_t n_rays, int32_t C) {
  // origins, dirs (3 each), near, far, out (C), tau, grad_out (C), grad_tau, bg (C); 256-B aligned pieces
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  const size_t M = n_rays > 0 ? (size_t)n_rays : 0;
  return al(M * 3 * 4) * 2 + al(M * 4) * 2 + al(M * C * 4) * 2 + al(M * 4) * 2 + al((size_t)C * 4);
}

lp_status lp_render_fwd_bwd_host(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays_host,
                                 const float* bg_host, const float* grad_out_host, const float* grad_tau_host,
                                 float* out_host, float* tau_host, float* const grad_data[3], float* grad_params,
                                 void* workspace, size_t workspace_bytes, void* stream) {
  // ---- every check before the first enqueue: nothing is copied or launched on error
  Inst in;
  lp_status st = validate(grid, mlp, rays_host, &in);
  if (st != LP_OK) return st;
  if ((st = check_grad_buffers(grid, grad_data, grad_params)) != LP_OK) return st;
  const int C = mlp->widths[mlp->n_layers] - 1;
  const int64_t M = rays_host->n_rays;
  if (!workspace || workspace_bytes < lp_fwd_bwd_host_workspace_bytes(M, C))
    return fail(LP_ERR_INVALID_ARG, "workspace too small (need %zu bytes)", lp_fwd_bwd_host_workspace_bytes(M, C));
  if ((reinterpret_cast<uintptr_t>(workspace) & 255u) != 0) return fail(LP_ERR_MISALIGNED, "workspace not 256-byte aligned");
  if (M > 0 && (!grad_out_host || !out_host || !tau_host)) return fail(LP_ERR_INVALID_ARG, "null host buffers");
  if (M == 0) return LP_OK;
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  char* w = static_cast<char*>(workspace);
  float* d_o = reinterpret_cast<float*>(w);   w += al(M * 12);
  float* d_d = reinterpret_cast<float*>(w);   w += al(M * 12);
  float* d_n = reinterpret_cast<float*>(w);   w += al(M * 4);
  float* d_f = reinterpret_cast<float*>(w);   w += al(M * 4);
  float* d_out = reinterpret_cast<float*>(w); w += al(M * C * 4);
  float* d_go = reinterpret_cast<float*>(w);  w += al(M * C * 4);
  float* d_tau = reinterpret_cast<float*>(w); w += al(M * 4);
  float* d_gt = reinterpret_cast<float*>(w);  w += al(M * 4);
  float* d_bg = reinterpret_cast<float*>(w);
  const float* dbg = bg_host ? d_bg : nullptr;

  // ---- pipelined over NCH ray chunks on the caller's stream `s` and two copy streams:
  //   h2d: bg, rays chunk 0..NCH-1 (event each), then grad_out / grad_tau
  //   s:   forward of chunk i after its rays land; backward over all M after grad_out lands
  //   d2h: out / tau of chunk i after its forward (overlaps the later chunks and the backward)
  // Exposed copies: the first rays chunk only. Rays are independent, so the chunked
  // forward computes exactly what one launch would.
  std::lock_guard<std::mutex> lock(host_entry_mutex());
  HostPipe* hp = nullptr;
  if ((st = host_pipe(&hp)) != LP_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t min_chunk = 1 << 20;   // below ~1M rays one chunk (the kernel tails would dominate)
  const int NCH = (int)(M >= kHostChunks * min_chunk ? kHostChunks : 1);
  const int64_t per = ((M + NCH - 1) / NCH + 127) / 128 * 128;   // whole 128-ray tiles per chunk
  const auto H2D = cudaMemcpyHostToDevice, D2H = cudaMemcpyDeviceToHost;
  cudaError_t ce = cudaSuccess;
  auto ok = [&](cudaError_t e) { if (ce == cudaSuccess) ce = e; return ce == cudaSuccess; };
  lp_status kst = LP_OK;
  ok(cudaEventRecord(hp->ev_start, s));                  // after the caller's earlier work on s
  ok(cudaStreamWaitEvent(hp->h2d, hp->ev_start, 0));
  ok(cudaStreamWaitEvent(hp->d2h, hp->ev_start, 0));
  if (bg_host) ok(cudaMemcpyAsync(d_bg, bg_host, C * 4, H2D, hp->h2d));
  for (int i = 0; i < NCH && ce == cudaSuccess; ++i) {
    const int64_t r0 = i * per, n = r0 + per < M ? per : M - r0;
    if (n <= 0) break;
    ok(cudaMemcpyAsync(d_o + 3 * r0, rays_host->origins + 3 * r0, n * 12, H2D, hp->h2d));
    ok(cudaMemcpyAsync(d_d + 3 * r0, rays_host->dirs + 3 * r0, n * 12, H2D, hp->h2d));
    ok(cudaMemcpyAsync(d_n + r0, rays_host->t_near + r0, n * 4, H2D, hp->h2d));
    ok(cudaMemcpyAsync(d_f + r0, rays_host->t_far + r0, n * 4, H2D, hp->h2d));
    ok(cudaEventRecord(hp->ev_in[i], hp->h2d));
  }
  ok(cudaMemcpyAsync(d_go, grad_out_host, M * C * 4, H2D, hp->h2d));
  if (grad_tau_host) ok(cudaMemcpyAsync(d_gt, grad_tau_host, M * 4, H2D, hp->h2d));
  ok(cudaEventRecord(hp->ev_grad, hp->h2d));
  for (int i = 0; i < NCH && ce == cudaSuccess && kst == LP_OK; ++i) {
    const int64_t r0 = i * per, n = r0 + per < M ? per : M - r0;
    if (n <= 0) break;
    if (!ok(cudaStreamWaitEvent(s, hp->ev_in[i], 0))) break;
    lp_rays dr = *rays_host;
    dr.n_rays = n;
    dr.origins = d_o + 3 * r0;
    dr.dirs = d_d + 3 * r0;
    dr.t_near = d_n + r0;
    dr.t_far = d_f + r0;
    if ((kst = lp_render_forward(grid, mlp, &dr, dbg, d_out + C * r0, d_tau + r0, nullptr, stream)) != LP_OK) break;
    ok(cudaEventRecord(hp->ev_fwd[i], s));
    ok(cudaStreamWaitEvent(hp->d2h, hp->ev_fwd[i], 0));
    ok(cudaMemcpyAsync(out_host + C * r0, d_out + C * r0, n * C * 4, D2H, hp->d2h));
    ok(cudaMemcpyAsync(tau_host + r0, d_tau + r0, n * 4, D2H, hp->d2h));
  }
  if (ce == cudaSuccess && kst == LP_OK && ok(cudaStreamWaitEvent(s, hp->ev_grad, 0))) {
    lp_rays dr = *rays_host;
    dr.origins = d_o;
    dr.dirs = d_d;
    dr.t_near = d_n;
    dr.t_far = d_f;
    kst = lp_render_backward(grid, mlp, &dr, dbg, d_tau, d_go, grad_tau_host ? d_gt : nullptr, nullptr, grad_data,
                             grad_params, stream);
  }
  // join the copy streams into s (also on failure: no copy may still be reading caller memory)
  const cudaError_t e1 = cudaEventRecord(hp->ev_end, hp->d2h);
  const cudaError_t e2 = e1 == cudaSuccess ? cudaStreamWaitEvent(s, hp->ev_end, 0) : e1;
  const cudaError_t e3 = cudaStreamSynchronize(hp->h2d);
  const cudaError_t e4 = cudaStreamSynchronize(hp->d2h);
  const cudaError_t e5 = cudaStreamSynchronize(s);
  if (kst != LP_OK) return kst;
  if (ce != cudaSuccess) return cuda_check(ce, "fwd_bwd_host enqueue");
  for (cudaError_t e : {e1, e2, e3, e4, e5})
    if (e != cudaSuccess) return cuda_check(e, "fwd_bwd_host sync");
  return LP_OK;
}

lp_status lp_set_l2_persist(float hit_ratio) {
  if (!(hit_ratio >= 0.0f && hit_ratio <= 1.0f)) return fail(LP_ERR_INVALID_ARG, "hit_ratio must be in [0,1]");
  if (hit_ratio > 0.0f) {
    int dev = 0, maxp = 0;
    lp_status e;
    if ((e = cuda_check(cudaGetDevice(&dev), "cudaGetDevice")) != LP_OK) return e;
    if ((e = cuda_check(cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, dev), "attr")) != LP_OK)
      return e;
    if ((e = cuda_check(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)maxp), "persisting L2 limit")) !=
        LP_OK)
      return e;
  }
  lpi::g_l2_hit.store(hit_ratio);
  return LP_OK;
}

#ifdef LP_PHASES
// Debug-only (variant builds): per-phase warp-cycle sums of the tensor-core kernels.
int lp_debug_phase_cycles(unsigned long long* host16, int reset) {
  unsigned long long* d = lpi::dbg_buffer();
  if (cudaMemcpy(host16, d, sizeof(unsigned long long) * 16, cudaMemcpyDeviceToHost) != cudaSuccess) return 1;
  if (reset && cudaMemset(d, 0, sizeof(unsigned long long) * 16) != cudaSuccess) return 1;
  return 0;
}
#endif

}  // extern "C"
