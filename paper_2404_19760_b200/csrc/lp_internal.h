// lp_internal.h -- declarations shared by the ABI translation unit and the
// per-instance kernel translation units (compiled in parallel).
#pragma once
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>

#include "../../include/lp.h"
#include "lp_kernels.cuh"

namespace lpi {

struct L2Window {
  const void* base = nullptr;
  size_t bytes = 0;
};

lp_status fail(lp_status s, const char* fmt, ...);
lp_status cuda_check(cudaError_t e, const char* what);
float l2_hit_ratio();

// Persistent grid size of one kernel = SMs x resident CTAs, computed once per
// device (cudaFuncSetAttribute and the occupancy query are per-device state).
struct LaunchShape {
  static constexpr int kMaxDevices = 64;
  std::once_flag once[kMaxDevices];
  int ctas[kMaxDevices] = {};
  cudaError_t err[kMaxDevices] = {};
};

// LP_MAX_CTAS: cap the persistent grid (tests of the multi-tile march, sanitizer runs).
inline int max_ctas_cap() {
  static const int cap = [] {
    const char* e = getenv("LP_MAX_CTAS");
    return e ? atoi(e) : 0;
  }();
  return cap;
}

// CTAs to launch for `work` independent work items (tiles or CTA-sized blocks) on the
// current device; 0 with LP_OK when there is no work.
template <typename KernelT>
lp_status persistent_grid(KernelT kernel, LaunchShape& sh, size_t smem, int threads, int64_t work, int& grid) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return cuda_check(e, "cudaGetDevice");
  if (dev < 0 || dev >= LaunchShape::kMaxDevices) return fail(LP_ERR_UNSUPPORTED, "device ordinal %d", dev);
  std::call_once(sh.once[dev], [&] {
    int sms = 0, occ = 0;
    cudaError_t& err = sh.err[dev];
    err = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (err == cudaSuccess && smem > 0)
      err = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (err == cudaSuccess) err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem);
    if (err == cudaSuccess && occ < 1) err = cudaErrorInvalidConfiguration;
    sh.ctas[dev] = sms * occ;
  });
  if (sh.err[dev] != cudaSuccess) return cuda_check(sh.err[dev], "kernel setup");
  int ctas = sh.ctas[dev];
  const int cap = max_ctas_cap();
  if (cap > 0 && cap < ctas) ctas = cap;
  grid = (int)(work < ctas ? work : ctas);
  return LP_OK;
}

template <int KIND, int K, int HID, int NH>
lp_status run_fwd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID, int NH>
lp_status run_bwd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID>
lp_status run_fwd_vd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID>
lp_status run_bwd_vd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K>
lp_status run_fwd_vd2(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K>
lp_status run_bwd_vd2(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);

}  // namespace lpi
