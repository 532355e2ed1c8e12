// lp_internal.h -- declarations shared by the ABI translation unit and the
// per-instance kernel translation units (compiled in parallel).
#pragma once
#include <cuda_runtime.h>

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

template <int KIND, int K, int HID, int NH>
lp_status run_fwd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID, int NH>
lp_status run_bwd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID>
lp_status run_fwd_vd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);
template <int KIND, int K, int HID>
lp_status run_bwd_vd(const lp::KernelArgs& a, const L2Window& w, cudaStream_t s);

}  // namespace lpi
