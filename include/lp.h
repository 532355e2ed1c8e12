/* lp.h -- C ABI of the B200-native Lightplane Renderer hot path.
 *
 * The library computes the fused emission-absorption (EA) renderer of
 * Cao et al., "Lightplane: Highly-Scalable Components for Neural 3D Fields"
 * (arXiv 2404.19760), forward and backward, for a hybrid field f = g o h
 * (PAPER.md P:197): a hashing scheme h on a triplane or voxel grid theta
 * followed by a tiny MLP g.
 *
 *   forward  (Eq. 1; fused per ray):
 *     v_i = sum_{j=1..R} (T_{i,j-1} - T_{ij}) f_v(x_ij) + T_{iR} bg,
 *     T_ij = exp(-sum_{n=0..j} Delta_i sigma(x_in)),  x_ij = o_i + (near_i + j Delta_i) d_i,
 *     Delta_i = max(far_i - near_i, 0) / R,  R = n_samples - 1.
 *   backward (Eq. 3; reverse march from the cached final
 *     transmittance, recomputing every activation).
 *
 * Readings of the paper used here are listed in DESIGN.md ("Readings"):
 * one MLP K -> hidden... -> 1 + C with output 0 the density logit (R6),
 * hidden ReLU, sigma = softplus, colour = sigmoid (R7), the cached per-ray
 * scalar is the optical depth tau_R = -ln T_R (R12), background term T_R bg (R5).
 *
 * Conventions for every entry point:
 *  - All array pointers are CUDA DEVICE pointers to fp32, C-contiguous,
 *    unless the name ends in _host. The caller owns every buffer; the library
 *    allocates no device memory and keeps no pointer after the call returns
 *    (apart from stream-ordered use by the kernels it enqueued).
 *  - Work is enqueued on `stream` (a cudaStream_t; NULL = legacy default
 *    stream) without host synchronisation, except lp_render_fwd_bwd_host.
 *    Kernel faults surface at the caller's next synchronisation.
 *  - Validation is host-side and happens before any launch, so nothing is
 *    written on error. Device-resident values (NaNs, near > far) are not
 *    inspected; they are documented preconditions.
 *  - Errors: a non-LP_OK status; lp_last_error() returns a thread-local
 *    message describing the last failure on the calling thread.
 *  - Reentrant: the only global state is per-device launch-shape caches.
 */
#ifndef LP_H_
#define LP_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define LP_ABI_VERSION 3
#define LP_MAX_LAYERS 8

typedef enum {
  LP_OK = 0,
  LP_ERR_INVALID_ARG = 1,  /* null pointer, bad size, broken width chain */
  LP_ERR_UNSUPPORTED = 2,  /* no compiled kernel instance for (kind, K, widths) */
  LP_ERR_MISALIGNED = 3,   /* a grid / gradient pointer is not 16-byte aligned */
  LP_ERR_CUDA = 4          /* a CUDA runtime call or launch failed */
} lp_status;

typedef enum { LP_GRID_TRIPLANE = 0, LP_GRID_VOXEL = 1 } lp_grid_kind;

/* Scene contraction applied to every sample point before hashing (Supp. Eq.
 * "contract"; reading R25):
 *   CC(x) = 0.5 a x                                   ||x|| <= 1
 *   CC(x) = 0.5 ((2 - a)(1 - 1/||x||) + a) x/||x||    otherwise,
 * mapping an unbounded scene into (-1,1)^3 with the foreground [-1,1] at
 * [-a/2, a/2]. PER_AXIS applies it to each coordinate with ||x|| -> |x_k|
 * (the paper's choice); RADIAL uses the Euclidean norm. */
typedef enum { LP_CONTRACT_NONE = 0, LP_CONTRACT_PER_AXIS = 1, LP_CONTRACT_RADIAL = 2 } lp_contraction;

/* theta, the 3D hash structure. Channel-last, K contiguous floats
 * per grid vertex. Axis convention (reading R9): x <-> H, y <-> W, z <-> D;
 * the world cube [-1,1]^3 maps to vertex index space [0, N-1] per axis
 * (align-corners, reading R8); a sample with any |x_a| > 1 reads zero (R11).
 *   triplane: data[0] = xy plane [H][W][K], data[1] = yz plane [W][D][K],
 *             data[2] = zx plane [D][H][K]; h = sum of the three bilinear samples.
 *   voxel:    data[0] = [H][W][D][K]; data[1], data[2] unused (may be NULL);
 *             h = trilinear sample.
 * Requirements: H, W, D >= 2; every data[] pointer 16-byte aligned;
 * elements per plane/volume < 2^31. Compiled K values: 8, 16, 32.
 * contraction / contract_scale: see lp_contraction; scale a in (0, 2) (SPEC S:
 *   ContractConfig: contracted points stay strictly inside the cube)
 * (ignored for LP_CONTRACT_NONE). */
typedef struct {
  int32_t kind;           /* lp_grid_kind */
  int32_t H, W, D;
  int32_t K;
  const float* data[3];
  int32_t contraction;    /* lp_contraction */
  float contract_scale;   /* a */
} lp_grid;

/* The tiny MLP g: n_layers Linear layers, ReLU between them,
 * widths[0] = K, widths[n_layers] = 1 + C (output 0 = density logit, then C
 * colour logits). params packs, per layer l, W_l as [widths[l+1]][widths[l]]
 * row-major then b_l [widths[l+1]]. Compiled widths:
 * (8,16,4), (16,32,4), (32,64,4) and (32,64,64,4).
 * dir_freqs = F > 0 selects the view-dependent field of P:249-250 (reading
 * R29): two networks with the hidden widths of `widths`, g_sigma: K -> H -> 1
 * and g_v: K + 6F -> H -> C fed [h, direnc(d)], direnc(d) = per axis k, per
 * frequency 2^i (i < F): sin(pi 2^i d_k), cos(pi 2^i d_k). params packs g_sigma
 * then g_v, each as above. Compiled: one hidden layer with (K, H) = (8, 16) or
 * (32, 64), and the paper's own networks ("3-layer MLPs with a width of
 * 64": widths (32, 64, 64, 4), g_sigma 32 -> 64 -> 64 -> 1, g_v 32 + 6F -> 64
 * -> 64 -> 3); F <= 5. */
typedef struct {
  int32_t n_layers;
  int32_t widths[LP_MAX_LAYERS + 1];
  const float* params;
  int32_t dir_freqs;
} lp_mlp;

/* The M rays r_i with R+1 = n_samples equispaced points each.
 * dirs are expected unit length (Delta is a distance); they are not
 * normalised. far <= near gives Delta = 0: out = bg, tau = 0, zero gradient. */
typedef struct {
  int64_t n_rays;         /* M >= 0 */
  const float* origins;   /* [M][3] */
  const float* dirs;      /* [M][3] */
  const float* t_near;    /* [M] */
  const float* t_far;     /* [M] */
  int32_t n_samples;      /* S = R + 1 >= 2 */
} lp_rays;

/* Forward render (Eq. 1). bg: [C] or NULL (= zeros).
 * out: [M][C], overwritten with v_i + T_iR bg.
 * tau_out: [M], overwritten with tau_iR = sum_j Delta_i sigma(x_ij) = -ln T_iR,
 * the one per-ray scalar the backward needs.
 * depth_out: [M] or NULL; if given, overwritten with the expected depth
 * sum_{j=1..R} (T_{i,j-1} - T_ij) t_ij, t_ij = near_i + j Delta_i (the "depths"
 * feature of P:234 rendered like a colour channel; reading R26; no background
 * term; the opacity is 1 - exp(-tau_out)). */
lp_status lp_render_forward(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays, const float* bg,
                            float* out, float* tau_out, float* depth_out, void* stream);

/* Backward (Eq. 3 by reverse marching) of the loss
 *   L = sum_i <grad_out_i, out_i> + grad_tau_i * tau_i + grad_depth_i * depth_i
 * w.r.t. theta and the MLP parameters. tau: [M] from lp_render_forward with the
 * same inputs. grad_out: [M][C]. grad_tau, grad_depth: [M] or NULL (= zeros).
 * grad_data: same shapes as grid->data (grad_data[1..2] unused for voxels);
 * grad_params: same packing as mlp->params. Both are ACCUMULATED (+=) with
 * fp32 atomics (summation order nondeterministic); the caller zeroes them.
 * No gradient is produced for rays, near/far or bg. */
lp_status lp_render_backward(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays, const float* bg,
                             const float* tau, const float* grad_out, const float* grad_tau,
                             const float* grad_depth, float* const grad_data[3], float* grad_params, void* stream);

/* End-to-end training step from HOST buffers (the e2e measurement path).
 * rays_host, bg_host, grad_out_host, grad_tau_host (may be NULL) are HOST
 * pointers (pinned memory recommended); grid, mlp, grad_data and grad_params
 * are device-resident. The call copies the ray batch and upstream gradients to
 * `workspace` (device, 256-byte aligned, >= lp_fwd_bwd_host_workspace_bytes(M, C)
 * bytes), runs forward and backward, copies out/tau back to out_host / tau_host
 * (HOST, [M][C] and [M]) and synchronises `stream` before returning.
 * Pipelined for M >= 4 Mi rays: the forward runs in 4 ray chunks, each
 * starting when its rays have landed (the upstream gradients copy under the
 * forward, out/tau copy back under the later chunks and the backward), on
 * `stream` plus two copy streams the library creates once per device. Every
 * argument is validated before the first copy; if a copy or launch fails
 * midway, all three streams are synchronised before the error returns, so no
 * copy still reads or writes the caller's host buffers. Calls serialise. */
size_t lp_fwd_bwd_host_workspace_bytes(int64_t n_rays, int32_t C);
lp_status lp_render_fwd_bwd_host(const lp_grid* grid, const lp_mlp* mlp, const lp_rays* rays_host,
                                 const float* bg_host, const float* grad_out_host, const float* grad_tau_host,
                                 float* out_host, float* tau_host, float* const grad_data[3], float* grad_params,
                                 void* workspace, size_t workspace_bytes, void* stream);

/* ---------------------------------------------------------------- Splatter
 * The dual of the renderer: M pixel rays, each
 * expanded into the renderer's R+1 equispaced points x_ij (same lp_rays
 * convention and contraction), every point inheriting the pixel feature v_i
 * (P:263). theta[c] += sum_ij w_c(x_ij) v_i with the sampling weights of h
 * ("the same as the sampling weights used in rendering"), and in a
 * second pass with the MLPs off theta_weight[c] += sum_ij w_c(x_ij)
 * (P:746-750); the result is theta / theta_weight. g_s of Eq. 2 is not
 * applied (the paper's benchmark disables it). grid->data is unused
 * (may be NULL); grid->K = feature channels (compiled: 8, 16, 32).
 * Layouts: theta / out / grad_out as grid->data (channel-last, 16-byte aligned);
 * theta_weight with the same planes and one channel ([H][W], [W][D], [D][H] or
 * [H][W][D]); features / grad_features [M][K] (16-byte aligned).
 * Forward: ACCUMULATES (+=, fp32 atomics) into theta and theta_weight; the
 * caller zeroes them. */
lp_status lp_splat_forward(const lp_grid* grid, const lp_rays* rays, const float* features, float* const theta[3],
                           float* const theta_weight[3], void* stream);

/* out = theta / theta_weight per cell, exactly 0 where theta_weight == 0
 * (reading R27). out may alias theta. */
lp_status lp_splat_normalize(const lp_grid* grid, const float* const theta[3], const float* const theta_weight[3],
                             float* const out[3], void* stream);

/* Backward of the normalised splat w.r.t. the features, theta_weight treated
 * as a constant cached from the forward:
 *   grad_features_i = sum_j h_{g'}(x_ij),  g' = grad_out / theta_weight (0 where 0),
 * the renderer's gather ("mirrors"). grad_features [M][K] is OVERWRITTEN. */
lp_status lp_splat_backward(const lp_grid* grid, const lp_rays* rays, const float* const grad_out[3],
                            const float* const theta_weight[3], float* grad_features, void* stream);

/* Splatter with its MLP g_s (Eq. 2; reading R30):
 *   v~_ij = g_s(v_i, h_prior(x_ij), direnc(d_i)),  theta += sum_ij w(x_ij) v~_ij,
 * theta_weight as in lp_splat_forward (the weight pass runs with the MLP off,
 * P:748). g_s = Linear(C_in + K_prior + 6F -> hidden) -> ReLU -> Linear(-> K)
 * (n_hidden = 1; 0 means 1), or with a second hidden layer Linear(hidden ->
 * hidden) -> ReLU before the output layer (n_hidden = 2: the paper's "3-layer
 * MLPs with a width of 64"). params packed layer by layer, W_l
 * [out][in] then b_l: W0 [hidden][C_in + K_prior + 6F] (input order: v,
 * h_prior, direnc as in lp_mlp), b0, (W1 [hidden][hidden], b1,) W_out
 * [K][hidden], b_out. The prior grid has the kind, dims and contraction of
 * `grid`, K_prior channels, channel-last, 16-byte aligned. Compiled: C_in =
 * K_prior = K = 32, hidden = 64, n_hidden 1 or 2, dir_freqs <= 5.
 * (ABI version 3 added n_hidden.) */
typedef struct {
  const float* params;
  int32_t hidden;
  int32_t C_in;
  int32_t dir_freqs;
  int32_t K_prior;
  const float* prior[3];
  int32_t n_hidden;
} lp_splat_mlp;

/* theta, theta_weight ACCUMULATED (+=). features [M][C_in]. */
lp_status lp_splat_forward_mlp(const lp_grid* grid, const lp_rays* rays, const float* features,
                               const lp_splat_mlp* gs, float* const theta[3], float* const theta_weight[3],
                               void* stream);

/* Backward of the normalised g_s splat (theta_weight constant):
 * grad_features [M][C_in] OVERWRITTEN; grad_prior (prior shapes) and
 * grad_params (params packing) ACCUMULATED (+=, fp32 atomics). */
lp_status lp_splat_backward_mlp(const lp_grid* grid, const lp_rays* rays, const float* features,
                                const lp_splat_mlp* gs, const float* const grad_out[3],
                                const float* const theta_weight[3], float* grad_features, float* const grad_prior[3],
                                float* grad_params, void* stream);

/* Optional: keep theta resident in L2 for kernels launched by this library on
 * the calling thread's current device (access-policy window on each launch,
 * hit ratio in (0,1]; 0 disables). Sets cudaLimitPersistingL2CacheSize. */
lp_status lp_set_l2_persist(float hit_ratio);

/* Thread-local description of the last non-OK status on this thread. */
const char* lp_last_error(void);
int lp_abi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* LP_H_ */
