// lp_tc_kernels.cuh -- tensor-core (tcgen05) versions of the fused ray march for
// one-hidden-layer MLPs: K1tc (forward, Eq. 1) and K2tc (backward, Eq. 3).
//
// Work decomposition. A CTA holds G independent "groups" of 128 threads; a group
// owns a tile of 128 rays (one ray per thread for the per-ray EA state) and
// marches it step by step (j = 0..R forward, q = R..0 backward).
// Per step:
//   taps     each thread turns its ray's point x_j (fp64) into compact
//            per-plane cell records (shared memory);
//   gather   the warp cooperatively reads the corner vectors of its 32 rays:
//            lane = (ray, 4-channel chunk), so one 16-byte load instruction
//            fetches whole 128-byte corner lines of 32/(K/4) rays, and the
//            lane accumulates its chunk over all corners of its ray
//            (h = sum_c w_c theta_c);
//            h is written as bf16 pieces into the A tile (sample-major);
//   MMA      one elected thread issues tcgen05.mma: Z = H W0^T into TMEM
//            (M = 128 samples, N = hidden, fp32 accumulate);
//   epilogue each thread loads its sample's row of Z from TMEM and runs bias,
//            ReLU, the 4-wide output layer, heads and the EA update.
// Backward additionally stages delta1, a1 and dL/do as bf16 pieces and issues
//   dH  = D1 W0            (M = 128, N = K, K = hidden)   -> grid gradient,
//   dW0 += D1^T H          (M = 64,  N = K, K = 128 samples) -- stays in TMEM,
//   dWo += A1^T DOUT       (M = 64,  N = 8, K = 128 samples) -- stays in TMEM,
// and scatters dH cooperatively with 16-byte vector reductions (one full
// 128-byte line per instruction group), the transpose of the gather.
// The weight-gradient accumulators live in TMEM for the CTA's lifetime and are
// flushed once (B7); bias gradients accumulate per thread in registers.
#pragma once

#include "lp_kernels.cuh"
#include "lp_tc.cuh"

#ifndef LP_GATHER_UNROLL
#define LP_GATHER_UNROLL 2
#endif

#ifdef LP_PHASES
// Debug-only phase timers (variant builds): per-warp clock64 deltas summed into
// a.dbg[kernel * 8 + phase]; read with lp_debug_phase_cycles().
#define LP_PT_DECL unsigned long long lp_pt_acc[8] = {0, 0, 0, 0, 0, 0, 0, 0}; long long lp_pt_t = clock64();
#define LP_PT(i)                                  \
  {                                               \
    long long now_ = clock64();                   \
    lp_pt_acc[i] += (unsigned long long)(now_ - lp_pt_t); \
    lp_pt_t = now_;                               \
  }
#define LP_PT_FLUSH(k)                                                              \
  if ((threadIdx.x & 31) == 0)                                                      \
    for (int i_ = 0; i_ < 8; ++i_) atomicAdd(a.dbg + (k) * 8 + i_, lp_pt_acc[i_]);
#else
#define LP_PT_DECL
#define LP_PT(i)
#define LP_PT_FLUSH(k)
#endif

#ifndef LP_PAIR_XO
#define LP_PAIR_XO 1
#endif

namespace lp {

// Exchange of the partial output-layer sums between the two threads of a ray (halves in
// warps wq and wq + 4 of a 256-thread group): with LP_PAIR_XO a named barrier over that warp
// pair only (64 threads, id `pair_id`), instead of the whole group; the next group-wide
// barrier (with its tcgen05 fence) still precedes the next MMA that overwrites TMEM.
__device__ __forceinline__ void xo_exchange_barrier(int group_id, int group_threads, int pair_id) {
#if LP_PAIR_XO
  tc::named_bar(pair_id, 64);
#else
  tc::fence_before_sync();
  tc::named_bar(group_id, group_threads);
#endif
}

// iterations of the cooperative gather whose loads are kept in flight together
constexpr int kGatherUnroll = LP_GATHER_UNROLL;
// ... in K1tc (all K/4 iterations: c4 fwd 129.3 -> 125.2 ms, c3 36.7 -> 36.0, c5 1606 -> 1584) and in
// K2tcp's producers (c4 bwd 342.8 -> 338.4 ms; 8 there: 379.5 ms)
#ifndef LP_FWD_GATHER_UNROLL
#define LP_FWD_GATHER_UNROLL 8
#endif
#ifndef LP_BWDP_UNROLL
#define LP_BWDP_UNROLL 4
#endif

#ifndef LP_BWD_HPIECES
#define LP_BWD_HPIECES 3
#endif
#ifndef LP_FWD_HPIECES
#define LP_FWD_HPIECES 3
#endif
// bf16 pieces of the sampled feature h in the H tiles of K1tc / K2tc. 3 (default): all 24
// significand bits, 6 products, fp32-class Z. 2 (experiment): 16 bits, 5 products, tiles
// 8 KB (fwd) / 12 KB (bwd) smaller per group: c4 fwd 133.6 -> 127.1 ms, bwd 379 -> 374 ms,
// but more hidden-unit ReLU decisions flip against the fp64 oracle (raw gradient error up
// to 3e-2 before the oracle's ambiguity slack, vs ~1e-5 with 3 pieces) -- kept off.
constexpr int kFwdHPieces = LP_FWD_HPIECES;
constexpr int kBwdHPieces = LP_BWD_HPIECES;

template <int KIND, int K, int HID>
struct TcShape {
  static constexpr int KP = K < 16 ? 16 : K;     // H tile columns / MMA K for Z, N for dH
  static constexpr int HP = HID < 64 ? 64 : HID; // D1 / A1 tile columns (M = 64 of dW MMAs)
  static constexpr int KC = K / 4;               // 16-byte chunks per corner vector
  static constexpr int RPI = 32 / KC;            // rays per cooperative iteration
  static constexpr int NPL = KIND == 0 ? 3 : 1;  // tap records per ray
  static constexpr int TILE = 128;
  // bytes
  static constexpr uint32_t W0_PIECE = HID * KP * 2;
  static constexpr uint32_t H_PIECE = TILE * KP * 2;
  // backward H tile [H | 1 | DO]: channels, an 8-wide group whose first column is 1
  // (so the weight-gradient contraction also yields db0 = sum_s delta1), and the
  // 8-wide dL/do group: one MMA set [D1 | A1]^T [H | 1 | DO] gives dW0, db0 and dWo
  static constexpr int HC = KP + 16;
  static constexpr uint32_t HB_PIECE = TILE * HC * 2;
  static constexpr uint32_t D_PIECE = TILE * HP * 2;
  static constexpr uint32_t DA_PIECE = TILE * 2 * HP * 2;   // [D1 | A1] tile
  static constexpr uint32_t DO_PIECE = TILE * 8 * 2;
  static constexpr uint32_t TAPS = TILE * NPL * 16;
  static_assert(HID % 16 == 0 && HID <= 64, "hidden width");
  static_assert(K % 4 == 0 && K <= 32, "channels");
};

// ---------------------------------------------------------------- taps (F2, F3)
// Compact per-plane record of a sample: (element offset of corner (0,0[,0]),
// f_a, f_b[, f_c | packed cell indices]) as float4; offset -1 marks a point
// outside the cube (R11).
template <int KIND, int K>
__device__ __forceinline__ void write_taps(float4* rec, const double x[3], const GridDims& g) {
  const bool inside = fabs(x[0]) <= 1.0 && fabs(x[1]) <= 1.0 && fabs(x[2]) <= 1.0;
  int ix, iy, iz;
  float fx, fy, fz;
  axis_cell(x[0], g.H, ix, fx);
  axis_cell(x[1], g.W, iy, fy);
  axis_cell(x[2], g.D, iz, fz);
  if constexpr (KIND == 1) {
    const int base = inside ? (((ix * g.W + iy) * g.D + iz) * K) : -1;
    rec[0] = make_float4(__int_as_float(base), fx, fy, fz);
  } else {
    // .w: the cell's (a, b) indices packed as a << 16 | b (window scatter, coop_gather)
    rec[0] = make_float4(__int_as_float(inside ? (ix * g.W + iy) * K : -1), fx, fy, __int_as_float((ix << 16) | iy));
    rec[1] = make_float4(__int_as_float(inside ? (iy * g.D + iz) * K : -1), fy, fz, __int_as_float((iy << 16) | iz));
    rec[2] = make_float4(__int_as_float(inside ? (iz * g.H + ix) * K : -1), fz, fx, __int_as_float((iz << 16) | ix));
  }
}

// Corner set of one record: up to 8 (element offset, weight) pairs.
template <int KIND, int K>
struct Corners {
  static constexpr int N = KIND == 1 ? 8 : 4;
  int off[N];
  float w[N];
};

template <int KIND, int K>
__device__ __forceinline__ void record_corners(const float4 rec, int p, const GridDims& g, Corners<KIND, K>& c) {
  int base = __float_as_int(rec.x);
  const float m = base >= 0 ? 1.0f : 0.0f;
  base = base >= 0 ? base : 0;
  if constexpr (KIND == 1) {
    const int sy = g.D * K, sx = g.W * g.D * K;
    const float ax[2] = {1.0f - rec.y, rec.y}, ay[2] = {1.0f - rec.z, rec.z}, az[2] = {1.0f - rec.w, rec.w};
#pragma unroll
    for (int cc = 0; cc < 8; ++cc) {
      const int dx = (cc >> 2) & 1, dy = (cc >> 1) & 1, dz = cc & 1;
      c.off[cc] = base + dx * sx + dy * sy + dz * K;
      c.w[cc] = ax[dx] * ay[dy] * az[dz] * m;
    }
  } else {
    const int sa = (p == 0 ? g.W : p == 1 ? g.D : g.H) * K;
    const float fa = rec.y, fb = rec.z;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
      const int a = (cc >> 1) & 1, b = cc & 1;
      c.off[cc] = base + a * sa + b * K;
      c.w[cc] = (a ? fa : 1.0f - fa) * (b ? fb : 1.0f - fb) * m;
    }
  }
}

// Row (tile slot) a lane serves in cooperative iteration `it`: consecutive slots, so the
// RPI rows of an iteration fall in distinct rows of a core matrix and its H-tile stores
// spread over the shared-memory banks.
template <int RPI>
__device__ __forceinline__ int coop_row(int row0, int it, int sub) {
  return row0 + it * RPI + sub;
}

#ifndef LP_RAY_SLOT16
#define LP_RAY_SLOT16 1
#endif
// Ray of tile slot rt (offset within the 128-ray tile). A warp's 32 rays are an
// 8x4-pixel block in raster order (workload `pixel_of`); with K = 32 (4 rays per
// cooperative iteration) slots 4i..4i+3 of the block take its 2x2-pixel quad i, whose
// corner sets overlap most (L1 reuse within an iteration). The
// permutation stays inside each 32-ray block, so tail tiles keep their valid rays.
template <int K>
__device__ __forceinline__ int ray_slot(int rt) {
  if constexpr (K == 32) {
    const int b = rt & ~31, it = (rt & 31) >> 2, s = rt & 3;
    return b + ((it >> 2) * 2 + (s >> 1)) * 8 + (it & 3) * 2 + (s & 1);
  } else if constexpr (K == 16 && LP_RAY_SLOT16) {   // 8 rays per iteration: 4x2-pixel blocks
    const int b = rt & ~31, it = (rt & 31) >> 3, s = rt & 7;
    return b + ((it >> 1) * 2 + (s >> 2)) * 8 + (it & 1) * 4 + (s & 3);
  } else {
    return rt;
  }
}


// Warp-cooperative gather of the warp's 32 rays: lane = (ray RPI-subgroup, chunk).
// Writes h into rows [row0, row0 + 32) of the H tile (NP bf16 pieces).
// With SCATTER, each iteration also issues the grid-gradient reductions of the
// previous march step for the same lane slot (records `ptaps`, dh rows `dhs`):
// the L2 reductions of step q+1 overlap the corner loads of step q (B6 || F3;
// the fused-scatter mode, SW = 0).
// Iterations [it0, it1) of the KC = K/4 per warp (two warps may split one row block).
template <int KIND, int K, int C, int NP, bool SCATTER = false, bool PAIR = true, int UNROLL = kGatherUnroll>
__device__ __forceinline__ void coop_gather(const float* const* planes, const float4* taps, const GridDims& g,
                                            uint8_t* Htile, uint32_t piece_stride, int row0, int lane,
                                            float* const* gplanes = nullptr, const float4* ptaps = nullptr,
                                            const float* dhs = nullptr, int it0 = 0, int it1 = K / 4,
                                            float* const* wplanes = nullptr) {
  constexpr int KC = K / 4, RPI = 32 / KC, NPL = KIND == 0 ? 3 : 1;
  const int ch = lane % KC, sub = lane / KC;
  // K = 32: an iteration's 4 rows fill half of each core matrix's 16-byte rows, so its
  // 8-byte piece stores hit the same 16 banks from all 4 channel blocks. Holding the even
  // iteration and storing it with the odd one, lanes of channel blocks 0-1 write one
  // iteration's rows and blocks 2-3 the other's (PAIR; measured: c4 fwd -1.6%, c4p bwd -1.7%;
  // off for K1tcv/K2tcv, +5% there). A half-warp still covers only 4 rows (2-way conflicts,
  // ncu); the conflict-free lane mapping was measured slower (DESIGN.md round-2 measurements).
  float pacc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
  int prow = 0;
#pragma unroll UNROLL
  for (int it = it0; it < it1; ++it) {
    const int row = coop_row<RPI>(row0, it, sub);
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int p = 0; p < NPL; ++p) {
      const float4 rec = taps[row * NPL + p];
      Corners<KIND, K> c;
      record_corners<KIND, K>(rec, p, g, c);
      const float* pl = planes[p] + 4 * ch;
      float4 v[Corners<KIND, K>::N];
#pragma unroll
      for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) v[cc] = __ldg(reinterpret_cast<const float4*>(pl + c.off[cc]));
      if constexpr (SCATTER) {
        const float4 prec = ptaps[row * NPL + p];
        if (__float_as_int(prec.x) >= 0) {
          const float4 d = *reinterpret_cast<const float4*>(dhs + row * (K + 4) + 4 * ch);
          Corners<KIND, K> pc;
          record_corners<KIND, K>(prec, p, g, pc);
          float* gpl = gplanes[p] + 4 * ch;
#pragma unroll
          for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
            const float w = pc.w[cc];
            atomicAdd(reinterpret_cast<float4*>(gpl + pc.off[cc]), make_float4(w * d.x, w * d.y, w * d.z, w * d.w));
          }
          if (wplanes && ch == 0) {   // the Splatter's weight pass (scalar 1 per sample)
#pragma unroll
            for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) atomicAdd(wplanes[p] + pc.off[cc] / K, pc.w[cc]);
          }
        }
      }
#pragma unroll
      for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
        acc[0] = fmaf(c.w[cc], v[cc].x, acc[0]);
        acc[1] = fmaf(c.w[cc], v[cc].y, acc[1]);
        acc[2] = fmaf(c.w[cc], v[cc].z, acc[2]);
        acc[3] = fmaf(c.w[cc], v[cc].w, acc[3]);
      }
    }
    if constexpr (RPI == 4 && PAIR) {
      if (((it - it0) & 1) == 0) {   // warp-uniform
        prow = row;
#pragma unroll
        for (int i = 0; i < 4; ++i) pacc[i] = acc[i];
      } else {
        const bool lo = ch < KC / 2;
        float va[4], vb[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          va[i] = lo ? pacc[i] : acc[i];
          vb[i] = lo ? acc[i] : pacc[i];
        }
        tc::store4<NP>(Htile, piece_stride, lo ? prow : row, 4 * ch, C, va);
        tc::store4<NP>(Htile, piece_stride, lo ? row : prow, 4 * ch, C, vb);
      }
    } else {
      tc::store4<NP>(Htile, piece_stride, row, 4 * ch, C, acc);
    }
  }
  if constexpr (RPI == 4 && PAIR) {
    if ((it1 - it0) & 1) tc::store4<NP>(Htile, piece_stride, prow, 4 * ch, C, pacc);   // odd count: the last one
  }
}

// Warp-cooperative scatter (B6): grad_theta[c] += w_c dh for the warp's 32 rays;
// dh rows are fp32 in `dhs` ([128][K + 4]).
template <int KIND, int K>
__device__ __forceinline__ void coop_scatter(float* const* gplanes, const float4* taps, const GridDims& g,
                                             const float* dhs, int row0, int lane, int it0 = 0, int it1 = K / 4,
                                             float* const* wplanes = nullptr) {
  constexpr int KC = K / 4, RPI = 32 / KC, NPL = KIND == 0 ? 3 : 1;
  const int ch = lane % KC, sub = lane / KC;
#pragma unroll 1
  for (int it = it0; it < it1; ++it) {
    const int row = coop_row<RPI>(row0, it, sub);
    const float4 d = *reinterpret_cast<const float4*>(dhs + row * (K + 4) + 4 * ch);
#pragma unroll
    for (int p = 0; p < NPL; ++p) {
      const float4 rec = taps[row * NPL + p];
      if (__float_as_int(rec.x) < 0) continue;
      Corners<KIND, K> c;
      record_corners<KIND, K>(rec, p, g, c);
      float* pl = gplanes[p] + 4 * ch;
#pragma unroll
      for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) {
        const float w = c.w[cc];
        atomicAdd(reinterpret_cast<float4*>(pl + c.off[cc]), make_float4(w * d.x, w * d.y, w * d.z, w * d.w));
      }
      if (wplanes && ch == 0) {
#pragma unroll
        for (int cc = 0; cc < Corners<KIND, K>::N; ++cc) atomicAdd(wplanes[p] + c.off[cc] / K, c.w[cc]);
      }
    }
  }
}

// ---------------------------------------------------------------- shared staging of the weights
template <int K, int HID>
struct TcParams {  // fp32 copies used on CUDA cores
  static constexpr int B0 = 0;               // [HID]
  static constexpr int WOT = HID;            // [HID][4]
  static constexpr int BO = HID + 4 * HID;   // [4]
  static constexpr int N = round4(BO + 4);
};

template <int K, int HID, int KP>
__device__ __forceinline__ void stage_tc_weights(uint8_t* w0p, float* fp, const float* __restrict__ g) {
  using P = PackedParams<K, HID, 1>;
  using F = TcParams<K, HID>;
  // W0 [HID][KP] as 3 bf16 pieces (columns >= K stay zero)
  for (int i = threadIdx.x; i < HID * K; i += blockDim.x) {
    const int r = i / K, c = i % K;
    float v = g[P::W0 + i];
#pragma unroll
    for (int pc = 0; pc < 3; ++pc) {
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      *reinterpret_cast<__nv_bfloat16*>(w0p + pc * (HID * KP * 2) + tc::cm_off(r, c, KP)) = b;
      v -= __bfloat162float(b);
    }
  }
  for (int i = threadIdx.x; i < HID; i += blockDim.x) fp[F::B0 + i] = g[P::B0 + i];
  for (int i = threadIdx.x; i < 4 * HID; i += blockDim.x) {
    const int r = i / HID, c = i % HID;
    fp[F::WOT + c * 4 + r] = g[P::WO + i];
  }
  if (threadIdx.x < 4) fp[F::BO + threadIdx.x] = g[P::BO + threadIdx.x];
}

// o = bo + Wo relu(z + b0); also returns a = relu(z + b0)
template <int HID>
__device__ __forceinline__ void tc_head_layer(const float* fp_b0, const float* fp_wot, const float* fp_bo,
                                              float (&z)[HID], float (&o)[kOut]) {
  lds<kOut>(fp_bo, o);
#pragma unroll
  for (int i = 0; i < HID; ++i) {
    z[i] = fmaxf(z[i] + fp_b0[i], 0.0f);
    const float4 w = reinterpret_cast<const float4*>(fp_wot)[i];
    o[0] = fmaf(w.x, z[i], o[0]);
    o[1] = fmaf(w.y, z[i], o[1]);
    o[2] = fmaf(w.z, z[i], o[2]);
    o[3] = fmaf(w.w, z[i], o[3]);
  }
}

// ================================================================= K1tc forward
template <int KIND, int K, int HID, int G>
struct FwdTcSmem {
  using S = TcShape<KIND, K, HID>;
  static constexpr uint32_t W0P = 0;                                   // 3 pieces
  static constexpr uint32_t FP = W0P + 3 * S::W0_PIECE;                // fp32 params
  static constexpr uint32_t GRP = (FP + TcParams<K, HID>::N * 4 + 127) & ~127u;
  static constexpr uint32_t H = 0;                                     // per group: H (kFwdHPieces), taps
  static constexpr uint32_t TAPS = H + kFwdHPieces * S::H_PIECE;
  static constexpr uint32_t GSIZE = (TAPS + S::TAPS + 127) & ~127u;
  static constexpr uint32_t BAR = GRP + G * GSIZE;                     // G mbarriers + tmem slot
  static constexpr uint32_t BYTES = BAR + 8 * G + 16;
  static constexpr uint32_t TMEM_COLS = G * 64 <= 32 ? 32 : G * 64 <= 64 ? 64 : G * 64 <= 128 ? 128 : 256;
};

template <int KIND, int K, int HID, int G>
__global__ void __launch_bounds__(128 * G, 1) lp_fwd_tc_kernel(const KernelArgs a) {
  using S = TcShape<KIND, K, HID>;
  using L = FwdTcSmem<KIND, K, HID, G>;
  using F = TcParams<K, HID>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 8 * G);

  const int g = threadIdx.x >> 7, gt = threadIdx.x & 127, wg = gt >> 5, lane = gt & 31;
  uint8_t* gsm = smem + L::GRP + g * L::GSIZE;
  uint8_t* Ht = gsm + L::H;
  float4* taps = reinterpret_cast<float4*>(gsm + L::TAPS);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tc_weights<K, HID, S::KP>(w0p, fp, a.params);
  if (threadIdx.x < G) tc::mbar_init(&bars[threadIdx.x], 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  const uint32_t tmem = *tslot + (uint32_t)(g * 64);
  const uint32_t tlane = (uint32_t)(wg * 32) << 16;

  const int R = a.S - 1;
  const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
  float bg[kC];
#pragma unroll
  for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
  const uint32_t idesc = tc::idesc_bf16(128, HID, 0, 0);
  const uint32_t h_addr = tc::smem_u32(Ht), w_addr = tc::smem_u32(w0p);
  uint32_t phase = 0;
  LP_PT_DECL

  const int64_t ntiles = (a.M + 127) / 128;
  for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < ntiles; tile += (int64_t)gridDim.x * G) {
    const int64_t r0 = tile * 128 + ray_slot<K>(gt);
    const bool valid = r0 < a.M;
    const int64_t r = valid ? r0 : a.M - 1;
    const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r, R);
    float tau = 0.0f, tau_e = 0.0f;
    float v[kC] = {0.0f, 0.0f, 0.0f};
    float dep = 0.0f;
    for (int j = 0; j <= R; ++j) {
      double x[3];
      sample_point(ray, j, a.contract, x);                                        // F2
      write_taps<KIND, K>(taps + gt * S::NPL, x, a.dims);          // F3 (cells)
      __syncwarp();
      LP_PT(0)
      coop_gather<KIND, K, S::KP, kFwdHPieces, false, true, LP_FWD_GATHER_UNROLL>(planes, taps, a.dims, Ht, S::H_PIECE,
                                                                               wg * 32, lane);  // F3 (gather)
      LP_PT(1)
      tc::fence_async_smem();
      tc::fence_before_sync();
      tc::named_bar(1 + g, 128);
      LP_PT(2)
      if (gt == 0) {                                               // F4: Z = H W0^T on the tensor core
        tc::fence_after_sync();
        constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
        constexpr int NPROD = kFwdHPieces == 3 ? 6 : 5;   // products with H piece < kFwdHPieces
        uint32_t acc = 0;
#pragma unroll
        for (int ks = 0; ks < S::KP / 16; ++ks)
#pragma unroll
          for (int c = 0; c < NPROD; ++c) {
            tc::mma_bf16(tmem, tc::desc_kmajor(h_addr + PA[c] * S::H_PIECE, S::KP, ks),
                         tc::desc_kmajor(w_addr + PB[c] * S::W0_PIECE, S::KP, ks), idesc, acc);
            acc = 1;
          }
        tc::mma_commit(&bars[g]);
      }
      LP_PT(3)
      tc::mbar_wait(&bars[g], phase);
      phase ^= 1;
      LP_PT(4)
      tc::fence_after_sync();
      float z[HID];
      tc::tmem_ld<HID>(tmem + tlane, z);
      tc::fence_before_sync();
      float o[kOut];
      tc_head_layer<HID>(fp + F::B0, fp + F::WOT, fp + F::BO, z, o);
      const float ds = (float)ray.delta * softplus_f(o[0]);       // F5
      if (j > 0) {                                                 // F6
        const float w = expf(-(tau + tau_e)) * (-expm1f(-ds));
#pragma unroll
        for (int c = 0; c < kC; ++c) v[c] = fmaf(w, sigmoid_f(o[1 + c]), v[c]);
        dep = fmaf(w, (float)ray_t(ray, j), dep);
      }
      two_sum_add(tau, tau_e, ds);
      LP_PT(5)
    }
    if (valid) {                                                   // F7
      const float tauR = tau + tau_e;
      const float TR = expf(-tauR);
#pragma unroll
      for (int c = 0; c < kC; ++c) a.out[3 * r + c] = fmaf(TR, bg[c], v[c]);
      a.tau[r] = tauR;
      if (a.depth) a.depth[r] = dep;
    }
  }
  LP_PT_FLUSH(0)
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

// ================================================================= K2tc backward
template <int KIND, int K, int HID, int G, int T>
struct BwdTcSmem {
  using S = TcShape<KIND, K, HID>;
  static constexpr uint32_t W0P = 0;
  static constexpr uint32_t FP = W0P + 3 * S::W0_PIECE;
  static constexpr uint32_t GRP = (FP + TcParams<K, HID>::N * 4 + 127) & ~127u;
  static constexpr uint32_t H = 0;                             // [H | 1 | DO], 3 pieces
  static constexpr uint32_t DA = H + kBwdHPieces * S::HB_PIECE;  // [D1 | A1], 2 pieces; after the
                                                               // MMAs: fp32 dH staging + tap records
  static constexpr uint32_t PTAPS = DA + S::DA_PIECE;
  static constexpr uint32_t TAPS = DA + 2 * S::DA_PIECE;      // [T halves][128][NPL]
  static constexpr uint32_t XO = TAPS + T * S::TAPS;           // T = 2: [2][128] float4 partial outputs
  static constexpr uint32_t GSIZE = (XO + (T == 2 ? 2 * 128 * 16 : 0) + 127) & ~127u;
  static constexpr uint32_t BAR = GRP + G * GSIZE;             // 4 mbarriers per group + tmem slot
  static constexpr uint32_t BYTES = BAR + 32 * G + 16;
  static constexpr uint32_t TMEM_COLS = G == 1 ? 256 : 512;
  static_assert(S::DA_PIECE >= 128 * (K + 4) * 4 && S::DA_PIECE >= 128 * S::NPL * 16, "staging fits the DA tile");
};

// TMEM columns of a group (bwd): Z [0,64), dH [64,96), W [96,96+HC): M = 128 rows
// [D1 units | A1 units] x [channels | 1 | dout] -> dW0, db0 (rows < 64), dWo^T (rows >= 64)
// T threads per ray (1 or 2): with T = 2 thread (half, row) takes hidden units
// [half*HID/2, (half+1)*HID/2) of every epilogue and half of the gather
// iterations, as in lp_tc2_kernels.cuh; the halves exchange their partial
// output-layer sums through shared memory.
#ifndef LP_BWD_SW
#define LP_BWD_SW 4
#endif
// Scatter warps of K2tc (T = 1): the grid-gradient reductions (B6) of each staged
// step are issued by dedicated warps (SW / G per group) while the group's compute
// warps gather and contract the next step, so the L2 reductions are not in the
// compute warps' instruction stream. 0: the compute warps issue them inside the
// next step's gather (fused scatter).
constexpr int kBwdScatterWarps = LP_BWD_SW;
template <int T>
constexpr int bwd_scatter_warps() { return T == 1 ? kBwdScatterWarps : 0; }

template <int KIND, int K, int HID, int G, int T>
__global__ void __launch_bounds__(128 * T * G + 32 * bwd_scatter_warps<T>(), 1) lp_bwd_tc_kernel(const KernelArgs a) {
  using S = TcShape<KIND, K, HID>;
  using L = BwdTcSmem<KIND, K, HID, G, T>;
  constexpr int GT = 128 * T, HH = HID / T, KC = K / 4;
  static_assert(T == 1 || T == 2, "threads per ray");
  static_assert(HH % 8 == 0 && KC % T == 0, "per-half split");
  using F = TcParams<K, HID>;
  using P = PackedParams<K, HID, 1>;
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + 32 * G);
  constexpr int SW = bwd_scatter_warps<T>(), SWG = SW / G;
  static_assert(SW % G == 0 && (SW == 0 || 4 % SWG == 0), "scatter warps per group");

  const int g = threadIdx.x / GT, gt = threadIdx.x % GT, hf = gt >> 7, rt = gt & 127;
  const int wg = (gt >> 5) & 3, lane = gt & 31;
  const int it0 = hf * (KC / T), it1 = it0 + KC / T;
  uint8_t* gsm = smem + L::GRP + g * L::GSIZE;
  uint8_t* Ht = gsm + L::H;
  uint8_t* DAt = gsm + L::DA;
  float4* xo = reinterpret_cast<float4*>(gsm + L::XO);
  // fp32 dH rows and tap records of the previous step (its scatter is fused into the
  // next gather): DA tile, free between the MMA2 completion and the next epilogue
  float* dhs = reinterpret_cast<float*>(gsm + L::DA);
  float4* ptaps = reinterpret_cast<float4*>(gsm + L::PTAPS);
  bool pending = false;
  float4* taps = reinterpret_cast<float4*>(gsm + L::TAPS) + hf * 128 * S::NPL;

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tc_weights<K, HID, S::KP>(w0p, fp, a.params);
  // per group: Z done, dH/dW done (tcgen05.commit), staged (128 compute threads),
  // drained (the group's scatter warps)
  if (threadIdx.x < 4 * G) tc::mbar_init(&bars[threadIdx.x], threadIdx.x % 4 == 2 ? 128 : threadIdx.x % 4 == 3 ? (SWG > 0 ? 32 * SWG : 1) : 1);
  if (threadIdx.x < 32) tc::tmem_alloc(tslot, L::TMEM_COLS);
  tc::fence_async_smem();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  tc::fence_before_sync();
  __syncthreads();
  tc::fence_after_sync();
  if constexpr (SW > 0) {
    if (threadIdx.x >= GT * G) {   // ---- scatter warps: B6 of every step the group stages
      const int sw = (threadIdx.x - GT * G) / 32, lane = threadIdx.x & 31;
      const int sg = sw / SWG, part = sw % SWG;
      const uint8_t* sgsm = smem + L::GRP + sg * L::GSIZE;
      const float* sdhs = reinterpret_cast<const float*>(sgsm + L::DA);
      const float4* sptaps = reinterpret_cast<const float4*>(sgsm + L::PTAPS);
      float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
      uint32_t ph = 0;
      const int64_t nt = (a.M + 127) / 128;
      for (int64_t tile = (int64_t)blockIdx.x * G + sg; tile < nt; tile += (int64_t)gridDim.x * G)
        for (int q = 0; q < a.S; ++q) {
          tc::mbar_wait(&bars[4 * sg + 2], ph);
          ph ^= 1;
          for (int rb = part; rb < 4; rb += SWG) coop_scatter<KIND, K>(sgpl, sptaps, a.dims, sdhs, rb * 32, lane);
          __syncwarp();
          tc::mbar_arrive(&bars[4 * sg + 3]);   // every lane: its own reads of the staging precede it
        }
    }
  }
  if (SW == 0 || threadIdx.x < GT * G) {   // ---- compute warps
    const uint32_t tbase = *tslot + (uint32_t)(g * 256);
    const uint32_t tZ = tbase, tDH = tbase + 64, tW = tbase + 96;
    // ones column of the H tile (piece 0 = 1, pieces 1, 2 = 0; written once, never overwritten)
    if (hf == 0) *reinterpret_cast<__nv_bfloat16*>(Ht + tc::cm_off(rt, S::KP, S::HC)) = __float2bfloat16_rn(1.0f);
    tc::fence_async_smem();
    const uint32_t tlane = (uint32_t)(wg * 32) << 16;
    uint64_t* bar_z = &bars[4 * g];
    uint64_t* bar_d = &bars[4 * g + 1];
    uint64_t* bar_st = &bars[4 * g + 2];
    uint64_t* bar_dr = &bars[4 * g + 3];
    uint32_t dphase = 0;
    bool staged = false;   // a step of this group is staged for the scatter warps

    const int R = a.S - 1;
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    float* gplanes[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id_z = tc::idesc_bf16(128, HID, 0, 0);
    const uint32_t id_dh = tc::idesc_bf16(128, S::KP, 0, 1);
    const uint32_t id_w = tc::idesc_bf16(128, S::HC, 1, 1);
    const uint32_t h_addr = tc::smem_u32(Ht), w_addr = tc::smem_u32(w0p), da_addr = tc::smem_u32(DAt);
    uint32_t phase = 0, wacc = 0;   // wacc: weight-gradient accumulators initialised (issuing thread)
    float dbo[kOut];
#pragma unroll
    for (int i = 0; i < kOut; ++i) dbo[i] = 0.0f;
    LP_PT_DECL

    const int64_t ntiles = (a.M + 127) / 128;
    for (int64_t tile = (int64_t)blockIdx.x * G + g; tile < ntiles; tile += (int64_t)gridDim.x * G) {
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
        // ---- B2: recompute sample q: taps, cooperative gather, Z = H W0^T
        double x[3];
        sample_point(ray, q, a.contract, x);
        write_taps<KIND, K>(taps + rt * S::NPL, x, a.dims);
        __syncwarp();
        LP_PT(0)
        if (SW == 0 && pending)   // warp-uniform
          coop_gather<KIND, K, S::HC, kBwdHPieces, true>(planes, taps, a.dims, Ht, S::HB_PIECE, wg * 32, lane, gplanes, ptaps, dhs,
                                               it0, it1);
        else
          coop_gather<KIND, K, S::HC, kBwdHPieces>(planes, taps, a.dims, Ht, S::HB_PIECE, wg * 32, lane, nullptr, nullptr,
                                         nullptr, it0, it1);
        pending = false;
        LP_PT(1)
        tc::fence_async_smem();
        tc::fence_before_sync();
        tc::named_bar(1 + g, GT);
        LP_PT(2)
        if (gt == 0) {
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
          constexpr int NPROD = kBwdHPieces == 3 ? 6 : 5;   // products with H piece < kBwdHPieces
          uint32_t acc = 0;
#pragma unroll
          for (int ks = 0; ks < S::KP / 16; ++ks)
#pragma unroll
            for (int c = 0; c < NPROD; ++c) {
              tc::mma_bf16(tZ, tc::desc_kmajor(h_addr + PA[c] * S::HB_PIECE, S::HC, ks),
                           tc::desc_kmajor(w_addr + PB[c] * S::W0_PIECE, S::KP, ks), id_z, acc);
              acc = 1;
            }
          tc::mma_commit(bar_z);
        }
        tc::mbar_wait(bar_z, phase);
        LP_PT(3)
        tc::fence_after_sync();
        float a1[HH];
        tc::tmem_ld<HH>(tZ + tlane + (uint32_t)(hf * HH), a1);
        float o[kOut];
        if constexpr (T == 1) {
          tc_head_layer<HID>(fp + F::B0, fp + F::WOT, fp + F::BO, a1, o);   // a1 = relu(z + b0)
        } else {   // this half's units: a1 = relu(z + b0), partial output layer, exchange
          float4 part = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < HH; ++i) {
            a1[i] = fmaxf(a1[i] + fp[F::B0 + hf * HH + i], 0.0f);
            const float4 w = reinterpret_cast<const float4*>(fp + F::WOT)[hf * HH + i];
            part.x = fmaf(w.x, a1[i], part.x);
            part.y = fmaf(w.y, a1[i], part.y);
            part.z = fmaf(w.z, a1[i], part.z);
            part.w = fmaf(w.w, a1[i], part.w);
          }
          xo[hf * 128 + rt] = part;
          tc::fence_before_sync();
          tc::named_bar(1 + g, GT);
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
        // ---- B3: Eq. 3, log-domain reverse update (R12)
        const float tau_q = (tauR - U) - Ue;
        two_sum_add(U, Ue, ds);
        const float tau_qm1 = (tauR - U) - Ue;
        float aq = 0.0f;
#pragma unroll
        for (int c = 0; c < kC; ++c) aq = fmaf(p[c], col[c], aq);
        aq = fmaf(gdep, (float)ray_t(ray, q), aq);   // depth channel: "colour" t_q, no MLP gradient
        const float wq = q > 0 ? expf(-tau_qm1) * (-expm1f(-ds)) : 0.0f;
        const float Tq_aq = q > 0 ? expf(-tau_q) * aq : 0.0f;
        const float dsig = (float)ray.delta * (gtau - (G_ - Tq_aq));
        G_ = fmaf(wq, aq, G_);
        // ---- B4: head VJP
        float dout[8];
        dout[0] = dsig * s_sig;
#pragma unroll
        for (int c = 0; c < kC; ++c) dout[1 + c] = wq * p[c] * col[c] * (1.0f - col[c]);
#pragma unroll
        for (int c = 4; c < 8; ++c) dout[c] = 0.0f;
        // ---- B5: per 8-unit chunk: stage a1, delta1 = ReLU'(z) (Wo^T dout), stage delta1
        if (hf == 0) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(Ht, S::HB_PIECE, rt, S::KP + 8, S::HC, dout);
        }
        if (SW > 0 && staged) {   // the DA tile still holds the previous step's staging
          LP_PT(4)
          tc::mbar_wait(bar_dr, dphase);
          dphase ^= 1;
          LP_PT(7)
        }
#pragma unroll
        for (int c = 0; c < HH / 8; ++c) {
          tc::store8<2>(DAt, S::DA_PIECE, rt, S::HP + hf * HH + 8 * c, 2 * S::HP, a1 + 8 * c);
          float d1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w = reinterpret_cast<const float4*>(fp + F::WOT)[hf * HH + 8 * c + u];
            float sacc = w.x * dout[0];
            sacc = fmaf(w.y, dout[1], sacc);
            sacc = fmaf(w.z, dout[2], sacc);
            sacc = fmaf(w.w, dout[3], sacc);
            d1[u] = a1[8 * c + u] > 0.0f ? sacc : 0.0f;
          }
          tc::store8<2>(DAt, S::DA_PIECE, rt, hf * HH + 8 * c, 2 * S::HP, d1);
        }
        LP_PT(4)
        tc::fence_async_smem();
        tc::fence_before_sync();
        tc::named_bar(1 + g, GT);
        if (gt == 0) {
          tc::fence_after_sync();
          constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
          // dH = D1 W0   (B = W0 viewed MN-major: MN = channel, K = hidden)
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tDH, tc::desc_kmajor(da_addr + QA[c] * S::DA_PIECE, 2 * S::HP, ks),
                           tc::desc_mnmajor(w_addr + QB[c] * S::W0_PIECE, S::KP, ks), id_dh, (ks | c) != 0);
          // [dW0 | db0 | . ; . | dWo^T] += [D1 | A1]^T [H | 1 | DOUT]   (K = the 128 samples of this step)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW, tc::desc_mnmajor(da_addr + QA[c] * S::DA_PIECE, 2 * S::HP, ks),
                           tc::desc_mnmajor(h_addr + QB[c] * S::HB_PIECE, S::HC, ks), id_w, wacc);
              wacc = 1;
            }
          tc::mma_commit(bar_d);
        }
        tc::mbar_wait(bar_d, phase);
        phase ^= 1;
        LP_PT(5)
        tc::fence_after_sync();
        // ---- B6: dH row -> fp32 staging -> cooperative scatter
        {
          constexpr int HK = S::KP / T;   // this thread's dH columns
          float dh[HK];
          tc::tmem_ld<HK>(tDH + tlane + (uint32_t)(hf * HK), dh);
#pragma unroll
          for (int k4 = 0; k4 < HK / 4; ++k4)
            if (hf * HK + 4 * k4 < K)
              *reinterpret_cast<float4*>(dhs + rt * (K + 4) + hf * HK + 4 * k4) =
                  make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        tc::fence_before_sync();
        // keep this step's tap records for its scatter, fused into the next gather
        if (hf == 0) {
#pragma unroll
          for (int pp = 0; pp < S::NPL; ++pp) ptaps[rt * S::NPL + pp] = taps[rt * S::NPL + pp];
        }
        pending = true;
        if constexpr (SW > 0) {
          tc::mbar_arrive(bar_st);
          staged = true;
        } else if constexpr (T == 1) {
          __syncwarp();
        } else {
          tc::named_bar(1 + g, GT);   // the other half's warps read these rows
        }
        LP_PT(6)
      }
    }
    if (SW == 0 && pending) {   // the last step's scatter
      __syncwarp();
      coop_scatter<KIND, K>(gplanes, ptaps, a.dims, dhs, wg * 32, lane, it0, it1);
      __syncwarp();
    }
    LP_PT_FLUSH(1)

    // ---- B7: flush this group's gradient partials (TMEM accumulators + register bias sums)
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x * G + g < ntiles;
    if (hf == 0) {
      // M = 128 accumulator: row i lives in TMEM lane i (warp i / 32); rows [0, HP) are
      // hidden units of D1 (dW0, db0), rows [HP, 2 HP) hidden units of A1 (dWo^T)
      float wrow[S::HC];
      tc::tmem_ld<S::HC>(tW + tlane, wrow);
      const int row = 32 * wg + lane;
      if (had_tiles && row < HID) {
#pragma unroll
        for (int c = 0; c < K; ++c) atomicAdd(a.gparams + P::W0 + row * K + c, wrow[c]);
        atomicAdd(a.gparams + P::B0 + row, wrow[S::KP]);   // ones column: db0
      }
      if (had_tiles && row >= S::HP && row - S::HP < HID) {
#pragma unroll
        for (int rr = 0; rr < kOut; ++rr) atomicAdd(a.gparams + P::WO + rr * HID + (row - S::HP), wrow[S::KP + 8 + rr]);
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
  }   // compute warps
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

// ================================================================= K2tc backward, warp-specialised
// The K2tc2 producer design (lp_tc2_kernels.cuh, lp_bwd_tc2p_kernel) for one hidden layer:
// one 128-ray group per CTA with two threads per ray (thread (half, row) owns hidden units
// [half*HID/2, (half+1)*HID/2) of its ray's sample), four producer warps that compute the
// taps and gather the next step into the other buffer of a double-buffered [H | 1 | DO]
// tile, and four scatter warps that reduce each step's dH, staged over the H buffer once
// Z and the weight-gradient MMAs are done with it. The compute warps never load from the
// grid and never wait for the scatter; per step they run Z = H W0^T, the epilogue (a1,
// partial output layer, exchange, heads, Eq. 3, delta1) and one MMA round
// dH = D1 W0, [dW0 db0 . ; . dWo^T] += [D1 | A1]^T [H | 1 | DO].
#ifndef LP_BWDP_NB
#define LP_BWDP_NB 3
#endif
// H / taps buffers in the producer -> compute -> scatter ring. Two are not enough here: the
// cycle staging(n) -> scatter(n) -> gather(n + NB) -> Z(n + NB) spans the scatter, the gather and
// the compute chain, ~2.5 steps of the short one-hidden-layer chain (c4 bwd 424 ms with NB = 2).
constexpr int kBwdpBuffers = LP_BWDP_NB;

template <int KIND, int K, int HID>
struct BwdTcpSmem {
  using S = TcShape<KIND, K, HID>;
  static constexpr int NB = kBwdpBuffers;
  static constexpr uint32_t W0P = 0;
  static constexpr uint32_t FP = W0P + 3 * S::W0_PIECE;
  static constexpr uint32_t H = (FP + TcParams<K, HID>::N * 4 + 127) & ~127u;   // 2 buffers x 3 pieces
  static constexpr uint32_t DA = H + NB * 3 * S::HB_PIECE;                     // [D1 | A1], 2 pieces
  static constexpr uint32_t TAPS = DA + 2 * S::DA_PIECE;                       // NB buffers [128][NPL]
  static constexpr uint32_t XO = TAPS + NB * S::TAPS;                          // [2 halves][128] float4
  static constexpr uint32_t BAR = (XO + 2 * 128 * 16 + 127) & ~127u;
  // mbarriers: MMA, staged[NB], full[NB], empty[NB], MMA (dH half, LP_TCP_SPLIT); then the TMEM slot
  static constexpr uint32_t SLOT = 8 * (2 + 3 * NB);
  static constexpr uint32_t BYTES = BAR + SLOT + 16;
  static constexpr uint32_t TMEM_COLS = 256;
  static_assert(2 * S::HB_PIECE >= 128 * (K + 4) * 4, "dH staging fits pieces 0-1 of an H buffer");
  static_assert(BYTES <= 227 * 1024, "shared memory");
};

#ifndef LP_TCP_SPLIT   // commit dH ahead of the weight-gradient MMAs
#define LP_TCP_SPLIT 0
#endif
#ifndef LP_BWDP_SW   // scatter warps of K2tcp: 2 measured better than 4 (c4 bwd 354 -> 340 ms; c3, c5 neutral), 1 worse (514 ms)
#define LP_BWDP_SW 2
#endif
constexpr int kBwdpScatterWarps = LP_BWDP_SW;

template <int KIND, int K, int HID>
__global__ void __launch_bounds__(256 + 128 + 32 * kBwdpScatterWarps, 1) lp_bwd_tcp_kernel(const KernelArgs a) {
  using L = BwdTcpSmem<KIND, K, HID>;
  using S = TcShape<KIND, K, HID>;
  using F = TcParams<K, HID>;
  using P = PackedParams<K, HID, 1>;
  constexpr int HH = HID / 2, KP = S::KP, HC = S::HC, HP = S::HP, NPL = S::NPL;
  constexpr int SW = kBwdpScatterWarps, NB = L::NB;
  static_assert(SW > 0 && 4 % SW == 0, "scatter warps");
  static_assert(HH % 8 == 0, "per-half hidden units");
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* w0p = smem + L::W0P;
  float* fp = reinterpret_cast<float*>(smem + L::FP);
  uint8_t* DAt = smem + L::DA;
  float4* xo = reinterpret_cast<float4*>(smem + L::XO);
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::BAR);
  uint64_t* staged = bar + 1;        // [NB] 256 compute threads: dH of the step staged in H[b]
  uint64_t* full = bar + 1 + NB;     // [NB] 128 producer threads: H / taps buffer written
  uint64_t* empty = bar + 1 + 2 * NB;  // [NB] every lane of the scatter warps: staging + taps read
  uint64_t* bar2 = bar + 1 + 3 * NB;   // dH complete (LP_TCP_SPLIT)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(smem + L::BAR + L::SLOT);

  for (uint32_t i = threadIdx.x * 16; i < L::BAR; i += blockDim.x * 16)
    *reinterpret_cast<uint4*>(smem + i) = make_uint4(0, 0, 0, 0);
  __syncthreads();
  stage_tc_weights<K, HID, KP>(w0p, fp, a.params);
  if (threadIdx.x == 0) {
    tc::mbar_init(bar, 1);
    tc::mbar_init(bar2, 1);
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
  const int R = a.S - 1;
  const int64_t ntiles = (a.M + 127) / 128;

  if (threadIdx.x >= 384) {   // ---- scatter warps: B6 of every staged step
    const int sw = (threadIdx.x - 384) / 32, sl = threadIdx.x & 31;
    float* sgpl[3] = {a.ggrid[0], a.ggrid[1], a.ggrid[2]};
    uint32_t b = 0, ph = 0;   // ring position of the step and the parity of its use
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x)
      for (int q = 0; q < a.S; ++q) {
        tc::mbar_wait(&staged[b], ph);
        const float4* staps = reinterpret_cast<const float4*>(smem + L::TAPS + b * S::TAPS);
        const float* dhs = reinterpret_cast<const float*>(smem + L::H + b * 3 * S::HB_PIECE);
        for (int rb = sw; rb < 4; rb += SW) coop_scatter<KIND, K>(sgpl, staps, a.dims, dhs, rb * 32, sl);
        __syncwarp();
        tc::mbar_arrive(&empty[b]);   // every lane: its own reads of the staging / taps precede it
        if (++b == NB) b = 0, ph ^= 1;
      }
  } else if (threadIdx.x >= 256) {   // ---- producers: taps + cooperative gather, one step ahead
    const int pw = (threadIdx.x - 256) >> 5, lane = threadIdx.x & 31, row = pw * 32 + lane;
    const float* planes[3] = {a.grid[0], a.grid[1], a.grid[2]};
    uint32_t b = 0, ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t r0 = tile * 128 + ray_slot<K>(row);
      const RayIn ray = load_ray(a.orig, a.dir, a.tnear, a.tfar, r0 < a.M ? r0 : a.M - 1, R);
      for (int q = R; q >= 0; --q) {
        float4* taps = reinterpret_cast<float4*>(smem + L::TAPS + b * S::TAPS);
        uint8_t* Hb = smem + L::H + b * 3 * S::HB_PIECE;
        tc::mbar_wait(&empty[b], ph ^ 1);
        {   // the staging of step n - NB overwrote pieces 0-1: restore this row's zero padding
            // columns [K, KP) (K = 8) and its ones column block
#pragma unroll
          for (int c8 = K; c8 < KP; c8 += 8)
#pragma unroll
            for (int pc = 0; pc < 2; ++pc)
              *reinterpret_cast<uint4*>(Hb + pc * S::HB_PIECE + tc::cm_off(row, c8, HC)) = make_uint4(0u, 0u, 0u, 0u);
          const uint32_t off = tc::cm_off(row, KP, HC);
          *reinterpret_cast<uint4*>(Hb + off) = make_uint4(0x3F80u, 0u, 0u, 0u);   // bf16 1.0, then zeros
          *reinterpret_cast<uint4*>(Hb + S::HB_PIECE + off) = make_uint4(0u, 0u, 0u, 0u);
        }
        double x[3];
        sample_point(ray, q, a.contract, x);
        write_taps<KIND, K>(taps + row * NPL, x, a.dims);
        __syncwarp();
        coop_gather<KIND, K, HC, kBwdHPieces, false, true, LP_BWDP_UNROLL>(planes, taps, a.dims, Hb, S::HB_PIECE, pw * 32, lane);
        tc::fence_async_smem();
        tc::mbar_arrive(&full[b]);
        if (++b == NB) b = 0, ph ^= 1;
      }
    }
  } else {   // ---- compute warps
    const int gt = threadIdx.x, hf = gt >> 7, rt = gt & 127, wq = (gt >> 5) & 3, lane = gt & 31;
    const uint32_t tbase = *tslot;
    const uint32_t tZ = tbase, tDH = tbase + 64, tW = tbase + 96;
    const uint32_t tq = (uint32_t)(wq * 32) << 16;
    float bg[kC];
#pragma unroll
    for (int c = 0; c < kC; ++c) bg[c] = a.bg ? __ldg(a.bg + c) : 0.0f;
    const uint32_t id_z = tc::idesc_bf16(128, HID, 0, 0);
    const uint32_t id_dh = tc::idesc_bf16(128, KP, 0, 1);
    const uint32_t id_w = tc::idesc_bf16(128, HC, 1, 1);
    const uint32_t h_addr = tc::smem_u32(smem + L::H), w_addr = tc::smem_u32(w0p), da_addr = tc::smem_u32(DAt);
    // base descriptors (the issuing thread adds compile-time piece / K-step offsets)
    const uint64_t kH = tc::kdesc0(h_addr, HC), kW0 = tc::kdesc0(w_addr, KP), kDA = tc::kdesc0(da_addr, 2 * HP);
    const uint64_t mW0 = tc::mdesc0(w_addr, KP), mDA = tc::mdesc0(da_addr, 2 * HP), mH = tc::mdesc0(h_addr, HC);
    constexpr uint32_t MSDA = 2 * (2 * HP / 8) * 128, MSW0 = 2 * (KP / 8) * 128, MSH = 2 * (HC / 8) * 128;
    constexpr int QA[3] = {0, 0, 1}, QB[3] = {0, 1, 0};
    uint32_t phase = 0, phase2 = 0, wacc = 0, b = 0, bph = 0;   // bph: parity of this use of ring buffer b
    float dbo[kOut] = {0.0f, 0.0f, 0.0f, 0.0f};
    const float* b0 = fp + F::B0 + hf * HH;
    const float4* wot = reinterpret_cast<const float4*>(fp + F::WOT) + hf * HH;
    LP_PT_DECL

    auto mma_done = [&]() {
      tc::mbar_wait(bar, phase);
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
        uint8_t* Hb = smem + L::H + b * 3 * S::HB_PIECE;
        const uint64_t kHb = tc::dplus(kH, (uint32_t)(b * 3) * S::HB_PIECE);
        const uint64_t mHb = tc::dplus(mH, (uint32_t)(b * 3) * S::HB_PIECE);
        // ---- B2: Z = H W0^T on the producers' H tile of this step
        if (gt == 0) {
          tc::mbar_wait(&full[b], bph);
          tc::fence_after_sync();
          constexpr int PA[6] = {0, 0, 1, 0, 1, 2}, PB[6] = {0, 1, 0, 2, 1, 0};
          constexpr int NPROD = kBwdHPieces == 3 ? 6 : 5;
#pragma unroll
          for (int ks = 0; ks < KP / 16; ++ks)
#pragma unroll
            for (int c = 0; c < NPROD; ++c)
              tc::mma_bf16(tZ, tc::dplus(kHb, PA[c] * S::HB_PIECE + ks * 256),
                           tc::dplus(kW0, PB[c] * S::W0_PIECE + ks * 256), id_z, (ks | c) != 0);
          tc::mma_commit(bar);
        }
        mma_done();
        LP_PT(2)
        float a1[HH];
        {   // this half's units: a1 = relu(z + b0), partial output layer, exchange
          tc::tmem_ld<HH>(tZ + tq + (uint32_t)(hf * HH), a1);
          float4 part = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
#pragma unroll
          for (int i = 0; i < HH; ++i) {
            a1[i] = fmaxf(a1[i] + b0[i], 0.0f);
            const float4 w = wot[i];
            part.x = fmaf(w.x, a1[i], part.x);
            part.y = fmaf(w.y, a1[i], part.y);
            part.z = fmaf(w.z, a1[i], part.z);
            part.w = fmaf(w.w, a1[i], part.w);
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
        // ---- B5: dL/do -> H[b] columns [KP + 8, KP + 16); a1 and delta1 = ReLU'(z) (Wo^T dout) -> [D1 | A1]
        if (hf == 0) {
#pragma unroll
          for (int i = 0; i < kOut; ++i) dbo[i] += dout[i];
          tc::store8<2>(Hb, S::HB_PIECE, rt, KP + 8, HC, dout);
        }
#pragma unroll
        for (int c = 0; c < HH / 8; ++c) {
          tc::store8<2>(DAt, S::DA_PIECE, rt, HP + hf * HH + 8 * c, 2 * HP, a1 + 8 * c);
          float d1[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const float4 w = wot[8 * c + u];
            float sacc = w.x * dout[0];
            sacc = fmaf(w.y, dout[1], sacc);
            sacc = fmaf(w.z, dout[2], sacc);
            sacc = fmaf(w.w, dout[3], sacc);
            d1[u] = a1[8 * c + u] > 0.0f ? sacc : 0.0f;
          }
          tc::store8<2>(DAt, S::DA_PIECE, rt, hf * HH + 8 * c, 2 * HP, d1);
        }
        LP_PT(3)
        tc::fence_async_smem();
        tc::fence_before_sync();
        tc::named_bar(1, 256);
        if (gt == 0) {
          tc::fence_after_sync();
          // dH = D1 W0   (B = W0 viewed MN-major: MN = channel, K = hidden)
#pragma unroll
          for (int ks = 0; ks < HID / 16; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c)
              tc::mma_bf16(tDH, tc::dplus(kDA, QA[c] * S::DA_PIECE + ks * 256), tc::dplus(mW0, QB[c] * S::W0_PIECE + ks * MSW0),
                           id_dh, (ks | c) != 0);
          if constexpr (LP_TCP_SPLIT) tc::mma_commit(bar2);   // dH complete
          // [dW0 | db0 | . ; . | dWo^T] += [D1 | A1]^T [H | 1 | DOUT]   (K = the 128 samples of this step)
#pragma unroll
          for (int ks = 0; ks < 8; ++ks)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
              tc::mma_bf16(tW, tc::dplus(mDA, QA[c] * S::DA_PIECE + ks * MSDA), tc::dplus(mHb, QB[c] * S::HB_PIECE + ks * MSH),
                           id_w, wacc);
              wacc = 1;
            }
          tc::mma_commit(bar);
        }
        if constexpr (LP_TCP_SPLIT) {   // dH first: its TMEM loads overlap the dW MMAs
          tc::mbar_wait(bar2, phase2);
          phase2 ^= 1;
          tc::fence_after_sync();
        } else {
          mma_done();
        }
        LP_PT(4)
        // ---- B6: this half's dH channels -> fp32 staging over H[b] (Z and dW are done with it)
        {
          float* dhs_b = reinterpret_cast<float*>(Hb);
          constexpr int HK = KP / 2;
          float dh[HK];
          tc::tmem_ld<HK>(tDH + tq + (uint32_t)(hf * HK), dh);
          if constexpr (LP_TCP_SPLIT) mma_done();   // dW has read H[b]
#pragma unroll
          for (int k4 = 0; k4 < HK / 4; ++k4)
            if (hf * HK + 4 * k4 < K)
              *reinterpret_cast<float4*>(dhs_b + rt * (K + 4) + hf * HK + 4 * k4) =
                  make_float4(dh[4 * k4], dh[4 * k4 + 1], dh[4 * k4 + 2], dh[4 * k4 + 3]);
        }
        tc::mbar_arrive(&staged[b]);
        if (++b == NB) b = 0, bph ^= 1;
        LP_PT(3)
      }
    }
    LP_PT_FLUSH(1)

    // ---- B7: flush the weight-gradient accumulator (M = 128: row i in TMEM lane i; rows [0, HP)
    // D1 units -> dW0, db0 (ones column); rows [HP, 2 HP) A1 units -> dWo^T) and the bias sums
    tc::fence_after_sync();
    const bool had_tiles = (int64_t)blockIdx.x < ntiles;
    if (hf == 0) {
      float wrow[HC];
      tc::tmem_ld<HC>(tW + tq, wrow);
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
  }
  tc::fence_before_sync();
  __syncthreads();
  if (threadIdx.x < 32) {
    tc::fence_after_sync();
    tc::tmem_dealloc(*tslot, L::TMEM_COLS);
  }
}

}  // namespace lp
