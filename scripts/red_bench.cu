// red_bench.cu -- throughput of full-line (128 B) gradient scatters into a 24 MB fp32 buffer:
//   A: 8 lanes x red.global.add.v4.f32 per line (4 lines per warp instruction)
//   B: stage the line in shared memory, cp.reduce.async.bulk (UBLKRED) per line
//   gran <bytes> <MB>: A with <bytes>-granules (corner vectors of K = bytes/4 channels,
//   bytes/16 lanes each) at random granule-aligned offsets of a <MB> buffer -- the
//   ceilings of the K = 16 voxel grid (c2: 64 B into 128 MB) and of the 2 GiB c5 grid
//   seq: A on sequential lines (warp w reduces a contiguous run of lines): is the
//   random-line rate the ceiling, or do conflicts of random lines cost throughput?
//   gather <window_lines>: the forward's load side -- 8 lanes x LDG.128 per 128-B
//   line, 4 lines per warp instruction, 4 instructions in flight per lane, lines
//   drawn at random from a per-warp window of <window_lines> lines (small window:
//   every load hits L1 -> the L1 line-gather ceiling; 0 = random over the 24 MB
//   buffer -> L1 misses served by L2, the L2->SM gather ceiling)
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void redA(float* g, const int* lines, int nl_per_warp, int nlines_total) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int* L = lines + (size_t)warp * nl_per_warp;
  const int sub = lane >> 3, ch = lane & 7;
  for (int i = 0; i < nl_per_warp; i += 4) {
    int line = L[i + sub];
    float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    atomicAdd(reinterpret_cast<float4*>(g + (size_t)line * 32 + 4 * ch), v);
  }
}

__global__ void redB(float* g, const int* lines, int nl_per_warp, int nlines_total) {
  __shared__ __align__(128) float st[8][4][32];
  const int w = threadIdx.x >> 5, warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int* L = lines + (size_t)warp * nl_per_warp;
  const int sub = lane >> 3, ch = lane & 7;
  for (int i = 0; i < nl_per_warp; i += 4) {
    *reinterpret_cast<float4*>(&st[w][sub][4 * ch]) = make_float4(1.f, 1.f, 1.f, 1.f);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    if (lane < 4) {
      int line = L[i + lane];
      asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], 128;" ::"l"(g + (size_t)line * 32),
                   "r"((unsigned)__cvta_generic_to_shared(&st[w][lane][0]))
                   : "memory");
      asm volatile("cp.async.bulk.commit_group;");
      asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    }
    __syncwarp();
  }
}

__global__ void redG(float* g, const long long* offs, int n_per_warp, int lanes_per_gran) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31, per_inst = 32 / lanes_per_gran;
  const int sub = lane / lanes_per_gran, ch = lane % lanes_per_gran;
  const long long* L = offs + warp * n_per_warp;
  for (int i = 0; i < n_per_warp; i += per_inst) {
    float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    atomicAdd(reinterpret_cast<float4*>(g + L[i + sub] + 4 * ch), v);
  }
}

__global__ void redSeq(float* g, int nl_per_warp) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 3, ch = lane & 7;
  const size_t base = (size_t)warp * nl_per_warp;
  for (int i = 0; i < nl_per_warp; i += 4) {
    float4 v = make_float4(1.f, 1.f, 1.f, 1.f);
    atomicAdd(reinterpret_cast<float4*>(g + (base + i + sub) * 32 + 4 * ch), v);
  }
}

__global__ void gatherK(const float* __restrict__ g, const int* lines, int nl_per_warp, float* sink) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  const int* L = lines + (size_t)warp * nl_per_warp;
  const int sub = lane >> 3, ch = lane & 7;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = 0; i < nl_per_warp; i += 16) {
    float4 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = __ldg(reinterpret_cast<const float4*>(g + (size_t)L[i + 4 * u + sub] * 32 + 4 * ch));
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.f) sink[0] = acc.x;
}

static int gather_mode(int window) {
  const int nlines = 24 * 1024 * 1024 / 128;
  const int blocks = 148 * 4, threads = 256, warps = blocks * threads / 32, per = 4096;
  float *g, *sink; int* lines;
  cudaMalloc(&g, (size_t)nlines * 128); cudaMemset(g, 0, (size_t)nlines * 128);
  cudaMalloc(&sink, 4);
  cudaMalloc(&lines, (size_t)warps * per * 4);
  int* h = new int[(size_t)warps * per];
  uint32_t s = 7;
  for (int w = 0; w < warps; ++w)
    for (int i = 0; i < per; ++i) {
      s = s * 1664525u + 1013904223u;
      h[(size_t)w * per + i] = window > 0 ? (int)(((size_t)w * window + (s >> 4) % window) % nlines) : (int)((s >> 4) % nlines);
    }
  cudaMemcpy(lines, h, (size_t)warps * per * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    gatherK<<<blocks, threads>>>(g, lines, per, sink);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double nl = (double)warps * per;
    printf("gather window %6d lines: %.3f ms  %.2f G lines/s  %.2f TB/s  (%s)\n", window, ms, nl / ms / 1e6,
           nl * 128 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

static int seq_mode() {
  const int blocks = 148 * 4, threads = 256, warps = blocks * threads / 32, per = 64;
  float* g;
  cudaMalloc(&g, (size_t)warps * per * 128); cudaMemset(g, 0, (size_t)warps * per * 128);   // 24 MB
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    for (int k = 0; k < 64; ++k) redSeq<<<blocks, threads>>>(g, per);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double nl = (double)warps * per * 64;
    printf("seq lines (24 MB, 64 launches): %.3f ms  %.2f G lines/s  %.2f TB/s payload  (%s)\n", ms, nl / ms / 1e6,
           nl * 128 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

static int gran_mode(int gbytes, long long mb) {
  const long long nfl = mb * 1024 * 1024 / 4, ngran = nfl / (gbytes / 4);
  const int blocks = 148 * 4, threads = 256, warps = blocks * threads / 32, per = 4096;
  float* g; long long* offs;
  if (cudaMalloc(&g, (size_t)nfl * 4) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(g, 0, (size_t)nfl * 4);
  cudaMalloc(&offs, (size_t)warps * per * 8);
  long long* h = new long long[(size_t)warps * per];
  unsigned long long s = 88172645463325252ull;
  for (size_t i = 0; i < (size_t)warps * per; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    h[i] = (long long)(s % (unsigned long long)ngran) * (gbytes / 4);
  }
  cudaMemcpy(offs, h, (size_t)warps * per * 8, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    redG<<<blocks, threads>>>(g, offs, per, gbytes / 16);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double n = (double)warps * per;
    printf("gran %3d B into %5lld MB: %.3f ms  %.2f G granules/s  %.2f TB/s payload  (%s)\n", gbytes, mb, ms,
           n / ms / 1e6, n * gbytes / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 3 && argv[1][0] == 'g' && argv[1][1] == 'r') return gran_mode(atoi(argv[2]), atoll(argv[3]));
  if (argc > 2 && argv[1][0] == 'g' && argv[1][1] == 'a') return gather_mode(atoi(argv[2]));
  if (argc > 1 && argv[1][0] == 's' && argv[1][1] == 'e') return seq_mode();
  // usage: red_bench [n_sm]  -- with n_sm < 148: one 1024-thread block per SM on n_sm SMs
  // (per-SM scaling of the reduction rate); default: 4 x 256-thread blocks per SM on all 148
  const int nlines = 24 * 1024 * 1024 / 128;  // 24 MB buffer
  const int n_sm = argc > 1 ? atoi(argv[1]) : 148;
  const int blocks = argc > 1 ? n_sm : 148 * 4, threads = argc > 1 ? 1024 : 256, warps = blocks * threads / 32;
  const int per = 4096;
  float* g; int* lines;
  cudaMalloc(&g, (size_t)nlines * 128); cudaMemset(g, 0, (size_t)nlines * 128);
  cudaMalloc(&lines, (size_t)warps * per * 4);
  int* h = new int[(size_t)warps * per];
  uint32_t s = 1;
  for (size_t i = 0; i < (size_t)warps * per; ++i) { s = s * 1664525u + 1013904223u; h[i] = (s >> 4) % nlines; }
  cudaMemcpy(lines, h, (size_t)warps * per * 4, cudaMemcpyHostToDevice);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int v = 0; v < 2; ++v) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (v == 0) redA<<<blocks, threads>>>(g, lines, per, nlines); else redB<<<blocks, threads>>>(g, lines, per, nlines);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double nl = (double)warps * per;
      printf("%s: %.3f ms  %.2f G lines/s  %.2f TB/s payload  (%s)\n", v == 0 ? "A red.v4 x8 lanes" : "B bulk reduce   ", ms,
             nl / ms / 1e6, nl * 128 / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
