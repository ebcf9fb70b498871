// Throughput probe of K2 cell-code variants with float2 rows in shared memory
// (no staging, no bookkeeping): % of the FFMA2 peak.
//   A: two accumulators per cell (the kernel's cells_f32), 8 warps x 1 CTA/SM
//   B: ONE accumulator per cell, (-+g.im, +-g.im) pair built once per G value, 16 warps
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cell_probe2 tools/cell_probe2.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1805_11775_b200/csrc/hos_kernels.cuh"
using namespace hos;

__device__ __forceinline__ float2 lds_conj(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  v.y = -v.y;
  return v;
}

template <int RS>
__device__ __forceinline__ void cells_two(const float2* rows, const float2* cols, const float2* gs, float2 (&aR)[4][8],
                                          float2 (&aI)[4][8]) {
  float2 fa[4], fac[4], fb[8];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    fa[i] = rows[RS * i];
    fac[i] = lds_conj(rows + RS * i);
  }
#pragma unroll
  for (int j = 0; j < 8; j++) fb[j] = cols[RS * j];
#pragma unroll
  for (int q = 0; q < 11; q++) {
    const float2 g = gs[RS * q];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int j = q - i;
      if (j < 0 || j > 7) continue;
      float2 p = fmul2(make_float2(fb[j].x, fb[j].x), fa[i]);
      p = ffma2(make_float2(fb[j].y, fb[j].y), make_float2(fac[i].y, fac[i].x), p);
      aR[i][j] = ffma2(make_float2(g.x, g.x), p, aR[i][j]);
      aI[i][j] = ffma2(make_float2(g.y, g.y), p, aI[i][j]);
    }
  }
}

// one accumulator: acc += p conj(G) = g.x * p + (g.y, -g.y) * (p.y, p.x)
template <int RS>
__device__ __forceinline__ void cells_one(const float2* rows, const float2* cols, const float2* gs, float2 (&acc)[4][8]) {
  float2 fa[4], fac[4], fb[8];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    fa[i] = rows[RS * i];
    fac[i] = lds_conj(rows + RS * i);
  }
#pragma unroll
  for (int j = 0; j < 8; j++) fb[j] = cols[RS * j];
#pragma unroll
  for (int q = 0; q < 11; q++) {
    const float2 g = gs[RS * q];
    const float2 gy = make_float2(g.y, -g.y);
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int j = q - i;
      if (j < 0 || j > 7) continue;
      float2 p = fmul2(make_float2(fb[j].x, fb[j].x), fa[i]);
      p = ffma2(make_float2(fb[j].y, fb[j].y), make_float2(fac[i].y, fac[i].x), p);
      acc[i][j] = ffma2(make_float2(g.x, g.x), p, acc[i][j]);
      acc[i][j] = ffma2(gy, make_float2(p.y, p.x), acc[i][j]);
    }
  }
}

template <int V, int NW, int MINB, int UNR>
__global__ void __launch_bounds__(32 * NW, MINB) kc(const float2* __restrict__ E, float2* out, int nseg, int Lp) {
  extern __shared__ float2 smf[];
  for (int i = threadIdx.x; i < 8 * Lp; i += blockDim.x) smf[i] = E[i % (4 * Lp)];
  __syncthreads();
  float2 acc[4][8], acc2[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = acc2[i][j] = make_float2(0.f, 0.f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane / 16, ra = (lane / 4) % 4, cb = lane % 4;
  const int base = (h ? 4 * Lp + 8 : 0) + (warp % 8) * 32;  // copy B 64 bytes further in the banks
  const float2* rows = smf + base + ra;
  const float2* cols = smf + base + 64 + cb;
  const float2* gs = smf + base + 128 + ra + cb;
  for (int s = 0; s < nseg; s += 4) {
#pragma unroll UNR
    for (int t = 0; t < 4; t++) {
      if (V == 0) cells_two<4>(rows + t * Lp, cols + t * Lp, gs + t * Lp, acc, acc2);
      else cells_one<4>(rows + t * Lp, cols + t * Lp, gs + t * Lp, acc);
    }
  }
  float2 r = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) { r.x += acc[i][j].x + acc2[i][j].x; r.y += acc[i][j].y + acc2[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int V, int NW, int MINB, int UNR>
void run(const char* name, const float2* E, float2* out, int Lp, double peak_tf) {
  auto k = kc<V, NW, MINB, UNR>;
  const size_t smem = 8 * (size_t)Lp * 8;
  cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = 148 * MINB, nseg = 2048;
  k<<<grid, 32 * NW, smem>>>(E, out, nseg, Lp);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    k<<<grid, 32 * NW, smem>>>(E, out, nseg, Lp);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double fma_instr = (double)grid * NW * 32 * nseg * 128;  // lane FMA-pipe instructions (x2 flops x2 lanes)
  const double tf = fma_instr * 4 / (best * 1e-3) / 1e12;
  printf("%-44s %8.3f ms  %6.2f TF/s (pipe)  %5.1f%% of FFMA2 peak  err=%s\n", name, best, tf, 100 * tf / peak_tf,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int Lp = 544;
  float2 *E, *out;
  cudaMalloc(&E, 4 * Lp * 8);
  cudaMemset(E, 0, 4 * Lp * 8);
  cudaMalloc(&out, 148 * 4 * 1024 * 8);
  const double peak = 73.0;
  run<0, 8, 1, 4>("A two acc, 8 warps, unroll 4 (kernel)", E, out, Lp, peak);
  run<0, 8, 1, 1>("A two acc, 8 warps, unroll 1", E, out, Lp, peak);
  run<1, 8, 1, 4>("B one acc, 8 warps, unroll 4", E, out, Lp, peak);
  run<1, 16, 1, 1>("B one acc, 16 warps, unroll 1", E, out, Lp, peak);
  run<1, 16, 1, 2>("B one acc, 16 warps, unroll 2", E, out, Lp, peak);
  run<1, 16, 1, 4>("B one acc, 16 warps, unroll 4", E, out, Lp, peak);
  run<1, 12, 1, 2>("B one acc, 12 warps, unroll 2", E, out, Lp, peak);
  run<1, 8, 2, 2>("B one acc, 8 warps x 2 CTAs, unroll 2", E, out, Lp, peak);
  run<0, 12, 1, 1>("A two acc, 12 warps (168 regs), unroll 1", E, out, Lp, peak);
  run<0, 12, 1, 2>("A two acc, 12 warps (168 regs), unroll 2", E, out, Lp, peak);
  run<0, 4, 1, 4>("A two acc, 4 warps (one per sub-partition)", E, out, Lp, peak);
  return 0;
}
