// Throughput probe of the K2 cell code with operands in shared memory
// (no staging, no bookkeeping): % of the FFMA2 peak per variant.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cell_probe tools/cell_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1805_11775_b200/csrc/hos_kernels.cuh"
using namespace hos;

template <bool CONJ, int RS>
__device__ __forceinline__ void cells_q(const float4* __restrict__ rows, const float4* __restrict__ cols,
                                        const float4* __restrict__ gs, float2 (&acc)[4][8]) {
  float4 fa[4];
  float2 fb[8];
#pragma unroll
  for (int i = 0; i < 4; i++) fa[i] = rows[RS * i];
#pragma unroll
  for (int j = 0; j < 8; j++) fb[j] = *reinterpret_cast<const float2*>(cols + RS * j);
#pragma unroll
  for (int q = 0; q < 11; q++) {
    const float4 g = gs[RS * q];
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int j = q - i;
      if (j < 0 || j > 7) continue;
      float2 p = fmul2(make_float2(fa[i].x, fa[i].x), fb[j]);
      p = ffma2(make_float2(-fa[i].z, fa[i].w), make_float2(fb[j].y, fb[j].x), p);
      acc[i][j] = ffma2(make_float2(g.x, g.x), p, acc[i][j]);
      if (CONJ) acc[i][j] = ffma2(make_float2(g.z, -g.w), make_float2(p.y, p.x), acc[i][j]);
      else acc[i][j] = ffma2(make_float2(-g.z, g.w), make_float2(p.y, p.x), acc[i][j]);
    }
  }
}

// variant: UNR segments unrolled per loop trip, NW warps per CTA, MINB CTAs per SM
template <int UNR, int NW, int MINB>
__global__ void __launch_bounds__(32 * NW, MINB) kq(const float4* __restrict__ E, float2* out, int nseg, int Lp) {
  extern __shared__ float4 sm[];
  for (int i = threadIdx.x; i < 8 * Lp; i += blockDim.x) sm[i] = E[i % (4 * Lp)];
  __syncthreads();
  float2 acc[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.f, 0.f);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int h = lane / 16, ra = (lane / 4) % 4, cb = lane % 4;
  const int base = (h ? 4 * Lp + 4 : 0) + (warp % 8) * 32;  // copy B 64 bytes further in the banks
  const float4* rows = sm + base + ra;
  const float4* cols = sm + base + 64 + cb;
  const float4* gs = sm + base + 128 + ra + cb;
  for (int s = 0; s < nseg; s += 4) {
#pragma unroll UNR
    for (int t = 0; t < 4; t++) cells_q<true, 4>(rows + (t % 4) * Lp, cols + (t % 4) * Lp, gs + (t % 4) * Lp, acc);
  }
  float2 r = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) { r.x += acc[i][j].x; r.y += acc[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int UNR, int NW, int MINB>
void run(const char* name, const float4* E, float2* out, int Lp, double peak_tf) {
  auto k = kq<UNR, NW, MINB>;
  const size_t smem = 8 * (size_t)Lp * 16;
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
  printf("%-34s %8.3f ms  %6.2f TF/s (pipe)  %5.1f%% of FFMA2 peak  err=%s\n", name, best, tf, 100 * tf / peak_tf,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int Lp = 544;
  float4* E;
  float2* out;
  cudaMalloc(&E, 4 * Lp * 16);
  cudaMemset(E, 0, 4 * Lp * 16);
  cudaMalloc(&out, 148 * 4 * 1024 * 8);
  const double peak = 73.0;  // TF/s (hos_peak_fp32 on this pool)
  run<1, 16, 1>("quad unroll1 16w x1", E, out, Lp, peak);
  run<2, 16, 1>("quad unroll2 16w x1", E, out, Lp, peak);
  run<1, 8, 2>("quad unroll1 8w x2", E, out, Lp, peak);
  run<1, 12, 1>("quad unroll1 12w x1", E, out, Lp, peak);
  run<1, 8, 1>("quad unroll1 8w x1", E, out, Lp, peak);
  run<4, 8, 1>("quad unroll4 8w x1", E, out, Lp, peak);
  return 0;
}
