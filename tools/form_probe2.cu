// Inner-loop ceilings of K2 cell formulations with fewer accumulator
// registers (so more warps fit per SM), operands already in shared memory.
// Exploration tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_11775_b200/csrc -o tools/form_probe2 tools/form_probe2.cu
// C48  : production form: 4x8 cells per lane, two accumulators per cell (aR += g.re p, aI += g.im p)
// C44  : 4x4 cells per lane, two accumulators per cell
// C48n : 4x8 cells, ONE complex accumulator, (g.im, -g.im) built by an FMUL2 per G value
// C48q : 4x8 cells, ONE complex accumulator, G staged as (re, im, im, -im) quads (LDS.128)
// FLAT : independent FFMA2s (pipe ceiling)
#include <cstdio>
#include <cuda_runtime.h>
#include "hos_kernels.cuh"
using namespace hos;

__device__ __forceinline__ float2 lds_conj(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  v.y = -v.y;
  return v;
}

__device__ __forceinline__ float2 lds_conj_x(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  v.y = __int_as_float(__float_as_int(v.y) ^ 0x80000000);
  return v;
}

// MODE 0: conj from a second load + FADD negation (production); 1: second load + sign-bit XOR (ALU pipe);
// 2: one load, conj built with XOR
template <int NI, int NJ, int MODE = 0>
__device__ __forceinline__ void cells2(const float2* __restrict__ rows, const float2* __restrict__ cols,
                                       const float2* __restrict__ gs, float2 (&aR)[NI][NJ], float2 (&aI)[NI][NJ]) {
  float2 fa[NI], fac[NI], fb[NJ];
#pragma unroll
  for (int i = 0; i < NI; i++) {
    fa[i] = rows[4 * i];
    if (MODE == 0) fac[i] = lds_conj(rows + 4 * i);
    if (MODE == 1) fac[i] = lds_conj_x(rows + 4 * i);
    if (MODE == 2) fac[i] = make_float2(fa[i].x, __int_as_float(__float_as_int(fa[i].y) ^ 0x80000000));
  }
#pragma unroll
  for (int j = 0; j < NJ; j++) fb[j] = cols[4 * j];
#pragma unroll
  for (int q = 0; q < NI + NJ - 1; q++) {
    const float2 g = gs[4 * q];
#pragma unroll
    for (int i = 0; i < NI; i++) {
      const int j = q - i;
      if (j < 0 || j >= NJ) continue;
      float2 p = fmul2(make_float2(fb[j].x, fb[j].x), fa[i]);
      p = ffma2(make_float2(fb[j].y, fb[j].y), make_float2(fac[i].y, fac[i].x), p);
      aR[i][j] = ffma2(make_float2(g.x, g.x), p, aR[i][j]);
      aI[i][j] = ffma2(make_float2(g.y, g.y), p, aI[i][j]);
    }
  }
}

// one accumulator: acc += p conj(g) = g.re (p.re, p.im) + (g.im, -g.im) (p.im, p.re)
template <bool QUAD>
__device__ __forceinline__ void cells1(const float2* __restrict__ rows, const float2* __restrict__ cols,
                                       const void* __restrict__ gs, float2 (&acc)[4][8]) {
  float2 fa[4], fac[4], fb[8];
#pragma unroll
  for (int i = 0; i < 4; i++) {
    fa[i] = rows[4 * i];
    fac[i] = lds_conj(rows + 4 * i);
  }
#pragma unroll
  for (int j = 0; j < 8; j++) fb[j] = cols[4 * j];
#pragma unroll
  for (int q = 0; q < 11; q++) {
    float gre;
    float2 gn;
    if (QUAD) {
      const float4 g = reinterpret_cast<const float4*>(gs)[4 * q];
      gre = g.x;
      gn = make_float2(g.z, g.w);
    } else {
      const float2 g = reinterpret_cast<const float2*>(gs)[4 * q];
      gre = g.x;
      gn = fmul2(make_float2(g.y, g.y), make_float2(1.f, -1.f));
    }
#pragma unroll
    for (int i = 0; i < 4; i++) {
      const int j = q - i;
      if (j < 0 || j > 7) continue;
      float2 p = fmul2(make_float2(fb[j].x, fb[j].x), fa[i]);
      p = ffma2(make_float2(fb[j].y, fb[j].y), make_float2(fac[i].y, fac[i].x), p);
      acc[i][j] = ffma2(make_float2(gre, gre), p, acc[i][j]);
      acc[i][j] = ffma2(gn, make_float2(p.y, p.x), acc[i][j]);
    }
  }
}

constexpr int NSEG = 4;
constexpr int TS = 104;  // tile stride (float2)

template <int MINB, int NJ, int MODE = 0>
__global__ void __launch_bounds__(128, MINB) k_c2(float2* out, int reps) {
  __shared__ float2 sm[4][NSEG * 2 * TS];  // per warp
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x & 31; i < NSEG * 2 * TS; i += 32) sm[warp][i] = make_float2(1e-3f * i, 1.f);
  __syncwarp();
  const int lane = threadIdx.x & 31, h = lane >> 4, ra = (lane >> 2) & 3, cb = lane & 3;
  float2 aR[4][NJ], aI[4][NJ];
  for (int i = 0; i < 4; i++) for (int j = 0; j < NJ; j++) aR[i][j] = aI[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps * 4 / NSEG * 8 / NJ; r++)
#pragma unroll
    for (int q = 0; q < NSEG; q++) {
      const float2* u = sm[warp] + q * 2 * TS + h * TS;
      cells2<4, NJ, MODE>(u + ra, u + 18 + cb, u + 52 + ra + cb, aR, aI);
    }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 4; i++) for (int j = 0; j < NJ; j++) { s.x += aR[i][j].x + aI[i][j].y; s.y += aR[i][j].y - aI[i][j].x; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MINB, bool QUAD>
__global__ void __launch_bounds__(128, MINB) k_c1(float2* out, int reps) {
  constexpr int GS = QUAD ? 2 : 1;  // float2 per G element
  constexpr int TSQ = 52 + GS * 52;
  __shared__ float2 sm[4][NSEG * 2 * TSQ];
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x & 31; i < NSEG * 2 * TSQ; i += 32) sm[warp][i] = make_float2(1e-3f * i, 1.f);
  __syncwarp();
  const int lane = threadIdx.x & 31, h = lane >> 4, ra = (lane >> 2) & 3, cb = lane & 3;
  float2 acc[4][8];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 8; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps * 4 / NSEG; r++)
#pragma unroll
    for (int q = 0; q < NSEG; q++) {
      const float2* u = sm[warp] + q * 2 * TSQ + h * TSQ;
      cells1<QUAD>(u + ra, u + 18 + cb, u + 52 + GS * (ra + cb), acc);
    }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 4; i++) for (int j = 0; j < 8; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_flat(float2* out, int reps) {
  const int lane = threadIdx.x & 31;
  float a[8];
  float2 b[4], acc[8][4];
  for (int i = 0; i < 8; i++) a[i] = 1e-3f * (lane + i);
  for (int j = 0; j < 4; j++) b[j] = make_float2(1e-3f * j, 1.f);
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps * 4 * 4; r++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i][j] = ffma2(make_float2(a[i], a[i]), b[j], acc[i][j]);
  }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

// flops_per_lane_rep: FFMA2-class instructions per lane per rep (x2 lanes x2 flops -> FMA lane-ops)
template <typename K>
void run(const char* name, K kern, double fma2_per_lane_rep, int sms, float2* buf) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  const int reps = 512;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int bps = 1; bps <= occ; bps++) {
    kern<<<sms * bps, 128>>>(buf, reps);
    cudaEventRecord(a);
    kern<<<sms * bps, 128>>>(buf, reps);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double lane_ops = (double)sms * bps * 128 * reps * fma2_per_lane_rep * 2;  // FMA lane-ops
    printf("%-6s regs=%3d occ=%d CTAs/SM=%d: FFMA-lane util %.1f%%\n", name, fa.numRegs, occ, bps,
           100.0 * lane_ops / (ms * 1e-3) / (148.0 * 128 * 1.965e9));
  }
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2* buf;
  cudaMalloc(&buf, sms * 16 * 128 * sizeof(float2));
  // useful FFMA2-class per lane per rep: 4 per cell, cells per rep = 32 x 4 (C48) ...
  run("FLAT", k_flat<4>, 8 * 4 * 16, sms, buf);
  run("C48", k_c2<2, 8>, 4 * 32 * 4, sms, buf);
  run("C48x", k_c2<2, 8, 1>, 4 * 32 * 4, sms, buf);
  run("C48s", k_c2<2, 8, 2>, 4 * 32 * 4, sms, buf);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
