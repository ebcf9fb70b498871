// Inner-loop ceilings of candidate K2 cell formulations on operands already in
// shared memory (no staging).  Exploration tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_11775_b200/csrc -o tools/form_probe tools/form_probe.cu
// Q : quad layout (re, im, -im, re) for cols and G, 8x4 cells per lane, 1 accumulator per cell
// D : float2 everywhere, 8x2 cells per lane, 2 accumulators per cell (accR += gr p, accI += gi p)
#include <cstdio>
#include <cuda_runtime.h>
#include "hos_kernels.cuh"
using namespace hos;

__device__ __forceinline__ float2 neg_swap(float2 v) { return make_float2(-v.y, v.x); }

__device__ __forceinline__ void cells_q(const float4* __restrict__ rows, const float4* __restrict__ cols,
                                        const float4* __restrict__ gs, int ta, int tb, float2 (&acc)[8][4]) {
  float2 fa[8];
  float4 fb[4];
#pragma unroll
  for (int i = 0; i < 8; i++) fa[i] = *reinterpret_cast<const float2*>(rows + ta + 4 * i);
#pragma unroll
  for (int j = 0; j < 4; j++) fb[j] = cols[tb + 8 * j];
  const float4* gq = gs + ta + tb;
#pragma unroll
  for (int q = 0; q < 14; q++) {
    const float4 g = gq[4 * q];
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const int i = q - 2 * j;
      if (i < 0 || i > 7) continue;
      float2 p = fmul2(make_float2(fa[i].x, fa[i].x), make_float2(fb[j].x, fb[j].y));
      p = ffma2(make_float2(fa[i].y, fa[i].y), make_float2(fb[j].z, fb[j].w), p);
      acc[i][j] = ffma2(make_float2(p.x, p.x), make_float2(g.w, g.z), acc[i][j]);
      acc[i][j] = ffma2(make_float2(p.y, p.y), make_float2(g.y, g.x), acc[i][j]);
    }
  }
}

template <int NJ>
__device__ __forceinline__ void cells_d(const float2* __restrict__ rows, const float2* __restrict__ cols,
                                        const float2* __restrict__ gs, int ta, int tb, float2 (&aR)[8][NJ],
                                        float2 (&aI)[8][NJ]) {
  float2 fa[8], fb[NJ], fbn[NJ];
#pragma unroll
  for (int i = 0; i < 8; i++) fa[i] = rows[ta + 4 * i];
#pragma unroll
  for (int j = 0; j < NJ; j++) {
    fb[j] = cols[tb + 8 * j];
    fbn[j] = neg_swap(fb[j]);
  }
  const float2* gq = gs + ta + tb;
#pragma unroll
  for (int q = 0; q < 8 + 2 * (NJ - 1); q++) {
    const float2 g = gq[4 * q];
#pragma unroll
    for (int j = 0; j < NJ; j++) {
      const int i = q - 2 * j;
      if (i < 0 || i > 7) continue;
      float2 p = fmul2(make_float2(fa[i].x, fa[i].x), fb[j]);
      p = ffma2(make_float2(fa[i].y, fa[i].y), fbn[j], p);
      aR[i][j] = ffma2(make_float2(g.x, g.x), p, aR[i][j]);
      aI[i][j] = ffma2(make_float2(g.y, g.y), p, aI[i][j]);
    }
  }
}

// operands in registers: the FMUL2 -> FFMA2 -> FFMA2 -> FFMA2 chain alone
template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_qreg(float2* out, int reps) {
  const int lane = threadIdx.x & 31;
  float2 fa[8];
  float4 fb[4], g[14];
  for (int i = 0; i < 8; i++) fa[i] = make_float2(1e-3f * (lane + i), 1.f);
  for (int j = 0; j < 4; j++) fb[j] = make_float4(1e-3f * j, 1.f, -1.f, 1e-3f * j);
  for (int q = 0; q < 14; q++) g[q] = make_float4(1e-4f * q, 1.f, -1.f, 1e-4f * q + lane);
  float2 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps * 4; r++) {
#pragma unroll
    for (int q = 0; q < 14; q++) {
#pragma unroll
      for (int j = 0; j < 4; j++) {
        const int i = q - 2 * j;
        if (i < 0 || i > 7) continue;
        float2 p = fmul2(make_float2(fa[i].x, fa[i].x), make_float2(fb[j].x, fb[j].y));
        p = ffma2(make_float2(fa[i].y, fa[i].y), make_float2(fb[j].z, fb[j].w), p);
        acc[i][j] = ffma2(make_float2(p.x, p.x), make_float2(g[q].w, g[q].z), acc[i][j]);
        acc[i][j] = ffma2(make_float2(p.y, p.y), make_float2(g[q].y, g[q].x), acc[i][j]);
      }
    }
  }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

// independent FFMA2 only (peak-like), same operand forms
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

__device__ __forceinline__ float2 lds_conj(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"((unsigned)__cvta_generic_to_shared(p)));
  v.y = -v.y;
  return v;
}

// the production K2 cell code (4x8 lane tile, rows/cols/G step 4, conj rows from a second load)
__device__ __forceinline__ void cells_48(const float2* __restrict__ rows, const float2* __restrict__ cols,
                                         const float2* __restrict__ gs, float2 (&aR)[4][8], float2 (&aI)[4][8]) {
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
    const float2 g = gs[4 * q];
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

template <int MINB, int NSEG>
__global__ void __launch_bounds__(128, MINB) k_48(float2* out, int reps) {
  __shared__ float2 sm[NSEG * 208];
  for (int i = threadIdx.x; i < NSEG * 208; i += 128) sm[i] = make_float2(1e-3f * i, 1.f);
  __syncthreads();
  const int lane = threadIdx.x & 31, h = lane >> 4, ra = (lane >> 2) & 3, cb = lane & 3;
  float2 aR[4][8], aI[4][8];
  for (int i = 0; i < 4; i++) for (int j = 0; j < 8; j++) aR[i][j] = aI[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps * 4 / NSEG; r++)
#pragma unroll
    for (int q = 0; q < NSEG; q++) {
      const float2* u = sm + q * 208 + h * 104;
      cells_48(u + ra, u + 18 + cb, u + 52 + ra + cb, aR, aI);
    }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 4; i++) for (int j = 0; j < 8; j++) { s.x += aR[i][j].x + aI[i][j].y; s.y += aR[i][j].y - aI[i][j].x; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_q(float2* out, int reps) {
  __shared__ float4 sm[4 * 320];
  for (int i = threadIdx.x; i < 4 * 320; i += 128) sm[i] = make_float4(1e-3f * i, 1.f, -1.f, 1e-3f * i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ta = lane >> 3, tb = lane & 7;
  float2 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps; r++)
    for (int q = 0; q < 4; q++)
      cells_q(sm + q * 32, sm + 128 + q * 128 + warp * 32, sm + 640 + q * 159 + warp * 32, ta, tb, acc);
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MINB, int NJ>
__global__ void __launch_bounds__(128, MINB) k_d(float2* out, int reps) {
  __shared__ float2 sm[4 * 320];
  for (int i = threadIdx.x; i < 4 * 320; i += 128) sm[i] = make_float2(1e-3f * i, 1.f);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ta = lane >> 3, tb = lane & 7;
  float2 aR[8][NJ], aI[8][NJ];
  for (int i = 0; i < 8; i++) for (int j = 0; j < NJ; j++) aR[i][j] = aI[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps; r++)
    for (int q = 0; q < 4; q++)
      cells_d<NJ>(sm + q * 32, sm + 128 + q * 128 + warp * 32, sm + 640 + q * 159 + warp * 32, ta, tb, aR, aI);
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 8; i++) for (int j = 0; j < NJ; j++) { s.x += aR[i][j].x + aI[i][j].y; s.y += aR[i][j].y - aI[i][j].x; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <typename K>
void run(const char* name, K kern, int cells_per_lane, int sms, float2* buf) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, 128, 0);
  cudaFuncAttributes fa; cudaFuncGetAttributes(&fa, kern);
  const int reps = 512;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int bps = 1; bps <= occ; bps++) {
    kern<<<sms * bps, 128>>>(buf, reps);
    cudaEventRecord(a);
    kern<<<sms * bps, 128>>>(buf, reps);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double cells = (double)sms * bps * 128 * reps * 4 * cells_per_lane;
    printf("%-6s regs=%3d occ=%d CTAs/SM=%d: %.3e cells/s  FFMA-lane util %.1f%%\n", name, fa.numRegs, occ, bps,
           cells / (ms * 1e-3), 100.0 * cells * 8 / (ms * 1e-3) / (148.0 * 128 * 1.965e9));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2* buf; cudaMalloc(&buf, sms * 16 * 128 * sizeof(float2));
  run("C48x4", k_48<2, 4>, 32, sms, buf);
  run("C48x1", k_48<2, 1>, 32, sms, buf);
  run("FLAT", k_flat<3>, 32, sms, buf);
  run("QREG", k_qreg<3>, 32, sms, buf);
  run("Q", k_q<3>, 32, sms, buf);
  run("D2", k_d<4, 2>, 16, sms, buf);
  run("D2m3", k_d<3, 2>, 16, sms, buf);
  run("D4", k_d<2, 4>, 32, sms, buf);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
