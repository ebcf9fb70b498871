// Inner-loop ceiling: cells_f32 (copied from hos_kernels.cu) on operands already
// in shared memory, no TMA / no pipeline.  Exploration tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_11775_b200/csrc -o tools/loop_probe tools/loop_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "hos_kernels.cuh"
using namespace hos;
// one segment of a lane's 8x4 micro-tile: rows/cols/g point at the segment's staged factors
template <bool CONJ, bool ORDER4>
__device__ __forceinline__ void cells_f32(const float4* __restrict__ rows, const float4* __restrict__ cols,
                                          const float4* __restrict__ gs, const float4* __restrict__ plane, int ta,
                                          int tb, float2 (&acc)[8][4]) {
  float2 fa[8];
  float4 fb[4];
#pragma unroll
  for (int i = 0; i < 8; i++) fa[i] = *reinterpret_cast<const float2*>(rows + ta + 4 * i);
  if (ORDER4) {
    const float4 pa = *plane;
#pragma unroll
    for (int i = 0; i < 8; i++) {
      float2 t = fmul2(make_float2(fa[i].x, fa[i].x), make_float2(pa.x, pa.y));
      fa[i] = ffma2(make_float2(fa[i].y, fa[i].y), make_float2(pa.z, pa.w), t);
    }
  }
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
      if (CONJ) {
        acc[i][j] = ffma2(make_float2(p.x, p.x), make_float2(g.w, g.z), acc[i][j]);
        acc[i][j] = ffma2(make_float2(p.y, p.y), make_float2(g.y, g.x), acc[i][j]);
      } else {
        acc[i][j] = ffma2(make_float2(p.x, p.x), make_float2(g.x, g.y), acc[i][j]);
        acc[i][j] = ffma2(make_float2(p.y, p.y), make_float2(g.z, g.w), acc[i][j]);
      }
    }
  }
}


template <int MINB>
__global__ void __launch_bounds__(128, MINB) k_loop(float2* out, int reps) {
  __shared__ float4 sm[4 * 320];
  for (int i = threadIdx.x; i < 4 * 320; i += 128) sm[i] = make_float4(1e-3f * i, 1.f, -1.f, 1e-3f * i);
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, ta = lane >> 3, tb = lane & 7;
  float2 acc[8][4];
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int r = 0; r < reps; r++)
    for (int q = 0; q < 4; q++)
      cells_f32<true, false>(sm + q * 32, sm + 128 + q * 128 + warp * 32, sm + 640 + q * 159 + warp * 32, sm, ta, tb, acc);
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 8; i++) for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * 128 + threadIdx.x] = s;
}

template <int MINB>
void run(int sms, float2* buf) {
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_loop<MINB>, 128, 0);
  const int reps = 512;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int blocks_per_sm = 1; blocks_per_sm <= occ; blocks_per_sm++) {
    k_loop<MINB><<<sms * blocks_per_sm, 128>>>(buf, reps);
    cudaEventRecord(a);
    k_loop<MINB><<<sms * blocks_per_sm, 128>>>(buf, reps);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double cells = (double)sms * blocks_per_sm * 4 /*warps*/ * reps * 4 /*segs*/ * 1024;
    const double lane_fma = cells * 8;  // 4 FFMA2-class per cell = 8 lane FMAs
    printf("MINB=%d occ=%d CTAs/SM=%d: %.3e cells/s  FFMA-lane util %.1f%% of 148x128x1.965GHz\n", MINB, occ,
           blocks_per_sm, cells / (ms * 1e-3), 100.0 * lane_fma / (ms * 1e-3) / (148.0 * 128 * 1.965e9));
  }
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  float2* buf; cudaMalloc(&buf, sms * 16 * 128 * sizeof(float2));
  run<1>(sms, buf);
  run<4>(sms, buf);
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
}
