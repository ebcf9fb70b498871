// FFMA2 issue-rate probe: which operand forms / dependency shapes reach the
// FP32 pipe peak (16 warps per SM, register-only, no memory).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ffma2_probe tools/ffma2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1805_11775_b200/csrc/hos_kernels.cuh"
using namespace hos;

// T: 0 = scalar A, pair B (peak-probe form); 1 = pair A with .NP, swapped B;
//    2 = cell chain FMUL2 -> FFMA2 -> FFMA2 -> FFMA2 (quad cells, register operands);
//    3 = cell chain of the old 4-float form (all-scalar A)
template <int T>
__global__ void __launch_bounds__(512, 1) kp(float2* out, int iters, float s) {
  float4 fa[4];
  float2 fb[8];
  float4 g[11];
  float2 acc[4][8], acc2[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++) fa[i] = make_float4(s + i, s * i, s - i, s * 0.5f + i);
#pragma unroll
  for (int j = 0; j < 8; j++) fb[j] = make_float2(s + j, s * j + threadIdx.x);
#pragma unroll
  for (int q = 0; q < 11; q++) g[q] = make_float4(s + q, s * q, s * q, s - q);
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = acc2[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int q = 0; q < 11; q++) {
#pragma unroll
      for (int i = 0; i < 4; i++) {
        const int j = q - i;
        if (j < 0 || j > 7) continue;
        if (T == 0) {
#pragma unroll
          for (int r = 0; r < 4; r++) acc[i][j] = ffma2(make_float2(g[q].x + r, g[q].x + r), fb[j], acc[i][j]);
        } else if (T == 1) {
#pragma unroll
          for (int r = 0; r < 4; r++)
            acc[i][j] = ffma2(make_float2(-fa[i].z, fa[i].w), make_float2(fb[j].y, fb[j].x), acc[i][j]);
        } else if (T == 2) {
          float2 p = fmul2(make_float2(fa[i].x, fa[i].x), fb[j]);
          p = ffma2(make_float2(-fa[i].z, fa[i].w), make_float2(fb[j].y, fb[j].x), p);
          acc[i][j] = ffma2(make_float2(g[q].x, g[q].x), p, acc[i][j]);
          acc[i][j] = ffma2(make_float2(g[q].z, -g[q].w), make_float2(p.y, p.x), acc[i][j]);
        } else {
          float2 p = fmul2(make_float2(fb[j].x, fb[j].x), make_float2(fa[i].x, fa[i].y));
          p = ffma2(make_float2(fb[j].y, fb[j].y), make_float2(fa[i].z, fa[i].w), p);
          acc[i][j] = ffma2(make_float2(g[q].x, g[q].x), p, acc[i][j]);
          acc2[i][j] = ffma2(make_float2(g[q].y, g[q].y), p, acc2[i][j]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < 8; j++) fb[j].x += 1e-7f;  // keep the loop honest
  }
  float2 r = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) { r.x += acc[i][j].x + acc2[i][j].x; r.y += acc[i][j].y + acc2[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int T>
void run(const char* name, float2* out, int nw) {
  const int iters = 400;
  kp<T><<<148, 32 * nw>>>(out, iters, 1.0001f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    kp<T><<<148, 32 * nw>>>(out, iters, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double instr = 148.0 * nw * 32 * iters * 128 + 148.0 * nw * 32 * iters * 8;  // FMA-pipe lane instr
  const double tf = instr * 4 / (best * 1e-3) / 1e12;
  printf("%-40s %2d warps %7.3f ms %6.2f TF/s %5.1f%% of 73 TF/s  %s\n", name, nw, best, tf, 100 * tf / 73.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float2* out;
  cudaMalloc(&out, 148 * 512 * 8);
  for (int nw : {8, 16}) {
    run<0>("T0 scalar A, pair B", out, nw);
    run<1>("T1 pair A .NP, swapped B", out, nw);
    run<2>("T2 quad cell chain", out, nw);
    run<3>("T3 old 4-float cell chain", out, nw);
  }
  return 0;
}
