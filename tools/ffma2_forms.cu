// FFMA2 operand-form issue-rate probe (register only, 32 independent accumulators per thread)
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1805_11775_b200/csrc/hos_kernels.cuh"
using namespace hos;

template <int F, int NT>
__global__ void __launch_bounds__(NT, 1) kf(float2* out, int iters, float s) {
  float sc[8];
  float2 w[8], v[4], acc[32];
#pragma unroll
  for (int i = 0; i < 8; i++) { sc[i] = s + i * threadIdx.x; w[i] = make_float2(s + i, s - i); }
#pragma unroll
  for (int i = 0; i < 4; i++) v[i] = make_float2(s * i, s + threadIdx.x);
#pragma unroll
  for (int c = 0; c < 32; c++) acc[c] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int c = 0; c < 32; c++) {
      if (F == 0) acc[c] = ffma2(make_float2(sc[c / 4], sc[c / 4]), v[c % 4], acc[c]);
      if (F == 1) acc[c] = ffma2(make_float2(-w[c / 4].x, w[c / 4].y), make_float2(v[c % 4].y, v[c % 4].x), acc[c]);
      if (F == 2) acc[c] = ffma2(w[c / 4], v[c % 4], acc[c]);
      if (F == 3) acc[c] = ffma2(make_float2(sc[c / 4], sc[c / 4]), make_float2(v[c % 4].y, v[c % 4].x), acc[c]);
      if (F == 4) acc[c] = ffma2(make_float2(sc[c % 8], sc[c % 8]), v[c / 8], acc[c]);
      if (F == 5) acc[c] = ffma2(w[c % 8], v[c / 8], acc[c]);
    }
  }
  float2 r = make_float2(0, 0);
#pragma unroll
  for (int c = 0; c < 32; c++) { r.x += acc[c].x; r.y += acc[c].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int F, int NT>
void run(const char* name, float2* out, int ctas_per_sm) {
  const int iters = 2000;
  const int grid = 148 * ctas_per_sm;
  kf<F, NT><<<grid, NT>>>(out, iters, 1.0001f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    kf<F, NT><<<grid, NT>>>(out, iters, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double tf = (double)grid * NT * iters * 32 * 4 / (best * 1e-3) / 1e12;
  printf("%-44s %4d warps/SM %6.2f TF/s %5.1f%%  %s\n", name, NT / 32 * ctas_per_sm, tf, 100 * tf / 73.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  float2* out;
  cudaMalloc(&out, 148 * 4 * 1024 * 8);
  run<0, 512>("F0 A=scalar(reuse-friendly), B=pair", out, 1);
  run<1, 512>("F1 A=pair.NP, B=pair swapped", out, 1);
  run<2, 512>("F2 A=pair, B=pair", out, 1);
  run<3, 512>("F3 A=scalar, B=pair swapped", out, 1);
  run<4, 512>("F4 A=scalar (cycling), B=pair (reuse)", out, 1);
  run<5, 512>("F5 A=pair (cycling), B=pair (reuse)", out, 1);
  run<0, 256>("F0 ", out, 4);
  run<2, 256>("F2 ", out, 4);
  return 0;
}
