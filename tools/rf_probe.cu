// Register-file probe of the FP32 pipe: which operand mixes of FFMA / FFMA2
// reach the pipe peak (register-only, no memory).  Every operand is a
// per-thread (vector-register) value unless the pattern says "uniform".
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rf_probe tools/rf_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_1805_11775_b200/csrc/hos_kernels.cuh"
using namespace hos;

// P: 0 scalar FFMA outer product 8x8
//    1 FFMA2 outer product, A pair, B pair (8x4 pairs)
//    2 FFMA2 outer product, A scalar broadcast, B pair
//    3 FFMA2 outer product, A scalar broadcast, B warp-uniform pair (peak probe form)
//    4 half scalar FFMA (8x4), half FFMA2 (4x4 pairs) interleaved
//    5 FFMA2 A pair, B pair, 4x8 pairs (A reused across 8)
//    6 scalar FFMA 4x16 (A reused across 16)
//    7 FFMA2 outer, i-inner ordering (B reused across 8 consecutive)
template <int P, int NT>
__global__ void __launch_bounds__(NT, 1) kp(float2* out, const float2* __restrict__ in, int iters, float s) {
  float a[8], bs[16];
  float2 a2[8], b2[8], acc[32];
  float accs[64];
  const float t = (float)threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = in[64 + 8 * threadIdx.x + i].x; a2[i] = in[8 * threadIdx.x + i]; }
#pragma unroll
  for (int j = 0; j < 8; j++) b2[j] = P == 3 ? in[j] : in[8192 + 8 * threadIdx.x + j];
#pragma unroll
  for (int j = 0; j < 16; j++) bs[j] = in[20000 + 16 * threadIdx.x + j].y;
#pragma unroll
  for (int c = 0; c < 32; c++) acc[c] = make_float2(0.f, 0.f);
#pragma unroll
  for (int c = 0; c < 64; c++) accs[c] = 0.f;
  for (int it = 0; it < iters; it++) {
    if (P == 0) {
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) accs[8 * i + j] = fmaf(a[i], bs[j], accs[8 * i + j]);
    } else if (P == 1) {
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[4 * i + j] = ffma2(a2[i], b2[j], acc[4 * i + j]);
    } else if (P == 2 || P == 3) {
#pragma unroll
      for (int i = 0; i < 8; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) acc[4 * i + j] = ffma2(make_float2(a[i], a[i]), b2[j], acc[4 * i + j]);
    } else if (P == 4) {
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 4; j++) {
          acc[4 * i + j] = ffma2(a2[i], b2[j], acc[4 * i + j]);
          accs[8 * i + 2 * j] = fmaf(a[i], bs[2 * j], accs[8 * i + 2 * j]);
          accs[8 * i + 2 * j + 1] = fmaf(a[i], bs[2 * j + 1], accs[8 * i + 2 * j + 1]);
        }
    } else if (P == 5) {
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 8; j++) acc[8 * i + j] = ffma2(a2[i], b2[j], acc[8 * i + j]);
    } else if (P == 6) {
#pragma unroll
      for (int i = 0; i < 4; i++)
#pragma unroll
        for (int j = 0; j < 16; j++) accs[16 * i + j] = fmaf(a[i], bs[j], accs[16 * i + j]);
    } else if (P == 8 || P == 9) {
      // K2 cell code on register operands: a2[0..3] = F(row), a2[4..7] = i F(row), b2[0..7] = F(col),
      // g from bs pairs.  P9: q-major (current kernel), P8: p formed column by column (scalar reuse)
      float2 (&aR)[32] = acc;
      float2* aI = reinterpret_cast<float2*>(accs);
      if (P == 9) {
#pragma unroll
        for (int q = 0; q < 11; q++) {
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int j = q - i;
            if (j < 0 || j > 7) continue;
            float2 p = fmul2(make_float2(b2[j].x, b2[j].x), a2[i]);
            p = ffma2(make_float2(b2[j].y, b2[j].y), make_float2(a2[4 + i].y, a2[4 + i].x), p);
            aR[8 * i + j] = ffma2(make_float2(bs[q], bs[q]), p, aR[8 * i + j]);
            aI[8 * i + j] = ffma2(make_float2(a[q % 8], a[q % 8]), p, aI[8 * i + j]);
          }
        }
      } else {
        float2 p[4][8];
#pragma unroll
        for (int q = 0; q < 11; q++) {
          if (q < 8) {
#pragma unroll
            for (int i = 0; i < 4; i++) p[i][q] = fmul2(make_float2(b2[q].x, b2[q].x), a2[i]);
#pragma unroll
            for (int i = 0; i < 4; i++)
              p[i][q] = ffma2(make_float2(b2[q].y, b2[q].y), make_float2(a2[4 + i].y, a2[4 + i].x), p[i][q]);
          }
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int j = q - i;
            if (j < 0 || j > 7) continue;
            aR[8 * i + j] = ffma2(make_float2(bs[q], bs[q]), p[i][j], aR[8 * i + j]);
          }
#pragma unroll
          for (int i = 0; i < 4; i++) {
            const int j = q - i;
            if (j < 0 || j > 7) continue;
            aI[8 * i + j] = ffma2(make_float2(a[q % 8], a[q % 8]), p[i][j], aI[8 * i + j]);
          }
        }
      }
    } else if (P == 7) {
#pragma unroll
      for (int j = 0; j < 4; j++)
#pragma unroll
        for (int i = 0; i < 8; i++) acc[4 * i + j] = ffma2(a2[i], b2[j], acc[4 * i + j]);
    }
  }
  float2 r = make_float2(0, 0);
#pragma unroll
  for (int c = 0; c < 32; c++) { r.x += acc[c].x; r.y += acc[c].y; }
#pragma unroll
  for (int c = 0; c < 64; c++) r.x += accs[c];
  out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}

template <int P, int NT>
void run(const char* name, float2* out, int lane_fma_per_iter) {
  const int iters = 4000;
  kp<P, NT><<<148, NT>>>(out, out + 148 * 1024, iters, 1.0001f);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9;
  for (int r = 0; r < 5; r++) {
    cudaEventRecord(a);
    kp<P, NT><<<148, NT>>>(out, out + 148 * 1024, iters, 1.0001f);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double tf = 148.0 * NT * iters * (double)lane_fma_per_iter * 2 / (best * 1e-3) / 1e12;
  printf("%-52s %2d warps/SM %6.2f TF/s %5.1f%% of 74.45  %s\n", name, NT / 32, tf, 100 * tf / 74.45,
         cudaGetErrorString(cudaGetLastError()));
}

#define RUN3(P, name, n)        \
  run<P, 256>(name, out, n);    \
  run<P, 512>(name, out, n);

int main() {
  float2* out;
  cudaMalloc(&out, 148 * 1024 * 8 + 8 * 65536);
  cudaMemset(out, 0, 148 * 1024 * 8 + 8 * 65536);
  RUN3(0, "P0 FFMA 8x8 outer (vector a, b)", 64)
  RUN3(6, "P6 FFMA 4x16 outer", 64)
  RUN3(1, "P1 FFMA2 8x4 pairs, A pair, B pair", 64)
  RUN3(7, "P7 FFMA2 as P1, B-major order", 64)
  RUN3(5, "P5 FFMA2 4x8 pairs", 64)
  RUN3(2, "P2 FFMA2 A scalar bcast, B pair", 64)
  RUN3(3, "P3 FFMA2 A scalar bcast, B uniform pair", 64)
  RUN3(4, "P4 mixed 16 FFMA2 + 32 FFMA", 64)
  run<9, 256>("P9 K2 cell code, q-major (kernel order)", out, 256);
  run<8, 256>("P8 K2 cell code, column-major p, scalar reuse", out, 256);
  return 0;
}
