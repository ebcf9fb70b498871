// FP32 / FFMA2 / FP64 pipe microbenchmarks for the triple-product roofline.
// Standalone exploration tool (the live peak used by bench.py is the
// hos_peak_* entry point of the product library).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp_pipes tools/fp_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b),
                     rc = *reinterpret_cast<unsigned long long*>(&c), rd;
  asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(rd) : "l"(ra), "l"(rb), "l"(rc));
  return *reinterpret_cast<float2*>(&rd);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long ra = *reinterpret_cast<unsigned long long*>(&a), rb = *reinterpret_cast<unsigned long long*>(&b), rd;
  asm volatile("mul.rn.f32x2 %0, %1, %2;" : "=l"(rd) : "l"(ra), "l"(rb));
  return *reinterpret_cast<float2*>(&rd);
}

__device__ unsigned long long g_clk[2];

// 1: 3-register outer product, 8x8 accumulators (SGEMM style)
__global__ void k_outer(float* out, int iters, float seed) {
  float a[8], b[8], acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; i++) { a[i] = seed + i * threadIdx.x; b[i] = seed * i + 1.0f; }
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) acc[i][j] = 0.f;
  long long t0 = clock64();
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
  }
  long long t1 = clock64();
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (blockIdx.x == 0 && threadIdx.x == 0) { g_clk[0] = t1 - t0; }
}

// 2: FFMA2 complex MAC, 8x4 complex cells: acc += (fa*fb)*conj(g)  (4 FFMA2 per cell)
__global__ void k_tri2(float2* out, int iters, float seed) {
  float2 fa[8], fb[4], fbr[4], g[11], gc[11], acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++) fa[i] = make_float2(seed + i, seed - threadIdx.x);
#pragma unroll
  for (int j = 0; j < 4; j++) { fb[j] = make_float2(seed * j, 1.f + j); fbr[j] = make_float2(-fb[j].y, fb[j].x); }
#pragma unroll
  for (int t = 0; t < 11; t++) { g[t] = make_float2(seed + t * 0.5f, seed * t); gc[t] = make_float2(g[t].x, -g[t].y); }
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        float2 p = fmul2(make_float2(fa[i].x, fa[i].x), fb[j]);
        p = ffma2(make_float2(fa[i].y, fa[i].y), fbr[j], p);
        acc[i][j] = ffma2(make_float2(p.x, p.x), gc[i + j], acc[i][j]);
        acc[i][j] = ffma2(make_float2(p.y, p.y), make_float2(g[i + j].y, g[i + j].x), acc[i][j]);
      }
  }
  float2 s = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 3: scalar complex triple product, 8x4 cells (2 FMUL + 6 FFMA per cell)
__global__ void k_tri1(float2* out, int iters, float seed) {
  float2 fa[8], fb[4], g[11], acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++) fa[i] = make_float2(seed + i, seed - threadIdx.x);
#pragma unroll
  for (int j = 0; j < 4; j++) fb[j] = make_float2(seed * j, 1.f + j);
#pragma unroll
  for (int t = 0; t < 11; t++) g[t] = make_float2(seed + t * 0.5f, seed * t);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) {
        float pr = fa[i].x * fb[j].x;
        pr = fmaf(-fa[i].y, fb[j].y, pr);
        float pi = fa[i].x * fb[j].y;
        pi = fmaf(fa[i].y, fb[j].x, pi);
        float2 c = g[i + j];
        acc[i][j].x = fmaf(pr, c.x, acc[i][j].x);
        acc[i][j].x = fmaf(pi, c.y, acc[i][j].x);
        acc[i][j].y = fmaf(pi, c.x, acc[i][j].y);
        acc[i][j].y = fmaf(-pr, c.y, acc[i][j].y);
      }
  }
  float2 s = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 4: FFMA2 plain outer product 8x8 pairs (peak FFMA2 issue)
__global__ void k_outer2(float2* out, int iters, float seed) {
  float a[8]; float2 b[4], acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; i++) a[i] = seed + i * threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; j++) b[j] = make_float2(seed * j + 1.f, seed - j);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = make_float2(0.f, 0.f);
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 8; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i][j] = ffma2(make_float2(a[i], a[i]), b[j], acc[i][j]);
  }
  float2 s = make_float2(0, 0);
#pragma unroll
  for (int i = 0; i < 8; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) { s.x += acc[i][j].x; s.y += acc[i][j].y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// 5: DFMA outer product 4x4
__global__ void k_dfma(double* out, int iters, double seed) {
  double a[4], b[4], acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; i++) { a[i] = seed + i * threadIdx.x; b[i] = seed * i + 1.0; }
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) acc[i][j] = 0.;
  for (int it = 0; it < iters; it++) {
#pragma unroll
    for (int i = 0; i < 4; i++)
#pragma unroll
      for (int j = 0; j < 4; j++) acc[i][j] = fma(a[i], b[j], acc[i][j]);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 4; j++) s += acc[i][j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_clock(unsigned long long* o, int spin) {
  unsigned long long g0, g1; long long c0 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  while (clock64() - c0 < spin) {}
  long long c1 = clock64();
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
  o[0] = c1 - c0; o[1] = g1 - g0;
}

template <typename F>
float timeit(F launch, int reps) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  launch();
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) launch();
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  void* buf; CK(cudaMalloc(&buf, 64 << 20));
  unsigned long long* ck; CK(cudaMalloc(&ck, 16));
  const int iters = 2048;
  for (int tpb : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int blocks = sms * bps;
      double thr = double(blocks) * tpb;
      float ms;
      ms = timeit([&] { k_outer<<<blocks, tpb>>>((float*)buf, iters, 1.001f); }, 5);
      double f1 = thr * iters * 64 * 2 / (ms * 1e-3) / 1e12;
      ms = timeit([&] { k_outer2<<<blocks, tpb>>>((float2*)buf, iters, 1.001f); }, 5);
      double f2 = thr * iters * 32 * 4 / (ms * 1e-3) / 1e12;
      ms = timeit([&] { k_tri1<<<blocks, tpb>>>((float2*)buf, iters, 1.001f); }, 5);
      double u1 = thr * iters * 32 / (ms * 1e-3);
      ms = timeit([&] { k_tri2<<<blocks, tpb>>>((float2*)buf, iters, 1.001f); }, 5);
      double u2 = thr * iters * 32 / (ms * 1e-3);
      ms = timeit([&] { k_dfma<<<blocks, tpb>>>((double*)buf, iters / 4, 1.001); }, 5);
      double fd = thr * (iters / 4) * 16 * 2 / (ms * 1e-3) / 1e12;
      cudaError_t e = cudaGetLastError();
      printf("tpb=%d bps=%d  FFMA outer %.2f TF | FFMA2 outer %.2f TF | tri scalar %.3e u/s (%.2f TF@14) | tri FFMA2 %.3e u/s (%.2f TF@14) | DFMA %.2f TF %s\n",
             tpb, bps, f1, f2, u1, u1 * 14 / 1e12, u2, u2 * 14 / 1e12, fd, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
  }
  k_clock<<<1, 1>>>(ck, 200000000);
  unsigned long long h[2]; CK(cudaMemcpy(h, ck, 16, cudaMemcpyDeviceToHost));
  printf("idle-ish clock: %.1f MHz\n", h[0] / (h[1] * 1e-3));
  // clock under load: run outer kernel concurrently on a second stream
  cudaStream_t s; cudaStreamCreate(&s);
  for (int r = 0; r < 20; r++) k_outer<<<sms * 2, 256, 0, s>>>((float*)buf, iters, 1.001f);
  k_clock<<<1, 1>>>(ck, 200000000);
  CK(cudaMemcpy(h, ck, 16, cudaMemcpyDeviceToHost));
  printf("loaded clock: %.1f MHz\n", h[0] / (h[1] * 1e-3));
  return 0;
}
