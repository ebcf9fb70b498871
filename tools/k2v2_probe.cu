// K2 staging experiment: one 8-warp CTA per SM, the CTA's warps share a ring
// of 4-segment stages, each stage = 2 bulk copies (cp.async.bulk) of the 4
// full E rows (copy B shifted 8 elements in banks so a warp's two tiles never
// conflict), last-arriving warp refills.  Cells as in production K2 (4x8 lane
// micro-tiles, step 4).  Exploration tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_1805_11775_b200/csrc -o tools/k2v2_probe tools/k2v2_probe.cu
#include <cstdio>
#include <cuda_runtime.h>
#include "hos_kernels.cuh"
using namespace hos;

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ float2 lds_conj(const float2* p) {
  float2 v;
  asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(su32(p)));
  v.y = -v.y;
  return v;
}

__device__ __forceinline__ void cells(const float2* __restrict__ rows, const float2* __restrict__ cols,
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

constexpr int NW = 8, GROUP = 4;

template <int LP, int DEPTH, bool COPY, int BOFF = 8, int ACTIVE = NW, int PERWARP = GROUP>
__global__ void __launch_bounds__(32 * NW, 1) k_v2(const float2* __restrict__ E, int K, int nstages, float2* out) {
  extern __shared__ __align__(128) float2 sm[];
  constexpr int SA = GROUP * LP;       // copy A elements
  constexpr int SS = 2 * SA + 32;      // stage stride (elements); copy B at SA + BOFF
  static_assert(SA % 16 == 0, "copy A must keep copy B at +8 banks");
  __shared__ __align__(8) unsigned long long full[DEPTH];
  __shared__ int cnt[DEPTH];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int seg0 = (blockIdx.x * 7 * GROUP) % (K - GROUP * nstages);
  constexpr unsigned bytes = SA * 8;
  auto issue = [&](int st, int d) {
    const float2* src = E + (size_t)(seg0 + st * GROUP) * LP;
    float2* dst = sm + d * SS;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[d])), "r"(2 * bytes)
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst)),
                 "l"(src), "r"(bytes), "r"(su32(&full[d]))
                 : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(dst + SA + BOFF)),
                 "l"(src), "r"(bytes), "r"(su32(&full[d]))
                 : "memory");
  };
  if (threadIdx.x == 0) {
    for (int d = 0; d < DEPTH; d++) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[d])));
      cnt[d] = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (COPY && threadIdx.x == 0)
    for (int d = 0; d < DEPTH && d < nstages; d++) issue(d, d);
  const int h = lane >> 4, ra = (lane >> 2) & 3, cb = lane & 3;
  const int row0 = 16 * warp, col0 = 32 * warp + 32 * h;
  const int bank = h * (SA + BOFF);
  const int o_r = bank + row0 + ra, o_c = bank + col0 + cb, o_g = bank + row0 + col0 + ra + cb;
  float2 aR[4][8], aI[4][8];
#pragma unroll
  for (int i = 0; i < 4; i++)
#pragma unroll
    for (int j = 0; j < 8; j++) aR[i][j] = aI[i][j] = make_float2(0.f, 0.f);
  for (int st = 0; st < nstages; st++) {
    const int d = st % DEPTH;
    if (COPY) {
      const unsigned par = (st / DEPTH) & 1;
      asm volatile(
          "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
              su32(&full[d])),
          "r"(par)
          : "memory");
    }
    const float2* q = sm + d * SS;
    if (warp < ACTIVE) {
#pragma unroll
      for (int t = 0; t < PERWARP; t++) {
        const int u = (warp * PERWARP + t) % GROUP;
        cells(q + u * LP + o_r, q + u * LP + o_c, q + u * LP + o_g, aR, aI);
      }
    }
    if (COPY) {
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();
        if (atomicAdd(&cnt[d], 1) == NW - 1) {
          cnt[d] = 0;
          if (st + DEPTH < nstages) issue(st + DEPTH, d);
        }
      }
    }
  }
  float2 s = make_float2(0, 0);
  for (int i = 0; i < 4; i++)
    for (int j = 0; j < 8; j++) {
      s.x += aR[i][j].x + aI[i][j].y;
      s.y += aR[i][j].y - aI[i][j].x;
    }
  out[blockIdx.x * 32 * NW + threadIdx.x] = s;
}

template <int LP, int DEPTH, bool COPY, int BOFF = 8, int ACTIVE = NW, int PERWARP = GROUP>
void run(const char* name, const float2* E, int K, int nstages, int sms, float2* out) {
  auto kern = k_v2<LP, DEPTH, COPY, BOFF, ACTIVE, PERWARP>;
  const size_t smem = (size_t)DEPTH * (2 * GROUP * LP + 32) * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncAttributes fa;
  cudaFuncGetAttributes(&fa, kern);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  kern<<<sms, 32 * NW, smem>>>(E, K, nstages, out);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaEventRecord(a);
    kern<<<sms, 32 * NW, smem>>>(E, K, nstages, out);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (ms < best) best = ms;
  }
  const double lane_ops = (double)sms * ACTIVE * 32 * nstages * PERWARP * 32 * 8;
  printf("%-10s LP=%d depth=%d stages=%4d us/stage=%.3f regs=%d smem=%zu: %.2f us  FFMA-lane util %.1f%%  (%s)\n", name, LP, DEPTH,
         nstages, best * 1e3 / nstages, fa.numRegs, smem, best * 1e3, 100.0 * lane_ops / (best * 1e-3) / (148.0 * 128 * 1.965e9),
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int K = 1024;
  float2 *E, *out;
  cudaMalloc(&E, (size_t)K * 544 * 8 * 4);
  cudaMemset(E, 0, (size_t)K * 544 * 8 * 4);
  cudaMalloc(&out, sms * 32 * NW * sizeof(float2));
  for (int ns : {18, 72}) {
    run<544, 6, true>("copy", E, K, ns, sms, out);
    run<544, 6, true, 16>("copyB+128", E, K, ns, sms, out);
    run<544, 6, false>("nocopy", E, K, ns, sms, out);
    run<544, 6, true, 8, 4, 1>("rem4x1", E, K, ns, sms, out);
    run<544, 6, false, 8, 4, 1>("rem-nocp", E, K, ns, sms, out);
    run<544, 6, true, 16, 4, 1>("rem+128", E, K, ns, sms, out);
  }
  return 0;
}
