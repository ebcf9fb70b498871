// Large-copy variant of tma_probe.cu (4-16 KB pieces, one CTA per SM).  Exploration tool.
// (LDGSTS) vs plain LDG->STS, copying `size`-byte pieces from an L2-resident
// buffer into shared memory, `ctas` CTAs per SM.  Exploration tool.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_probe tools/tma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned su32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_bulk(const char* src, int size, int per_batch, int batches, unsigned long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  long long t0 = clock64();
  const char* base = src + (size_t)blockIdx.x * 262144;
  for (int b = 0; b < batches; b++) {
    if (threadIdx.x < 32) {
      if (threadIdx.x == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(size * per_batch)
                     : "memory");
      __syncwarp();
      for (int q = threadIdx.x; q < per_batch; q += 32)
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                         su32(sm + q * size)),
                     "l"(base + ((b * per_batch + q) % 16) * size), "r"(size), "r"(su32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@!P1 bra W_%=;\n}\n" ::"r"(
            su32(&bar)),
        "r"(b & 1)
        : "memory");
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

__global__ void k_ldgsts(const char* src, int size, int per_batch, int batches, unsigned long long* cyc) {
  extern __shared__ __align__(128) char sm[];
  long long t0 = clock64();
  const char* base = src + (size_t)blockIdx.x * 262144;
  const int n16 = size / 16;
  for (int b = 0; b < batches; b++) {
    for (int e = threadIdx.x; e < per_batch * n16; e += blockDim.x) {
      const int q = e / n16, k = e % n16;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + q * size + k * 16)),
                   "l"(base + ((b * per_batch + q) % 16) * size + k * 16));
    }
    asm volatile("cp.async.commit_group;");
    asm volatile("cp.async.wait_group 0;");
    __syncthreads();
  }
  if (threadIdx.x == 0) cyc[blockIdx.x] = clock64() - t0;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  char* src;
  cudaMalloc(&src, (size_t)sms * 4 * 262144 + (1 << 20));
  cudaMemset(src, 1, (size_t)sms * 4 * 262144 + (1 << 20));
  unsigned long long* cyc;
  cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 4);
  cudaFuncSetAttribute(k_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaFuncSetAttribute(k_ldgsts, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int ctas : {1}) {
    for (int size : {4096, 8192, 16384}) {
      for (int per : {1, 2, 4, 8}) {
        if (size * per > 200 * 1024) continue;
        const int batches = 2000;
        float ms[2];
        for (int kind = 0; kind < 2; kind++) {
          auto launch = [&] {
            if (kind == 0) k_bulk<<<sms * ctas, 128, size * per>>>(src, size, per, batches, cyc);
            else k_ldgsts<<<sms * ctas, 128, size * per>>>(src, size, per, batches, cyc);
          };
          launch();
          cudaEventRecord(e0);
          launch();
          cudaEventRecord(e1);
          cudaEventSynchronize(e1);
          cudaEventElapsedTime(&ms[kind], e0, e1);
        }
        const double bytes = (double)sms * ctas * batches * per * size;
        printf("ctas/SM=%d size=%5d per_batch=%d : bulk %.1f ns/batch (%.2f TB/s)  ldgsts %.1f ns/batch (%.2f TB/s)\n",
               ctas, size, per, ms[0] * 1e6 / batches, bytes / (ms[0] * 1e-3) / 1e12, ms[1] * 1e6 / batches,
               bytes / (ms[1] * 1e-3) / 1e12);
      }
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
