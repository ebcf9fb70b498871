// Zero-copy PCIe bandwidth probe: how fast can kernels read a page-locked,
// device-mapped host buffer (the e2e path's input) and write one (its output)?
// Variants: scalar / float4 loads, TMA bulk copies (cp.async.bulk) into shared
// memory, and the copy engine for comparison.  Exploration tool:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/pcie tools/pcie_probe.cu && /tmp/pcie
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x)                                                                   \
  do {                                                                          \
    cudaError_t e_ = (x);                                                       \
    if (e_ != cudaSuccess) {                                                    \
      printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));         \
      return 1;                                                                 \
    }                                                                           \
  } while (0)

__global__ void k_read_scalar(const float* __restrict__ x, size_t n, float* out) {
  float s = 0.f;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) s += x[i];
  if (s == 12345.f) out[0] = s;
}

template <int U>
__global__ void k_read_v4(const float4* __restrict__ x, size_t n4, float* out) {
  float s = 0.f;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; u++) v[u] = x[i + u * stride];
#pragma unroll
    for (int u = 0; u < U; u++) s += v[u].x + v[u].y + v[u].z + v[u].w;
  }
  for (; i < n4; i += stride) s += x[i].x;
  if (s == 12345.f) out[0] = s;
}

// one thread per CTA issues bulk copies of `chunk` bytes into a shared ring
__global__ void k_read_bulk(const char* __restrict__ x, size_t n, int chunk, float* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  const unsigned d = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(b));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  float s = 0.f;
  unsigned phase = 0;
  for (size_t off = (size_t)blockIdx.x * chunk; off < n; off += (size_t)gridDim.x * chunk) {
    const int bytes = (int)((n - off) < (size_t)chunk ? (n - off) : (size_t)chunk);
    if (threadIdx.x == 0) {
      asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(bytes));
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(d),
                   "l"(x + off), "r"(bytes), "r"(b)
                   : "memory");
    }
    unsigned done = 0;
    while (!done)
      asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                   : "=r"(done)
                   : "r"(b), "r"(phase));
    phase ^= 1;
    s += reinterpret_cast<const float*>(sm)[threadIdx.x];
    __syncthreads();
  }
  if (s == 12345.f) out[0] = s;
}

__global__ void k_write_v4(float4* __restrict__ y, size_t n4) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n4; i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_float4(1.f, 2.f, 3.f, (float)i);
}

__global__ void k_write_v2(float2* __restrict__ y, size_t n2) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x)
    y[i] = make_float2(1.f, (float)i);
}

template <typename F>
float time_us(F f, int reps = 20) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  cudaEventRecord(a);
  for (int r = 0; r < reps; r++) f();
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / reps;
}

int main() {
  const size_t n = 1 << 20;  // 4 MiB of fp32 (cfg2's series)
  const size_t bytes = n * 4;
  float *h, *hd, *dev, *out;
  CK(cudaHostAlloc(&h, bytes, cudaHostAllocMapped));
  for (size_t i = 0; i < n; i++) h[i] = (float)(i % 977);
  CK(cudaHostGetDevicePointer(&hd, h, 0));
  CK(cudaMalloc(&dev, bytes));
  CK(cudaMalloc(&out, 64));
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto gbs = [&](float us, size_t b) { return b / (us * 1e-6) / 1e9; };

  for (int ctas : {sms, 2 * sms, 4 * sms, 8 * sms}) {
    float t = time_us([&] { k_read_scalar<<<ctas, 256>>>(hd, n, out); });
    printf("scalar   ctas %4d: %7.1f us %6.1f GB/s\n", ctas, t, gbs(t, bytes));
  }
  for (int ctas : {sms, 2 * sms, 4 * sms}) {
    float t1 = time_us([&] { k_read_v4<1><<<ctas, 256>>>((const float4*)hd, n / 4, out); });
    float t4 = time_us([&] { k_read_v4<4><<<ctas, 256>>>((const float4*)hd, n / 4, out); });
    printf("v4 U1/U4 ctas %4d: %7.1f / %7.1f us  %6.1f / %6.1f GB/s\n", ctas, t1, t4, gbs(t1, bytes), gbs(t4, bytes));
  }
  for (int chunk : {4096, 16384, 32768}) {
    CK(cudaFuncSetAttribute(k_read_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, chunk));
    for (int ctas : {sms, 2 * sms}) {
      float t = time_us([&] { k_read_bulk<<<ctas, 128, chunk>>>((const char*)hd, bytes, chunk, out); });
      printf("bulk chunk %5d ctas %4d: %7.1f us %6.1f GB/s\n", chunk, ctas, t, gbs(t, bytes));
    }
  }
  CK(cudaGetLastError());
  {
    float t = time_us([&] { cudaMemcpyAsync(dev, h, bytes, cudaMemcpyHostToDevice); });
    printf("copy engine H2D 4 MiB: %7.1f us %6.1f GB/s\n", t, gbs(t, bytes));
    float t2 = time_us([&] { cudaMemcpyAsync(h, dev, 700000, cudaMemcpyDeviceToHost); });
    printf("copy engine D2H 700 KB: %7.1f us %6.1f GB/s\n", t2, gbs(t2, 700000));
  }
  for (int ctas : {sms, 4 * sms}) {
    float t = time_us([&] { k_write_v4<<<ctas, 256>>>((float4*)hd, 700000 / 16); });
    float t2 = time_us([&] { k_write_v2<<<ctas, 256>>>((float2*)hd, 700000 / 8); });
    printf("zero-copy write 700 KB ctas %4d: v4 %7.1f us (%5.1f GB/s)  v2 %7.1f us (%5.1f GB/s)\n", ctas, t,
           gbs(t, 700000), t2, gbs(t2, 700000));
  }
  // small-launch latency floor
  {
    float t = time_us([&] { k_write_v2<<<1, 32>>>((float2*)dev, 32); });
    printf("empty-ish launch: %.1f us\n", t);
  }
  CK(cudaDeviceSynchronize());
  return 0;
}
