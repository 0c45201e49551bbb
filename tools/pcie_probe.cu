// pcie_probe.cu — PCIe rates on the box: copy engines vs SM loads/stores to
// mapped pinned host memory, alone and concurrently.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/pcie_probe.cu -o /tmp/pcie_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void copy_kernel(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += stride) {
    int4 v = __ldcs(src + i);
    __stcs(dst + i, v);
  }
}

// 4 independent 16B loads in flight per thread (host reads are latency bound)
__global__ void copy_kernel_ilp(const int4* __restrict__ src, int4* __restrict__ dst, size_t n) {
  size_t stride = (size_t)gridDim.x * blockDim.x;
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n; i += 4 * stride) {
    int4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride),
         d = __ldcs(src + i + 3 * stride);
    __stcs(dst + i, a); __stcs(dst + i + stride, b); __stcs(dst + i + 2 * stride, c);
    __stcs(dst + i + 3 * stride, d);
  }
  for (; i < n; i += stride) __stcs(dst + i, __ldcs(src + i));
}

int main() {
  const size_t B = 2ull << 30;
  void *hin, *hout, *d0, *d1;
  CK(cudaHostAlloc(&hin, B, cudaHostAllocDefault));
  CK(cudaHostAlloc(&hout, B, cudaHostAllocDefault));
  CK(cudaMalloc(&d0, B));
  CK(cudaMalloc(&d1, B));
  cudaMemset(d0, 1, B);
  memset(hin, 2, B);
  cudaStream_t s1, s2;
  cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
  cudaEvent_t a, b, c, d;
  cudaEventCreate(&a); cudaEventCreate(&b); cudaEventCreate(&c); cudaEventCreate(&d);
  auto ms = [&](cudaEvent_t x, cudaEvent_t y) { float t; cudaEventElapsedTime(&t, x, y); return t; };
  const size_t n16 = B / 16;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s1); cudaMemcpyAsync(d1, hin, B, cudaMemcpyHostToDevice, s1); cudaEventRecord(b, s1);
    cudaEventSynchronize(b); printf("CE H2D            : %.1f GB/s\n", B / ms(a, b) / 1e6);
    cudaEventRecord(a, s1); cudaMemcpyAsync(hout, d0, B, cudaMemcpyDeviceToHost, s1); cudaEventRecord(b, s1);
    cudaEventSynchronize(b); printf("CE D2H            : %.1f GB/s\n", B / ms(a, b) / 1e6);
    for (int ctas : {16, 32, 64, 148, 296, 592}) {
      cudaEventRecord(a, s1); copy_kernel<<<ctas, 256, 0, s1>>>((const int4*)d0, (int4*)hout, n16); cudaEventRecord(b, s1);
      cudaEventSynchronize(b); printf("SM store D2H %4d : %.1f GB/s\n", ctas, B / ms(a, b) / 1e6);
    }
    for (int ctas : {148, 296, 592, 1184}) {
      cudaEventRecord(a, s1); copy_kernel_ilp<<<ctas, 256, 0, s1>>>((const int4*)hin, (int4*)d1, n16); cudaEventRecord(b, s1);
      cudaEventSynchronize(b); printf("SM load  H2D %4d : %.1f GB/s\n", ctas, B / ms(a, b) / 1e6);
    }
    // concurrent: CE H2D + CE D2H
    cudaEventRecord(a, s1); cudaEventRecord(c, s2);
    cudaMemcpyAsync(d1, hin, B, cudaMemcpyHostToDevice, s1);
    cudaMemcpyAsync(hout, d0, B, cudaMemcpyDeviceToHost, s2);
    cudaEventRecord(b, s1); cudaEventRecord(d, s2); cudaDeviceSynchronize();
    printf("CE H2D || CE D2H  : %.1f ms (H2D %.1f, D2H %.1f)\n", std::max(ms(a, b), ms(c, d)), ms(a, b), ms(c, d));
    for (int ctas : {32, 64, 148}) {
      cudaEventRecord(a, s1); cudaEventRecord(c, s2);
      cudaMemcpyAsync(d1, hin, B, cudaMemcpyHostToDevice, s1);
      copy_kernel<<<ctas, 256, 0, s2>>>((const int4*)d0, (int4*)hout, n16);
      cudaEventRecord(b, s1); cudaEventRecord(d, s2); cudaDeviceSynchronize();
      printf("CE H2D || SM D2H %3d: %.1f ms (H2D %.1f, D2H %.1f)\n", ctas, std::max(ms(a, b), ms(c, d)), ms(a, b), ms(c, d));
    }
    for (int ctas : {148, 296}) {
      cudaEventRecord(a, s1); cudaEventRecord(c, s2);
      copy_kernel_ilp<<<ctas, 256, 0, s1>>>((const int4*)hin, (int4*)d1, n16);
      copy_kernel<<<64, 256, 0, s2>>>((const int4*)d0, (int4*)hout, n16);
      cudaEventRecord(b, s1); cudaEventRecord(d, s2); cudaDeviceSynchronize();
      printf("SM H2D %3d || SM D2H 64: %.1f ms (H2D %.1f, D2H %.1f)\n", ctas, std::max(ms(a, b), ms(c, d)), ms(a, b), ms(c, d));
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
  }
  return 0;
}
