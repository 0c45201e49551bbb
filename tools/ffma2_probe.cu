// ffma2_probe.cu — peak FMA-pipe rates of FFMA vs FFMA2 (broadcast + uniform
// weight pair operand form used by the filter kernel).
#include <cstdio>
#include <cstdint>
struct __align__(16) W { float w[64]; };
__device__ __forceinline__ uint64_t pk(float a, float b) { uint64_t r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b)); return r; }
__device__ __forceinline__ uint64_t ffma2(float x, uint64_t w, uint64_t c) {
  uint64_t r; asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk(x, x)), "l"(w), "l"(c)); return r; }
template <int NA>
__global__ void k2(float* out, const __grid_constant__ W wt, int n, float x0) {
  uint64_t acc[NA];
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = x0 + threadIdx.x + j;
  for (int a = 0; a < NA; ++a) acc[a] = pk(a, a);
  for (int i = 0; i < n; ++i) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(wt.w) + (i & 7) * 4;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      uint64_t wv = w[d];
#pragma unroll
      for (int a = 0; a < NA; ++a) acc[a] = ffma2(v[(a + d) & 7], wv, acc[a]);
    }
  }
  float s = 0; for (int a = 0; a < NA; ++a) { float2 f = *reinterpret_cast<float2*>(&acc[a]); s += f.x + f.y; }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <int NA>
__global__ void k1(float* out, const __grid_constant__ W wt, int n, float x0) {
  float acc[NA];
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = x0 + threadIdx.x + j;
  for (int a = 0; a < NA; ++a) acc[a] = a;
  for (int i = 0; i < n; ++i) {
    const float* w = wt.w + (i & 7) * 8;
#pragma unroll
    for (int d = 0; d < 8; ++d) {
      float wv = w[d];
#pragma unroll
      for (int a = 0; a < NA; ++a) asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(acc[a]) : "f"(v[(a + d) & 7]), "f"(wv));
    }
  }
  float s = 0; for (int a = 0; a < NA; ++a) s += acc[a];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// mixed stream: per weight, NA FFMA2 on pairs + NS FFMA on singles
template <int NA, int NS>
__global__ void kmix(float* out, const __grid_constant__ W wt, int n, float x0) {
  uint64_t acc[NA];
  float accs[NS];
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = x0 + threadIdx.x + j;
  for (int a = 0; a < NA; ++a) acc[a] = pk(a, a);
  for (int a = 0; a < NS; ++a) accs[a] = a;
  for (int i = 0; i < n; ++i) {
    const uint64_t* w = reinterpret_cast<const uint64_t*>(wt.w) + (i & 7) * 4;
#pragma unroll
    for (int d = 0; d < 4; ++d) {
      uint64_t wv = w[d];
      float ws = wt.w[(i & 7) * 8 + d];
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        acc[a] = ffma2(v[(a + d) & 7], wv, acc[a]);
        if (a % (NA / NS) == 0)
          asm volatile("fma.rn.f32 %0, %1, %2, %0;" : "+f"(accs[a / (NA / NS)]) : "f"(v[(a + d + 1) & 7]), "f"(ws));
      }
    }
  }
  float s = 0; for (int a = 0; a < NA; ++a) { float2 f = *reinterpret_cast<float2*>(&acc[a]); s += f.x + f.y; }
  for (int a = 0; a < NS; ++a) s += accs[a];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  W w; for (int i = 0; i < 64; ++i) w.w[i] = 1e-3f * i;
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int n = 20000;
  for (int warps : {4, 8, 16}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); kmix<24, 8><<<148, 32 * warps>>>(out, w, n, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fma = 148.0 * 32 * warps * n * 4 * (24 * 2 + 8);
      if (rep) printf("warps/SM %2d: mix 24 FFMA2 + 8 FFMA: %.1f TFMA/s  (%s)\n", warps, fma / ms / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  for (int warps : {4, 8, 12}) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a); k2<32><<<148, 32 * warps>>>(out, w, n, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      double fma = 148.0 * 32 * warps * n * 4 * 32 * 2;
      double ms2 = ms;
      cudaEventRecord(a); k1<32><<<148, 32 * warps>>>(out, w, n, 1.f); cudaEventRecord(b); cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      double fma1 = 148.0 * 32 * warps * n * 8 * 32;
      if (rep) printf("warps/SM %2d: FFMA2 %.1f TFMA/s  FFMA %.1f TFMA/s  (peak at %d MHz: %.1f)\n", warps,
                      fma / ms2 / 1e9, fma1 / ms / 1e9, clk / 1000, 148.0 * 128 * clk / 1e9);
    }
  }
  return 0;
}
