// tma_probe.cu — standalone checks of the TMA / mbarrier idioms used by
// filter_tma.cuh (run one variant per process: ./tma_probe <variant> <x> <boxx> <nx>).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap map, uint8_t* out, int bytes, int x, int y, int z, int variant) {
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    if (variant == 3) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map)) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1));
    if (variant == 1) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (variant == 2) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(bytes) : "memory");
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(smem_u32(smem)), "l"(reinterpret_cast<uint64_t>(&map)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(smem_u32(&bar)), "r"(0) : "memory");
  for (int i = threadIdx.x; i < bytes; i += blockDim.x) out[i] = smem[i];
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                             const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                             CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 0;
  int x = argc > 2 ? atoi(argv[2]) : 0;
  int bx = argc > 3 ? atoi(argv[3]) : 80;
  int nx = argc > 4 ? atoi(argv[4]) : 80;
  void* p = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn fn = (EncodeFn)p;
  const int ny = 37, nz = 23, by = 18;
  std::vector<uint8_t> h((size_t)nx * ny * nz);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (uint8_t)(i * 7 + 3);
  uint8_t *d, *o; cudaMalloc(&d, h.size()); cudaMalloc(&o, 8192);
  cudaMemcpy(d, h.data(), h.size(), cudaMemcpyHostToDevice);
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)nx, ny, nz}; cuuint64_t str[2] = {(cuuint64_t)nx, (cuuint64_t)nx * ny};
  cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)by, 1}; cuuint32_t es[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, d, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaMemset(o, 0xEE, 8192);
  probe<<<1, 128, 8192>>>(m, o, bx * by, x, -1, 2, variant);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<uint8_t> ho(bx * by);
  cudaMemcpy(ho.data(), o, ho.size(), cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int yy = 0; yy < by; ++yy) for (int xx = 0; xx < bx; ++xx) {
    int gx = x + xx, gy = -1 + yy, gz = 2;
    uint8_t want = (gx >= 0 && gx < nx && gy >= 0 && gy < ny) ? h[((size_t)gz * ny + gy) * nx + gx] : 0;
    bad += ho[yy * bx + xx] != want;
  }
  printf("variant %d x=%d box=%d nx=%d encode=%d: %s bad=%d\n", variant, x, bx, nx, (int)r, cudaGetErrorString(e), bad);
  return e != cudaSuccess;
}
