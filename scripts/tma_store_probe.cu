// TMA tile store with partially out-of-bounds boxes: which coordinates are
// legal on sm_100a?  nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>

__global__ void k_store(const __grid_constant__ CUtensorMap map, int c0,
                        int c1, int c2) {
  __shared__ __align__(1024) double tile[512];
  for (int i = threadIdx.x; i < 512; i += blockDim.x) tile[i] = 1.0 + i;
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned s = (unsigned)__cvta_generic_to_shared(tile);
    asm volatile(
        "cp.async.bulk.tensor.3d.global.shared::cta.tile.bulk_group"
        " [%0, {%2, %3, %4}], [%1];" ::"l"(&map), "r"(s), "r"(c0), "r"(c1),
        "r"(c2)
        : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }
}

int main() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)fn;
  const int pz = 24, py = 20, px = 20;
  double* d;
  cudaMalloc(&d, sizeof(double) * pz * py * px);
  cuuint64_t dims[3] = {pz, py, px};
  cuuint64_t str[2] = {pz * 8, pz * py * 8};
  cuuint32_t box[3] = {8, 8, 8}, es[3] = {1, 1, 1};
  int coords[][3] = {{4, 2, 2}, {4, 18, 2}, {20, 2, 2}, {4, 2, 18},
                     {4, -6, 2}, {-4, 2, 2}, {4, 2, -6}};
  for (int sw = 0; sw < 2; ++sw) {
    CUtensorMap m;
    CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, str, box,
                     es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     sw ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_NONE,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (auto& c : coords) {
      k_store<<<1, 64>>>(m, c[0], c[1], c[2]);
      cudaError_t e = cudaDeviceSynchronize();
      printf("swizzle %s  coords z=%d y=%d x=%d  encode %d  -> %s\n",
             sw ? "64B" : "none", c[0], c[1], c[2], (int)r,
             cudaGetErrorString(e));
      if (e != cudaSuccess) return 1;
    }
  }
  return 0;
}
