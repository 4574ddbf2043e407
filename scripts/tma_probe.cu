// tma_probe.cu — isolate the TMA/mbarrier failure modes on a B200.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -std=c++17 tma_probe.cu -o tma_probe
// Run:   ./tma_probe <variant>   (each variant in its own process)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

template <int MODE>
__global__ void probe(const __grid_constant__ CUtensorMap tmap,
                      const CUtensorMap* gmap, double* out, int g, unsigned tx5 = 32*32*4) {
  extern __shared__ __align__(128) double sbox[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (MODE == 0) {  // arrive only, no TMA
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&bar)));
    } else {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                       sa(&bar)),
                   "r"(MODE == 5 ? (int)tx5 : 12 * 12 * 12 * 8));
      const void* m = MODE == 1 || MODE >= 3 ? (const void*)&tmap : (const void*)gmap;
      if (MODE == 4) {
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(sbox)), "l"((uint64_t)(gmap)), "r"(12*12*12*8), "r"(sa(&bar)) : "memory");
      } else if (MODE == 5) {
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(sa(sbox)), "l"((uint64_t)m), "r"(0), "r"(0), "r"(sa(&bar)) : "memory");
      } else if (MODE == 3) {
        asm volatile("cp.async.bulk.tensor.4d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                     ::"r"(sa(sbox)), "l"((uint64_t)m), "r"(1), "r"(1), "r"(1), "r"(g), "r"(sa(&bar)) : "memory");
      } else
      asm volatile(
          "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::"
          "bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(sa(sbox)),
          "l"((uint64_t)m), "r"(1), "r"(1), "r"(1), "r"(g), "r"(sa(&bar))
          : "memory");
    }
  }
  asm volatile(
      "{\n.reg .pred P1;\nLAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
      "@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(sa(&bar))
      : "memory");
  if (MODE != 0)
    for (int i = threadIdx.x; i < (MODE == 5 ? 0 : 1728); i += blockDim.x) out[i] = sbox[i];
}

int main(int argc, char** argv) {
  int variant = argc > 1 ? atoi(argv[1]) : 1;
  const int E = 14, S = 4;
  double* pool;
  cudaMalloc(&pool, sizeof(double) * S * E * E * E);
  double* h = (double*)malloc(sizeof(double) * S * E * E * E);
  for (int i = 0; i < S * E * E * E; ++i) h[i] = i;
  cudaMemcpy(pool, h, sizeof(double) * S * E * E * E, cudaMemcpyHostToDevice);
  double* out;
  cudaMalloc(&out, sizeof(double) * 1728);
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
  CUtensorMap m;
  cuuint64_t dims[4] = {E, E, E, S};
  cuuint64_t str[3] = {E * 8, E * E * 8, E * E * E * 8};
  cuuint32_t box[4] = {12, 12, 12, 1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  CUtensorMapDataType dt = variant == 3 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                                        : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = enc(&m, dt, 4, pool, dims, str, box, es,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                   variant == 4 ? CU_TENSOR_MAP_L2_PROMOTION_NONE
                                : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("variant %d encode=%d\n", variant, (int)r);
  CUtensorMap* gmap;
  cudaMalloc(&gmap, sizeof(CUtensorMap));
  cudaMemcpy(gmap, &m, sizeof(m), cudaMemcpyHostToDevice);
  size_t smem = 1728 * 8;
  if (variant == 5 || variant == 7) {
    // classic 2D: 64x64 fp32 matrix, box 24x36 (inner 96 B) or 32x32 (inner 128 B)
    float* f; cudaMalloc(&f, 64 * 64 * 4);
    cuuint64_t d2[2] = {64, 64}; cuuint64_t s2[1] = {256};
    cuuint32_t b2[2] = {variant == 5 ? 32u : 24u, variant == 5 ? 32u : 36u}; cuuint32_t e2[2] = {1, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, f, d2, s2, b2, e2, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant %d 2d encode=%d\n", variant, (int)r);
  }
  if (variant == 6) {  // inner box 16 doubles = 128 B over dim 14 (OOB fill)
    cuuint32_t b6[4] = {16, 12, 12, 1};
    r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, pool, dims, str, b6, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("variant 6 encode=%d\n", (int)r);
    smem = 16 * 12 * 12 * 8;
  }
  if (variant == 0)
    probe<0><<<1, 128, smem>>>(m, gmap, out, 2);
  else if (variant == 3 || variant == 8)
    probe<3><<<1, 128, smem>>>(m, gmap, out, 2);
  else if (variant == 4)
    probe<4><<<1, 128, smem>>>(m, (const CUtensorMap*)pool, out, 2);
  else if (variant == 5 || variant == 7)
    probe<5><<<1, 128, 32 * 36 * 4>>>(m, gmap, out, 2, variant == 5 ? 32*32*4 : 24*36*4);
  else if (variant == 6)
    probe<1><<<1, 128, smem>>>(m, gmap, out, 2);
  else if (variant == 2)
    probe<2><<<1, 128, smem>>>(m, gmap, out, 2);
  else
    probe<1><<<1, 128, smem>>>(m, gmap, out, 2);
  cudaError_t e = cudaDeviceSynchronize();
  printf("variant %d sync=%s\n", variant, cudaGetErrorString(e));
  if (e == cudaSuccess && (variant == 1 || variant == 2 || variant == 3)) {
    double o[1728];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    // box (1,1,1) of slice 2: ext (1+i, 1+j, 1+k)
    int bad = 0;
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j)
        for (int k = 0; k < 12; ++k) {
          double want = 2 * E * E * E + (1 + i) * E * E + (1 + j) * E + 1 + k;
          if (o[(i * 12 + j) * 12 + k] != want) ++bad;
        }
    printf("variant %d mismatches=%d\n", variant, bad);
  }
  return 0;
}
