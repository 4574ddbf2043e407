// tma_probe2.cu — which tensor-map shapes load a (12,12,12) box of a pool of
// (14,14,14) FP64 sub-grids on sm_100a.  ./tma_probe2 <elem_bytes 4|8> <rank 2|3|4>
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>

__device__ __forceinline__ uint32_t sa(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

__global__ void probe(const __grid_constant__ CUtensorMap tmap, int rank,
                      int c0, int c1, int c2, int c3, unsigned bytes,
                      double* out) {
  extern __shared__ __align__(128) double sbox[];
  __shared__ __align__(8) uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&bar)), "r"(bytes));
    const uint64_t m = (uint64_t)&tmap;
    if (rank == 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(sa(sbox)), "l"(m), "r"(c0), "r"(c1), "r"(sa(&bar)) : "memory");
    else if (rank == 3)
      asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                   ::"r"(sa(sbox)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(sa(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
                   ::"r"(sa(sbox)), "l"(m), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(sa(&bar)) : "memory");
  }
  __syncthreads();
  asm volatile("{\n.reg .pred P1;\nLAB_WAIT:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra DONE;\nbra LAB_WAIT;\nDONE:\n}\n" ::"r"(sa(&bar)) : "memory");
  for (int i = threadIdx.x; i < (int)(bytes / 8); i += blockDim.x) out[i] = sbox[i];
}

int main(int argc, char** argv) {
  const int eb = atoi(argv[1]), rank = atoi(argv[2]);
  const int E = 14, S = 4, k = 8 / eb, g = 2;
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
  cuuint64_t dims[4], str[3];
  cuuint32_t box[4], es[4] = {1, 1, 1, 1};
  int c[4] = {0, 0, 0, 0};
  dims[0] = E * k; box[0] = 12 * k; c[0] = 1 * k;
  str[0] = E * 8;
  if (rank == 2) {
    dims[1] = (cuuint64_t)E * E * S; box[1] = 12; c[1] = g * E * E + 1 * E + 1;  // one y-row strip only
  } else if (rank == 3) {
    dims[1] = E; dims[2] = (cuuint64_t)E * S; str[1] = E * E * 8;
    box[1] = 12; box[2] = 12; c[1] = 1; c[2] = g * E + 1;
  } else {
    dims[1] = E; dims[2] = E; dims[3] = S; str[1] = E * E * 8; str[2] = E * E * E * 8;
    box[1] = 12; box[2] = 12; box[3] = 1; c[1] = 1; c[2] = 1; c[3] = g;
  }
  CUresult r = enc(&m, eb == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32,
                   rank, pool, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  unsigned bytes = eb;
  for (int i = 0; i < rank; ++i) bytes *= box[i];
  probe<<<1, 128, 13824>>>(m, rank, c[0], c[1], c[2], c[3], bytes, out);
  cudaError_t e = cudaDeviceSynchronize();
  int bad = -1;
  if (e == cudaSuccess && rank == 4) {
    double o[1728];
    cudaMemcpy(o, out, sizeof(o), cudaMemcpyDeviceToHost);
    bad = 0;
    for (int i = 0; i < 12; ++i)
      for (int j = 0; j < 12; ++j)
        for (int kk = 0; kk < 12; ++kk)
          if (o[(i * 12 + j) * 12 + kk] != g * E * E * E + (1 + i) * E * E + (1 + j) * E + 1 + kk) ++bad;
  }
  printf("elem=%d rank=%d encode=%d bytes=%u sync=%s mismatches=%d\n", eb, rank, (int)r, bytes,
         cudaGetErrorString(e), bad);
  return 0;
}
