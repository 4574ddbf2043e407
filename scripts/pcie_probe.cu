// PCIe probe: GPU-initiated (zero-copy) reads from / writes to pinned host
// memory vs the copy engines.  Built by scripts/probe_pcie2.py with nvcc.
#include <cuda_runtime.h>
#include <stdint.h>

__global__ void k_copy16(const double2* __restrict__ src, double2* __restrict__ dst,
                         int64_t n2) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // four independent loads in flight per thread
  for (; i + 3 * stride < n2; i += 4 * stride) {
    double2 a = src[i], b = src[i + stride], c = src[i + 2 * stride],
            d = src[i + 3 * stride];
    dst[i] = a;
    dst[i + stride] = b;
    dst[i + 2 * stride] = c;
    dst[i + 3 * stride] = d;
  }
  for (; i < n2; i += stride) dst[i] = src[i];
}

extern "C" int probe_copy(const void* src, void* dst, int64_t bytes, int blocks,
                          int threads, void* stream) {
  k_copy16<<<blocks, threads, 0, (cudaStream_t)stream>>>(
      (const double2*)src, (double2*)dst, bytes / 16);
  return (int)cudaGetLastError();
}
