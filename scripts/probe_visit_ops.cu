// Per-visit device-op chain of the per-task path (HydroSim at A = 1): an
// h2d copy of a 21 952 B lease, a small kernel, a d2h copy of 4 096 B, 320
// visits per iteration on one stream.  DMA copies (cudaMemcpyAsync) vs copy
// kernels reading / writing the pinned leases zero-copy.
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

__global__ void k_copy(double* __restrict__ dst, const double* __restrict__ src,
                       int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x)
    dst[i] = src[i];
}
__global__ void k_work(double* a, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += gridDim.x * blockDim.x)
    a[i] = a[i] * 1.0000001 + 1.0;
}

int main() {
  const int V = 320, in = 2744, out = 512;
  double *h_in, *h_out, *d_in, *d_out;
  cudaHostAlloc(&h_in, sizeof(double) * in * V, 0);
  cudaHostAlloc(&h_out, sizeof(double) * out * V, 0);
  cudaMalloc(&d_in, sizeof(double) * in * V);
  cudaMalloc(&d_out, sizeof(double) * out * V);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int variant = 0; variant < 3; ++variant) {
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a, s);
      for (int v = 0; v < V; ++v) {
        double* hi = h_in + (size_t)v * in;
        double* di = d_in + (size_t)v * in;
        double* ho = h_out + (size_t)v * out;
        double* dout = d_out + (size_t)v * out;
        if (variant == 0) {
          cudaMemcpyAsync(di, hi, sizeof(double) * in, cudaMemcpyHostToDevice, s);
        } else {
          k_copy<<<variant == 1 ? 4 : 22, 128, 0, s>>>(di, hi, in);
        }
        k_work<<<8, 128, 0, s>>>(dout, out);
        if (variant == 0) {
          cudaMemcpyAsync(ho, dout, sizeof(double) * out, cudaMemcpyDeviceToHost, s);
        } else {
          k_copy<<<4, 128, 0, s>>>(ho, dout, out);
        }
      }
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (rep == 3)
        printf("%s: %.1f us per iteration of %d visits (%.2f us per visit)\n",
               variant == 0 ? "DMA copies" : variant == 1 ? "copy kernels, 4 CTAs"
                                                          : "copy kernels, 22 CTAs",
               ms * 1e3, V, ms * 1e3 / V);
    }
  }
  return 0;
}
