// Speed-of-light probe for the recon+flux traffic shape: per CTA (one 8^3
// sub-grid) read R bytes, write W bytes (W = 72 000 = um+up+F), same grid
// (4096 CTAs x 512 threads, 4 CTAs/SM), trivial arithmetic.  Tells how much
// of the measured copy peak a write-dominated kernel of this shape can reach.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a scripts/sol_probe.cu
//        -o scripts/_sol_probe
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W2 = 72000 / 16;  // double2 stores per CTA
constexpr int R2 = 16128 / 16;  // double2 loads per CTA ((n+4)^2 (n+6) cells)

template <int MODE>  // 0 = write only, 1 = read then write, 2 = write .wb
__global__ void __launch_bounds__(512, 4)
k_shape(const double2* __restrict__ in, double2* __restrict__ out) {
  __shared__ double2 s[R2];
  const int64_t b = blockIdx.x;
  double2 acc = make_double2(0.0, 0.0);
  if (MODE == 1) {
    for (int i = threadIdx.x; i < R2; i += 512) s[i] = in[b * R2 + i];
    __syncthreads();
    acc = s[threadIdx.x];
  }
  double2* o = out + b * W2;
  for (int i = threadIdx.x; i < W2; i += 512) {
    double2 v = make_double2(acc.x + i, acc.y - i);
    if (MODE == 2)
      o[i] = v;
    else
      asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(o + i),
                   "d"(v.x), "d"(v.y)
                   : "memory");
  }
}

template <int MODE>
float run(const double2* in, double2* out, int grid, int reps) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) k_shape<MODE><<<grid, 512>>>(in, out);
  cudaEventRecord(a);
  for (int i = 0; i < reps; ++i) k_shape<MODE><<<grid, 512>>>(in, out);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  return ms / reps;
}

int main() {
  const int grid = 4096;
  double2 *in, *out;
  cudaMalloc(&in, (size_t)grid * R2 * 16);
  cudaMalloc(&out, (size_t)grid * W2 * 16);
  cudaMemset(in, 0, (size_t)grid * R2 * 16);
  const int reps = 50;
  const double wb = (double)grid * W2 * 16, rb = (double)grid * R2 * 16;
  float t0 = run<0>(in, out, grid, reps);
  float t1 = run<1>(in, out, grid, reps);
  float t2 = run<2>(in, out, grid, reps);
  printf("write-only .cs : %.2f us  %.0f GB/s\n", t0 * 1e3, wb / t0 / 1e6);
  printf("read+write .cs : %.2f us  %.0f GB/s (alg %.0f GB/s incl. 84.8 KB/sub-grid)\n",
         t1 * 1e3, (wb + rb) / t1 / 1e6, grid * 84800.0 / t1 / 1e6);
  printf("write-only .wb : %.2f us  %.0f GB/s\n", t2 * 1e3, wb / t2 / 1e6);
  // larger grids (multiple waves of the same shape)
  for (int g : {4096 * 4, 4096 * 8}) {
    double2 *in2, *out2;
    cudaMalloc(&in2, (size_t)g * R2 * 16);
    cudaMalloc(&out2, (size_t)g * W2 * 16);
    float t = run<1>(in2, out2, g, 10);
    printf("read+write .cs grid %d: %.2f us  %.0f GB/s\n", g, t * 1e3,
           ((double)g * (W2 + R2) * 16) / t / 1e6);
    cudaFree(in2);
    cudaFree(out2);
  }
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
