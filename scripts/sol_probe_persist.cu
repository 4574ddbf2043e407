// Is a persistent grid slower than one CTA per slice for the recon+flux
// traffic shape?  Same per-slice work as scripts/sol_probe.cu (read 16 KB
// into smem, write 72 KB with 16-B streaming stores), 4096 slices:
//   A: 4096 CTAs, one slice each;  B: 592 CTAs looping (static stride);
//   C: 592 CTAs looping, dynamic atomic claim.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
//        scripts/sol_probe_persist.cu -o scripts/_sol_probe_persist
#include <cstdio>
#include <cuda_runtime.h>

constexpr int W2 = 72000 / 16;
constexpr int R2 = 16128 / 16;

__device__ __forceinline__ void slice(const double2* in, double2* out,
                                      int64_t b, double2* s) {
  for (int i = threadIdx.x; i < R2; i += 512) s[i] = in[b * R2 + i];
  __syncthreads();
  const double2 acc = s[threadIdx.x];
  double2* o = out + b * W2;
  for (int i = threadIdx.x; i < W2; i += 512) {
    const double2 v = make_double2(acc.x + i, acc.y - i);
    asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(o + i),
                 "d"(v.x), "d"(v.y)
                 : "memory");
  }
  __syncthreads();
}

__device__ __forceinline__ long long ld_acq(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_rlx(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

template <int MODE>
__global__ void __launch_bounds__(512, 4)
k(const double2* __restrict__ in, double2* __restrict__ out, int S,
  unsigned* claim) {
  __shared__ double2 s[R2];
  __shared__ int next;
  if (MODE == 0) {
    slice(in, out, blockIdx.x, s);
  } else if (MODE == 1) {
    for (int b = blockIdx.x; b < S; b += gridDim.x) slice(in, out, b, s);
  } else if (MODE == 5) {
    // dynamic claim, double-buffered read: the next slice's 16 KB is read
    // (cp.async into the other buffer) while this slice's 72 KB are written
    __shared__ double2 s2[R2];
    double2* buf[2] = {s, s2};
    __shared__ int nxt2;
    if (threadIdx.x == 0) next = (int)atomicAdd(claim, 1u);
    __syncthreads();
    int b = next, t = 0;
    if (b < S)
      for (int i = threadIdx.x; i < R2; i += 512) buf[0][i] = in[(int64_t)b * R2 + i];
    while (b < S) {
      if (threadIdx.x == 0) nxt2 = (int)atomicAdd(claim, 1u);
      __syncthreads();
      const int bn = nxt2;
      double2* cur = buf[t & 1];
      double2* nb = buf[(t + 1) & 1];
      if (bn < S)
        for (int i = threadIdx.x; i < R2; i += 512) {
          const double2* src = in + (int64_t)bn * R2 + i;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                           (unsigned)__cvta_generic_to_shared(nb + i)),
                       "l"(src)
                       : "memory");
        }
      asm volatile("cp.async.commit_group;" ::: "memory");
      const double2 acc = cur[threadIdx.x];
      double2* o = out + (int64_t)b * W2;
      for (int i = threadIdx.x; i < W2; i += 512) {
        const double2 v = make_double2(acc.x + i, acc.y - i);
        asm volatile("st.global.cs.v2.f64 [%0], {%1, %2};" ::"l"(o + i),
                     "d"(v.x), "d"(v.y)
                     : "memory");
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      __syncthreads();
      b = bn;
      ++t;
    }
  } else if (MODE == 2) {
    for (;;) {
      if (threadIdx.x == 0) next = (int)atomicAdd(claim, 1u);
      __syncthreads();
      const int b = next;
      if (b >= S) break;
      slice(in, out, b, s);
    }
  } else {
    // queue-like: claim, poll a published counter, look the slot up in a ring
    const long long* pub = reinterpret_cast<const long long*>(claim + 64);
    const int* ring = reinterpret_cast<const int*>(claim + 128);
    for (;;) {
      if (threadIdx.x == 0) {
        const int kk = (int)atomicAdd(claim, 1u);
        int g = S;
        if (kk < S) {
          if (MODE == 3) { while (kk >= ld_acq(pub)) {} g = ring[kk]; }
          else { while (kk >= ld_rlx(pub)) {} g = __ldcg(ring + kk); }
        }
        next = g;
      }
      __syncthreads();
      const int b = next;
      if (b >= S) break;
      slice(in, out, b, s);
    }
  }
}

template <int MODE>
float run(const double2* in, double2* out, int S, int grid, unsigned* claim) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float best = 1e9, sum = 0;
  for (int i = 0; i < 23; ++i) {
    cudaMemsetAsync(claim, 0, 4);
    cudaEventRecord(a);
    k<MODE><<<grid, 512>>>(in, out, S, claim);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (i >= 3) { sum += ms; best = ms < best ? ms : best; }
  }
  return sum / 20;
}

int main() {
  const int S = 4096;
  double2 *in, *out;
  unsigned* claim;
  cudaMalloc(&in, (size_t)S * R2 * 16);
  cudaMalloc(&out, (size_t)S * W2 * 16);
  cudaMalloc(&claim, 4 * (128 + S));
  {  // published = S at word 64 (as long long), ring = identity at word 128
    long long pubv = S;
    cudaMemcpy(claim + 64, &pubv, 8, cudaMemcpyHostToDevice);
    int* ring = new int[S];
    for (int i = 0; i < S; ++i) ring[i] = i;
    cudaMemcpy(claim + 128, ring, 4 * S, cudaMemcpyHostToDevice);
    delete[] ring;
  }
  cudaMemset(in, 0, (size_t)S * R2 * 16);
  int per_sm = 0, sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k<1>, 512, 0);
  const int P = sms * per_sm;
  printf("one CTA per slice (4096 CTAs): %.2f us\n", 1e3 * run<0>(in, out, S, S, claim));
  printf("persistent static (%d CTAs): %.2f us\n", P, 1e3 * run<1>(in, out, S, P, claim));
  printf("persistent claim  (%d CTAs): %.2f us\n", P, 1e3 * run<2>(in, out, S, P, claim));
  printf("claim + double-buffered read (%d CTAs): %.2f us\n", P, 1e3 * run<5>(in, out, S, P, claim));
  {
    int ps = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&ps, k<5>, 512, 0);
    printf("  (mode 5 occupancy %d CTAs/SM)\n", ps);
  }
  printf("claim+acquire poll+ring (%d CTAs): %.2f us\n", P, 1e3 * run<3>(in, out, S, P, claim));
  printf("claim+relaxed poll+cg ring (%d CTAs): %.2f us\n", P, 1e3 * run<4>(in, out, S, P, claim));
  printf("err: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
