// halo.cu — slab-partitioned ghost exchange for multi-GPU runs.
//
// The sub-grid lattice (m per axis) is cut into x-slabs of mx sub-grid
// layers per rank.  A rank's ghost shell needs, in x, the 3 cell layers
// adjacent to its slab on either side (the ring neighbours' boundary layers,
// periodic: scenario.py:134); in y and z the rank holds the full periodic
// extent.  Per iteration:  pack own boundary layers -> exchange planes with
// the two ring neighbours (NCCL P2P) -> fill every ghost cell from the local
// pool or the received halo planes.  With one rank the halo planes are the
// rank's own opposite boundary layers, so the fill reduces exactly to
// exchange_ghosts (scenario.py:124-142) — decomposition invariance
// (test_hydro.py:139-142) is the parity anchor.
//
// Plane layout: (3, G, G) FP64, G = m*n (global y, z), layer 0 lowest x.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/taskfuse_b200.h"

namespace {

template <int N>
__global__ void __launch_bounds__(256)
    k_halo_pack(const double* __restrict__ pool, int mx, int m,
                double* __restrict__ lo, double* __restrict__ hi) {
  constexpr int E = N + 6;
  const int G = m * N;
  const int64_t per = 3LL * G * G;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < 2 * per;
       t += (int64_t)gridDim.x * blockDim.x) {
    const bool upper = t >= per;
    const int64_t r = upper ? t - per : t;
    const int l = (int)(r / ((int64_t)G * G));
    const int gy = (int)((r / G) % G), gz = (int)(r % G);
    // lo: local x = l (sub-grid 0, ext 3+l); hi: local x = mx*N-3+l
    const int lbx = upper ? mx - 1 : 0;
    const int ex = upper ? N + l : 3 + l;
    const int64_t id = ((int64_t)lbx * m + gy / N) * m + gz / N;
    const double v =
        pool[id * E * E * E + ((int64_t)ex * E + (gy % N + 3)) * E + (gz % N + 3)];
    (upper ? hi : lo)[r] = v;
  }
}

template <int N>
__global__ void __launch_bounds__(256)
    k_ghost_fill_slab(double* __restrict__ pool, int mx, int m,
                      const double* __restrict__ halo_lo,
                      const double* __restrict__ halo_hi, int first) {
  constexpr int E = N + 6;
  const int G = m * N, X = mx * N;
  const int g = first + blockIdx.x;
  const int bx = g / (m * m), by = (g / m) % m, bz = g % m;
  double* __restrict__ dst = pool + (int64_t)g * E * E * E;
  // loads issued in groups before their stores: sources (neighbours' owned
  // cells, halo planes) never overlap destinations (this sub-grid's ghost
  // cells), but through one pointer the compiler would serialise each load
  // behind the previous store (the same fix as k_ghost_fill)
  constexpr int TH = 256, PER = (E * E * E + TH - 1) / TH;
  constexpr int GRP = PER < 12 ? PER : 12;
#pragma unroll 1
  for (int q0 = 0; q0 < PER; q0 += GRP) {
    double v[GRP];
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int c = threadIdx.x + (q0 + q) * TH;
      const int i = c / (E * E), j = (c / E) % E, k = c % E;
      if (c >= E * E * E ||
          (i >= 3 && i < N + 3 && j >= 3 && j < N + 3 && k >= 3 && k < N + 3))
        continue;
      const int lx = bx * N + i - 3;  // slab-local x, in [-3, X+3)
      const int gy = (by * N + j - 3 + G) % G;
      const int gz = (bz * N + k - 3 + G) % G;
      if (lx < 0) {
        v[q] = halo_lo[((int64_t)(lx + 3) * G + gy) * G + gz];
      } else if (lx >= X) {
        v[q] = halo_hi[((int64_t)(lx - X) * G + gy) * G + gz];
      } else {
        const int64_t src = ((int64_t)(lx / N) * m + gy / N) * m + gz / N;
        v[q] = pool[src * E * E * E + ((int64_t)(lx % N + 3) * E +
                                      (gy % N + 3)) * E + (gz % N + 3)];
      }
    }
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int c = threadIdx.x + (q0 + q) * TH;
      const int i = c / (E * E), j = (c / E) % E, k = c % E;
      if (c < E * E * E &&
          !(i >= 3 && i < N + 3 && j >= 3 && j < N + 3 && k >= 3 && k < N + 3))
        dst[c] = v[q];
    }
  }
}

}  // namespace

extern "C" {

int tf_halo_pack_f64(const double* pool_ext, int32_t n, int32_t mx, int32_t m,
                     double* lo_plane, double* hi_plane, tf_stream_t stream) {
  if ((n != 8 && n != 16) || mx < 1 || m < 1 || !pool_ext || !lo_plane ||
      !hi_plane)
    return TF_E_INVALID;
  const int64_t total = 2LL * 3 * (int64_t)m * n * m * n;
  const int blocks = (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256
                                                          : 148 * 32);
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8)
    k_halo_pack<8><<<blocks, 256, 0, st>>>(pool_ext, mx, m, lo_plane, hi_plane);
  else
    k_halo_pack<16><<<blocks, 256, 0, st>>>(pool_ext, mx, m, lo_plane,
                                            hi_plane);
  return cudaGetLastError();
}

int tf_ghost_fill_slab_f64(double* pool_ext, int32_t n, int32_t mx, int32_t m,
                           const double* halo_lo, const double* halo_hi,
                           int32_t first, int32_t count, tf_stream_t stream) {
  if ((n != 8 && n != 16) || mx < 1 || m < 1 || !pool_ext || !halo_lo ||
      !halo_hi || first < 0 || count < 0 || first + count > mx * m * m)
    return TF_E_INVALID;
  if (count == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8)
    k_ghost_fill_slab<8><<<count, 256, 0, st>>>(pool_ext, mx, m, halo_lo,
                                                halo_hi, first);
  else
    k_ghost_fill_slab<16><<<count, 256, 0, st>>>(pool_ext, mx, m, halo_lo,
                                                 halo_hi, first);
  return cudaGetLastError();
}

}  // extern "C"
