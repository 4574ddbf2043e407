// hydro_kernels.cu — sm_100a kernels for the strategy-3 hydro hot path.
//
// Batched re-statements of the reference per-sub-grid numpy bodies
// (/root/reference/pkg/src/taskfuse/hydro/kernels.py), indexed by
// (aggregated slice, cell).  The arithmetic is the reference's, operation
// for operation, with FMA contraction forbidden (explicit __d*_rn
// intrinsics), so every output is bit-identical to the CPU path:
//   minmod      kernels.py:58-60   where(a*b<=0, 0, where(|a|<|b|, a, b))
//   reconstruct kernels.py:73-81   um = base - 0.5*s ; up = base + 0.5*s
//   flux        kernels.py:84-93   F = a*up  |  a*roll(um, -1, axis)
//   update      kernels.py:100-111 u - dt_dx*((dFx) + (dFy)) + (dFz)
//   ghosts      scenario.py:124-142 periodic 26-neighbour fill
//
// Data movement (B200): the fused reconstruct+flux kernel stages each
// slice's (n+4)^2 x (n+6) stencil box — the smallest TMA-legal box covering
// the 6-point star the stencil reads (the inner z extent is the
// full 16-byte-aligned row) — from HBM into shared memory with ONE TMA
// tensor load (cp.async.bulk.tensor.4d, mbarrier completion), so a gather
// of strided team members costs nothing extra: the slice's
// sub-grid id is just the 4th TMA coordinate.  Outputs (um, up, F: 90% of
// the bytes) leave through coalesced streaming stores.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <atomic>
#include <cstdlib>
#include <mutex>
#include <unordered_map>

#include "../../include/taskfuse_b200.h"
#include "internal.h"
#include "sm100_common.cuh"
#include "recon_flux.cuh"

namespace {

// ------------------------------------------ reference launch geometry
// reconstruct_body + flux_body with the REFERENCE's launch geometry
// (blocks_for, kernels.py:39-55): ceil((n+2)^3 / 128) blocks of 128
// threads per slice, one face-cube cell per thread, every stencil value
// read straight from the slice's ghosted sub-grid in global memory (L1 /
// L2), no staging.  Used for the strategy-1 baseline (n = 16: 46 blocks per
// sub-grid) so that a larger sub-grid's launch is spread over as many CTAs
// as the reference assumes.  Same arithmetic as cell_axis (bit-identical).
template <int N>
__global__ void __launch_bounds__(128)
    k_recon_flux_refgeo(const double* __restrict__ pool,
                        const __grid_constant__ TeamIds team, int out_mode,
                        double ax, double ay, double az,
                        double* __restrict__ um, double* __restrict__ up,
                        double* __restrict__ F, double* __restrict__ amax,
                        int flux_form) {
  using G = Geo<N>;
  constexpr int C = G::C, E = G::E, CELLS = G::CELLS;
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int s = blockIdx.y;
  const int g = team.id[s];
  const int c = blockIdx.x * 128 + threadIdx.x;
  const int64_t slot = out_mode ? (int64_t)g : (int64_t)s;
  if (c < CELLS) {
    const double* __restrict__ w = pool + (int64_t)g * G::EXT3;
    const int ci = c / (C * C), cj = (c / C) % C, ck = c % C;
    // cube (ci,cj,ck) = ext (ci+2, cj+2, ck+2)
    const int b = ((ci + 2) * E + (cj + 2)) * E + (ck + 2);
    const int stv[3] = {E * E, E, 1};
    const int pos[3] = {ci, cj, ck};
    const double av[3] = {ax, ay, az};
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      const Faces r = cell_axis(w, b, stv[axis], pos[axis], C, av[axis], 0,
                                flux_form);
      um[(slot * 3 + axis) * CELLS + c] = r.vm;
      up[(slot * 3 + axis) * CELLS + c] = r.vp;
      F[(slot * 3 + axis) * CELLS + c] = r.f;
    }
  }
  if (amax != nullptr && blockIdx.x == 0 && threadIdx.x == 0)
    amax[slot] = fmax(fmax(fabs(ax), fabs(ay)), fabs(az));
}

// ------------------------------------------------ PPM reconstruction
// Piecewise-parabolic reconstruction (Colella & Woodward 1984), the scheme
// north_star names for Octo-Tiger; the reference artifact has no PPM
// (SURVEY F1), so parity is against the self-written oracle/ppm_oracle.py
// (UNPINNED), whose operation order this follows exactly.
// numpy maximum/minimum semantics: first operand on ties, NaN propagates.
__device__ __forceinline__ double np_max(double a, double b) {
  return (a >= b || a != a) ? a : b;
}
__device__ __forceinline__ double np_min(double a, double b) {
  return (a <= b || a != a) ? a : b;
}
// clipped 4th-order interface value between cells b and b+st
__device__ __forceinline__ double ppm_interface(const double* __restrict__ s,
                                                int b, int st) {
  const double u0 = s[b], u1 = s[b + st];
  const double a = __dsub_rn(__dmul_rn(7.0 / 12.0, __dadd_rn(u0, u1)),
                             __dmul_rn(1.0 / 12.0,
                                       __dadd_rn(s[b - st], s[b + 2 * st])));
  return np_min(np_max(a, np_min(u0, u1)), np_max(u0, u1));
}
// CW84 limiting of cell value u between its interface values l and r
__device__ __forceinline__ void ppm_limit(double u, double l, double r,
                                          double& ul, double& ur) {
  const double dq = __dsub_rn(r, l);
  const double mid = __dsub_rn(u, __dmul_rn(0.5, __dadd_rn(l, r)));
  const bool flat = __dmul_rn(__dsub_rn(r, u), __dsub_rn(u, l)) <= 0.0;
  const double lhs = __dmul_rn(dq, mid);
  const double rhs = __dmul_rn(__dmul_rn(dq, dq), 1.0 / 6.0);
  const bool over_l = lhs > rhs;
  const bool over_r = lhs < -rhs;
  ul = flat ? u : (over_l ? __dsub_rn(__dmul_rn(3.0, u), __dmul_rn(2.0, r)) : l);
  ur = flat ? u
            : ((!over_l && over_r)
                   ? __dsub_rn(__dmul_rn(3.0, u), __dmul_rn(2.0, l))
                   : r);
}
// CW84-limited left/right states of the cell at b along st
__device__ __forceinline__ void ppm_states(const double* __restrict__ s, int b,
                                           int st, double& ul, double& ur) {
  ppm_limit(s[b], ppm_interface(s, b - st, st), ppm_interface(s, b, st), ul,
            ur);
}

// Batched PPM reconstruct + (upwind | KT) flux, one CTA per slice, the whole
// ghosted sub-grid staged by one TMA box load.
template <int N, int THREADS, bool DEV_IDS, int MINB = 1>
__global__ void __launch_bounds__(THREADS, MINB)
    k_recon_flux_ppm(const __grid_constant__ CUtensorMap tmap,
                     const int32_t* __restrict__ dev_ids, int out_mode,
                     double ax, double ay, double az, double* __restrict__ um,
                     double* __restrict__ up, double* __restrict__ F,
                     double* __restrict__ amax, int flux_form) {
  using G = Geo<N>;
  constexpr int C = G::C, E = G::E, CELLS = G::CELLS;
  extern __shared__ __align__(128) double sbox[];  // E^3
  __shared__ __align__(8) uint64_t bar;
  __shared__ double red[THREADS / 32];
  __shared__ double s_ul[CELLS];  // one axis' left states (KT / a < 0)
  const int s = blockIdx.x;
  const int g = dev_ids ? dev_ids[s] : s;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  __syncthreads();  // initialised before the arrive (see k_recon_flux)
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, G::EXT3 * (uint32_t)sizeof(double));
    tma_load_box(sbox, &tmap, 0, 0, 0, g, &bar);
  }
  mbar_wait(&bar, 0);
  const int64_t slot = out_mode ? (int64_t)g : (int64_t)s;
  double* um_s = um + slot * 3 * CELLS;
  double* up_s = up + slot * 3 * CELLS;
  double* F_s = F + slot * 3 * CELLS;
  const double av[3] = {ax, ay, az};
  const int stv[3] = {E * E, E, 1};
  const int cst[3] = {C * C, C, 1};  // cube strides
  constexpr int PER = (CELLS + THREADS - 1) / THREADS;
  double speed = 0.0;
  if (flux_form == 0 && ax >= 0.0 && ay >= 0.0 && az >= 0.0) {
    // upwind with a >= 0 on every axis: F = a * up needs no neighbour, so
    // one cell-major pass (measured faster than the axis phases below)
    for (int c = threadIdx.x; c < CELLS; c += THREADS) {
      const int ci = c / (C * C), cj = (c / C) % C, ck = c % C;
      const int b = ((ci + 2) * E + (cj + 2)) * E + (ck + 2);
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        double ul, ur;
        ppm_states(sbox, b, stv[axis], ul, ur);
        __stcs(um_s + axis * CELLS + c, ul);
        __stcs(up_s + axis * CELLS + c, ur);
        __stcs(F_s + axis * CELLS + c, __dmul_rn(av[axis], ur));
      }
    }
    speed = fmax(fmax(fabs(ax), fabs(ay)), fabs(az));
    if (amax != nullptr) block_max_store<THREADS>(speed, red, amax + slot);
    return;
  }
#pragma unroll 1
  for (int axis = 0; axis < 3; ++axis) {
    const int st = stv[axis];
    const double a = av[axis];
    // KT form or a < 0: F needs the NEXT cell's limited left state.  Every
    // cell's left state is formed once (phase 1, into s_ul) and the flux
    // read from there (phase 2) — instead of each cell re-limiting its
    // neighbour.
    const bool next = a < 0.0 || flux_form == 1;
    double urk[PER];
#pragma unroll
    for (int k = 0; k < PER; ++k) {
      const int c = threadIdx.x + k * THREADS;
      if (c >= CELLS) break;
      const int ci = c / (C * C), cj = (c / C) % C, ck = c % C;
      // cube c = extended index c + 2 in every axis
      const int b = ((ci + 2) * E + (cj + 2)) * E + (ck + 2);
      double ul, ur;
      ppm_states(sbox, b, st, ul, ur);
      __stcs(um_s + axis * CELLS + c, ul);
      __stcs(up_s + axis * CELLS + c, ur);
      urk[k] = ur;
      if (next) s_ul[c] = ul;
      else __stcs(F_s + axis * CELLS + c, __dmul_rn(a, ur));
    }
    if (next) {
      __syncthreads();
#pragma unroll
      for (int k = 0; k < PER; ++k) {
        const int c = threadIdx.x + k * THREADS;
        if (c >= CELLS) break;
        const int ci = c / (C * C), cj = (c / C) % C, ck = c % C;
        const int pos = axis == 0 ? ci : (axis == 1 ? cj : ck);
        // np.roll(um, -1): the last layer wraps onto layer 0
        const double next_l =
            s_ul[pos == C - 1 ? c - (C - 1) * cst[axis] : c + cst[axis]];
        const double ur = urk[k];
        double f;
        if (flux_form == 0) {
          f = __dmul_rn(a, next_l);
        } else {
          const double fl = __dmul_rn(a, ur), fr = __dmul_rn(a, next_l);
          f = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl, fr)),
                        __dmul_rn(__dmul_rn(0.5, fabs(a)),
                                  __dsub_rn(next_l, ur)));
        }
        __stcs(F_s + axis * CELLS + c, f);
      }
      __syncthreads();  // s_ul is rewritten for the next axis
    }
    speed = fmax(speed, fabs(a));
  }
  if (amax != nullptr) block_max_store<THREADS>(speed, red, amax + slot);
}

// flux_body alone (kernels.py:84-93), elementwise over (slot, axis, cell).
template <int N>
__global__ void __launch_bounds__(256)
    k_flux(const int32_t* __restrict__ ids, int T, int out_mode, double ax,
           double ay, double az, const double* __restrict__ um,
           const double* __restrict__ up, double* __restrict__ F) {
  using G = Geo<N>;
  constexpr int C = G::C, CELLS = G::CELLS;
  const int64_t total = (int64_t)T * 3 * CELLS;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int s = (int)(i / (3 * CELLS));
    const int r = (int)(i % (3 * CELLS));
    const int axis = r / CELLS;
    const int c = r % CELLS;
    const int64_t slot = out_mode ? (int64_t)(ids ? ids[s] : s) : (int64_t)s;
    const double a = axis == 0 ? ax : (axis == 1 ? ay : az);
    const int64_t off = slot * 3 * CELLS + (int64_t)axis * CELLS;
    double f;
    if (a >= 0.0) {
      f = __dmul_rn(a, up[off + c]);
    } else {
      const int st = axis == 0 ? C * C : (axis == 1 ? C : 1);
      const int pos = (c / st) % C;
      const int cn = pos == C - 1 ? c - (C - 1) * st : c + st;
      f = __dmul_rn(a, um[off + cn]);
    }
    F[off + c] = f;
  }
}

// update_body (kernels.py:100-111): no FMA anywhere, x,y,z accumulation order.
template <int N>
__global__ void __launch_bounds__(256)
    k_update(const double* __restrict__ pool, const int32_t* __restrict__ ids,
             int out_mode, const double* __restrict__ F, double dt_dx,
             double* __restrict__ next) {
  using G = Geo<N>;
  constexpr int C = G::C, E = G::E, CELLS = G::CELLS;
  const int s = blockIdx.x;
  const int g = ids ? ids[s] : s;
  const int64_t slot = out_mode ? (int64_t)g : (int64_t)s;
  const double* __restrict__ Fs = F + slot * 3 * CELLS;
  const double* __restrict__ u = pool + (int64_t)g * G::EXT3;
  double* __restrict__ o = next + (int64_t)g * G::EXT3;
  for (int c = threadIdx.x; c < G::OWN; c += blockDim.x) {
    const int i = c / (N * N), j = (c / N) % N, k = c % N;
    const int own = ((i + 1) * C + (j + 1)) * C + (k + 1);
    double div = __dsub_rn(Fs[own], Fs[own - C * C]);
    div = __dadd_rn(div, __dsub_rn(Fs[CELLS + own], Fs[CELLS + own - C]));
    div = __dadd_rn(div, __dsub_rn(Fs[2 * CELLS + own], Fs[2 * CELLS + own - 1]));
    const int e = ((i + 3) * E + (j + 3)) * E + (k + 3);
    o[e] = __dsub_rn(u[e], __dmul_rn(dt_dx, div));
  }
}

// exchange_ghosts (scenario.py:124-142): every ghost cell of sub-grid g is
// the periodic global cell it overlays, i.e. a neighbour's owned cell.
template <int N>
__global__ void __launch_bounds__(256)
    k_ghost_fill(double* __restrict__ pool, const int32_t* __restrict__ ids,
                 int per_axis) {
  using G = Geo<N>;
  constexpr int E = G::E;
  const int s = blockIdx.x;
  const int g = ids ? ids[s] : s;
  // the 27 periodic neighbours' base offsets, once per CTA (no division or
  // wrap arithmetic per cell); a ghost cell (i,j,k) of direction
  // d = (di,dj,dk) in {-1,0,1}^3 is the neighbour's ext cell (i,j,k) - d*N
  __shared__ int64_t nbase[27];
  if (threadIdx.x < 27) {
    const int m = per_axis;
    const int bx = g / (m * m), by = (g / m) % m, bz = g % m;
    const int t = threadIdx.x;
    const int di = t / 9 - 1, dj = (t / 3) % 3 - 1, dk = t % 3 - 1;
    const int nx = (bx + di + m) % m, ny = (by + dj + m) % m,
              nz = (bz + dk + m) % m;
    nbase[t] = ((int64_t)(nx * m + ny) * m + nz) * G::EXT3 -
               (int64_t)((di * E + dj) * E + dk) * N;
  }
  __syncthreads();
  double* __restrict__ dst = pool + (int64_t)g * G::EXT3;
  // every load issued before any store: sources are neighbours' OWNED
  // cells, destinations this sub-grid's GHOST cells, so they never overlap
  // — but through one pointer the compiler would otherwise serialise each
  // load behind the previous store
  constexpr int TH = 256, PER = (G::EXT3 + TH - 1) / TH;
  constexpr int GRP = PER < 12 ? PER : 12;  // loads in flight per thread
#pragma unroll 1
  for (int q0 = 0; q0 < PER; q0 += GRP) {
    double v[GRP];
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int c = threadIdx.x + (q0 + q) * TH;
      const int i = c / (E * E), j = (c / E) % E, k = c % E;  // constexpr E
      const int t = (((i >= 3) + (i >= N + 3)) * 3 + (j >= 3) +
                     (j >= N + 3)) * 3 + (k >= 3) + (k >= N + 3);
      if (c < G::EXT3 && t != 13) v[q] = pool[nbase[t] + c];  // 13 = owned
    }
#pragma unroll
    for (int q = 0; q < GRP; ++q) {
      const int c = threadIdx.x + (q0 + q) * TH;
      const int i = c / (E * E), j = (c / E) % E, k = c % E;
      const bool owned = i >= 3 && i < N + 3 && j >= 3 && j < N + 3 &&
                         k >= 3 && k < N + 3;
      if (c < G::EXT3 && !owned) dst[c] = v[q];
    }
  }
}

// prep_body (kernels.py:69-70): whole-extended-array copy, 16 B vectors.
template <int N>
__global__ void __launch_bounds__(256)
    k_prep(const double* __restrict__ pool, const int32_t* __restrict__ ids,
           int out_mode, double* __restrict__ w) {
  using G = Geo<N>;
  const int s = blockIdx.x;
  const int g = ids ? ids[s] : s;
  const int64_t slot = out_mode ? (int64_t)g : (int64_t)s;
  const double2* __restrict__ src =
      reinterpret_cast<const double2*>(pool + (int64_t)g * G::EXT3);
  double2* __restrict__ dst = reinterpret_cast<double2*>(w + slot * G::EXT3);
  for (int c = threadIdx.x; c < G::EXT3 / 2; c += blockDim.x) dst[c] = src[c];
}

// make_state / assemble (scenario.py:83-106) on the device: the global
// (G,G,G) field <-> the owned cells of the (S,E,E,E) pool.  DIR 0: field ->
// pool (ghosts untouched), DIR 1: pool -> field.  One thread per owned cell,
// consecutive threads along z in both layouts.
// Sub-grid layers [layer0, layer0 + layers) along x only (the chunks of a
// pipelined upload); the whole field is layer0 = 0, layers = per_axis.
template <int N, int DIR>
__global__ void __launch_bounds__(256)
    k_field_pool(double* __restrict__ field, double* __restrict__ pool,
                 int per_axis, int layer0, int layers) {
  using G = Geo<N>;
  constexpr int E = G::E;
  const int m = per_axis, Gn = per_axis * N;
  const int64_t plane = (int64_t)Gn * Gn;
  const int64_t first = (int64_t)layer0 * N * plane;
  const int64_t total = first + (int64_t)layers * N * plane;
  for (int64_t t = first + blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
       t < total; t += (int64_t)gridDim.x * blockDim.x) {
    const int x = (int)(t / ((int64_t)Gn * Gn));
    const int y = (int)((t / Gn) % Gn), z = (int)(t % Gn);
    const int64_t id = ((int64_t)(x / N) * m + y / N) * m + z / N;
    const int64_t e = id * G::EXT3 +
                      ((int64_t)(x % N + 3) * E + (y % N + 3)) * E + (z % N + 3);
    if (DIR == 0)
      pool[e] = field[t];
    else
      field[t] = pool[e];
  }
}

__global__ void k_reduce(const int32_t* __restrict__ ids, int T, int out_mode,
                         double v, double* __restrict__ out) {
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= T) return;
  const int64_t slot = out_mode ? (int64_t)(ids ? ids[s] : s) : (int64_t)s;
  out[slot] = v;
}

// ------------------------------------------------------------ host side
struct MapKey {
  const void* ptr;
  int64_t slices;
  int n;
  bool operator==(const MapKey& o) const {
    return ptr == o.ptr && slices == o.slices && n == o.n;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.ptr) ^ (size_t)(k.slices * 131 + k.n);
  }
};

// 4-D view (slice, x, y, z) of the pool; box = the (n+4)^2 x (n+6) minmod
// stencil box, or (full) the whole (n+6)^3 ghosted sub-grid (PPM's stencil
// reaches the ghost depth 3).
int pool_map(const double* pool, int64_t slices, int n, CUtensorMap* out,
             bool full = false) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{pool, slices, full ? -n : n};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return 0;
  }
  auto fn = encode_fn();
  if (!fn) return TF_E_NO_TMA;
  const cuuint64_t E = (cuuint64_t)(n + 6);
  const cuuint32_t Bx = (cuuint32_t)(full ? n + 6 : n + 4);
  cuuint64_t dims[4] = {E, E, E, (cuuint64_t)slices};
  cuuint64_t strides[3] = {E * 8, E * E * 8, E * E * E * 8};
  cuuint32_t box[4] = {(cuuint32_t)E, Bx, Bx, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  CUtensorMap m;
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4,
                  const_cast<double*>(pool), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                  // 64-B L2 promotion: each x plane of the box is one
                  // contiguous 1.3 KB run, and 256-B promotion over-fetched
                  // its ends (A/B on B200: +0.8% HBM fraction, 64 vs 256)
                  CU_TENSOR_MAP_L2_PROMOTION_L2_64B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return TF_E_INVALID;
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return 0;
}

template <int N>
constexpr int recon_threads() {
  // 512 threads: every z-pair of an 8^3 slice (500) in flight at once;
  // measured best of 128/256/512 on B200
  return 512;
}

template <int N, int MODE, bool DEV_IDS>
int launch_recon(const CUtensorMap& map, const int32_t* dev_ids,
                     const TeamIds& team, int T, int out_mode, double ax,
                     double ay, double az, double* um, double* up, double* F,
                     double* amax, int flux_form, cudaStream_t st, int flags) {
  constexpr int TH = recon_threads<N>();
  constexpr size_t smem = Geo<N>::BOX * sizeof(double);
  auto kern = k_recon_flux<N, TH, MODE, DEV_IDS>;
  // set once per instantiation (a function-local static: thread-safe init)
  static const cudaError_t smem_attr = cudaFuncSetAttribute(
      kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (smem_attr != cudaSuccess) return smem_attr;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)T);
  cfg.blockDim = dim3(TH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // TF_LAUNCH_OVERLAP_PREV: programmatic dependent launch — this team may
  // start while the previous (independent) team kernel on the stream is
  // still running; the kernel never calls griddepcontrol.wait.
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (flags & TF_LAUNCH_OVERLAP_PREV) ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, map, dev_ids, team, out_mode, ax, ay,
                            az, um, up, F, amax, flux_form);
}

template <int MODE, bool DEV_IDS>
int dispatch_recon(const double* pool, int64_t slices, const int32_t* dev_ids,
                   const TeamIds& team, int T, int n, int out_mode, double ax,
                   double ay, double az, double* um, double* up, double* F,
                   double* amax, int flux_form, cudaStream_t st,
                   int flags = 0) {
  if (T == 0) return 0;
  CUtensorMap map;
  int rc = pool_map(pool, slices, n, &map);
  if (rc) return rc;
  if (n == 8)
    return launch_recon<8, MODE, DEV_IDS>(map, dev_ids, team, T, out_mode, ax,
                                          ay, az, um, up, F, amax, flux_form,
                                          st, flags);
  return launch_recon<16, MODE, DEV_IDS>(map, dev_ids, team, T, out_mode, ax,
                                         ay, az, um, up, F, amax, flux_form,
                                         st, flags);
}

bool valid_n(int n) { return n == 8 || n == 16; }

// ------------------------------------------------- device work queue
// Strategy 3 with a device-side queue: a resident grid consumes the slices
// the host's formation core publishes, team by team, into a ring in mapped
// pinned memory — a team closure costs a few host stores instead of a
// kernel launch.  Control block (mapped pinned memory):
struct QueueCtl {
  long long published;    // (host bookkeeping; the fetcher reads the tags)
  long long final_count;  // host -> GPU: the run's count once closed, or -1
  long long completed;    // GPU -> host: (epoch << 32) | slices done (the
                          //   fetcher is its only writer)
  long long status;       // 0 ok; 1 a fetcher / consumer timed out
};
// device-side mirror, polled by the consumers through L2 (only the fetcher
// CTA ever touches host memory, so the pollers do not flood PCIe)
// Each word on its own 128-B line: the consumers poll `final_count` while
// every CTA hits `done` with atomics — on one shared line those polls and
// atomics serialised in the same L2 slice.
struct QueueDev {
  alignas(128) long long published;
  alignas(128) long long final_count;    // (epoch << 32) | count
  alignas(128) unsigned long long spare; // (the dynamic claim counter once)
  alignas(128) unsigned long long done;  // monotonic over the slot's runs
};
static_assert(sizeof(QueueDev) == 512, "QueueDev layout (aggregator.cpp)");

__device__ __forceinline__ long long ld_relaxed_gpu(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed_gpu_u64(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ long long ld_acquire_gpu(const long long* p) {
  long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acquire_gpu_u64(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_gpu(long long* p, long long v) {
  asm volatile("st.release.gpu.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void st_relaxed_sys(long long* p, long long v) {
  asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// Programmatic dependent launch between consecutive runs of the queue: run
// k+1's CTAs take the SM slots run k's CTAs leave during its tail, mirror
// and fetch their first ring entries (and, with early_loads, load their
// stencil boxes) while run k finishes; a consumer waits for run k
// (griddepcontrol.wait: complete, its writes visible) before its first
// output store.  The fetcher waits before it triggers the NEXT run, so a
// launched run k+2 implies run k is complete — the invariant that lets the
// queue slot of run k be reused by run k+2 without any counter reset (the
// `done` count is monotonic, done_base; final_count carries the epoch).
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void pdl_trigger() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// final_count mirror on the device, tagged with the run's epoch so that a
// slot's counters never need resetting: (epoch << 32) | count
__device__ __forceinline__ long long fin_of(long long tagged, unsigned epoch) {
  return (unsigned)((unsigned long long)tagged >> 32) == epoch
             ? (long long)(unsigned)tagged
             : -1;
}

__device__ __forceinline__ unsigned long long ld_relaxed_sys_u64(
    const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Block 0 is the fetcher: it mirrors the host ring into device memory and
// reports the device-side completion count back to the host.  Host entries
// carry the run's epoch like the device ones ((epoch << 32) | id), so a
// round reads the ring SPECULATIVELY — no round trip for a published count
// first: every entry read with this run's tag is mirrored (all threads,
// several independent PCIe reads in flight each), the valid prefix advances
// the cursor, and the close marker (final_count) rides in the same round
// trip.  Blocks 1.. compute the slices (k_queue_consumer).  The slot's
// `done` counter is monotonic across runs: this run counts from done_base.
template <int THREADS>
__device__ void queue_fetcher(const unsigned long long* __restrict__ ring_h,
                              QueueCtl* ctl,
                              unsigned long long* __restrict__ ring_d,
                              long long ring_cap, QueueDev* qd, unsigned epoch,
                              unsigned long long done_base,
                              long long timeout_ns, int sort_shift) {
  __shared__ long long s_fin;
  __shared__ int s_bad, s_stop;
  // sort_shift >= 0: each round's entries go to the device ring ordered by
  // sub-grid id (buckets of 2^sort_shift ids, a counting sort): the formed
  // teams' members are the reference's strided parents (arrival % P), and
  // consecutive CTAs then work on sub-grids far apart in memory — in id
  // order the grid streams the pool and the outputs like a one-launch team
  constexpr int NBUCKET = 1024;
  __shared__ int s_hist[NBUCKET];
  constexpr int U = 8;                  // loads in flight per thread
  constexpr int CHUNK = THREADS * U;    // entries read per round
  long long fetched = 0, fin_sent = -1, reported = -1;
  int span = CHUNK;                     // 32 after a round without progress
  bool triggered = false;
  unsigned long long last_change = globaltimer();
  // phase 1: mirror entries as the host publishes them, until the queue is
  // closed and every entry below the close is mirrored
  for (;;) {
    const long long end = fin_sent >= 0 ? fin_sent : ring_cap;
    const long long lim = fetched + span < end ? fetched + span : end;
    if (threadIdx.x == 0) {
      s_bad = CHUNK;
      s_fin = (long long)ld_relaxed_sys_u64(
          reinterpret_cast<const unsigned long long*>(&ctl->final_count));
    }
    unsigned long long v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = fetched + u * THREADS + threadIdx.x;
      v[u] = k < lim ? ld_relaxed_sys_u64(ring_h + k) : 0ULL;
    }
    if (sort_shift >= 0)
      for (int b = threadIdx.x; b < NBUCKET; b += THREADS) s_hist[b] = 0;
    __syncthreads();  // s_bad (and the histogram) initialised
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = fetched + u * THREADS + threadIdx.x;
      if (k < lim) {
        // a consumer that sees its run's epoch in the slot has the id —
        // no fence, no acquire (and no L1 invalidation) needed
        if ((unsigned)(v[u] >> 32) == epoch) {
          if (sort_shift < 0) ring_d[k] = v[u];
        } else {
          atomicMin(&s_bad, u * THREADS + (int)threadIdx.x);
        }
      }
    }
    __syncthreads();
    const long long fin = s_fin;
    const long long valid = s_bad < lim - fetched ? s_bad : lim - fetched;
    if (sort_shift >= 0 && valid > 0) {
      // counting sort of the round's valid prefix by id bucket
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = u * THREADS + threadIdx.x;
        if (i < valid)
          atomicAdd(&s_hist[min((int)((unsigned)v[u] >> sort_shift),
                                NBUCKET - 1)], 1);
      }
      __syncthreads();
      if (threadIdx.x < 32) {
        // exclusive scan of the histogram by one warp (32 buckets a lane)
        constexpr int PER = NBUCKET / 32;
        int sum = 0;
#pragma unroll
        for (int j = 0; j < PER; ++j) sum += s_hist[threadIdx.x * PER + j];
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int t = __shfl_up_sync(0xffffffffu, incl, o);
          if ((int)threadIdx.x >= o) incl += t;
        }
        int run = incl - sum;
#pragma unroll
        for (int j = 0; j < PER; ++j) {
          const int c = s_hist[threadIdx.x * PER + j];
          s_hist[threadIdx.x * PER + j] = run;
          run += c;
        }
      }
      __syncthreads();
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int i = u * THREADS + threadIdx.x;
        if (i < valid) {
          const int pos = atomicAdd(
              &s_hist[min((int)((unsigned)v[u] >> sort_shift), NBUCKET - 1)],
              1);
          ring_d[fetched + pos] = v[u];
        }
      }
    }
    fetched += valid;
    span = valid > 0 ? CHUNK : 32;
    if (valid > 0) last_change = globaltimer();
    if (!triggered) {
      // the first entries are out: wait for the previous run (its tail
      // overlaps this mirror), then let the next run launch
      pdl_wait();
      pdl_trigger();
      triggered = true;
    }
    if (threadIdx.x == 0) {
      if (fin >= 0 && fin_sent < 0)
        // the close marker as soon as it is known: CTAs beyond it exit
        st_release_gpu(&qd->final_count,
                       (long long)(((unsigned long long)epoch << 32) |
                                   (unsigned long long)fin));
      const long long done =
          (long long)(ld_relaxed_gpu_u64(&qd->done) - done_base);
      if (done != reported) {
        st_relaxed_sys(&ctl->completed,
                       (long long)(((unsigned long long)epoch << 32) |
                                   (unsigned long long)done));
        reported = done;
        last_change = globaltimer();
      }
      int stop = fin >= 0 && fetched >= fin ? 1 : 0;
      if (!stop && (long long)(globaltimer() - last_change) > timeout_ns) {
        st_release_gpu(&qd->final_count,
                       (long long)(((unsigned long long)epoch << 32) |
                                   (unsigned long long)fetched));
        st_release_sys(&ctl->status, 1);
        stop = 2;
      }
      s_stop = stop;
    }
    if (fin >= 0 && fin_sent < 0) fin_sent = fin;
    __syncthreads();
    if (s_stop) break;
    if (valid == 0) __nanosleep(100);
  }
  if (threadIdx.x != 0) return;
  // phase 2 (one thread): every entry is on the device; post completions to
  // the host until all are done — relaxed device loads and relaxed posted
  // stores (a system-scope release per update cost microseconds each, and
  // the run's grid ends only when this loop sees the last slice)
  if (s_stop != 2) {
    const long long fin = fin_sent;
    const unsigned long long tag = (unsigned long long)epoch << 32;
    unsigned long long last_post = 0;
    for (;;) {
      const long long done =
          (long long)(ld_relaxed_gpu_u64(&qd->done) - done_base);
      const unsigned long long now = globaltimer();
      // at most one post per microsecond until the last one: every post
      // takes the line from the host core that polls it (a miss there per
      // post, in the formation loop's busy test)
      if (done != reported && (done >= fin || now - last_post >= 1000)) {
        st_relaxed_sys(&ctl->completed,
                       (long long)(tag | (unsigned long long)done));
        reported = done;
        last_change = now;
        last_post = now;
      }
      if (done >= fin) break;
      if ((long long)(globaltimer() - last_change) > timeout_ns) {
        st_release_sys(&ctl->status, 1);
        break;
      }
      __nanosleep(32);
    }
  }
}

// One CTA per ring entry: CTA k (blocks 1..) computes the k-th published
// slice, so the hardware's block scheduler — not a software claim loop —
// hands slices to free SM slots, exactly as in a one-launch team kernel.
// A persistent consumer grid (each CTA looping over claimed slices) ran
// 6 us (10%) slower than the one-launch kernel on the same pre-published
// slices: every slice ended in a block barrier waiting for the service
// thread's warp, whether the slice was claimed dynamically (atomic + ring
// poll) or statically with the entry prefetched (67.7 vs 61.4 us).
//
// Wait until ring entry k carries this run's epoch: returns the sub-grid
// id, -1 once the queue is closed below k, -2 on timeout.
__device__ __noinline__ int queue_poll(const QueueDev* qd,
                                       const unsigned long long* ring_d,
                                       long long k, long long ring_cap,
                                       unsigned epoch, long long timeout_ns) {
  const unsigned long long t0 = globaltimer();
  for (;;) {
    // this run publishes at most ring_cap ids: a slot beyond them is never
    // filled (and lies outside the ring)
    if (k >= ring_cap) return -1;
    // relaxed polls only: an acquire would invalidate the SM's L1
    const unsigned long long v = ld_relaxed_gpu_u64(ring_d + k);
    if ((unsigned)(v >> 32) == epoch) return (int)(unsigned)v;
    const long long fin = fin_of(ld_relaxed_gpu(&qd->final_count), epoch);
    if (fin >= 0 && k >= fin) return -1;  // queue closed and drained
    if ((long long)(globaltimer() - t0) > timeout_ns) return -2;
    __nanosleep(200);
  }
}

template <int N, int THREADS>
__global__ void __launch_bounds__(THREADS, recon_min_blocks<THREADS>())
    k_queue_consumer(const __grid_constant__ CUtensorMap tmap,
                     const unsigned long long* __restrict__ ring_h,
                     QueueCtl* ctl, unsigned long long* __restrict__ ring_d,
                     long long ring_cap, QueueDev* qd,
                     unsigned long long done_base, unsigned epoch, double ax,
                     double ay, double az, double* __restrict__ um,
                     double* __restrict__ up, double* __restrict__ F,
                     double* __restrict__ amax, int flux_form,
                     long long timeout_ns, int early_loads, int sort_shift) {
  using G = Geo<N>;
  constexpr int CELLS = G::CELLS;
  if (blockIdx.x == 0) {
    queue_fetcher<THREADS>(ring_h, ctl, ring_d, ring_cap, qd, epoch,
                           done_base, timeout_ns, sort_shift);
    return;
  }
  // slice CTAs never gate the next run's launch: the fetcher does
  pdl_trigger();
  extern __shared__ __align__(128) double sbox[];
  __shared__ __align__(8) uint64_t bar;
  __shared__ double red[THREADS / 32];
  __shared__ int s_g;
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  // the box load waits for the previous kernel on the stream unless the
  // caller vouched that it does not produce the pool (early_loads)
  if (!early_loads) pdl_wait();
  __syncthreads();  // initialised before the first arrive (k_recon_flux)
  if (threadIdx.x == 0) {
    const int g = queue_poll(qd, ring_d, (long long)blockIdx.x - 1, ring_cap,
                             epoch, timeout_ns);
    s_g = g;
    if (g >= 0) {
      mbar_expect_tx(&bar, G::BOX * (uint32_t)sizeof(double));
      tma_load_box(sbox, &tmap, 0, 1, 1, g, &bar);
    } else if (g == -2) {
      // nothing arrived in time: give the GPU back and tell the host
      st_release_sys(&ctl->status, 1);
    }
  }
  __syncthreads();
  const int g = s_g;
  if (g < 0) return;
  mbar_wait(&bar, 0);
  // the previous run on the stream writes the same outputs: its writes
  // land first
  if (early_loads) pdl_wait();
  const double speed = slice_compute<N, THREADS, 0, true>(
      sbox, um + (int64_t)g * 3 * CELLS, up + (int64_t)g * 3 * CELLS,
      F + (int64_t)g * 3 * CELLS, ax, ay, az, flux_form);
  if (amax != nullptr)
    block_max_store<THREADS>(speed, red, amax + g);  // thread 0 stores last
  else
    __syncthreads();
  // the completion count is the host's busy signal only (the kernel's exit
  // orders the outputs for the stream), so no fence before it: a fence (or
  // a system-scope store) here holds the CTA until its stores drain
  if (threadIdx.x == 0) atomicAdd(&qd->done, 1ULL);
}

}  // namespace

extern "C" {

int tf_internal_pool_map(const double* pool, int64_t slices, int n,
                         CUtensorMap* out) {
  if (!valid_n(n) || !pool || slices < 1 || !out) return TF_E_INVALID;
  return pool_map(pool, slices, n, out);
}

int tf_recon_flux_f64(const double* pool_ext, int64_t pool_slices,
                      const int32_t* ids, int32_t T, int32_t n, double ax,
                      double ay, double az, double* um, double* up, double* F,
                      int32_t out_mode, double* amax, int32_t flux_form,
                      tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !pool_ext || !um || !up || !F ||
      (flux_form != 0 && flux_form != 1) || pool_slices < 1 ||
      (ids == nullptr && T > pool_slices))
    return TF_E_INVALID;
  static const TeamIds none{};
  return dispatch_recon<0, true>(pool_ext, pool_slices, ids, none, T, n,
                                 out_mode, ax, ay, az, um, up, F, amax,
                                 flux_form, (cudaStream_t)stream);
}

int tf_recon_flux_team_f64(const double* pool_ext, int64_t pool_slices,
                           const int32_t* host_ids, int32_t T, int32_t n,
                           double ax, double ay, double az, double* um,
                           double* up, double* F, int32_t out_mode,
                           double* amax, int32_t flux_form,
                           tf_stream_t stream) {
  return tf_recon_flux_team_ex_f64(pool_ext, pool_slices, host_ids, T, n, ax,
                                   ay, az, um, up, F, out_mode, amax,
                                   flux_form, 0, stream);
}

int tf_recon_flux_team_ex_f64(const double* pool_ext, int64_t pool_slices,
                              const int32_t* host_ids, int32_t T, int32_t n,
                              double ax, double ay, double az, double* um,
                              double* up, double* F, int32_t out_mode,
                              double* amax, int32_t flux_form, int32_t flags,
                              tf_stream_t stream) {
  if (!valid_n(n) || T < 1 || T > TF_MAX_TEAM || !host_ids || !pool_ext ||
      !um || !up || !F || (flux_form != 0 && flux_form != 1))
    return TF_E_INVALID;
  TeamIds team;
  for (int i = 0; i < T; ++i) {
    if (host_ids[i] < 0 || host_ids[i] >= pool_slices) return TF_E_INVALID;
    team.id[i] = host_ids[i];
  }
  return dispatch_recon<0, false>(pool_ext, pool_slices, nullptr, team, T, n,
                                  out_mode, ax, ay, az, um, up, F, amax,
                                  flux_form, (cudaStream_t)stream, flags);
}

int tf_recon_flux_refgeo_f64(const double* pool_ext, int64_t pool_slices,
                             const int32_t* host_ids, int32_t T, int32_t n,
                             double ax, double ay, double az, double* um,
                             double* up, double* F, int32_t out_mode,
                             double* amax, int32_t flux_form, int32_t flags,
                             tf_stream_t stream) {
  if (!valid_n(n) || T < 1 || T > TF_MAX_TEAM || !host_ids || !pool_ext ||
      !um || !up || !F || (flux_form != 0 && flux_form != 1))
    return TF_E_INVALID;
  TeamIds team;
  for (int i = 0; i < T; ++i) {
    if (host_ids[i] < 0 || host_ids[i] >= pool_slices) return TF_E_INVALID;
    team.id[i] = host_ids[i];
  }
  const int C = n + 2;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((C * C * C + 127) / 128), (unsigned)T);
  cfg.blockDim = dim3(128);
  cfg.stream = (cudaStream_t)stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (flags & TF_LAUNCH_OVERLAP_PREV) ? 1 : 0;
  if (n == 8)
    return cudaLaunchKernelEx(&cfg, k_recon_flux_refgeo<8>, pool_ext, team,
                              out_mode, ax, ay, az, um, up, F, amax,
                              flux_form);
  return cudaLaunchKernelEx(&cfg, k_recon_flux_refgeo<16>, pool_ext, team,
                            out_mode, ax, ay, az, um, up, F, amax, flux_form);
}

int tf_reconstruct_f64(const double* pool_ext, int64_t pool_slices,
                       const int32_t* ids, int32_t T, int32_t n, double* um,
                       double* up, int32_t out_mode, tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !pool_ext || !um || !up || pool_slices < 1 ||
      (ids == nullptr && T > pool_slices))
    return TF_E_INVALID;
  static const TeamIds none{};
  return dispatch_recon<1, true>(pool_ext, pool_slices, ids, none, T, n,
                                 out_mode, 0, 0, 0, um, up, nullptr, nullptr,
                                 0, (cudaStream_t)stream);
}

int tf_flux_f64(const int32_t* ids, int32_t T, int32_t n, double ax, double ay,
                double az, const double* um, const double* up, double* F,
                int32_t out_mode, tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !um || !up || !F) return TF_E_INVALID;
  if (T == 0) return 0;
  const int64_t total = (int64_t)T * 3 * (n + 2) * (n + 2) * (n + 2);
  const int blocks = (int)((total + 255) / 256 < 148 * 16 ? (total + 255) / 256
                                                          : 148 * 16);
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8)
    k_flux<8><<<blocks, 256, 0, st>>>(ids, T, out_mode, ax, ay, az, um, up, F);
  else
    k_flux<16><<<blocks, 256, 0, st>>>(ids, T, out_mode, ax, ay, az, um, up, F);
  return cudaGetLastError();
}

int tf_update_f64(const double* pool_ext, const int32_t* ids, int32_t T,
                  int32_t n, const double* F, int32_t out_mode, double dt_dx,
                  double* next_ext, tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !pool_ext || !F || !next_ext)
    return TF_E_INVALID;
  if (T == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8)
    k_update<8><<<T, 256, 0, st>>>(pool_ext, ids, out_mode, F, dt_dx, next_ext);
  else
    k_update<16><<<T, 256, 0, st>>>(pool_ext, ids, out_mode, F, dt_dx,
                                    next_ext);
  return cudaGetLastError();
}

int tf_ghost_fill_f64(double* pool_ext, const int32_t* ids, int32_t T,
                      int32_t n, int32_t per_axis, tf_stream_t stream) {
  if (!valid_n(n) || per_axis < 1 || !pool_ext) return TF_E_INVALID;
  const int64_t S = (int64_t)per_axis * per_axis * per_axis;
  if (ids == nullptr) T = (int32_t)S;
  if (T < 0 || (ids == nullptr && T != S)) return TF_E_INVALID;
  if (T == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  // (a variant walking a compile-time table of the ghost shell instead of
  // the per-cell index math measured the same: 27.8-28.2 vs 28.2-28.7 us at
  // config 2, 186 vs 179 us at grid 256 — DESIGN.md §4)
  if (n == 8)
    k_ghost_fill<8><<<T, 256, 0, st>>>(pool_ext, ids, per_axis);
  else
    k_ghost_fill<16><<<T, 256, 0, st>>>(pool_ext, ids, per_axis);
  return cudaGetLastError();
}

int tf_prep_f64(const double* pool_ext, const int32_t* ids, int32_t T,
                int32_t n, double* w, int32_t out_mode, tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !pool_ext || !w) return TF_E_INVALID;
  if (T == 0) return 0;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8)
    k_prep<8><<<T, 256, 0, st>>>(pool_ext, ids, out_mode, w);
  else
    k_prep<16><<<T, 256, 0, st>>>(pool_ext, ids, out_mode, w);
  return cudaGetLastError();
}

int tf_reduce_f64(const int32_t* ids, int32_t T, double ax, double ay,
                  double az, double* reduce_out, int32_t out_mode,
                  tf_stream_t stream) {
  if (T < 0 || !reduce_out) return TF_E_INVALID;
  if (T == 0) return 0;
  // max_speed (scenario.py:40-41): max(|v|) over the velocity components
  double v = fabs(ax);
  v = fabs(ay) > v ? fabs(ay) : v;
  v = fabs(az) > v ? fabs(az) : v;
  k_reduce<<<(T + 127) / 128, 128, 0, (cudaStream_t)stream>>>(
      ids, T, out_mode, v, reduce_out);
  return cudaGetLastError();
}

static int field_pool(double* field, double* pool, int32_t grid_n, int32_t n,
                      int dir, tf_stream_t stream, int layer0 = 0,
                      int layers = -1) {
  if (!valid_n(n) || grid_n < n || grid_n % n || !field || !pool)
    return TF_E_INVALID;
  const int m = grid_n / n;
  if (layers < 0) layers = m;
  if (layer0 < 0 || layer0 + layers > m) return TF_E_INVALID;
  if (layers == 0) return 0;
  const int64_t total = (int64_t)layers * n * grid_n * grid_n;
  const int blocks =
      (int)((total + 255) / 256 < 148 * 32 ? (total + 255) / 256 : 148 * 32);
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8) {
    if (dir == 0)
      k_field_pool<8, 0><<<blocks, 256, 0, st>>>(field, pool, m, layer0, layers);
    else
      k_field_pool<8, 1><<<blocks, 256, 0, st>>>(field, pool, m, layer0, layers);
  } else {
    if (dir == 0)
      k_field_pool<16, 0><<<blocks, 256, 0, st>>>(field, pool, m, layer0,
                                                  layers);
    else
      k_field_pool<16, 1><<<blocks, 256, 0, st>>>(field, pool, m, layer0,
                                                  layers);
  }
  return cudaGetLastError();
}

int tf_field_to_pool_layers_f64(const double* field, int32_t grid_n,
                                int32_t n, int32_t layer0, int32_t layers,
                                double* pool_ext, tf_stream_t stream) {
  return field_pool(const_cast<double*>(field), pool_ext, grid_n, n, 0,
                    stream, layer0, layers);
}

int tf_field_to_pool_f64(const double* field, int32_t grid_n, int32_t n,
                         double* pool_ext, tf_stream_t stream) {
  return field_pool(const_cast<double*>(field), pool_ext, grid_n, n, 0,
                    stream);
}

int tf_pool_to_field_f64(const double* pool_ext, int32_t grid_n, int32_t n,
                         double* field, tf_stream_t stream) {
  return field_pool(field, const_cast<double*>(pool_ext), grid_n, n, 1,
                    stream);
}

int tf_recon_flux_ppm_f64(const double* pool_ext, int64_t pool_slices,
                          const int32_t* ids, int32_t T, int32_t n, double ax,
                          double ay, double az, double* um, double* up,
                          double* F, int32_t out_mode, double* amax,
                          int32_t flux_form, tf_stream_t stream) {
  if (!valid_n(n) || T < 0 || !pool_ext || !um || !up || !F ||
      (flux_form != 0 && flux_form != 1) || pool_slices < 1 ||
      (ids == nullptr && T > pool_slices))
    return TF_E_INVALID;
  if (T == 0) return 0;
  CUtensorMap map;
  int rc = pool_map(pool_ext, pool_slices, n, &map, /*full=*/true);
  if (rc) return rc;
  constexpr int TH = 512;
  cudaStream_t st = (cudaStream_t)stream;
  if (n == 8) {
    constexpr size_t smem = Geo<8>::EXT3 * sizeof(double);
    // 256 threads at <= 64 registers, 4 CTAs/SM: measured best of 128 /
    // 256 / 512 threads x register budgets (config 2, one launch: PPM +
    // upwind 68.6% -> 88.5% of HBM, PPM + KT 52.8% -> 54.7%)
    k_recon_flux_ppm<8, 256, true, 4><<<T, 256, smem, st>>>(
        map, ids, out_mode, ax, ay, az, um, up, F, amax, flux_form);
  } else {
    constexpr size_t smem = Geo<16>::EXT3 * sizeof(double);
    static const cudaError_t smem_attr = cudaFuncSetAttribute(
        k_recon_flux_ppm<16, TH, true>,
        cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (smem_attr != cudaSuccess) return smem_attr;
    k_recon_flux_ppm<16, TH, true><<<T, TH, smem, st>>>(
        map, ids, out_mode, ax, ay, az, um, up, F, amax, flux_form);
  }
  return cudaGetLastError();
}

}  // extern "C"

namespace {

template <int N>
int consumer_launch(const CUtensorMap& map, cudaStream_t st,
                    const int64_t* ring_h, QueueCtl* c, int64_t* ring_d,
                    int64_t ring_cap, QueueDev* q, uint64_t done_base,
                    int32_t epoch, double ax, double ay, double az,
                    double* um, double* up, double* F, double* amax,
                    int32_t flux_form, int64_t timeout_ns, int32_t flags,
                    int sort_shift) {
  // flags: TF_QUEUE_CHAIN — launched as a programmatic dependent of the
  // previous kernel on the stream; TF_LAUNCH_OVERLAP_PREV — and the first
  // stencil boxes may load before that kernel completes.  sort_shift: the
  // fetcher's id-bucket width for TF_QUEUE_SORTED, or -1
  constexpr int TH = 512;
  const int smem = Geo<N>::BOX * (int)sizeof(double);
  static const cudaError_t attr_ok = cudaFuncSetAttribute(
      k_queue_consumer<N, TH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      smem);
  if (attr_ok != cudaSuccess) return attr_ok;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)ring_cap + 1);  // the fetcher + a CTA per entry
  cfg.blockDim = dim3(TH);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = (flags & (TF_QUEUE_CHAIN | TF_LAUNCH_OVERLAP_PREV)) ? 1 : 0;
  return cudaLaunchKernelEx(
      &cfg, k_queue_consumer<N, TH>, map,
      reinterpret_cast<const unsigned long long*>(ring_h), c,
      reinterpret_cast<unsigned long long*>(ring_d), (long long)ring_cap, q,
      (unsigned long long)done_base, (unsigned)epoch, ax, ay, az, um, up, F,
      amax, (int)flux_form, (long long)timeout_ns,
      (flags & TF_LAUNCH_OVERLAP_PREV) ? 1 : 0, sort_shift);
}

}  // namespace

extern "C" {

int tf_queue_consumer_launch(const double* pool_ext, int64_t pool_slices,
                             int32_t n, const int64_t* ring_h, void* ctl_h,
                             int64_t* ring_d, int64_t ring_cap, void* qdev,
                             uint64_t done_base, int32_t epoch, double ax,
                             double ay, double az, double* um, double* up,
                             double* F, double* amax, int32_t flux_form,
                             int64_t timeout_ns, int32_t flags,
                             tf_stream_t stream) {
  if (!valid_n(n) || !pool_ext || !ring_h || !ctl_h || !ring_d || !qdev ||
      ring_cap < 0 || ring_cap >= (1LL << 31) - 1 || epoch < 1 || !um ||
      !up || !F ||
      (flags & ~(TF_QUEUE_CHAIN | TF_LAUNCH_OVERLAP_PREV | TF_QUEUE_SORTED)))
    return TF_E_INVALID;
  // TF_QUEUE_SORTED: the id-bucket width that fits the pool in 1024 buckets
  int sort_shift = -1;
  if (flags & TF_QUEUE_SORTED) {
    sort_shift = 0;
    while (((pool_slices - 1) >> sort_shift) >= 1024) ++sort_shift;
  }
  CUtensorMap map;
  int rc = pool_map(pool_ext, pool_slices, n, &map);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;
  QueueCtl* c = static_cast<QueueCtl*>(ctl_h);
  QueueDev* q = static_cast<QueueDev*>(qdev);
  auto go = [&](auto launch) {
    return launch(map, st, ring_h, c, ring_d, ring_cap, q, done_base, epoch,
                  ax, ay, az, um, up, F, amax, flux_form, timeout_ns,
                  flags & ~TF_QUEUE_SORTED, sort_shift);
  };
  return n == 8 ? go(consumer_launch<8>) : go(consumer_launch<16>);
}

// device.py:237-252 enqueue_copy: a real stream-ordered copy (pinned host
// <-> device, or device <-> device), direction inferred from the pointers.
int tf_memcpy_async(void* dst, const void* src, int64_t bytes,
                    tf_stream_t stream) {
  if (bytes < 0 || (bytes > 0 && (!dst || !src))) return TF_E_INVALID;
  if (bytes == 0) return 0;
  return cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault,
                         (cudaStream_t)stream);
}

const char* tf_version(void) { return "taskfuse_b200 0.1 sm_100a"; }

int tf_check_device(int32_t dev) {
  cudaDeviceProp p;
  cudaError_t e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) return e;
  return (p.major == 10 && p.minor == 0) ? 0 : TF_E_INVALID;
}

}  // extern "C"
