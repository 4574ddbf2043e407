// recon_flux.cuh — the fused reconstruct+flux kernel (k_recon_flux) and
// its numerics, shared by the translation units that launch it: the host
// launch paths (hydro_kernels.cu) and the device-side team launcher
// (device_launch.cu, relocatable device code).  Header-only, anonymous
// namespace: each translation unit keeps its own copy.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/taskfuse_b200.h"
#include "sm100_common.cuh"

namespace {

template <int N>
struct Geo {
  static constexpr int C = N + 2;      // face / flux cube edge
  static constexpr int E = N + 6;      // ghosted edge (GHOST = 3)
  static constexpr int B = N + 4;      // stencil box x/y edge, ext 1..N+4
  // TMA needs the box's inner (z) start 16-byte aligned, so the box spans
  // the full z row (ext 0..E-1) — the same DRAM sectors as z 1..N+4.
  static constexpr int BZ = E;
  static constexpr int CELLS = C * C * C;
  static constexpr int BOX = B * B * BZ;
  static constexpr int EXT3 = E * E * E;
  static constexpr int OWN = N * N * N;
};

// ---------------------------------------------------------------- PTX glue
__device__ __forceinline__ void tma_load_box(void* dst, const CUtensorMap* map,
                                             int c0, int c1, int c2, int c3,
                                             uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::"
      "complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
}

// --------------------------------------------------------------- numerics
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Face states and fluxes of one cell along one axis from the staged box.
// minus state of the next cell along the axis: np.roll(.., -1) wraps the
// last layer onto layer 0 (kernels.py:90-93).
struct Faces {
  double vm, vp, f;
};

__device__ __forceinline__ Faces cell_axis(const double* __restrict__ sbox,
                                           int b, int st, int pos, int C,
                                           double a, int mode, int flux_form) {
  const double base = sbox[b];
  const double half = __dmul_rn(0.5, slope(sbox, b, st));
  Faces r;
  r.vm = __dsub_rn(base, half);
  r.vp = __dadd_rn(base, half);
  r.f = 0.0;
  if (mode == 0) {
    double next_m = 0.0;
    if (a < 0.0 || flux_form == 1) {
      const int bn = (pos == C - 1) ? b - (C - 1) * st : b + st;
      next_m = __dsub_rn(sbox[bn], __dmul_rn(0.5, slope(sbox, bn, st)));
    }
    if (flux_form == 0) {
      r.f = (a >= 0.0) ? __dmul_rn(a, r.vp) : __dmul_rn(a, next_m);
    } else {
      // Kurganov-Tadmor central-upwind: 1/2(f_L+f_R) - 1/2 a_max (u_R-u_L)
      const double fl = __dmul_rn(a, r.vp), fr = __dmul_rn(a, next_m);
      r.f = __dsub_rn(__dmul_rn(0.5, __dadd_rn(fl, fr)),
                      __dmul_rn(__dmul_rn(0.5, fabs(a)), __dsub_rn(next_m, r.vp)));
    }
  }
  return r;
}

// reconstruct_body + flux_body for one slice whose stencil box is staged in
// shared memory.  Work is split in z-pairs of cells so every store is a
// 16-byte streaming store (C = n+2 is even; slot bases are 16-B aligned).
// Returns this thread's max signal speed over the faces it produced.
template <int N, int THREADS, int MODE, bool PAIR = true>
__device__ __forceinline__ double slice_compute(
    const double* __restrict__ sbox, double* __restrict__ um_s,
    double* __restrict__ up_s, double* __restrict__ F_s, double ax, double ay,
    double az, int flux_form) {
  using G = Geo<N>;
  constexpr int C = G::C, B = G::B, BZ = G::BZ, CELLS = G::CELLS;
  constexpr int HP = C / 2;           // pairs per z row
  constexpr int PAIRS = C * C * HP;
  const double av[3] = {ax, ay, az};
  const int stv[3] = {B * BZ, BZ, 1};
  double speed = 0.0;
  if constexpr (!PAIR) {
    // one cell per thread-iteration, 8-byte stores
    for (int c = threadIdx.x; c < CELLS; c += THREADS) {
      const int ci = c / (C * C), cj = (c / C) % C, ck = c % C;
      const int b = ((ci + 1) * B + (cj + 1)) * BZ + (ck + 2);
#pragma unroll
      for (int axis = 0; axis < 3; ++axis) {
        const int pos = axis == 0 ? ci : (axis == 1 ? cj : ck);
        const Faces r = cell_axis(sbox, b, stv[axis], pos, C, av[axis], MODE,
                                  flux_form);
        __stcs(um_s + axis * CELLS + c, r.vm);
        __stcs(up_s + axis * CELLS + c, r.vp);
        if (MODE == 0) {
          __stcs(F_s + axis * CELLS + c, r.f);
          speed = fmax(speed, fabs(av[axis]));
        }
      }
    }
    return speed;
  } else {
  for (int p = threadIdx.x; p < PAIRS; p += THREADS) {
    const int ci = p / (C * HP);
    const int cj = (p / HP) % C;
    const int ck = 2 * (p % HP);
    const int c = (ci * C + cj) * C + ck;
    // cube (ci,cj,ck) = ext (ci+2,cj+2,ck+2) = box (ci+1, cj+1, ck+2)
    const int b = ((ci + 1) * B + (cj + 1)) * BZ + (ck + 2);
#pragma unroll
    for (int axis = 0; axis < 3; ++axis) {
      const int st = stv[axis];
      const int pos0 = axis == 0 ? ci : (axis == 1 ? cj : ck);
      const int pos1 = axis == 2 ? ck + 1 : pos0;
      const Faces r0 = cell_axis(sbox, b, st, pos0, C, av[axis], MODE, flux_form);
      const Faces r1 = cell_axis(sbox, b + 1, st, pos1, C, av[axis], MODE, flux_form);
      __stcs(reinterpret_cast<double2*>(um_s + axis * CELLS + c),
             make_double2(r0.vm, r1.vm));
      __stcs(reinterpret_cast<double2*>(up_s + axis * CELLS + c),
             make_double2(r0.vp, r1.vp));
      if (MODE == 0) {
        __stcs(reinterpret_cast<double2*>(F_s + axis * CELLS + c),
               make_double2(r0.f, r1.f));
        speed = fmax(speed, fabs(av[axis]));  // local signal speed
      }
    }
  }
  return speed;
  }
}

// Block-wide max of the per-thread signal speeds -> one store (reduce stage).
template <int THREADS>
__device__ __forceinline__ void block_max_store(double v, double* red,
                                                double* out) {
  v = warp_max(v);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < THREADS / 32 ? red[threadIdx.x] : 0.0;
    w = warp_max(w);
    if (threadIdx.x == 0) *out = w;
  }
}

// Register budget: <= 32 registers/thread so 2048 threads (4 CTAs of 512)
// are resident per SM — measured best on B200 (DESIGN.md §4 table).
template <int THREADS>
constexpr int recon_min_blocks() {
  return 2048 / THREADS > 0 ? 2048 / THREADS : 1;
}

// One CTA's share of a team: stage slice g's stencil box with one TMA load,
// then reconstruct (+ flux for MODE 0) into output slot `slot`.
// `sbox`: the CTA's BOX doubles of shared memory, 128-byte aligned (the
// TMA destination rule).
template <int N, int THREADS, int MODE>
__device__ __forceinline__ void recon_flux_cta(
    double* sbox, const CUtensorMap* tmap, int g, int64_t slot, double ax,
    double ay, double az, double* __restrict__ um, double* __restrict__ up,
    double* __restrict__ F, double* __restrict__ amax, int flux_form) {
  using G = Geo<N>;
  constexpr int CELLS = G::CELLS;
  __shared__ __align__(8) uint64_t bar;
  __shared__ double red[THREADS / 32];
  if (threadIdx.x == 0) mbar_init(&bar, 1);
  // the barrier is initialised (and the init fenced) before anyone arrives
  // on it or polls it — also the order compute-sanitizer's racecheck
  // models: an arrive by the initialising thread before a block barrier is
  // reported as a warp-level RAW hazard on the mbarrier word
  __syncthreads();
  if (threadIdx.x == 0) {
    mbar_expect_tx(&bar, G::BOX * (uint32_t)sizeof(double));
    // box origin = extended index (x,y,z) = (1,1,0) of sub-grid g;
    // coordinates innermost first
    tma_load_box(sbox, tmap, 0, 1, 1, g, &bar);
  }
  mbar_wait(&bar, 0);
  const double speed = slice_compute<N, THREADS, MODE>(
      sbox, um + slot * 3 * CELLS, up + slot * 3 * CELLS,
      MODE == 0 ? F + slot * 3 * CELLS : nullptr, ax, ay, az, flux_form);
  if (MODE == 0 && amax != nullptr)
    block_max_store<THREADS>(speed, red, amax + slot);
}

// Fused reconstruct + flux.  MODE 0: um, up and F; MODE 1: um, up only
// (reconstruct_body alone).  One CTA per aggregated slice.
template <int N, int THREADS, int MODE, bool DEV_IDS>
__global__ void __launch_bounds__(THREADS, recon_min_blocks<THREADS>())
    k_recon_flux(const __grid_constant__ CUtensorMap tmap,
                 const int32_t* __restrict__ dev_ids,
                 const __grid_constant__ TeamIds team, int out_mode, double ax,
                 double ay, double az, double* __restrict__ um,
                 double* __restrict__ up, double* __restrict__ F,
                 double* __restrict__ amax, int flux_form) {
  // let a programmatically-dependent next team launch as soon as every CTA
  // of this one is resident (no-op unless the next launch opted in)
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  extern __shared__ __align__(128) double sbox[];
  const int s = blockIdx.x;
  const int g = DEV_IDS ? (dev_ids ? dev_ids[s] : s) : team.id[s];
  recon_flux_cta<N, THREADS, MODE>(sbox, &tmap, g, out_mode ? (int64_t)g : s,
                                   ax, ay, az, um, up, F, amax, flux_form);
}

}  // namespace
