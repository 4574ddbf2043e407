// field_march.cu — the fused full iteration over a WHOLE padded slab by
// x-marching warp columns (SURVEY §8(f) rank 2 at config-5 scale; the
// multi-GPU step of §8(e)).
//
// k_step_cols8s (field_step.cu) gives every 8^3 sub-grid its own CTA and
// one 11 x 11 x 16 TMA box: 15.5 KB through shared memory per 4 KB of owned
// cells, and a CTA that waits on one box load then retires — latency-bound
// at 0.60 of the 16 B/cell DRAM floor on 262 144 sub-grids.  When a launch
// covers every sub-grid of the slab (the config-5 iteration: one team = the
// whole slab) the sub-grid boxes tile the field, and the work can be cut the
// other way:
//
//  * a WARP owns a column of the field: R = 8 rows (y) x 32 cells (z, one
//    per lane), and marches it along x through a chunk of xc = 16 planes (a
//    work item = 2 x 1 x 4 sub-grids); warps claim items from a counter,
//    chunk-major, so neighbouring columns march side by side (their shared
//    halo rows are L2 hits: DRAM traffic 2.16 GB per 2.15 GB floor) and
//    the tail is one item long (round-robin items ran 700+ us: stragglers
//    and columns drifting apart);
//  * each x plane of the column arrives as ONE TMA box (R+4 rows x 36 z,
//    the star stencil's halo included) into a per-warp ring of NB = 4
//    plane buffers (one mbarrier each); lane 0 keeps NB-1-D planes in
//    flight and refills a buffer the moment the warp is done with it — no
//    block barrier anywhere, warps never wait for each other;
//  * every value along x lives in registers (shift register of the
//    column's owned rows), every y face is formed once and carried row to
//    row in the lane, every z face once and taken from lane-1 by shuffle;
//    the faces the column cannot get that way (row y0-1's y face, z0-1's z
//    faces) are formed once per plane: 1/R and 1/(3R) extra.  A one-sided
//    difference shared by two faces (y; x for a >= 0) is formed once.
//
// Shared-memory traffic per owned cell: (R+4)*36/(32 R) = 1.7 x (R = 8) vs
// 3.8 x for the per-sub-grid boxes.  Results leave as whole 256-B rows per
// warp store (coalesced), together with the next field's periodic y/z halo
// copies (TF_STEP_HALO_YZ) and the x halo layers — the periodic copy on one
// GPU (TF_STEP_HALO_X) or the ring neighbours' halos over peer memory
// (peer_lo / peer_hi), so the exchange rides on the compute.
//
// TF_MARCH_ALONG_Y swaps the roles of x and y (the TMA map's two outer
// dimensions and the strides exchanged, the x halo copies made by the items
// on the row faces): a rank's thin x slab is marched along its long y
// extent.  The update sums (dFx + dFy) + dFz either way — addition is
// commutative, so the result is bit-identical.
//
// Work items are ordered interior first (no halo copies), then the items
// on the field's faces; an interior item runs a loop unrolled twice whose
// two register sets alternate (no register moves for the x shift), a face
// item a single-copy loop with the halo-writing finalise — the two loops
// together outgrow the instruction cache, so the phases are kept apart.
//
// Config 5 (grid 512, one B200, full clock): 0.444-0.448 ms per iteration
// vs 0.541 ms for k_step_cols8s = 0.73-0.74 of the 16 B/cell DRAM floor.
// The kernel is issue-bound (IPC ~2.7 of 4, FP64 pipe ~50%, 15 warps/SM at
// 128 registers).
//
// Arithmetic: face3 / the update are exactly cols8s_body's (kernels.py:73-111
// face_flux and update_body, no FMA contraction): bit-identical to the
// reference's advect_once on the whole grid (tests/test_gpu_march.py).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <stdint.h>

#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "../../include/taskfuse_b200.h"
#include "sm100_common.cuh"

namespace {

constexpr int HX = 2, HY = 2, HZ = 4;  // halo widths of the padded field
constexpr int MZ = 32;                 // owned z per warp column (lanes)
constexpr int BZW = MZ + 4;            // plane box z: z0-2 .. z0+33 (288 B)

template <int R, int NB_ = 4>
struct MGeo {
  static constexpr int ROWS = R + 4;                  // y0-2 .. y0+R+1
  static constexpr int PLANE = ROWS * BZW * 8;        // bytes per plane box
  static constexpr int NB = NB_;                      // ring depth per warp
  static constexpr int W = 1;                         // warps per CTA
  // boxes, then per warp NB mbarriers and the R-entry z-boundary strip
  static constexpr int SMEM = W * (NB * (PLANE + 8) + R * 8 + 16);
};

// Face between cells with values (v0, v1, v2) taken upwind-first
// (face_flux, kernels.py:73-93; identical to field_step.cu's face3)
template <bool POS>
__device__ __forceinline__ double face3(double v0, double v1, double v2,
                                        double a) {
  const double h =
      __dmul_rn(0.5, minmod(__dsub_rn(v2, v1), __dsub_rn(v1, v0)));
  return __dmul_rn(a, POS ? __dadd_rn(v1, h) : __dsub_rn(v1, h));
}

// The same face from the upwind-first value v1 and its two one-sided
// differences fwd = v2 - v1, bwd = v1 - v0, when a difference shared by two
// faces has been formed once (the same rounded value: bit-identical)
template <bool POS>
__device__ __forceinline__ double face_d(double v1, double fwd, double bwd,
                                         double a) {
  const double h = __dmul_rn(0.5, minmod(fwd, bwd));
  return __dmul_rn(a, POS ? __dadd_rn(v1, h) : __dsub_rn(v1, h));
}

__device__ __forceinline__ void tma_plane(void* dst, const CUtensorMap* map,
                                          int pz, int py, int px,
                                          uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::"
      "complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(pz), "r"(py), "r"(px),
      "r"(smem_u32(bar))
      : "memory");
}

// The kernel marches along its "plane" axis and stacks R "rows" per column:
// physical x and y by default, y and x with TF_MARCH_ALONG_Y (a thin x slab
// marched along its long y extent).  Names below are the default's.
struct MarchArgs {
  double* out;      // next padded field
  // halo copies of the owned layers next to each face, or null: the plane
  // axis's low / high faces go to plo[+pw] / phi[-pw] (x: the ring
  // neighbours' next fields, or this one), the row axis's to qlo / qhi [+-qw]
  double *plo, *phi, *qlo, *qhi;
  int64_t pw, qw;
  int64_t pyz;      // padded stride of the plane axis
  int pz;           // padded stride of the row axis
  int X, Gy, Gz;    // owned extents: plane axis, row axis, z
  int xc;           // planes per work item
  int nzb;          // z blocks (Gz / 32)
  int ncols;        // warp columns per plane (Gy / R * nzb)
  int nitems;       // ceil(X / xc) * ncols
  // item order: the n_int interior items (no halo copies: chunks [cl, ch)
  // x the nyi x nzi columns off the y/z faces) first, then the rest
  int n_int, cl, ch, nyb, nyi, nzi, yoff, zoff;
  int halo_yz;      // also write the next field's periodic z halos
  int pdl_edge;     // PDL: 1 = items on the plane axis's faces wait for the
                    // previous kernel, 2 = items on the row axis's faces
  unsigned* work;   // {claim, done} counters (zero at launch), or null
  double ax, ay, az, dt_dx;
};

// Work item `it` -> its first plane xa, length len and column origin
// (y0, z0).  Interior items come first so that, while they last, the warps
// run only the interior loop (march_warp): the halo-writing loop is a
// second copy of the plane body, and both together outgrow the SM's
// instruction cache.  Returns whether the item is interior.
template <int R>
__device__ __forceinline__ bool item_geo(const MarchArgs& A, int it, int& xa,
                                         int& len, int& y0, int& z0) {
  int chunk, yg, zb;
  bool interior = it < A.n_int;
  if (interior) {
    const int per = A.nyi * A.nzi;
    chunk = A.cl + it / per;
    const int r = it - (chunk - A.cl) * per;
    yg = A.yoff + r / A.nzi;
    zb = A.zoff + r % A.nzi;
  } else {
    int e = it - A.n_int;
    const int nch = (A.X + A.xc - 1) / A.xc;
    const int edge_chunks = nch - (A.ch - A.cl);
    if (e < edge_chunks * A.ncols) {
      // the chunks holding x-halo planes, every column
      const int k = e / A.ncols, col = e - k * A.ncols;
      chunk = k < A.cl ? k : A.ch + (k - A.cl);
      yg = col / A.nzb;
      zb = col - yg * A.nzb;
    } else {
      // the interior chunks' columns on the y/z faces (the frame)
      e -= edge_chunks * A.ncols;
      const int frame = A.ncols - A.nyi * A.nzi;
      chunk = A.cl + e / frame;
      int f = e - (chunk - A.cl) * frame;
      if (f < A.nzb) {
        yg = 0, zb = f;
      } else if (A.nyb > 1 && f < 2 * A.nzb) {
        yg = A.nyb - 1, zb = f - A.nzb;
      } else {
        f -= A.nyb > 1 ? 2 * A.nzb : A.nzb;
        const int sides = A.nzb < 2 ? A.nzb : 2;
        yg = 1 + f / sides;
        zb = (f % sides) ? A.nzb - 1 : 0;
      }
    }
  }
  xa = chunk * A.xc;
  len = min(A.xc, A.X - xa);
  y0 = yg * R;
  z0 = zb * MZ;
  return interior;
}

// The owned rows of plane p (values c = u(p), x faces fx / fxm of its
// +-1/2 sides) finalised from the plane's buffer `cb`: y and z faces, the
// update, the store — and, EDGE only, the halo copies of a column / plane on
// the field's faces.
template <int R, bool PY, bool PZ, bool EDGE>
__device__ __forceinline__ void finalise(const MarchArgs& A,
                                         const double* cb, double* strip,
                                         const double (&c)[R],
                                         const double (&fx)[R],
                                         const double (&fxm)[R], int p, int y0,
                                         int z0, bool hy, bool hz, bool hlo,
                                         bool hhi) {
  const int lane = threadIdx.x & 31;
  const int z = z0 + lane;
  const double ay = A.ay, az = A.az, dt = A.dt_dx;
  const double* col = cb + 2 + lane;  // own z, row index 0 = y0-2
  // y: the column's values w[k] = row y0+k-2 (owned rows from c) and their
  // forward differences d[k] = w[k+1] - w[k], each formed once: the y face
  // of row r uses d[r+1] (forward) and d[r] (backward) (a >= 0), one row
  // up for a < 0 — face3's own operations, shared by two faces
  double w[R + 4];
  w[0] = PY ? col[0] : 0.0;
  w[1] = col[BZW];
#pragma unroll
  for (int r = 0; r < R; ++r) w[r + 2] = c[r];
  w[R + 2] = col[(R + 2) * BZW];
  w[R + 3] = PY ? 0.0 : col[(R + 3) * BZW];
  double d[R + 3];
#pragma unroll
  for (int k = PY ? 0 : 1; k < (PY ? R + 2 : R + 3); ++k)
    d[k] = __dsub_rn(w[k + 1], w[k]);
  // Phi_y(r), r = -1..R-1 (row r is w[r+2])
  auto fy_of = [&](int r) {
    return PY ? face_d<true>(w[r + 2], d[r + 2], d[r + 1], ay)
              : face_d<false>(w[r + 3], d[r + 3], d[r + 2], ay);
  };
  double fym = fy_of(-1);
  // z faces below z0 (row `lane` of the column, lanes < R), parked in the
  // warp's strip for lane 0 (one broadcast load per row, not two shuffles)
  {
    const double* zb = cb + (2 + (lane & (R - 1))) * BZW;
    const double bz = PZ ? face3<true>(zb[0], zb[1], zb[2], az)
                         : face3<false>(zb[1], zb[2], zb[3], az);
    if (lane < R) strip[lane] = bz;
  }
  __syncwarp();
  const int64_t pz = A.pz;
  double* o = A.out + (int64_t)(p + HX) * A.pyz + (int64_t)(y0 + HY) * pz +
              (z + HZ);
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const double fy = fy_of(r);
    const double* zr = col + (r + 2) * BZW;
    const double fz = PZ ? face3<true>(zr[-1], c[r], zr[1], az)
                         : face3<false>(c[r], zr[1], zr[2], az);
    double fzm = __shfl_up_sync(0xffffffffu, fz, 1);
    const double fzb = strip[r];
    fzm = lane == 0 ? fzb : fzm;
    // update_body order: ((dFx + dFy) + dFz), kernels.py:100-111
    double div = __dsub_rn(fx[r], fxm[r]);
    div = __dadd_rn(div, __dsub_rn(fy, fym));
    div = __dadd_rn(div, __dsub_rn(fz, fzm));
    fym = fy;
    const double v = __dsub_rn(c[r], __dmul_rn(dt, div));
    double* orow = o + r * pz;
    *orow = v;
    if (EDGE) {
      // periodic y/z copies of the next field, and the slab's two lowest /
      // highest x layers as the ring neighbours' next x halo (one GPU: this
      // field's own); halo edges / corners are never read
      const int y = y0 + r;
      const int64_t off = orow - A.out;
      if (hy && A.qlo && y < HY) A.qlo[off + A.qw] = v;
      if (hy && A.qhi && y >= A.Gy - HY) A.qhi[off - A.qw] = v;
      if (hz && z < HZ) orow[A.Gz] = v;
      if (hz && z >= A.Gz - HZ) orow[-A.Gz] = v;
      if (hlo) A.plo[off + A.pw] = v;
      if (hhi) A.phi[off - A.pw] = v;
    }
  }
}

// One warp's whole share of the slab.  PX/PY/PZ: velocity signs (a >= 0).
// Items come from the launch's work counter (A.work: dynamic, balanced) or
// round-robin by warp (A.work == nullptr).
template <int R, int NB_, bool PX, bool PY, bool PZ, bool PDL>
__device__ __forceinline__ void march_warp(const CUtensorMap* map,
                                           const MarchArgs& A,
                                           unsigned char* wbuf,
                                           uint64_t* bars, double* strip,
                                           int* iq, int slot0, int nslots) {
  using G = MGeo<R, NB_>;
  constexpr int NB = G::NB, PLANE = G::PLANE;
  constexpr int D = PX ? 1 : 2;  // x look-ahead of a +1/2 face
  constexpr int IQ = 4;          // item queue: producer ahead <= 3 items
  const int lane = threadIdx.x & 31;

  // ---- producer (lane 0): claims items, issues their planes in order ----
  int p_item = -1, p_t = 0, p_q0 = 0, p_n = 0, p_py = 0, p_pz = 0;
  int p_next = slot0;   // next round-robin item (static mode)
  unsigned p_claims = 0;
  auto p_claim = [&]() {
    int it;
    if (A.work != nullptr) {
      it = (int)atomicAdd(A.work, 1u);
      if (it >= A.nitems) {
        // the last warp to run dry resets the counters for the next launch
        if (atomicAdd(A.work + 1, 1u) == gridDim.x * G::W - 1) {
          A.work[0] = 0;
          A.work[1] = 0;
        }
      }
    } else {
      it = p_next;
      p_next += nslots;
    }
    p_item = it < A.nitems ? it : -1;
    iq[p_claims++ % IQ] = p_item;
    if (p_item < 0) return;
    int xa, len, y0, z0;
    item_geo<R>(A, p_item, xa, len, y0, z0);
    if (PDL && (A.pdl_edge == 1 ? (xa < A.cl * A.xc || xa + len > A.ch * A.xc)
                                : (y0 < HY || y0 + R > A.Gy - HY))) {
      // an x-edge item reads the halo layers the ring neighbours store and
      // stores theirs: only it waits for the ring barrier before it loads
      // (a separate instantiation: the branch costs the plain kernel ~2.5%
      // in register pressure)
      asm volatile("griddepcontrol.wait;" ::: "memory");
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    p_q0 = xa - (PX ? 2 : 1) + HX;  // padded x of the item's first plane
    p_n = len + 3;
    p_py = y0 + HY - 2;             // padded origin of the box rows
    p_pz = z0 + HZ - 2;             // and of its z extent
  };
  unsigned gi = 0;  // planes issued
  auto issue = [&]() {
    if (p_item < 0) return;
    const unsigned s = gi % NB;
    mbar_expect_tx(&bars[s], PLANE);
    tma_plane(wbuf + s * PLANE, map, p_pz, p_py, p_q0 + p_t, &bars[s]);
    ++gi;
    if (++p_t == p_n) {
      p_t = 0;
      p_claim();
    }
  };
  if (lane == 0) {
    p_claim();
    for (int k = 0; k < NB; ++k) issue();
  }
  __syncwarp();

  unsigned gc = 0;  // planes consumed
  const double ax = A.ax;
  for (unsigned ci = 0;; ++ci) {
    const int it = iq[ci % IQ];
    if (it < 0) break;
    int xa, len, y0, z0;
    const bool interior = item_geo<R>(A, it, xa, len, y0, z0);
    // warp-uniform: does this column touch a periodic y / z face?
    const bool hy = (A.qlo && y0 < HY) || (A.qhi && y0 + R > A.Gy - HY);
    const bool hz = A.halo_yz && (z0 == 0 || z0 + MZ == A.Gz);
    // One x plane of the march: the state carried from plane to plane
    // (s0 = u(p-1) or, a >= 0, the backward difference u(p) - u(p-1);
    // s1 = u(p); sm = the -1/2 x face) comes in as (s0, s1, sm) and the
    // next state goes out as (d0, d1, dm).
    auto plane = [&](auto edge_tag, int t, const auto& s0, const auto& s1,
                     const auto& sm, auto& d0, auto& d1, auto& dm) {
      constexpr bool EDGE = decltype(edge_tag)::value;
      const unsigned s = gc % NB;
      mbar_wait(&bars[s], (gc / NB) & 1);
      const double* nb =
          reinterpret_cast<const double*>(wbuf + s * PLANE) + 2 * BZW + 2 +
          lane;  // (row 0, own z) of the new plane
#pragma unroll
      for (int r = 0; r < R; ++r) d1[r] = nb[r * BZW];
      int nfree = 0;
      // a >= 0: the backward difference u(p) - u(p-1) is carried instead of
      // u(p-1) — the forward difference of the previous plane, formed once
#pragma unroll
      for (int r = 0; r < R; ++r)
        d0[r] = PX ? __dsub_rn(d1[r], s1[r]) : s1[r];
      if (t >= 2) {
#pragma unroll
        for (int r = 0; r < R; ++r)
          dm[r] = PX ? face_d<true>(s1[r], d0[r], s0[r], ax)
                     : face3<false>(s0[r], s1[r], d1[r], ax);
        if (t >= 3) {
          // finalise plane p = q - D from its own buffer (D planes ago)
          const int p = xa + t - 3;
          const double* cb = reinterpret_cast<const double*>(
              wbuf + ((gc - D) % NB) * PLANE);
          const auto& c = PX ? s1 : s0;
          if (EDGE) {
            const bool hlo = A.plo != nullptr && p < HX;
            const bool hhi = A.phi != nullptr && p >= A.X - HX;
            finalise<R, PY, PZ, true>(A, cb, strip, c, dm, sm, p, y0, z0, hy,
                                      hz, hlo, hhi);
          } else {
            finalise<R, PY, PZ, false>(A, cb, strip, c, dm, sm, p, y0, z0,
                                       false, false, false, false);
          }
          nfree = 1;  // the finalised plane's buffer
        }
        // the item's last plane: the look-ahead planes are done too
        if (t == len + 2) nfree += D;
      } else {
        // POS: planes xa-2, xa-1 feed only the x faces; NEG: xa-1 only
        nfree = (PX || t == 0) ? 1 : 0;
      }
      // every lane's reads of the freed buffer are done (their values are
      // consumed above) before lane 0 lets the TMA rewrite it.  No proxy
      // fence: fence.proxy.async compiles to MEMBAR.ALL.CTA, which would
      // wait for the plane's global stores too
      __syncwarp();
      if (lane == 0)
        for (int k = 0; k < nfree; ++k) issue();
      __syncwarp();  // the item queue entry lane 0 may have written
      ++gc;
    };
    double a0[R], a1[R], am[R], b0[R], b1[R], bm[R];
    const int n = len + 3;
    if (interior) {
      // two register sets alternate, so the x shift costs no register
      // moves (rotating one set in place is 48 moves per plane, 9% of the
      // instructions).  Plane 0 only loads: n - 1 = len + 2 is even for an
      // even chunk, so the pair loop's remainder copy stays cold
      {
        const unsigned s = gc % NB;
        mbar_wait(&bars[s], (gc / NB) & 1);
        const double* nb = reinterpret_cast<const double*>(wbuf + s * PLANE) +
                           2 * BZW + 2 + lane;
#pragma unroll
        for (int r = 0; r < R; ++r) a1[r] = nb[r * BZW];
        __syncwarp();
        if (lane == 0) issue();  // plane xa-2 (POS) / xa-1 (NEG) is done
        __syncwarp();
        ++gc;
      }
      int t = 1;
      for (; t + 1 < n; t += 2) {
        plane(std::false_type{}, t, a0, a1, am, b0, b1, bm);
        plane(std::false_type{}, t + 1, b0, b1, bm, a0, a1, am);
      }
      if (t < n) plane(std::false_type{}, t, a0, a1, am, b0, b1, bm);
    } else {
      for (int t = 0; t < n; ++t) {
        plane(std::true_type{}, t, a0, a1, am, b0, b1, bm);
#pragma unroll
        for (int r = 0; r < R; ++r) {
          a0[r] = b0[r];
          a1[r] = b1[r];
          am[r] = bm[r];
        }
      }
    }
  }
}

// <= 128 registers: the register file is split between the SM's four
// schedulers (16 K each), so 129-136 registers hold 3 warps per scheduler
// and <= 128 hold 4 — with the shared-memory carveout at its maximum the
// ring buffers then fit 15 warps per SM instead of 12 (config 5: 458 ->
// 444 us; the ptxas budget costs 16 bytes of spills in one of the eight
// velocity-sign variants)
template <int R, int NB, bool PX, bool PY, bool PZ, bool PDL>
__global__ void __launch_bounds__(MGeo<R, NB>::W * 32, 16)
    k_step_march(const __grid_constant__ CUtensorMap map,
                 const __grid_constant__ MarchArgs A) {
  using G = MGeo<R, NB>;
  extern __shared__ __align__(128) unsigned char smem[];
  const int w = threadIdx.x >> 5;
  unsigned char* wbuf = smem + w * G::NB * G::PLANE;
  uint64_t* bars =
      reinterpret_cast<uint64_t*>(smem + G::W * G::NB * G::PLANE) + w * G::NB;
  double* strip = reinterpret_cast<double*>(
                      smem + G::W * G::NB * (G::PLANE + 8)) + w * R;
  int* iq = reinterpret_cast<int*>(smem + G::W * (G::NB * (G::PLANE + 8) +
                                                  R * 8)) + w * 4;
  if ((threadIdx.x & 31) == 0)
    for (int k = 0; k < G::NB; ++k) mbar_init(&bars[k], 1);
  __syncwarp();
  march_warp<R, NB, PX, PY, PZ, PDL>(&map, A, wbuf, bars, strip, iq,
                                blockIdx.x * G::W + w, gridDim.x * G::W);
}

struct MapKey {
  const void* p;
  int X, Gy, Gz, R, ym;
  bool operator==(const MapKey& o) const {
    return p == o.p && X == o.X && Gy == o.Gy && Gz == o.Gz && R == o.R &&
           ym == o.ym;
  }
};
struct MapKeyHash {
  size_t operator()(const MapKey& k) const {
    return std::hash<const void*>()(k.p) ^ ((size_t)k.X * 1315423911u) ^
           ((size_t)k.Gy << 20) ^ ((size_t)k.Gz << 40) ^ (size_t)k.R ^
           ((size_t)k.ym << 8);
  }
};

// plane box of a padded field: (36 z, R+4 y, 1 x), no swizzle; ym: the
// tensor's two outer dimensions swapped, (36 z, R+4 x, 1 y)
int plane_map(const double* P, int X, int Gy, int Gz, int R, int ym,
              CUtensorMap* out) {
  static std::mutex mu;
  static std::unordered_map<MapKey, CUtensorMap, MapKeyHash> cache;
  const MapKey key{P, X, Gy, Gz, R, ym};
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(key);
  if (it != cache.end()) {
    *out = it->second;
    return 0;
  }
  auto fn = encode_fn();
  if (!fn) return TF_E_NO_TMA;
  const cuuint64_t pz = Gz + 2 * HZ, py = Gy + 2 * HY, px = X + 2 * HX;
  cuuint64_t dims[3] = {pz, ym ? px : py, ym ? py : px};
  cuuint64_t strides[2] = {(ym ? pz * py : pz) * 8, (ym ? pz : pz * py) * 8};
  cuuint32_t box[3] = {(cuuint32_t)BZW, (cuuint32_t)(R + 4), 1};
  cuuint32_t es[3] = {1, 1, 1};
  CUtensorMap m;
  if (fn(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(P), dims,
         strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return TF_E_INVALID;
  if (cache.size() > 256) cache.clear();
  cache.emplace(key, m);
  *out = m;
  return 0;
}

template <int R, int NB>
int launch_march(const CUtensorMap& map, const MarchArgs& A, int sg,
                 cudaStream_t st) {
  using G = MGeo<R, NB>;
  using K = void (*)(const CUtensorMap, const MarchArgs);
  static const K kerns[16] = {
      k_step_march<R, NB, false, false, false, false>,
      k_step_march<R, NB, true, false, false, false>,
      k_step_march<R, NB, false, true, false, false>,
      k_step_march<R, NB, true, true, false, false>,
      k_step_march<R, NB, false, false, true, false>,
      k_step_march<R, NB, true, false, true, false>,
      k_step_march<R, NB, false, true, true, false>,
      k_step_march<R, NB, true, true, true, false>,
      k_step_march<R, NB, false, false, false, true>,
      k_step_march<R, NB, true, false, false, true>,
      k_step_march<R, NB, false, true, false, true>,
      k_step_march<R, NB, true, true, false, true>,
      k_step_march<R, NB, false, false, true, true>,
      k_step_march<R, NB, true, false, true, true>,
      k_step_march<R, NB, false, true, true, true>,
      k_step_march<R, NB, true, true, true, true>};
  const K kern = kerns[sg + (A.pdl_edge ? 8 : 0)];
  // persistent grid: as many CTAs as fit on the device at once (per-kernel
  // occupancy and SM count cached once per device)
  static std::mutex mu;
  static std::unordered_map<int64_t, int> grids;
  int dev = 0;
  cudaGetDevice(&dev);
  const int64_t key = ((int64_t)dev << 16) | (A.pdl_edge << 12) | (NB << 8) |
                      (sg << 4) | R;
  int grid = 0;
  {
    std::lock_guard<std::mutex> lock(mu);
    auto it = grids.find(key);
    if (it != grids.end()) {
      grid = it->second;
    } else {
      cudaError_t e = cudaFuncSetAttribute(
          reinterpret_cast<const void*>(kern),
          cudaFuncAttributeMaxDynamicSharedMemorySize, G::SMEM);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(reinterpret_cast<const void*>(kern),
                               cudaFuncAttributePreferredSharedMemoryCarveout,
                               cudaSharedmemCarveoutMaxShared);
      if (e != cudaSuccess) return e;
      int per_sm = 0, sms = 0;
      e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(
          &per_sm, reinterpret_cast<const void*>(kern), G::W * 32, G::SMEM);
      if (e != cudaSuccess) return e;
      e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (e != cudaSuccess) return e;
      grid = (per_sm < 1 ? 1 : per_sm) * sms;
      grids[key] = grid;
    }
  }
  const int need = (A.nitems + G::W - 1) / G::W;
  if (grid > need) grid = need;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(G::W * 32);
  cfg.dynamicSmemBytes = G::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = A.pdl_edge ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, map, A);
}

}  // namespace

extern "C" {

int tf_field_march_f64(const double* padded_in, int32_t X, int32_t Gy,
                       int32_t Gz, double ax, double ay, double az,
                       double dt_dx, double* padded_out, double* peer_lo,
                       double* peer_hi, int32_t flags, int32_t xc,
                       uint32_t* work, tf_stream_t stream) {
  const int R = (flags & TF_MARCH_ROWS4) ? 4 : 8;
  const bool ym = (flags & TF_MARCH_ALONG_Y) != 0;
  const bool hyz = (flags & TF_STEP_HALO_YZ) != 0;
  // the kernel's plane / row extents
  const int P = ym ? Gy : X, Q = ym ? X : Gy;
  if (!padded_in || !padded_out || padded_in == padded_out || P < 1 ||
      Q < R || Gz < MZ || Q % R || Gz % MZ || xc < 0 ||
      (flags & ~(TF_STEP_HALO_YZ | TF_STEP_HALO_X | TF_MARCH_ROWS4 |
                 TF_MARCH_PDL_EDGE | TF_MARCH_ALONG_Y)))
    return TF_E_INVALID;
  if (flags & TF_STEP_HALO_X) {
    if (peer_lo || peer_hi) return TF_E_INVALID;
    peer_lo = peer_hi = padded_out;
  }
  if ((peer_lo || peer_hi) && X < HX) return TF_E_INVALID;
  // along y: both x faces and the y/z halos (the item order's frame is the
  // row axis's and z's faces together)
  if (ym && !(hyz && peer_lo && peer_hi)) return TF_E_INVALID;
  CUtensorMap map;
  int rc = plane_map(padded_in, X, Gy, Gz, R, ym ? 1 : 0, &map);
  if (rc) return rc;
  const int64_t pz = Gz + 2 * HZ, pyz = (int64_t)(Gy + 2 * HY) * pz;
  MarchArgs A;
  A.out = padded_out;
  double* own = hyz ? padded_out : nullptr;
  const int64_t xw = (int64_t)X * pyz, yw = (int64_t)Gy * pz;
  A.plo = ym ? own : peer_lo;
  A.phi = ym ? own : peer_hi;
  A.pw = ym ? yw : xw;
  A.qlo = ym ? peer_lo : own;
  A.qhi = ym ? peer_hi : own;
  A.qw = ym ? xw : yw;
  A.pz = (int)(ym ? pyz : pz);
  A.pyz = ym ? pz : pyz;
  A.X = P;
  A.Gy = Q;
  A.Gz = Gz;
  A.nzb = Gz / MZ;
  A.nyb = Q / R;
  A.ncols = A.nyb * A.nzb;
  // default chunk: 16 planes, or 8 when 16-plane chunks would give at most
  // 8192 items (under ~4 per warp of the grid: a rank's share of config 5
  // at N >= 4, 128 planes 166 -> 152 us along x, 151 -> 143 along y; at 256
  // planes 16 stays ahead, 236 vs 240 us)
  A.xc = xc > 0 ? xc
                : ((int64_t)((P + 15) / 16) * A.ncols > 8192 ? 16 : 8);
  const int nch = (P + A.xc - 1) / A.xc;
  const int64_t items = (int64_t)nch * A.ncols;
  if (items > (1 << 30)) return TF_E_INVALID;
  A.nitems = (int)items;
  A.halo_yz = hyz ? 1 : 0;
  A.pdl_edge = (flags & TF_MARCH_PDL_EDGE) ? (ym ? 2 : 1) : 0;
  // interior items: no halo copy on the row axis / z (the frame) and no
  // halo layer of the plane axis
  A.yoff = A.zoff = A.halo_yz;
  A.nyi = A.halo_yz ? (A.nyb > 2 ? A.nyb - 2 : 0) : A.nyb;
  A.nzi = A.halo_yz ? (A.nzb > 2 ? A.nzb - 2 : 0) : A.nzb;
  // chunk c is clear of the low plane-axis halo iff c * xc >= HX, of the
  // high one iff (c + 1) * xc <= P - HX
  A.cl = A.plo ? (HX + A.xc - 1) / A.xc : 0;
  A.ch = A.phi ? (P - HX) / A.xc : nch;
  if (A.ch < A.cl) A.ch = A.cl;
  if (A.cl > nch) A.cl = A.ch = nch;
  A.n_int = (A.ch - A.cl) * A.nyi * A.nzi;
  A.work = work;
  A.ax = ym ? ay : ax;  // the plane axis's velocity
  A.ay = ym ? ax : ay;
  A.az = az;
  A.dt_dx = dt_dx;
  const int sg =
      (A.ax >= 0.0 ? 1 : 0) | (A.ay >= 0.0 ? 2 : 0) | (az >= 0.0 ? 4 : 0);
  cudaStream_t st = (cudaStream_t)stream;
  // ring depth 4 for both column heights (A/B on config 5, R = 8, xc 16,
  // 128 registers: NB 3 / 4 / 5 = 450 / 448 / 477 us; more buffers cost
  // warps, fewer leave one plane in flight).  TF_MARCH_NB: tuning builds
#ifndef TF_MARCH_NB
#define TF_MARCH_NB 4
#endif
  return R == 4 ? launch_march<4, TF_MARCH_NB>(map, A, sg, st)
                : launch_march<8, TF_MARCH_NB>(map, A, sg, st);
}

}  // extern "C"
