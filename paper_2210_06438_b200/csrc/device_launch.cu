// device_launch.cu — strategy 3 with DEVICE-SIDE team launches.
//
// The reference's aggregated launch (aggregator.py:157-165): when the last
// member of a closed team arrives, ONE kernel of blocks_per_slice x T blocks
// is enqueued for the whole team.  On a B200 the host launch costs more than
// a team's work, so here the host only FORMS teams (the C++
// formation core, real-time starvation signal) and publishes each closed
// team — its sub-grid ids and its end offset — into mapped pinned memory.
// A one-CTA launcher kernel, resident for the run, mirrors the published
// ids into device memory and launches each team as its own grid from the
// device (CUDA dynamic parallelism, fire-and-forget stream): T CTAs of the
// same fused reconstruct+flux kernel the captured plans use (recon_flux.cuh),
// so a team is still ONE aggregated kernel, and the team size A still
// decides how many launches an iteration needs — without a host launch or
// a host-side graph.  Child grids signal completion through a device
// counter that the launcher mirrors to host memory: the formation core's
// busy signal ("published slices not all completed").
//
// Relocatable device code (nvcc -rdc=true), device-linked with cudadevrt.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdlib>
#include <vector>

#include "../../include/taskfuse_b200.h"
#include "internal.h"
#include "recon_flux.cuh"
#include "tf_nvtx.h"

namespace {

constexpr int kThreads = 512;   // child CTA: the plan kernel's shape
constexpr int kLauncher = 256;  // launcher CTA threads
constexpr int kTeamsPerRound = 64;

// Control block in mapped pinned memory (host writes teams / final_teams /
// published, the launcher writes completed / status).  `teams` and
// `final_teams` are adjacent and 16-byte aligned: one PCIe read gets both.
struct alignas(16) DlCtl {
  long long teams;        // teams published so far
  long long final_teams;  // -1 while more may come
  long long published;    // slices published so far
  long long completed;    // slices completed (launcher mirror)
  long long status;       // 1: the launcher timed out
  long long pad;
};

__device__ __forceinline__ long long dl_ld_sys64(const long long* p) {
  long long v;
  asm volatile("ld.relaxed.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int dl_ld_sys32(const int* p) {
  int v;
  asm volatile("ld.relaxed.sys.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void dl_st_sys64(long long* p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long dl_clock() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// One team = one grid of T CTAs (launched from the device).
// The tensor map lives in global memory (written by the host before the
// run): a device-side launch's parameter buffer does not guarantee the
// 64-byte alignment a TMA descriptor needs (cudaErrorMisalignedAddress).
template <int N>
__global__ void __launch_bounds__(kThreads, recon_min_blocks<kThreads>())
    k_team_child(const CUtensorMap* __restrict__ tmap,
                 const int32_t* __restrict__ ids, double ax, double ay,
                 double az, double* __restrict__ um, double* __restrict__ up,
                 double* __restrict__ F, double* __restrict__ amax,
                 int flux_form, unsigned long long* done) {
  // relocatable device code does not place the dynamic shared memory on a
  // 128-byte boundary (the TMA destination rule): the launch carries 128
  // spare bytes and the box starts at the next boundary
  extern __shared__ __align__(16) unsigned char dyn[];
  double* sbox = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(dyn) + 127) & ~uintptr_t(127));
  const int g = ids[blockIdx.x];
  recon_flux_cta<N, kThreads, 0>(sbox, tmap, g, (int64_t)g, ax, ay, az, um, up,
                                 F, amax, flux_form);
  __syncthreads();
  // completion is the host's busy hint only: no fence (the parent grid's
  // completion orders the outputs for the stream)
  if (threadIdx.x == 0) atomicAdd(done, 1ULL);
}

template <int N>
__global__ void __launch_bounds__(kLauncher)
    k_team_launcher(const CUtensorMap* tmap, const int* __restrict__ ring_h,
                    const long long* __restrict__ ends_h, DlCtl* ctl,
                    int32_t* __restrict__ ids_d, unsigned long long* done,
                    double ax, double ay, double az, double* um, double* up,
                    double* F, double* amax, int flux_form,
                    long long timeout_ns) {
  __shared__ long long s_teams, s_fin;
  __shared__ long long s_end[kTeamsPerRound];
  __shared__ int s_stop;
  constexpr size_t smem = Geo<N>::BOX * sizeof(double) + 128;
  const int t = threadIdx.x;
  if (t == 0) *done = 0;  // this slot's counter; no child of the run yet
  long long seen = 0, mirrored = 0, reported = -1;
  unsigned long long last_change = dl_clock();
  for (;;) {
    if (t == 0) {
      long long tp, fin;
      asm volatile("ld.relaxed.sys.global.v2.b64 {%0, %1}, [%2];"
                   : "=l"(tp), "=l"(fin)
                   : "l"(&ctl->teams)
                   : "memory");
      asm volatile("fence.acq_rel.sys;" ::: "memory");
      s_teams = tp < seen + kTeamsPerRound ? tp : seen + kTeamsPerRound;
      s_fin = fin;
    }
    __syncthreads();
    const long long tp = s_teams;
    if (tp > seen) {
      if (t < tp - seen) s_end[t] = dl_ld_sys64(ends_h + seen + t);
      __syncthreads();
      const long long end = s_end[tp - seen - 1];
      for (long long k = mirrored + t; k < end; k += kLauncher)
        ids_d[k] = dl_ld_sys32(ring_h + k);
      __threadfence();
      __syncthreads();  // every id of these teams is in device memory
      // one launching thread per new team: device-side launches from
      // different threads proceed in parallel (one thread issuing them
      // all serialised them at ~8 us each)
      if (t < tp - seen) {
        const long long start = t == 0 ? mirrored : s_end[t - 1];
        const long long e = s_end[t];
        k_team_child<N><<<(unsigned)(e - start), kThreads, smem,
                          cudaStreamFireAndForget>>>(
            tmap, ids_d + start, ax, ay, az, um, up, F, amax, flux_form,
            done);
      }
      mirrored = end;
      seen = tp;
      last_change = dl_clock();
    }
    if (t == 0) {
      const long long d = (long long)atomicAdd(done, 0ULL);
      if (d != reported) {
        dl_st_sys64(&ctl->completed, d);
        reported = d;
        last_change = dl_clock();
      }
      int stop = (s_fin >= 0 && seen >= s_fin) ? 1 : 0;
      if (!stop && (long long)(dl_clock() - last_change) > timeout_ns) {
        dl_st_sys64(&ctl->status, 1);
        stop = 2;
      }
      s_stop = stop;
    }
    __syncthreads();
    if (s_stop) break;
    __nanosleep(200);
  }
  if (t != 0 || s_stop == 2) return;
  // every team launched: keep the host's completion count fresh until the
  // children are done (the parent grid completes after them anyway)
  for (;;) {
    const long long d = (long long)atomicAdd(done, 0ULL);
    if (d != reported) {
      dl_st_sys64(&ctl->completed, d);
      reported = d;
      last_change = dl_clock();
    }
    if (d >= mirrored) break;
    if ((long long)(dl_clock() - last_change) > timeout_ns) {
      dl_st_sys64(&ctl->status, 1);
      break;
    }
    __nanosleep(100);
  }
}

struct DlSlot {
  CUtensorMap* map_h = nullptr;  // pinned staging of the pool's map
  CUtensorMap* map_d = nullptr;  // the copy the team grids read
  DlCtl* ctl_h = nullptr;
  void* ctl_d = nullptr;
  int32_t* ring_h = nullptr;
  int32_t* ring_hd = nullptr;
  long long* ends_h = nullptr;
  long long* ends_hd = nullptr;
  int32_t* ids_d = nullptr;
  unsigned long long* done_d = nullptr;
  int64_t cap = 0;
  cudaEvent_t done_ev = nullptr;
  cudaStream_t stream = nullptr;
  bool in_flight = false;
};

void free_ring(DlSlot& S) {
  if (S.ring_h) cudaFreeHost(S.ring_h);
  if (S.ends_h) cudaFreeHost(S.ends_h);
  if (S.ids_d) cudaFree(S.ids_d);
  S.ring_h = nullptr;
  S.ends_h = nullptr;
  S.ids_d = nullptr;
  S.cap = 0;
}

}  // namespace

struct tf_dlexec {
  tf_region* region = nullptr;
  int32_t n = 8;
  DlSlot slots[2];
  int cur = 1;
  int64_t published = 0, teams = 0, seen_published = 0;
  DlSlot& slot() { return slots[cur]; }
};

namespace {

int dl_busy(void* ctx, int32_t) {
  tf_dlexec* q = static_cast<tf_dlexec*>(ctx);
  if (q->published != q->seen_published) {  // new work cannot be done yet
    q->seen_published = q->published;
    return 1;
  }
  return __atomic_load_n(&q->slot().ctl_h->completed, __ATOMIC_ACQUIRE) <
         q->published;
}

void dl_publish(tf_dlexec* q, int64_t team) {
  tf_region* r = q->region;
  const int size = tf_region_team_size(r, team);
  if (size < 1) return;
  DlSlot& S = q->slot();
  tf_nvtx::TeamRange range("team publish (device launch)", size);
  std::vector<int64_t> tags(size);
  tf_region_team_members(r, team, tags.data(), size);
  for (int64_t tag : tags) S.ring_h[q->published++] = (int32_t)tag;
  S.ends_h[q->teams++] = q->published;
  // ids and end first, then the team count (release): the launcher
  // acquires the count
  __atomic_store_n(&S.ctl_h->published, (long long)q->published,
                   __ATOMIC_RELEASE);
  __atomic_store_n(&S.ctl_h->teams, (long long)q->teams, __ATOMIC_RELEASE);
  tf_region_release_team(r, team);
}

}  // namespace

extern "C" {

int tf_dlexec_create(tf_region* region, int32_t n, tf_dlexec** out) {
  if (!region || !out || n != 8) return TF_E_INVALID;
  // a run may leave up to one fire-and-forget launch per slice pending
  static const cudaError_t lim =
      cudaDeviceSetLimit(cudaLimitDevRuntimePendingLaunchCount, 1 << 16);
  if (lim != cudaSuccess) return lim;
  static const cudaError_t attr = cudaFuncSetAttribute(
      k_team_child<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
      (int)(Geo<8>::BOX * sizeof(double) + 128));
  if (attr != cudaSuccess) return attr;
  tf_dlexec* q = new tf_dlexec();
  q->region = region;
  q->n = n;
  cudaError_t e = cudaSuccess;
  for (DlSlot& S : q->slots) {
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&S.ctl_h), sizeof(DlCtl),
                        cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&S.ctl_d, S.ctl_h, 0);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&S.done_d),
                     sizeof(unsigned long long));
    if (e == cudaSuccess)
      e = cudaEventCreateWithFlags(&S.done_ev, cudaEventDisableTiming);
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&S.map_h),
                        sizeof(CUtensorMap), 0);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&S.map_d), sizeof(CUtensorMap));
  }
  if (e != cudaSuccess) {
    tf_dlexec_destroy(q);
    return e;
  }
  *out = q;
  return 0;
}

void tf_dlexec_destroy(tf_dlexec* q) {
  if (!q) return;
  for (DlSlot& S : q->slots) {
    if (S.in_flight) cudaEventSynchronize(S.done_ev);
    free_ring(S);
    if (S.ctl_h) cudaFreeHost(S.ctl_h);
    if (S.done_d) cudaFree(S.done_d);
    if (S.done_ev) cudaEventDestroy(S.done_ev);
    if (S.map_h) cudaFreeHost(S.map_h);
    if (S.map_d) cudaFree(S.map_d);
  }
  delete q;
}

int tf_dlexec_run_recon_flux(tf_dlexec* q, const double* pool_ext,
                             int64_t pool_slices, const int32_t* ids,
                             int64_t count, double ax, double ay, double az,
                             double* um, double* up, double* F, double* amax,
                             int32_t flux_form, tf_stream_t stream,
                             int64_t* teams_published) {
  if (!q || !ids || count < 0 || !teams_published || !pool_ext || !um ||
      !up || !F)
    return TF_E_INVALID;
  for (int64_t i = 0; i < count; ++i)
    if (ids[i] < 0 || ids[i] >= pool_slices) return TF_E_INVALID;
  CUtensorMap map;
  int rc = tf_internal_pool_map(pool_ext, pool_slices, q->n, &map);
  if (rc) return rc;
  // alternate slots: this run publishes while the previous run's teams may
  // still execute; the slot's own previous run must be finished
  q->cur ^= 1;
  DlSlot& S = q->slot();
  if (S.in_flight) {
    cudaError_t e = cudaEventSynchronize(S.done_ev);
    if (e != cudaSuccess) return e;
    S.in_flight = false;
    if (__atomic_load_n(&S.ctl_h->status, __ATOMIC_ACQUIRE)) {
      S.ctl_h->status = 0;
      return TF_E_TIMEOUT;
    }
  }
  if (count > S.cap || !S.ring_h) {
    free_ring(S);
    const int64_t cap = count > 0 ? count : 1;
    cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&S.ring_h),
                                  sizeof(int32_t) * cap, cudaHostAllocMapped);
    if (e == cudaSuccess)
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.ring_hd),
                                   S.ring_h, 0);
    if (e == cudaSuccess)
      e = cudaHostAlloc(reinterpret_cast<void**>(&S.ends_h),
                        sizeof(long long) * cap, cudaHostAllocMapped);
    if (e == cudaSuccess)
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.ends_hd),
                                   S.ends_h, 0);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&S.ids_d), sizeof(int32_t) * cap);
    if (e != cudaSuccess) return e;
    S.cap = cap;
  }
  q->published = 0;
  q->teams = 0;
  q->seen_published = 0;
  S.ctl_h->teams = 0;
  S.ctl_h->final_teams = -1;
  S.ctl_h->published = 0;
  S.ctl_h->completed = 0;
  S.ctl_h->status = 0;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  cudaStream_t st = (cudaStream_t)stream;
  *S.map_h = map;  // the slot's previous run is complete: safe to rewrite
  cudaError_t me = cudaMemcpyAsync(S.map_d, S.map_h, sizeof(CUtensorMap),
                                   cudaMemcpyHostToDevice, st);
  if (me != cudaSuccess) return me;
  k_team_launcher<8><<<1, kLauncher, 0, st>>>(
      S.map_d, S.ring_hd, S.ends_hd, static_cast<DlCtl*>(S.ctl_d), S.ids_d,
      S.done_d, ax, ay, az, um, up, F, amax, flux_form,
      /*timeout_ns=*/2000000000LL);
  cudaError_t ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = cudaEventRecord(S.done_ev, st);
  if (ce != cudaSuccess) return ce;
  S.in_flight = true;
  S.stream = st;
  tf_region* r = q->region;
  int64_t teams = 0;
  std::vector<int64_t> closed;
  auto drain = [&]() {
    const int32_t cap = tf_region_watch_count(r, 0);
    if (cap <= 0) return;
    closed.resize(cap);
    const int k = tf_region_stream_idle(r, 0, closed.data(), cap);
    for (int i = 0; i < k; ++i, ++teams) dl_publish(q, closed[i]);
  };
  for (int64_t i = 0; i < count; ++i) {
    if (tf_region_watch_count(r, 0) > 0 && !dl_busy(q, 0)) drain();
    tf_enter_result res;
    rc = tf_region_enter(r, ids[i], dl_busy, q, &res);
    if (rc) break;
    if (res.closed) {
      dl_publish(q, res.team);
      ++teams;
    }
  }
  drain();  // arrivals done: the device drains, closing what is left
  // close the run even on error so the launcher exits
  __atomic_store_n(&S.ctl_h->final_teams, (long long)q->teams,
                   __ATOMIC_RELEASE);
  *teams_published = teams;
  return rc;
}

int tf_dlexec_wait(tf_dlexec* q) {
  if (!q) return TF_E_INVALID;
  int rc = 0;
  for (DlSlot& S : q->slots) {
    if (!S.in_flight) continue;
    cudaError_t e = cudaEventSynchronize(S.done_ev);
    if (e != cudaSuccess) return e;
    S.in_flight = false;
    if (__atomic_load_n(&S.ctl_h->status, __ATOMIC_ACQUIRE)) {
      S.ctl_h->status = 0;
      rc = TF_E_TIMEOUT;
    }
  }
  return rc;
}

}  // extern "C"
