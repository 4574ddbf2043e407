// hydro_engine.cpp — the HydroSim task iteration run natively.
//
// The reference's per-sub-grid task body (hydro/step.py:83-123) visits the
// five aggregation regions in KERNEL_ORDER; each visit is
//     member = enter(region) -> slice_alloc x4 -> slice_copy(h2d)
//     -> slice_launch -> slice_copy(d2h) -> await(d2h) -> leave
// and the driver runs one such task per sub-grid per iteration
// (step.py:126-143) under a cooperative FIFO scheduler (sched.py:243-271).
// In Python every visit costs ~100 us of interpreter time, so on a B200 the
// parent stream has always drained by the next arrival and the starvation
// rule closes almost every team solo.  This engine executes
// the same task state machine in C++ against the SAME rules — the
// tf_region formation core (cap / solo fast path / stream-drain closure)
// and the tf_team member bookkeeping (SPMD signatures, lease per step,
// release when all members left and no op is in flight) — with real CUDA
// streams, real pinned/device staging leases from an exact-size recycling
// pool (bufferpool.py:112-159), one aggregated cudaMemcpyAsync per team
// copy and ONE batched sm_100a launch per team, so the arrivals come as
// fast as the formation core can take them and teams actually form.
//
// Scheduling semantics follow the Python scheduler the mirror uses: tasks
// run FIFO until they park (team still forming, or d2h not landed); the
// streams are polled only when no task is runnable; a polled stream with
// no op left in flight fires its idle watches (tf_region_stream_idle).
#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstring>
#include <deque>
#include <map>
#include <string>
#include <utility>
#include <vector>

#include "../../include/taskfuse_b200.h"
#include "tf_nvtx.h"

namespace {

constexpr int kRegions = 5;  // KERNEL_ORDER, kernels.py:22
const char* const kNames[kRegions] = {"prep", "reconstruct", "flux",
                                      "reduce", "update"};
enum { K_PREP = 0, K_RECON, K_FLUX, K_REDUCE, K_UPDATE };
enum { KIND_PINNED = 0, KIND_DEVICE = 1 };

int ceil_div(int a, int b) { return (a + b - 1) / b; }

// kernels.py:39-55 at THREADS_PER_BLOCK = 128
int blocks_for(int k, int n) {
  const int ext = n + 6, cube = n + 2;
  switch (k) {
    case K_PREP: return ceil_div(ext * ext * ext, 128);
    case K_RECON: return ceil_div(cube * cube * cube, 128);
    case K_FLUX: return 3 * ceil_div(cube * cube * cube, 128);
    case K_REDUCE: return 1;
    default: return ceil_div(n * n * n, 128);
  }
}

// Exact-size recycling pool over real memory (bufferpool.py:112-159):
// buckets keyed by (kind, bytes), most recently returned record first; a
// bucket miss creates a buffer record (a "raw allocation", the reference's
// count).  Storage is managed apart from the records: a lease takes a chunk
// of the next power-of-two size class from a per-kind free list, or carves
// a new one from the kind's pre-allocated arena (bump pointer), and gives
// it back on release.  Real-time formation produces many distinct team
// sizes; with storage bound to exact-size records every new size held its
// own memory for good, the arena ran dry and each further size cost a
// cudaHostAlloc of up to a millisecond — enough to drain the streams and
// turn formation into solo launches.  Only an exhausted arena falls back to
// a real allocation per chunk.
class StagingPool {
 public:
  ~StagingPool() {
    for (auto& kv : owned_)
      for (void* p : kv.second) {
        if (kv.first == KIND_DEVICE) cudaFree(p);
        else cudaFreeHost(p);
      }
    if (arena_[KIND_DEVICE]) cudaFree(arena_[KIND_DEVICE]);
    if (arena_[KIND_PINNED]) cudaFreeHost(arena_[KIND_PINNED]);
  }
  int reserve(int64_t bytes_per_kind) {
    cudaError_t e = cudaMalloc(&arena_[KIND_DEVICE], (size_t)bytes_per_kind);
    if (e == cudaSuccess)
      e = cudaHostAlloc(&arena_[KIND_PINNED], (size_t)bytes_per_kind, 0);
    if (e != cudaSuccess) return e;
    cap_ = bytes_per_kind;
    return 0;
  }
  int acquire(int kind, int64_t bytes, void** out) {
    take(kind, bytes);  // the record (bucket accounting)
    const int cls = size_class(bytes);
    auto& fl = free_[kind][cls];
    void* p;
    if (!fl.empty()) {
      p = fl.back();
      fl.pop_back();
    } else {
      const int64_t chunk = int64_t(1) << cls;
      if (arena_[kind] && used_[kind] + chunk <= cap_) {
        p = static_cast<char*>(arena_[kind]) + used_[kind];
        used_[kind] += chunk;
      } else {
        cudaError_t e = kind == KIND_DEVICE ? cudaMalloc(&p, (size_t)chunk)
                                            : cudaHostAlloc(&p, (size_t)chunk, 0);
        if (e != cudaSuccess) {
          give(kind, bytes);
          return e;
        }
        owned_[kind].push_back(p);
        spilled_[kind] += 1;
      }
      materialised_[kind] += 1;
    }
    leased_[p] = Lease{kind, bytes, cls};
    *out = p;
    return 0;
  }
  int release(void* p) {
    auto it = leased_.find(p);
    if (it == leased_.end()) return TF_E_INVALID;
    const Lease l = it->second;
    leased_.erase(it);
    free_[l.kind][l.cls].push_back(p);
    give(l.kind, l.bytes);
    return 0;
  }
  // bufferpool.py:154-159: `count` records of this bucket exist afterwards
  void ensure(int kind, int64_t bytes, int count) {
    for (int i = 0; i < count; ++i) take(kind, bytes);
    for (int i = 0; i < count; ++i) give(kind, bytes);
  }
  int64_t raw(int kind) const { return raw_[kind]; }
  int64_t materialised(int kind) const { return materialised_[kind]; }
  int64_t spilled() const { return spilled_[0] + spilled_[1]; }
  int64_t outstanding() const { return (int64_t)leased_.size(); }
  int64_t acquisitions() const { return acquisitions_; }

 private:
  struct Lease {
    int kind;
    int64_t bytes;
    int cls;
  };
  static int size_class(int64_t bytes) {
    int c = 8;  // 256 B minimum chunk
    while ((int64_t(1) << c) < bytes) ++c;
    return c;
  }
  // records: per bucket, the number of idle records (LIFO order is moot
  // once storage is decoupled; the counts are the reference's accounting)
  void take(int kind, int64_t bytes) {
    acquisitions_ += 1;
    int64_t& idle = idle_[{kind, bytes}];
    if (idle > 0) {
      idle -= 1;
    } else {
      raw_[kind] += 1;
    }
  }
  void give(int kind, int64_t bytes) { idle_[{kind, bytes}] += 1; }
  std::map<std::pair<int, int64_t>, int64_t> idle_;
  std::map<int, std::vector<void*>> free_[2];
  std::map<void*, Lease> leased_;
  std::map<int, std::vector<void*>> owned_;
  int64_t raw_[2] = {0, 0}, materialised_[2] = {0, 0}, spilled_[2] = {0, 0};
  int64_t acquisitions_ = 0;
  void* arena_[2] = {nullptr, nullptr};
  int64_t used_[2] = {0, 0};
  int64_t cap_ = 0;
};

// Engine-side objects of one live core team (the rules are in tf_team_*).
struct TeamCtx {
  bool live = false;
  bool closed = false;
  bool landed = false;         // the visit's d2h copy completed
  std::vector<int32_t> members;  // task indices, slice order
  std::vector<int32_t> waiters;  // tasks parked on the d2h proxy
  void* lease[4] = {nullptr, nullptr, nullptr, nullptr};
};

struct Task {
  int32_t g = 0;       // sub-grid id
  int32_t visit = 0;   // region index in KERNEL_ORDER
  int32_t phase = 0;   // ENTER / OPS / LEAVE
  int64_t team = -1;
  int32_t slice = 0;
};
enum { P_ENTER = 0, P_OPS, P_LEAVE };

struct Op {
  cudaEvent_t ev;
  int32_t region;
  int64_t team;
};

}  // namespace

struct tf_hydro {
  int32_t n = 8, m = 1, S = 1, E = 1, max_team = 1;
  double ax = 1, ay = 1, az = 1, dt_dx = 0.3;
  double *w = nullptr, *um = nullptr, *up = nullptr, *F = nullptr,
         *reduce_out = nullptr;
  tf_region* regions[kRegions] = {};
  std::vector<cudaStream_t> streams;
  bool own_streams = false;
  std::vector<std::deque<Op>> inflight;  // per executor stream, issue order
  std::vector<cudaEvent_t> free_events;
  std::vector<std::deque<TeamCtx>> ctx;   // [region][core team id]
  // (a deque: growing it never moves a live TeamCtx a caller holds)
  StagingPool pool;
  std::string sig[kRegions][7];           // the visit's 7 step signatures
  int32_t* ids_h = nullptr;                // pinned team-id ring
  int64_t ids_cap = 0, ids_pos = 0;
  cudaEvent_t fork = nullptr;
  std::vector<Task> tasks;
  std::deque<int32_t> runnable;
  // counters (device.py:168-173 + the bench columns)
  int64_t kernels = 0, copies = 0, bytes = 0, polls = 0;
  // host nanoseconds in device-op issue (copies, launches, events), in
  // device polls that found no progress, and whole iterations
  int64_t ns_issue = 0, ns_idle_poll = 0, ns_iter = 0;
  // per-iteration state
  const double* u = nullptr;
  double* u_next = nullptr;
  int32_t finished = 0;
};

namespace {

int64_t host_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

int busy_cb(void* ctx, int32_t e) {
  tf_hydro* h = static_cast<tf_hydro*>(ctx);
  auto& q = h->inflight[e];
  return !q.empty() && cudaEventQuery(q.back().ev) == cudaErrorNotReady;
}

TeamCtx& team_ctx(tf_hydro* h, int k, int64_t team) {
  auto& v = h->ctx[k];
  if ((int64_t)v.size() <= team) v.resize(team + 1);
  return v[team];
}

void close_team(tf_hydro* h, int k, int64_t team, int32_t self) {
  TeamCtx& c = team_ctx(h, k, team);
  c.closed = true;
  for (int32_t m : c.members)
    if (m != self) h->runnable.push_back(m);
}

int release_team(tf_hydro* h, int k, int64_t team) {
  TeamCtx& c = team_ctx(h, k, team);
  for (void*& p : c.lease) {
    if (p) {
      int rc = h->pool.release(p);
      if (rc) return rc;
      p = nullptr;
    }
  }
  c.live = false;
  c.members.clear();
  c.waiters.clear();
  return tf_region_release_team(h->regions[k], team);
}

int launch(tf_hydro* h, int k, const int32_t* ids, int T, cudaStream_t s) {
  const int n = h->n;
  switch (k) {
    case K_PREP:
      return tf_prep_f64(h->u, ids, T, n, h->w, 1, s);
    case K_RECON:
      return tf_reconstruct_f64(h->w, h->S, ids, T, n, h->um, h->up, 1, s);
    case K_FLUX:
      return tf_flux_f64(ids, T, n, h->ax, h->ay, h->az, h->um, h->up, h->F,
                         1, s);
    case K_REDUCE:
      return tf_reduce_f64(ids, T, h->ax, h->ay, h->az, h->reduce_out, 1, s);
    default:
      return tf_update_f64(h->u, ids, T, n, h->F, 1, h->dt_dx, h->u_next, s);
  }
}

// The visit's device ops, issued by the LAST member to reach each step.
int issue_step(tf_hydro* h, int k, int64_t team, int step, cudaStream_t s) {
  TeamCtx& c = team_ctx(h, k, team);
  const int T = (int)c.members.size();
  const int64_t ext3 = (int64_t)(h->n + 6) * (h->n + 6) * (h->n + 6);
  const int64_t n3 = (int64_t)h->n * h->n * h->n;
  tf_region* r = h->regions[k];
  int rc = 0;
  if (step == 4 || step == 6) {
    // h2d: pinned ext^3 lease -> device ext^3 lease; d2h: device n^3 ->
    // pinned n^3 (step.py:111-117), one copy of T * bytes_per_slice
    const bool h2d = step == 4;
    const int64_t nbytes = 8 * T * (h2d ? ext3 : n3);
    void* dst = h2d ? c.lease[1] : c.lease[2];
    void* src = h2d ? c.lease[0] : c.lease[3];
    rc = cudaMemcpyAsync(dst, src, (size_t)nbytes,
                         h2d ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToHost,
                         s);
    h->copies += 1;
    h->bytes += nbytes;
  } else {
    if (h->ids_pos + T > h->ids_cap) return TF_E_CAPACITY;
    int32_t* ids = h->ids_h + h->ids_pos;
    h->ids_pos += T;
    for (int i = 0; i < T; ++i) ids[i] = h->tasks[c.members[i]].g;
    tf_nvtx::TeamRange range(kNames[k], T);
    rc = launch(h, k, ids, T, s);
    h->kernels += 1;
  }
  if (rc) return rc;
  rc = tf_team_op_begin(r, team);
  if (rc) return rc;
  if (step == 6) {  // the visit's last op: its completion lands all three
    cudaEvent_t ev;
    if (!h->free_events.empty()) {
      ev = h->free_events.back();
      h->free_events.pop_back();
    } else {
      rc = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
      if (rc) return rc;
    }
    rc = cudaEventRecord(ev, s);
    if (rc) return rc;
    const int32_t parent = tf_region_team_parent(r, team);
    h->inflight[tf_region_parent_executor(r, parent)].push_back({ev, k, team});
  }
  return 0;
}

// Run task t until it parks or finishes (sched.py _step).
int run_task(tf_hydro* h, int32_t ti) {
  Task& t = h->tasks[ti];
  for (;;) {
    const int k = t.visit;
    tf_region* r = h->regions[k];
    if (t.phase == P_ENTER) {
      tf_enter_result res;
      int rc = tf_region_enter(r, t.g, busy_cb, h, &res);
      if (rc) return rc;
      t.team = res.team;
      t.slice = res.slice_id;
      TeamCtx& c = team_ctx(h, k, res.team);
      if (!c.live) {
        c.live = true;
        c.closed = false;
        c.landed = false;
      }
      c.members.push_back(ti);
      t.phase = P_OPS;
      if (!res.closed) return 0;  // parked until the team closes
      close_team(h, k, res.team, ti);
    }
    if (t.phase == P_OPS) {
      TeamCtx& c = team_ctx(h, k, t.team);
      const int T = (int)c.members.size();
      const int64_t ext3 = (int64_t)(h->n + 6) * (h->n + 6) * (h->n + 6);
      const int64_t n3 = (int64_t)h->n * h->n * h->n;
      const cudaStream_t s =
          h->streams[tf_region_parent_executor(r, tf_region_team_parent(
                                                      r, t.team))];
      for (int step = 0; step < 7; ++step) {
        int32_t idx, arrivals;
        int rc = tf_team_issue(r, t.team, step, h->sig[k][step].c_str(), &idx,
                               &arrivals);
        if (rc) return rc;
        if (step < 4) {
          if (arrivals == 1) {  // first arrival leases len * T
            const int kind = (step % 2 == 0) ? KIND_PINNED : KIND_DEVICE;
            const int64_t len = step < 2 ? ext3 : n3;
            rc = h->pool.acquire(kind, 8 * len * T, &c.lease[step]);
            if (rc) return rc;
          }
        } else if (arrivals == T) {
          const int64_t t0 = host_ns();
          rc = issue_step(h, k, t.team, step, s);
          h->ns_issue += host_ns() - t0;
          if (rc) return rc;
        }
      }
      t.phase = P_LEAVE;
      if (!c.landed) {
        c.waiters.push_back(ti);
        return 0;  // await(d2h)
      }
    }
    // P_LEAVE
    int32_t release = 0;
    int rc = tf_team_leave(r, t.team, 7, &release);
    if (rc) return rc;
    if (release) {
      rc = release_team(h, k, t.team);
      if (rc) return rc;
    }
    t.visit += 1;
    t.phase = P_ENTER;
    if (t.visit == kRegions) {
      h->finished += 1;
      return 0;
    }
  }
}

// Device progress: retire landed visits, fire idle watches of drained
// streams (device.py:356-373).  Returns 1 on any progress.
int poll(tf_hydro* h, int* err) {
  int progress = 0;
  h->polls += 1;
  for (int e = 0; e < h->E; ++e) {
    auto& q = h->inflight[e];
    while (!q.empty()) {
      const cudaError_t st = cudaEventQuery(q.front().ev);
      if (st == cudaErrorNotReady) break;
      if (st != cudaSuccess) {
        *err = st;
        return 0;
      }
      const Op op = q.front();
      q.pop_front();
      h->free_events.push_back(op.ev);
      progress = 1;
      TeamCtx& c = team_ctx(h, op.region, op.team);
      c.landed = true;
      for (int32_t w : c.waiters) h->runnable.push_back(w);
      c.waiters.clear();
      int32_t release = 0;
      for (int i = 0; i < 3 && !*err; ++i)  // h2d, launch, d2h
        *err = tf_team_op_end(h->regions[op.region], op.team, &release);
      if (!*err && release) *err = release_team(h, op.region, op.team);
      if (*err) return 0;
    }
    if (q.empty()) {
      for (int k = 0; k < kRegions; ++k) {
        const int32_t cap = tf_region_watch_count(h->regions[k], e);
        if (cap <= 0) continue;
        std::vector<int64_t> closed(cap);
        const int got = tf_region_stream_idle(h->regions[k], e, closed.data(),
                                              cap);
        if (got < 0) {
          *err = -got;
          return 0;
        }
        for (int i = 0; i < got; ++i) close_team(h, k, closed[i], -1);
        if (got) progress = 1;
      }
    }
  }
  return progress;
}

std::string fmt_sig(const char* a, const char* b, int64_t c) {
  return std::string(a) + ":" + b + ":" + std::to_string(c);
}

}  // namespace

extern "C" {

int tf_hydro_create(int32_t n, int32_t per_axis, int32_t max_team,
                    int32_t executors, const tf_stream_t* streams, double ax,
                    double ay, double az, double dt_dx, double* w, double* um,
                    double* up, double* F, double* reduce_out,
                    tf_hydro** out) {
  if (!out || (n != 8 && n != 16) || per_axis < 1 || executors < 1 ||
      max_team < 1 || max_team > TF_MAX_TEAM || !w || !um || !up || !F ||
      !reduce_out)
    return TF_E_INVALID;
  tf_hydro* h = new tf_hydro();
  h->n = n;
  h->m = per_axis;
  h->S = per_axis * per_axis * per_axis;
  h->E = executors;
  h->max_team = max_team;
  h->ax = ax;
  h->ay = ay;
  h->az = az;
  h->dt_dx = dt_dx;
  h->w = w;
  h->um = um;
  h->up = up;
  h->F = F;
  h->reduce_out = reduce_out;
  const int parents = h->S / max_team > 1 ? h->S / max_team : 1;  // step.py:61
  int rc = 0;
  for (int k = 0; k < kRegions && !rc; ++k)
    rc = tf_region_create(kNames[k], max_team, parents, executors,
                          &h->regions[k]);
  h->ctx.resize(kRegions);
  h->inflight.resize(executors);
  h->streams.resize(executors);
  h->own_streams = streams == nullptr;
  for (int e = 0; e < executors && !rc; ++e) {
    if (streams)
      h->streams[e] = (cudaStream_t)streams[e];
    else
      rc = cudaStreamCreateWithFlags(&h->streams[e], cudaStreamNonBlocking);
  }
  if (!rc) rc = cudaEventCreateWithFlags(&h->fork, cudaEventDisableTiming);
  // every visit launches one team kernel per region per task at most
  h->ids_cap = (int64_t)kRegions * h->S;
  if (!rc) rc = cudaHostAlloc(&h->ids_h, sizeof(int32_t) * h->ids_cap, 0);
  const int64_t ext3 = (int64_t)(n + 6) * (n + 6) * (n + 6), n3 = n * n * n;
  for (int k = 0; k < kRegions; ++k) {
    // step.py:106-117 in the reference's signature format (aggregator.py
    // _fmt_sig): alloc x4, copy h2d, launch, copy d2h
    h->sig[k][0] = fmt_sig("alloc:pinned_host", "<f8", ext3);
    h->sig[k][1] = fmt_sig("alloc:device", "<f8", ext3);
    h->sig[k][2] = fmt_sig("alloc:pinned_host", "<f8", n3);
    h->sig[k][3] = fmt_sig("alloc:device", "<f8", n3);
    h->sig[k][4] = "copy:h2d:" + std::to_string(ext3 * 8);
    h->sig[k][5] = std::string("launch:") + kNames[k] + ":" +
                   std::to_string(blocks_for(k, n)) + ":1";
    h->sig[k][6] = "copy:d2h:" + std::to_string(n3 * 8);
  }
  h->tasks.resize(h->S);
  // staging arenas: buckets are exact sizes and a buffer keeps its storage
  // (the reference's pool), so real-time formation with many distinct team
  // sizes needs several times one iteration's live leases (S x (ext^3+n^3)
  // per kind): 8x, capped at 1 GiB per kind
  if (!rc) {
    int64_t arena = 8LL * h->S * (ext3 + n3) * 8;
    if (arena > (1LL << 30)) arena = 1LL << 30;
    rc = h->pool.reserve(arena);
  }
  if (rc) {
    tf_hydro_destroy(h);
    return rc;
  }
  *out = h;
  return 0;
}

void tf_hydro_destroy(tf_hydro* h) {
  if (!h) return;
  for (auto& q : h->inflight) {
    for (auto& op : q) {
      cudaEventSynchronize(op.ev);
      cudaEventDestroy(op.ev);
    }
  }
  for (cudaEvent_t e : h->free_events) cudaEventDestroy(e);
  if (h->own_streams)
    for (cudaStream_t s : h->streams)
      if (s) cudaStreamDestroy(s);
  if (h->fork) cudaEventDestroy(h->fork);
  if (h->ids_h) cudaFreeHost(h->ids_h);
  for (auto* r : h->regions)
    if (r) tf_region_destroy(r);
  delete h;
}

// bench.py:142-153 _presize_pools: every (kind, len * team size) bucket the
// run can touch, count = ceil(tasks / size), so steady state never
// raw-allocates.
int tf_hydro_presize(tf_hydro* h) {
  if (!h) return TF_E_INVALID;
  const int n = h->n;
  const int64_t ext3 = (int64_t)(n + 6) * (n + 6) * (n + 6), n3 = n * n * n;
  const int top = h->max_team < h->S ? h->max_team : h->S;
  for (int size = 1; size <= top; ++size) {
    const int count = ceil_div(h->S, size);
    for (int kind = 0; kind < 2; ++kind)
      for (int64_t len : {ext3, n3}) h->pool.ensure(kind, 8 * len * size, count);
  }
  return 0;
}

int tf_hydro_iteration(tf_hydro* h, const double* u_pool, double* u_next_pool,
                       tf_stream_t stream) {
  if (!h || !u_pool || !u_next_pool) return TF_E_INVALID;
  const int64_t t_begin = host_ns();
  h->u = u_pool;
  h->u_next = u_next_pool;
  h->ids_pos = 0;
  h->finished = 0;
  // the executor streams start after the work issued on `stream` so far
  // (the ghost exchange that produced u_pool)
  int rc = cudaEventRecord(h->fork, (cudaStream_t)stream);
  for (int e = 0; e < h->E && !rc; ++e)
    rc = cudaStreamWaitEvent(h->streams[e], h->fork, 0);
  if (rc) return rc;
  // driver (step.py:133-137): one task per sub-grid, lexicographic order
  h->runnable.clear();
  for (int32_t g = 0; g < h->S; ++g) {
    Task& t = h->tasks[g];
    t = Task();
    t.g = g;
    h->runnable.push_back(g);
  }
  while (h->finished < h->S) {
    if (!h->runnable.empty()) {
      const int32_t ti = h->runnable.front();
      h->runnable.pop_front();
      rc = run_task(h, ti);
      if (rc) return rc;
      continue;
    }
    int err = 0;
    const int64_t t0 = host_ns();
    const int progress = poll(h, &err);
    if (!progress) h->ns_idle_poll += host_ns() - t0;
    if (err) return err;
    if (!progress) {
      bool any = false;
      for (auto& q : h->inflight) any = any || !q.empty();
      for (int k = 0; k < kRegions && !any; ++k)
        for (int e = 0; e < h->E && !any; ++e)
          any = tf_region_watch_count(h->regions[k], e) > 0;
      if (!any) return TF_E_ORDERING;  // parked tasks, nothing to wake them
    }
  }
  // the caller's stream continues after every team's work
  for (int e = 0; e < h->E && !rc; ++e) {
    rc = cudaEventRecord(h->fork, h->streams[e]);
    if (!rc) rc = cudaStreamWaitEvent((cudaStream_t)stream, h->fork, 0);
  }
  h->ns_iter += host_ns() - t_begin;
  return rc;
}

int tf_hydro_region(const tf_hydro* h, int32_t k, tf_region** out) {
  if (!h || k < 0 || k >= kRegions || !out) return TF_E_INVALID;
  *out = h->regions[k];
  return 0;
}

int tf_hydro_host_times(const tf_hydro* h, int64_t* out3) {
  if (!h || !out3) return TF_E_INVALID;
  out3[0] = h->ns_issue;
  out3[1] = h->ns_idle_poll;
  out3[2] = h->ns_iter;
  return 0;
}

int tf_hydro_counters(const tf_hydro* h, int64_t* out8) {
  if (!h || !out8) return TF_E_INVALID;
  out8[0] = h->kernels;
  out8[1] = h->copies;
  out8[2] = h->bytes;
  out8[3] = h->pool.raw(KIND_DEVICE);
  out8[4] = h->pool.raw(KIND_PINNED);
  out8[5] = h->pool.outstanding();
  // real cudaMalloc / cudaHostAlloc calls past the reserved arenas (a chunk
  // carved from an arena is not an allocation)
  out8[6] = h->pool.spilled();
  out8[7] = h->polls;
  return 0;
}

}  // extern "C"
