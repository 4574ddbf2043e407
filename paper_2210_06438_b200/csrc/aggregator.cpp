// aggregator.cpp — strategy-3 team formation core and the real-time bulk
// executor that feeds the batched sm_100a kernels.
//
// The formation state machine restates AggregationRegion.enter/_close/
// _close_if_forming (reference aggregator.py:284-345) with the device
// queries abstracted behind two signals:
//   * stream_busy(executor)   -> device.stream_busy        (device.py:187-194)
//   * tf_region_stream_idle() <- the stream-drain callback (device.py:364-370)
// Fed the same signal sequence, it produces the same teams, parents and
// slice ids as the reference (checked against recorded reference traces in
// tests/test_abi.py).  The executor wires the signals to real
// CUDA streams: busy == the parent stream's last event has not completed.
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstddef>
#include <chrono>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/taskfuse_b200.h"
#include "tf_nvtx.h"

namespace {

// zlib crc32 (IEEE 802.3, reflected 0xEDB88320) — the reference derives each
// region's lead executor from crc32(name) (aggregator.py:273).
struct Crc32Table {
  uint32_t t[256];
  Crc32Table() {
    for (uint32_t i = 0; i < 256; ++i) {
      uint32_t c = i;
      for (int k = 0; k < 8; ++k) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
      t[i] = c;
    }
  }
};

uint32_t crc32_ieee(const char* s) {
  static const Crc32Table table;  // thread-safe one-time init
  uint32_t c = 0xFFFFFFFFu;
  for (const unsigned char* p = (const unsigned char*)s; *p; ++p)
    c = table.t[(c ^ *p) & 0xFFu] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

enum { FORMING = 0, CAP = 1, SOLO = 2, DRAIN = 3 };

// One step of a team's SPMD op sequence (aggregator.py:64-74): every member
// issues the same signature at the same cursor; the first arrival owns the
// step's lease, the last one issues its device op.
struct TeamStep {
  std::string sig;
  int32_t arrivals = 0;
  int64_t lease = -1;
};

struct Team {
  int32_t parent = 0;
  int32_t state = FORMING;  // FORMING or the closure reason
  uint32_t gen = 0;         // bumped each time the slot is reused
  bool watching = false;    // holds a stream-idle watch (forming only)
  std::vector<int64_t> tags;
  // member bookkeeping after closure (aggregator.py:76-99,168-234)
  std::vector<TeamStep> steps;
  int32_t final_cursor = -1;  // cursor of the first member to leave
  int32_t left = 0;
  int32_t pending_ops = 0;
  bool released = false;
};

struct Parent {
  int32_t executor = 0;
  int64_t forming = -1;
};

// Live teams in reusable slots: a team id is its slot index while alive
// (ids are unique among live teams; a released slot is recycled, keeping
// its tag vector's capacity, so steady-state formation never allocates).
class TeamTable {
 public:
  int64_t create(int32_t parent) {
    int64_t id;
    if (!free_.empty()) {
      id = free_.back();
      free_.pop_back();
    } else {
      id = (int64_t)slots_.size();
      slots_.emplace_back();
    }
    Slot& s = slots_[id];
    s.alive = true;
    Team& t = s.team;
    t.gen += 1;
    t.watching = false;
    t.parent = parent;
    t.state = FORMING;
    t.tags.clear();
    t.steps.clear();   // keeps capacity (and the strings' buffers below)
    t.final_cursor = -1;
    t.left = 0;
    t.pending_ops = 0;
    t.released = false;
    return id;
  }
  Team* get(int64_t id) {
    if (id < 0 || id >= (int64_t)slots_.size() || !slots_[id].alive)
      return nullptr;
    return &slots_[id].team;
  }
  const Team* get(int64_t id) const {
    return const_cast<TeamTable*>(this)->get(id);
  }
  void release(int64_t id) {
    slots_[id].alive = false;
    free_.push_back(id);
  }

 private:
  struct Slot {
    bool alive = false;
    Team team;
  };
  std::vector<Slot> slots_;
  std::vector<int64_t> free_;
};

// A stream-idle watch: the team's slot id and its generation, so a watch
// left behind by a team that closed at its cap (the slot since recycled)
// is recognised as stale instead of searched for and erased at the close.
struct Watch {
  int64_t id;
  uint32_t gen;
};

}  // namespace

struct tf_region {
  std::string name;
  int32_t max_team = 1;
  int32_t executors = 1;
  std::vector<Parent> parents;
  int64_t arrivals = 0;
  int32_t next_parent = 0;  // == arrivals % parents.size(), kept incrementally
  TeamTable teams;
  // per executor: forming teams holding a stream-idle watch, in watch order
  // (plus stale watches of teams that closed at their cap since, skipped
  // and dropped by the next tf_region_stream_idle), and the live count
  std::vector<std::vector<Watch>> watchers;
  std::vector<int32_t> live_watch;
  std::vector<Watch> fire_scratch;  // tf_region_stream_idle's swap buffer
  int64_t teams_formed = 0;
  int64_t solo_fast_path = 0;
  int64_t histogram[TF_MAX_TEAM + 1] = {0};
  int64_t violations = 0;
  std::string error;  // last ordering violation: "expected\ngot"
};

namespace {

void close_team(tf_region* r, int64_t id, Team& t, int reason) {
  t.state = reason;
  r->teams_formed += 1;
  r->histogram[t.tags.size()] += 1;
  (void)id;
}

// O(1): the watch entry stays in the list, stale (a linear search + erase
// per cap closure made formation quadratic in the forming teams — A = 4 on
// 4096 arrivals keeps ~1000 teams forming)
void unwatch(tf_region* r, int32_t executor, Team& t) {
  if (!t.watching) return;
  t.watching = false;
  r->live_watch[executor] -= 1;
}

}  // namespace

extern "C" {

int tf_region_create(const char* name, int32_t max_team, int32_t parent_count,
                     int32_t executors, tf_region** out) {
  if (!name || !out || max_team < 1 || max_team > TF_MAX_TEAM ||
      parent_count < 1 || executors < 1)
    return TF_E_INVALID;
  tf_region* r = new tf_region();
  r->name = name;
  r->max_team = max_team;
  r->executors = executors;
  const uint32_t lead = crc32_ieee(name) % (uint32_t)executors;
  r->parents.resize(parent_count);
  for (int32_t i = 0; i < parent_count; ++i)
    r->parents[i].executor = (int32_t)((lead + (uint32_t)i) % (uint32_t)executors);
  r->watchers.resize(executors);
  r->live_watch.assign(executors, 0);
  *out = r;
  return 0;
}

void tf_region_destroy(tf_region* r) { delete r; }

int32_t tf_region_parent_executor(const tf_region* r, int32_t parent) {
  if (!r || parent < 0 || parent >= (int32_t)r->parents.size()) return -1;
  return r->parents[parent].executor;
}

int tf_region_enter(tf_region* r, int64_t tag, tf_busy_fn busy, void* ctx,
                    tf_enter_result* out) {
  if (!r || !out) return TF_E_INVALID;
  const int32_t pi = r->next_parent;  // parents[arrivals % P]
  r->arrivals += 1;
  if (++r->next_parent == (int32_t)r->parents.size()) r->next_parent = 0;
  Parent& p = r->parents[pi];
  int64_t id = p.forming;
  if (id < 0) id = r->teams.create(pi);
  Team& t = *r->teams.get(id);
  out->parent = pi;
  out->executor = p.executor;
  out->team = id;
  out->slice_id = (int32_t)t.tags.size();
  out->closed = FORMING;
  out->queried = 0;
  t.tags.push_back(tag);
  if ((int32_t)t.tags.size() >= r->max_team) {
    // cap reached (max_team 1 closes instantly)           aggregator.py:310
    if (p.forming == id) {
      p.forming = -1;
      unwatch(r, p.executor, t);
    }
    close_team(r, id, t, CAP);
    out->closed = CAP;
  } else if (p.forming < 0) {
    out->queried = 1;
    const int is_busy = busy ? busy(ctx, p.executor) : 1;
    if (!is_busy) {
      // device is starving: run alone rather than wait     aggregator.py:317
      r->solo_fast_path += 1;
      close_team(r, id, t, SOLO);
      out->closed = SOLO;
    } else {
      p.forming = id;  // watch the stream for its drain  aggregator.py:321
      auto& w = r->watchers[p.executor];
      if (w.size() > 2 * (size_t)r->live_watch[p.executor] + 64) {
        // drop the stale watches (order kept) so that a stream that never
        // drains does not grow the list without bound
        w.erase(std::remove_if(w.begin(), w.end(),
                               [&](const Watch& x) {
                                 const Team* u = r->teams.get(x.id);
                                 return !u || u->gen != x.gen || !u->watching;
                               }),
                w.end());
      }
      w.push_back(Watch{id, t.gen});
      t.watching = true;
      r->live_watch[p.executor] += 1;
    }
  }
  return 0;
}

int tf_region_stream_idle(tf_region* r, int32_t executor, int64_t* out_teams,
                          int32_t cap) {
  if (!r || executor < 0 || executor >= r->executors) return -TF_E_INVALID;
  if (cap < 0 || (cap > 0 && !out_teams)) return -TF_E_INVALID;
  std::vector<Watch>& fire = r->fire_scratch;
  fire.swap(r->watchers[executor]);  // keeps both buffers' capacity
  int32_t n = 0;
  for (const Watch& w : fire) {
    const int64_t id = w.id;
    Team* t = r->teams.get(id);
    // stale: the team closed at its cap (and its slot may be reused)
    if (!t || t->gen != w.gen || !t->watching || t->state != FORMING)
      continue;
    if (n == cap) {
      // no room to report it: it keeps watching, so the caller's next call
      // (sized by tf_region_watch_count) closes it — a team is never closed
      // without its id reaching the caller
      r->watchers[executor].push_back(w);
      continue;
    }
    Parent& p = r->parents[t->parent];
    if (p.forming == id) p.forming = -1;  // aggregator.py:328-332
    t->watching = false;
    r->live_watch[executor] -= 1;
    close_team(r, id, *t, DRAIN);
    out_teams[n++] = id;
  }
  fire.clear();
  return n;
}

int32_t tf_region_watch_count(const tf_region* r, int32_t executor) {
  if (!r || executor < 0 || executor >= r->executors) return -TF_E_INVALID;
  return r->live_watch[executor];
}

int tf_region_team_size(const tf_region* r, int64_t team) {
  if (!r) return -TF_E_INVALID;
  const Team* t = r->teams.get(team);
  if (!t) return -TF_E_INVALID;
  return (int)t->tags.size();
}

int tf_region_team_members(const tf_region* r, int64_t team, int64_t* tags,
                           int32_t cap) {
  if (!r || !tags) return -TF_E_INVALID;
  const Team* t = r->teams.get(team);
  if (!t) return -TF_E_INVALID;
  const auto& v = t->tags;
  const int32_t n = std::min<int32_t>(cap, (int32_t)v.size());
  std::copy(v.begin(), v.begin() + n, tags);
  return (int)v.size();
}

int tf_region_team_parent(const tf_region* r, int64_t team) {
  if (!r) return -TF_E_INVALID;
  const Team* t = r->teams.get(team);
  if (!t) return -TF_E_INVALID;
  return t->parent;
}

int tf_region_stats(const tf_region* r, int64_t* teams_formed,
                    int64_t* solo_fast_path, int64_t* histogram129) {
  if (!r) return TF_E_INVALID;
  if (teams_formed) *teams_formed = r->teams_formed;
  if (solo_fast_path) *solo_fast_path = r->solo_fast_path;
  if (histogram129)
    for (int i = 0; i <= TF_MAX_TEAM; ++i) histogram129[i] = r->histogram[i];
  return 0;
}

// Frees the bookkeeping of a closed team (the executor does this after the
// launch; the Python facade after every member left).
int tf_region_release_team(tf_region* r, int64_t team) {
  if (!r) return TF_E_INVALID;
  const Team* t = r->teams.get(team);
  if (!t || t->state == FORMING) return TF_E_INVALID;
  r->teams.release(team);
  return 0;
}

// ---- member-side bookkeeping of a closed team ----------------------------
// The reference keeps this per team in Python (TeamMember._issue / leave /
// _chain / _maybe_release, aggregator.py:168-234); here it lives next to the
// formation state, so the Python facade and the native HydroSim engine run
// the same rules.

namespace {

int violation(tf_region* r, const std::string& expected, const char* got) {
  r->violations += 1;
  r->error = expected;
  r->error += '\n';
  r->error += got;
  return TF_E_ORDERING;
}

// left == size and nothing in flight: the team's leases may go back
int release_due(Team& t) {
  if (t.released || t.left < (int32_t)t.tags.size() || t.pending_ops > 0)
    return 0;
  t.released = true;
  return 1;
}

}  // namespace

int tf_team_issue(tf_region* r, int64_t team, int32_t cursor, const char* sig,
                  int32_t* step, int32_t* arrivals) {
  if (!r || !sig || cursor < 0) return TF_E_INVALID;
  Team* t = r->teams.get(team);
  if (!t || t->state == FORMING || t->released) return TF_E_INVALID;
  // a member may not issue past the point where another already left
  if (t->final_cursor >= 0 && cursor >= t->final_cursor)
    return violation(r, "leave", sig);
  if (cursor < (int32_t)t->steps.size()) {
    if (t->steps[cursor].sig != sig)
      return violation(r, t->steps[cursor].sig, sig);
  } else if (cursor == (int32_t)t->steps.size()) {
    t->steps.emplace_back();
    t->steps.back().sig = sig;
  } else {
    return TF_E_INVALID;  // a member skipped a step: caller bug
  }
  TeamStep& st = t->steps[cursor];
  st.arrivals += 1;
  if (step) *step = cursor;
  if (arrivals) *arrivals = st.arrivals;
  return 0;
}

int tf_team_leave(tf_region* r, int64_t team, int32_t cursor,
                  int32_t* release) {
  if (!r || cursor < 0) return TF_E_INVALID;
  Team* t = r->teams.get(team);
  if (!t || t->state == FORMING || t->released) return TF_E_INVALID;
  if ((int32_t)t->steps.size() > cursor)
    return violation(r, t->steps[cursor].sig, "leave");
  t->final_cursor = cursor;
  t->left += 1;
  const int due = release_due(*t);
  if (release) *release = due;
  return 0;
}

int tf_team_op_begin(tf_region* r, int64_t team) {
  Team* t = r ? r->teams.get(team) : nullptr;
  if (!t || t->released) return TF_E_INVALID;
  t->pending_ops += 1;
  return 0;
}

int tf_team_op_end(tf_region* r, int64_t team, int32_t* release) {
  Team* t = r ? r->teams.get(team) : nullptr;
  if (!t || t->pending_ops < 1) return TF_E_INVALID;
  t->pending_ops -= 1;
  const int due = release_due(*t);
  if (release) *release = due;
  return 0;
}

int tf_team_set_lease(tf_region* r, int64_t team, int32_t step,
                      int64_t lease) {
  Team* t = r ? r->teams.get(team) : nullptr;
  if (!t || step < 0 || step >= (int32_t)t->steps.size()) return TF_E_INVALID;
  t->steps[step].lease = lease;
  return 0;
}

int64_t tf_team_lease(const tf_region* r, int64_t team, int32_t step) {
  const Team* t = r ? r->teams.get(team) : nullptr;
  if (!t || step < 0 || step >= (int32_t)t->steps.size()) return -1;
  return t->steps[step].lease;
}

int tf_team_leases(const tf_region* r, int64_t team, int64_t* out,
                   int32_t cap) {
  const Team* t = r ? r->teams.get(team) : nullptr;
  if (!t) return -TF_E_INVALID;
  int32_t n = 0;
  for (const TeamStep& st : t->steps)
    if (st.lease >= 0) {
      if (out && n < cap) out[n] = st.lease;
      ++n;
    }
  return n;
}

int tf_team_step_info(const tf_region* r, int64_t team, int32_t step,
                      int32_t* arrivals, char* sig, int32_t sig_cap) {
  const Team* t = r ? r->teams.get(team) : nullptr;
  if (!t || step < 0 || step >= (int32_t)t->steps.size()) return TF_E_INVALID;
  const TeamStep& st = t->steps[step];
  if (arrivals) *arrivals = st.arrivals;
  if (sig && sig_cap > 0) {
    const size_t k = std::min<size_t>((size_t)sig_cap - 1, st.sig.size());
    std::copy(st.sig.begin(), st.sig.begin() + k, sig);
    sig[k] = 0;
  }
  return 0;
}

int64_t tf_region_violations(const tf_region* r) {
  return r ? r->violations : -1;
}

const char* tf_region_error(const tf_region* r) {
  return r ? r->error.c_str() : "";
}

}  // extern "C"

// ------------------------------------------------------------ executor
struct tf_executor {
  tf_region* region = nullptr;
  std::vector<cudaStream_t> streams;
  std::vector<cudaEvent_t> last;
  std::vector<char> recorded;
  std::vector<char> overlap_ok;  // previous op on the stream is a team kernel
  cudaEvent_t fork = nullptr;
  int32_t flags = 0;
  std::vector<int64_t> busy_until;  // steady-clock ns; see rt_busy
};

namespace {

int64_t now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// A stream observed busy is not re-queried for kRecheckNs: no kernel
// finishes faster than that, and cudaEventQuery (~0.3-1 us) would otherwise
// dominate the arrival loop.
constexpr int64_t kRecheckNs = 2000;

int rt_busy(void* ctx, int32_t e) {
  tf_executor* ex = static_cast<tf_executor*>(ctx);
  if (!ex->recorded[e]) return 0;
  const int64_t t = now_ns();
  if (t < ex->busy_until[e]) return 1;
  if (cudaEventQuery(ex->last[e]) == cudaErrorNotReady) {
    ex->busy_until[e] = t + kRecheckNs;
    return 1;
  }
  return 0;
}

struct ReconArgs {
  const double* pool;
  int64_t slices;
  int32_t n;
  double ax, ay, az;
  double *um, *up, *F, *amax;
  int32_t flux_form;
};

int launch_team(tf_executor* ex, int64_t team, const ReconArgs& a,
                int64_t* launches) {
  tf_region* r = ex->region;
  const Team* tp = r->teams.get(team);
  if (!tp) return TF_E_INVALID;
  const Team& t = *tp;
  int32_t ids[TF_MAX_TEAM];
  const int T = (int)t.tags.size();
  for (int i = 0; i < T; ++i) ids[i] = (int32_t)t.tags[i];
  const int32_t e = r->parents[t.parent].executor;
  const int f = ex->overlap_ok[e] ? (ex->flags & TF_LAUNCH_OVERLAP_PREV) : 0;
  tf_nvtx::TeamRange range("team launch", T);
  int rc = tf_recon_flux_team_ex_f64(a.pool, a.slices, ids, T, a.n, a.ax,
                                     a.ay, a.az, a.um, a.up, a.F,
                                     /*out_mode=*/1, a.amax, a.flux_form, f,
                                     (tf_stream_t)ex->streams[e]);
  if (rc) return rc;
  ex->overlap_ok[e] = 1;
  cudaError_t ce = cudaEventRecord(ex->last[e], ex->streams[e]);
  if (ce != cudaSuccess) return ce;
  ex->recorded[e] = 1;
  ex->busy_until[e] = now_ns() + kRecheckNs;  // just launched: busy
  r->teams.release(team);
  *launches += 1;
  return 0;
}

int drain_executor(tf_executor* ex, int32_t e, const ReconArgs& a,
                   int64_t* launches) {
  std::vector<int64_t> closed(ex->region->live_watch[e]);
  if (closed.empty()) return 0;
  const int n = tf_region_stream_idle(ex->region, e, closed.data(),
                                      (int32_t)closed.size());
  if (n < 0) return -n;
  for (int i = 0; i < n; ++i) {
    int rc = launch_team(ex, closed[i], a, launches);
    if (rc) return rc;
  }
  return 0;
}

}  // namespace

extern "C" {

int tf_executor_create(tf_region* region, int32_t count, tf_executor** out) {
  if (!region || !out || count < 1 || count != region->executors)
    return TF_E_INVALID;
  tf_executor* ex = new tf_executor();
  ex->region = region;
  ex->streams.resize(count);
  ex->last.resize(count);
  ex->recorded.assign(count, 0);
  ex->overlap_ok.assign(count, 0);
  ex->busy_until.assign(count, 0);
  if (cudaEventCreateWithFlags(&ex->fork, cudaEventDisableTiming) !=
      cudaSuccess) {
    delete ex;
    return TF_E_INVALID;
  }
  for (int i = 0; i < count; ++i) {
    cudaError_t e = cudaStreamCreateWithFlags(&ex->streams[i], cudaStreamNonBlocking);
    if (e == cudaSuccess)
      e = cudaEventCreateWithFlags(&ex->last[i], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      delete ex;
      return e;
    }
  }
  *out = ex;
  return 0;
}

void tf_executor_destroy(tf_executor* ex) {
  if (!ex) return;
  for (auto s : ex->streams) cudaStreamDestroy(s);
  for (auto e : ex->last) cudaEventDestroy(e);
  if (ex->fork) cudaEventDestroy(ex->fork);
  delete ex;
}

tf_stream_t tf_executor_stream(const tf_executor* ex, int32_t executor) {
  if (!ex || executor < 0 || executor >= (int32_t)ex->streams.size())
    return nullptr;
  return (tf_stream_t)ex->streams[executor];
}

int tf_executor_run_recon_flux(tf_executor* ex, const double* pool_ext,
                               int64_t pool_slices, const int32_t* ids,
                               int64_t count, int32_t n, double ax, double ay,
                               double az, double* um, double* up, double* F,
                               double* amax, int32_t flux_form,
                               int64_t* launches) {
  if (!ex || !ids || count < 0 || !launches) return TF_E_INVALID;
  ReconArgs a{pool_ext, pool_slices, n, ax, ay, az, um, up, F, amax, flux_form};
  tf_region* r = ex->region;
  const int32_t E = (int32_t)ex->streams.size();
  *launches = 0;
  for (int64_t i = 0; i < count; ++i) {
    // real-time drain signal: before the arrival joins its parent's forming
    // team, observe whether that parent's stream has gone idle meanwhile
    const int32_t pi = r->next_parent;
    const int32_t pe = r->parents[pi].executor;
    if (r->live_watch[pe] > 0 && !rt_busy(ex, pe)) {
      int rc = drain_executor(ex, pe, a, launches);
      if (rc) return rc;
    }
    if ((i & 31) == 31) {
      for (int32_t e = 0; e < E; ++e)
        if (e != pe && r->live_watch[e] > 0 && !rt_busy(ex, e)) {
          int rc = drain_executor(ex, e, a, launches);
          if (rc) return rc;
        }
    }
    tf_enter_result res;
    int rc = tf_region_enter(r, ids[i], rt_busy, ex, &res);
    if (rc) return rc;
    if (res.closed != FORMING) {
      rc = launch_team(ex, res.team, a, launches);
      if (rc) return rc;
    }
  }
  // no more arrivals: every stream eventually drains, closing what is left
  for (int32_t e = 0; e < E; ++e) {
    int rc = drain_executor(ex, e, a, launches);
    if (rc) return rc;
  }
  return 0;
}

int tf_executor_set_flags(tf_executor* ex, int32_t flags) {
  if (!ex) return TF_E_INVALID;
  ex->flags = flags;
  return 0;
}

int tf_executor_fork(tf_executor* ex, tf_stream_t stream) {
  if (!ex) return TF_E_INVALID;
  cudaError_t ce = cudaEventRecord(ex->fork, (cudaStream_t)stream);
  for (size_t e = 0; e < ex->streams.size() && ce == cudaSuccess; ++e) {
    ce = cudaStreamWaitEvent(ex->streams[e], ex->fork, 0);
    ex->overlap_ok[e] = 0;  // next team follows a full dependency
  }
  return ce;
}

int tf_executor_join(tf_executor* ex, tf_stream_t stream) {
  if (!ex) return TF_E_INVALID;
  for (size_t e = 0; e < ex->streams.size(); ++e) {
    cudaError_t ce = cudaEventRecord(ex->last[e], ex->streams[e]);
    if (ce == cudaSuccess)
      ce = cudaStreamWaitEvent((cudaStream_t)stream, ex->last[e], 0);
    if (ce != cudaSuccess) return ce;
    ex->recorded[e] = 1;
  }
  return 0;
}

int tf_executor_sync(tf_executor* ex) {
  if (!ex) return TF_E_INVALID;
  for (auto s : ex->streams) {
    cudaError_t ce = cudaStreamSynchronize(s);
    if (ce != cudaSuccess) return ce;
  }
  return 0;
}

}  // extern "C"

// ------------------------------------------------- device-queue executor
// Strategy 3 where closing a team publishes its sub-grid ids into a ring the
// GPU's resident consumer grid drains (tf_queue_consumer_launch), instead of
// launching a kernel.  The reference's signals map to the queue:
//   busy  == published slices not all completed (per-CTA progress counters
//            the consumer writes to mapped pinned memory)
//   drain == observed by polling busy at arrivals (as the stream executor).
// One queue == one executor (the region must have executors == 1).
struct QueueCtlHost {   // mirrors QueueCtl (hydro_kernels.cu)
  long long published;
  long long final_count;
  long long completed;    // (epoch << 32) | slices done
  long long status;       // 1: the consumer grid timed out
};
struct QueueDevInit {   // mirrors QueueDev (one 128-B line per word)
  alignas(128) long long published;
  alignas(128) long long final_count;  // (epoch << 32) | count
  alignas(128) unsigned long long spare;
  alignas(128) unsigned long long done;
};

// One queue instance; runs alternate between two so that run k+1 can
// publish while run k's consumer grid is still draining its tail.  A slot's
// device completion count is monotonic across its runs (the host passes
// each run the slices of the slot's earlier runs) and its close marker is
// tagged with the run's epoch, so nothing is reset between runs and
// consecutive runs can overlap (programmatic dependent launch,
// k_queue_consumer).
struct QueueSlot {
  QueueCtlHost* ctl_h = nullptr;   // mapped pinned
  void* ctl_hd = nullptr;          // its device alias
  int64_t* ring_h = nullptr;       // mapped pinned, tagged (epoch << 32 | id)
  int64_t* ring_hd = nullptr;      // its device alias
  int64_t* ring_d = nullptr;       // device mirror, tagged (epoch << 32 | id)
  int32_t epoch = 0;               // last epoch launched on this slot
  int64_t ring_cap = 0;
  void* qdev = nullptr;            // QueueDevInit on the device
  uint64_t done_base = 0;          // slices of the slot's earlier runs
  int64_t count = 0;               // slices the last run published
  cudaEvent_t ev = nullptr;        // recorded only to order other streams
  cudaStream_t stream = nullptr;   // where this slot's last run went
  bool in_flight = false;
};

struct tf_qexec {
  tf_region* region = nullptr;
  QueueSlot slots[2];
  int cur = 1;
  int32_t n = 0;
  int32_t flags = 0;               // TF_LAUNCH_OVERLAP_PREV: early box loads
  int64_t published = 0;
  int64_t seen_published = 0;
  // host time per phase, summed over runs: waiting for a slot's previous
  // run, the launch, the formation + publish loop
  int64_t runs = 0, ns_wait = 0, ns_launch = 0, ns_publish = 0;
  QueueSlot& slot() { return slots[cur]; }
  const QueueSlot& slot() const { return slots[cur]; }
};

namespace {

int64_t q_now_ns() {
  return std::chrono::duration_cast<std::chrono::nanoseconds>(
             std::chrono::steady_clock::now().time_since_epoch())
      .count();
}

// a GPU-written count, if it carries the slot's current epoch
int64_t q_tagged(const long long* word, int32_t epoch) {
  const uint64_t v = (uint64_t)__atomic_load_n(word, __ATOMIC_ACQUIRE);
  return (uint32_t)(v >> 32) == (uint32_t)epoch ? (int64_t)(uint32_t)v : 0;
}

int64_t q_slot_done(const QueueSlot& S) {
  return q_tagged(&S.ctl_h->completed, S.epoch);
}

int64_t q_done(const tf_qexec* q) { return q_slot_done(q->slot()); }

// busy = published slices not all completed.  No clock: the completion
// count lives in host memory (the fetcher CTA writes it), so a read costs a
// cache hit, or one miss per device-side update — unlike cudaEventQuery there
// is nothing to throttle.
int q_busy(void* ctx, int32_t) {
  tf_qexec* q = static_cast<tf_qexec*>(ctx);
  // work published since the last look cannot be finished yet
  if (q->published != q->seen_published) {
    q->seen_published = q->published;
    return 1;
  }
  return q_done(q) < q->published;
}

void q_publish(tf_qexec* q, int64_t team) {
  tf_region* r = q->region;
  const Team* t = r->teams.get(team);
  if (!t) return;
  QueueSlot& S = q->slot();
  tf_nvtx::TeamRange range("team publish", (int64_t)t->tags.size());
  // entries carry the run's epoch: the fetcher reads them speculatively and
  // takes the tagged ones, so a team costs its stores and no shared counter
  // (a release store per team to a line the GPU polls was the cost of a
  // closure at small A)
  const int64_t tagged = (int64_t)((uint64_t)(uint32_t)S.epoch << 32);
  for (int64_t tag : t->tags)
    S.ring_h[q->published++] = tagged | (int64_t)(uint32_t)tag;
  r->teams.release(team);
}

// A timed-out run leaves unprocessed slices and claims the host cannot
// count: once the stream is idle, start the slot's counters afresh.
int q_reset_slot(QueueSlot& S) {
  cudaError_t e = cudaStreamSynchronize(S.stream);
  QueueDevInit init{};
  if (e == cudaSuccess)
    e = cudaMemcpy(S.qdev, &init, sizeof(init), cudaMemcpyHostToDevice);
  S.done_base = 0;
  S.ctl_h->status = 0;
  S.in_flight = false;
  return e != cudaSuccess ? (int)e : TF_E_TIMEOUT;
}

// The slot's previous run has completed every slice it published (host
// view: the fetcher's completion count), or reported a timeout.  Its host
// memory (ring, control block) is then free; its device-side stragglers
// (consumers seeing the queue closed) are ordered before the slot's next
// run by the stream (PDL chain) or by q_order_streams.
int q_drain_slot(QueueSlot& S) {
  if (!S.in_flight) return 0;
  for (uint64_t spins = 0;; ++spins) {
    if (__atomic_load_n(&S.ctl_h->status, __ATOMIC_ACQUIRE))
      return q_reset_slot(S);
    if (S.count == 0 ||
        q_slot_done(S) >= S.count)
      break;
    if ((spins & 1023) == 1023) {
      // a failed or finished stream that never reported every slice
      const cudaError_t e = cudaStreamQuery(S.stream);
      if (e == cudaSuccess &&
          q_slot_done(S) < S.count)
        return q_reset_slot(S);
      if (e != cudaSuccess && e != cudaErrorNotReady) return e;
    }
    __builtin_ia32_pause();
  }
  S.in_flight = false;
  return 0;
}

// Order a launch on `st` after a slot's last run on another stream.
int q_order_streams(QueueSlot& S, cudaStream_t st) {
  if (S.stream == nullptr || S.stream == st) return 0;
  cudaError_t e = cudaEventRecord(S.ev, S.stream);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(st, S.ev, 0);
  return e;
}

}  // namespace

extern "C" {

int tf_qexec_create(tf_region* region, int32_t n, tf_qexec** out) {
  if (!region || !out || region->executors != 1 || (n != 8 && n != 16))
    return TF_E_INVALID;
  tf_qexec* q = new tf_qexec();
  q->region = region;
  q->n = n;
  cudaError_t e = cudaSuccess;
  for (QueueSlot& S : q->slots) {
    if (e == cudaSuccess)
      e = cudaHostAlloc(&S.ctl_h, sizeof(QueueCtlHost), cudaHostAllocMapped);
    if (e == cudaSuccess) e = cudaHostGetDevicePointer(&S.ctl_hd, S.ctl_h, 0);
    if (e == cudaSuccess) e = cudaMalloc(&S.qdev, sizeof(QueueDevInit));
    if (e == cudaSuccess) {  // all zero: final_count's epoch tag 0 = open
      QueueDevInit init{};
      e = cudaMemcpy(S.qdev, &init, sizeof(init), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess)
      e = cudaEventCreateWithFlags(&S.ev, cudaEventDisableTiming);
  }
  if (e != cudaSuccess) {
    tf_qexec_destroy(q);
    return e;
  }
  *out = q;
  return 0;
}

int tf_qexec_set_flags(tf_qexec* q, int32_t flags) {
  if (!q || (flags & ~(TF_LAUNCH_OVERLAP_PREV | TF_QUEUE_SORTED)))
    return TF_E_INVALID;
  q->flags = flags;
  return 0;
}

void tf_qexec_destroy(tf_qexec* q) {
  if (!q) return;
  for (QueueSlot& S : q->slots)
    if (S.in_flight && S.stream) cudaStreamSynchronize(S.stream);
  for (QueueSlot& S : q->slots) {
    if (S.ctl_h) cudaFreeHost(S.ctl_h);
    if (S.ring_h) cudaFreeHost(S.ring_h);
    if (S.ring_d) cudaFree(S.ring_d);
    if (S.qdev) cudaFree(S.qdev);
    if (S.ev) cudaEventDestroy(S.ev);
  }
  delete q;
}

int tf_qexec_run_recon_flux(tf_qexec* q, const double* pool_ext,
                            int64_t pool_slices, const int32_t* ids,
                            int64_t count, double ax, double ay, double az,
                            double* um, double* up, double* F, double* amax,
                            int32_t flux_form, tf_stream_t stream,
                            int64_t* teams_published) {
  if (!q || !ids || count < 0 || !teams_published) return TF_E_INVALID;
  for (int64_t i = 0; i < count; ++i)
    if (ids[i] < 0 || ids[i] >= pool_slices) return TF_E_INVALID;
  // alternate queue slots: this run publishes while the previous run's
  // consumer may still drain its tail; the slot's own previous use (two
  // runs ago) must have completed its slices before its host ring and
  // control block are rewritten
  const int64_t t0 = q_now_ns();
  q->cur ^= 1;
  QueueSlot& S = q->slot();
  int drc = q_drain_slot(S);
  if (drc) return drc;
  const int64_t t1 = q_now_ns();
  cudaStream_t st = (cudaStream_t)stream;
  if (count > S.ring_cap || !S.ring_h) {
    // the device mirror is reallocated: nothing of the slot may be running
    if (S.stream) {
      cudaError_t e = cudaStreamSynchronize(S.stream);
      if (e != cudaSuccess) return e;
    }
    if (S.ring_h) cudaFreeHost(S.ring_h);
    if (S.ring_d) cudaFree(S.ring_d);
    S.ring_h = nullptr;
    S.ring_d = nullptr;
    const int64_t cap = count > 0 ? count : 1;
    cudaError_t e = cudaHostAlloc(&S.ring_h, sizeof(int64_t) * cap,
                                  cudaHostAllocMapped);
    // no host entry may carry a live epoch before it is published
    if (e == cudaSuccess) std::fill(S.ring_h, S.ring_h + cap, int64_t{0});
    if (e == cudaSuccess)
      e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.ring_hd),
                                   S.ring_h, 0);
    if (e == cudaSuccess)
      e = cudaMalloc(reinterpret_cast<void**>(&S.ring_d), sizeof(int64_t) * cap);
    // no stale entry may carry a live epoch (tag 0); the epoch itself keeps
    // counting — the slot's final_count still carries the last run's tag
    if (e == cudaSuccess) e = cudaMemset(S.ring_d, 0, sizeof(int64_t) * cap);
    if (e != cudaSuccess) return e;
    S.ring_cap = cap;
  }
  q->published = 0;
  q->seen_published = 0;
  S.ctl_h->published = 0;
  S.ctl_h->final_count = -1;
  S.ctl_h->completed = 0;
  S.ctl_h->status = 0;
  __atomic_thread_fence(__ATOMIC_SEQ_CST);
  // runs of this queue on another stream: this one goes after them (the
  // PDL chain orders runs on one stream)
  QueueSlot& other = q->slots[q->cur ^ 1];
  int orc = q_order_streams(S, st);
  if (!orc && other.in_flight) orc = q_order_streams(other, st);
  if (orc) return orc;
  const bool chain = S.stream == st && (!other.in_flight || other.stream == st);
  S.stream = st;
  int rc = tf_queue_consumer_launch(
      pool_ext, pool_slices, q->n, S.ring_hd, S.ctl_hd, S.ring_d, count,
      S.qdev, S.done_base, ++S.epoch, ax, ay, az, um,
      up, F, amax, flux_form,
      /*timeout_ns=*/2000000000LL,
      chain ? (TF_QUEUE_CHAIN | q->flags) : (q->flags & TF_QUEUE_SORTED),
      stream);
  if (rc) return rc;
  S.in_flight = true;
  const int64_t t2 = q_now_ns();
  tf_region* r = q->region;
  int64_t teams = 0;
  std::vector<int64_t> closed;
  auto drain = [&]() {
    closed.resize(r->live_watch[0]);
    const int k = tf_region_stream_idle(r, 0, closed.data(),
                                        (int32_t)closed.size());
    for (int i = 0; i < k; ++i, ++teams) q_publish(q, closed[i]);
  };
  for (int64_t i = 0; i < count; ++i) {
    if (r->live_watch[0] > 0 && !q_busy(q, 0)) drain();
    tf_enter_result res;
    rc = tf_region_enter(r, ids[i], q_busy, q, &res);
    if (rc) break;
    if (res.closed != FORMING) {
      q_publish(q, res.team);
      ++teams;
    }
  }
  drain();  // arrivals done: the queue drains, closing what is left
  // close the queue even on error so the consumer grid exits
  S.count = q->published;
  S.done_base += (uint64_t)q->published;
  __atomic_store_n(&S.ctl_h->final_count, (long long)q->published,
                   __ATOMIC_RELEASE);
  *teams_published = teams;
  const int64_t t3 = q_now_ns();
  q->runs += 1;
  q->ns_wait += t1 - t0;
  q->ns_launch += t2 - t1;
  q->ns_publish += t3 - t2;
  return rc;
}

int tf_qexec_host_times(const tf_qexec* q, int64_t* out4) {
  if (!q || !out4) return TF_E_INVALID;
  out4[0] = q->runs;
  out4[1] = q->ns_wait;
  out4[2] = q->ns_launch;
  out4[3] = q->ns_publish;
  return 0;
}

int64_t tf_qexec_completed(const tf_qexec* q) { return q ? q_done(q) : -1; }

int tf_qexec_wait(tf_qexec* q) {
  if (!q) return TF_E_INVALID;
  int rc = 0;
  for (QueueSlot& S : q->slots) {
    if (!S.in_flight) continue;
    cudaError_t e = cudaStreamSynchronize(S.stream);
    if (e != cudaSuccess) return e;
    if (__atomic_load_n(&S.ctl_h->status, __ATOMIC_ACQUIRE)) {
      rc = q_reset_slot(S);
      continue;
    }
    S.in_flight = false;
  }
  return rc;
}

}  // extern "C"

// ------------------------------------------------------- captured plans
// A formed team plan (the teams the formation core closed for one
// iteration's arrival sequence) captured once into a CUDA graph: one kernel
// node per team, each team on its parent's executor branch, so replaying an
// iteration costs one graph launch instead of one host launch per team.
struct tf_plan {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

namespace {

// Capture nteams team launches (launch(ids, T, flags, stream)) as a graph:
// fork to one branch per executor, teams in order on their branch (the first
// one after the fork is a full dependency, later ones may overlap their
// predecessor via PDL when flags ask for it), join.
template <typename Launch>
int capture_teams(const int32_t* ids, const int64_t* team_offsets,
                  const int32_t* team_executor, int64_t nteams,
                  int32_t executors, int32_t flags, Launch launch,
                  tf_plan** out) {
  if (!ids || !team_offsets || !team_executor || nteams < 0 || executors < 1 ||
      !out)
    return TF_E_INVALID;
  for (int64_t t = 0; t < nteams; ++t) {
    const int64_t sz = team_offsets[t + 1] - team_offsets[t];
    if (sz < 1 || sz > TF_MAX_TEAM || team_executor[t] < 0 ||
        team_executor[t] >= executors)
      return TF_E_INVALID;
  }
  std::vector<cudaStream_t> br(executors + 1);
  std::vector<cudaEvent_t> ev(executors + 1);
  int rc = 0;
  for (int i = 0; i <= executors && !rc; ++i) {
    rc = cudaStreamCreateWithFlags(&br[i], cudaStreamNonBlocking);
    if (!rc) rc = cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
  }
  tf_plan* plan = new tf_plan();
  cudaStream_t origin = br[executors];
  if (!rc) rc = cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal);
  if (!rc) {
    int crc = cudaEventRecord(ev[executors], origin);
    for (int e = 0; e < executors && !crc; ++e)
      crc = cudaStreamWaitEvent(br[e], ev[executors], 0);
    std::vector<char> started(executors, 0);
    for (int64_t t = 0; t < nteams && !crc; ++t) {
      const int64_t lo = team_offsets[t];
      const int T = (int)(team_offsets[t + 1] - lo);
      const int e = team_executor[t];
      const int f = (started[e] ? (flags & TF_LAUNCH_OVERLAP_PREV) : 0) |
                    (flags & (TF_STEP_HALO_YZ | TF_STEP_HALO_X));
      crc = launch(ids + lo, T, f, (tf_stream_t)br[e]);
      started[e] = 1;
      plan->kernels += 1;
    }
    for (int e = 0; e < executors && !crc; ++e) {
      crc = cudaEventRecord(ev[e], br[e]);
      if (!crc) crc = cudaStreamWaitEvent(origin, ev[e], 0);
    }
    int erc = cudaStreamEndCapture(origin, &plan->graph);
    rc = crc ? crc : erc;
  }
  if (!rc) rc = cudaGraphInstantiate(&plan->exec, plan->graph, 0);
  for (int i = 0; i <= executors; ++i) {
    if (br[i]) cudaStreamDestroy(br[i]);
    if (ev[i]) cudaEventDestroy(ev[i]);
  }
  if (rc) {
    if (plan->exec) cudaGraphExecDestroy(plan->exec);
    if (plan->graph) cudaGraphDestroy(plan->graph);
    delete plan;
    return rc;
  }
  *out = plan;
  return 0;
}

}  // namespace

extern "C" {

int tf_plan_capture_field_step(const int32_t* ids, const int64_t* team_offsets,
                               const int32_t* team_executor, int64_t nteams,
                               int32_t executors, const double* padded_in,
                               int32_t X, int32_t Gy, int32_t Gz, int32_t n,
                               double ax, double ay, double az, double dt_dx,
                               double* padded_out, int32_t flags,
                               tf_plan** out) {
  return capture_teams(
      ids, team_offsets, team_executor, nteams, executors, flags,
      [&](const int32_t* tid, int T, int f, tf_stream_t s) {
        return tf_field_step_f64(padded_in, X, Gy, Gz, n, nullptr, tid, T, ax,
                                 ay, az, dt_dx, padded_out, f, s);
      },
      out);
}

int tf_plan_capture_recon_flux(const int32_t* ids, const int64_t* team_offsets,
                               const int32_t* team_executor, int64_t nteams,
                               int32_t executors, const double* pool_ext,
                               int64_t pool_slices, int32_t n, double ax,
                               double ay, double az, double* um, double* up,
                               double* F, double* amax, int32_t flux_form,
                               int32_t flags, tf_plan** out) {
  const int64_t per = 3LL * (n + 2) * (n + 2) * (n + 2);
  const bool team_buffers = (flags & TF_PLAN_TEAM_BUFFERS) != 0;
  // TF_PLAN_REFGEO: the reference's launch geometry instead of one TMA CTA
  // per slice (the strategy-1 baseline)
  auto team_launch = (flags & TF_PLAN_REFGEO) ? tf_recon_flux_refgeo_f64
                                              : tf_recon_flux_team_ex_f64;
  return capture_teams(
      ids, team_offsets, team_executor, nteams, executors, flags,
      [&](const int32_t* tid, int T, int f, tf_stream_t s) {
        if (!team_buffers)
          return team_launch(pool_ext, pool_slices, tid, T, n, ax, ay, az, um,
                             up, F, 1, amax, flux_form, f, s);
        // the team's lease: slices [lo, lo+T) of the iteration's packed
        // team buffers (aggregator.py:121-128), slice s at lo + s
        const int64_t lo = tid - ids;
        return team_launch(pool_ext, pool_slices, tid, T, n, ax, ay, az,
                           um + lo * per, up + lo * per, F + lo * per, 0,
                           amax ? amax + lo : nullptr, flux_form, f, s);
      },
      out);
}

int tf_plan_launch(tf_plan* plan, tf_stream_t stream) {
  if (!plan || !plan->exec) return TF_E_INVALID;
  return cudaGraphLaunch(plan->exec, (cudaStream_t)stream);
}

int64_t tf_plan_kernels(const tf_plan* plan) { return plan ? plan->kernels : -1; }

void tf_plan_destroy(tf_plan* plan) {
  if (!plan) return;
  if (plan->exec) cudaGraphExecDestroy(plan->exec);
  if (plan->graph) cudaGraphDestroy(plan->graph);
  delete plan;
}

}  // extern "C"
