/*
 * taskfuse_b200.h — C ABI of the B200-native strategy-3 hydro hot path.
 *
 * Drop-in boundary for the per-sub-grid numerics and the aggregation
 * executor of the reference `taskfuse` package (arXiv 2210.06438 artifact,
 * /root/reference/pkg/src/taskfuse).  Every entry point is `extern "C"`,
 * takes plain pointers and sizes (no torch types), is stream-ordered and
 * returns an int: 0 on success, otherwise a cudaError_t value or one of the
 * TF_E* codes below.  Nothing throws across this boundary.
 *
 * Memory layout (all FP64, C order, z fastest — the reference layout):
 *   pool_ext : (pool_slices, E, E, E)      E = n + 6, ghost width 3
 *              == HydroState.u[block] stacked in lexicographic block order
 *              (reference scenario.py:52-96).
 *   um/up/F  : (slots, 3, C, C, C)         C = n + 2
 *              == make_scratch(n)["um"/"up"/"F"] stacked per slot
 *              (reference kernels.py:27-36).
 *   A "slot" is either the slice index inside the team (out_mode 0, the
 *   team-buffer layout of aggregator.py:121-128: slice s owns
 *   [s*len, (s+1)*len)) or the sub-grid id itself (out_mode 1: per-sub-grid
 *   scratch, HydroSim.scratch[block], step.py:53).
 *
 * Supported sub-grid edges: n = 8 and n = 16 (strategy 1).
 */
#ifndef TASKFUSE_B200_H
#define TASKFUSE_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* tf_stream_t; /* == cudaStream_t */

enum {
  TF_OK = 0,
  TF_E_INVALID = 1001,     /* bad argument (n, T, pointer, id range) */
  TF_E_NO_TMA = 1002,      /* cuTensorMapEncodeTiled unavailable */
  TF_E_ORDERING = 1003,    /* aggregation: replay diverged / misuse */
  TF_E_CAPACITY = 1004,    /* aggregation: out of slots */
  TF_E_TIMEOUT = 1005      /* a device queue / barrier gave up waiting */
};

#define TF_MAX_TEAM 128 /* aggregator.py:42 MAX_TEAM */

/* ---- numerics (reference hydro/kernels.py) ------------------------------ */

/* Fused reconstruct + flux over T aggregated slices.
 * Replaces reconstruct_body (kernels.py:73-81) followed by flux_body
 * (kernels.py:84-93), batched over a team as slice_launch would
 * (aggregator.py:143-166).  Slice s reads pool_ext[ids[s]] (ids == NULL:
 * identity).  ids is a DEVICE pointer.  flux_form 0 = reference upwind
 * (bit-exact), 1 = Kurganov-Tadmor central-upwind form (equal to upwind in
 * exact arithmetic for f = a u; checked at 1e-12 relative).
 * amax (may be NULL): per-slot max signal speed over all faces, the value
 * reduce_body stores (kernels.py:96-97).                                   */
int tf_recon_flux_f64(const double* pool_ext, int64_t pool_slices,
                      const int32_t* ids, int32_t T, int32_t n,
                      double ax, double ay, double az,
                      double* um, double* up, double* F, int32_t out_mode,
                      double* amax, int32_t flux_form, tf_stream_t stream);

/* Same, with the team's sub-grid ids given in HOST memory (T <= 128); they
 * travel inside the kernel parameters, so a team launch needs no copy.     */
int tf_recon_flux_team_f64(const double* pool_ext, int64_t pool_slices,
                           const int32_t* host_ids, int32_t T, int32_t n,
                           double ax, double ay, double az,
                           double* um, double* up, double* F,
                           int32_t out_mode, double* amax, int32_t flux_form,
                           tf_stream_t stream);

/* Launch flags for tf_recon_flux_team_ex_f64.
 * TF_LAUNCH_OVERLAP_PREV: programmatic dependent launch — the team kernel may
 * start while the previous kernel on the stream still runs.  Only valid when
 * that kernel does not produce this team's inputs (e.g. it is another team
 * of the same region); the executor and the captured plans use it between
 * consecutive teams of one executor stream.                                */
#define TF_LAUNCH_OVERLAP_PREV 1
int tf_recon_flux_team_ex_f64(const double* pool_ext, int64_t pool_slices,
                              const int32_t* host_ids, int32_t T, int32_t n,
                              double ax, double ay, double az,
                              double* um, double* up, double* F,
                              int32_t out_mode, double* amax,
                              int32_t flux_form, int32_t flags,
                              tf_stream_t stream);

/* The same team launch with the REFERENCE's launch geometry (blocks_for,
 * kernels.py:39-55): ceil((n+2)^3/128) blocks of 128 threads per slice
 * (46 at n = 16), one cell per thread, stencil read from global memory.
 * The strategy-1 baseline kernel (a 16^3 sub-grid spread over 46 CTAs).   */
int tf_recon_flux_refgeo_f64(const double* pool_ext, int64_t pool_slices,
                             const int32_t* host_ids, int32_t T, int32_t n,
                             double ax, double ay, double az,
                             double* um, double* up, double* F,
                             int32_t out_mode, double* amax,
                             int32_t flux_form, int32_t flags,
                             tf_stream_t stream);

/* PPM variant (north_star's "batched PPM reconstruction"; Colella-Woodward
 * 1984 with CW84 limiting) of tf_recon_flux_f64, same arguments and layout.
 * The reference has no PPM (its scheme is minmod): parity is
 * against oracle/ppm_oracle.py and is UNPINNED.                            */
int tf_recon_flux_ppm_f64(const double* pool_ext, int64_t pool_slices,
                          const int32_t* ids, int32_t T, int32_t n,
                          double ax, double ay, double az,
                          double* um, double* up, double* F, int32_t out_mode,
                          double* amax, int32_t flux_form,
                          tf_stream_t stream);

/* reconstruct_body alone (kernels.py:73-81): w = pool_ext[ids[s]].          */
int tf_reconstruct_f64(const double* pool_ext, int64_t pool_slices,
                       const int32_t* ids, int32_t T, int32_t n,
                       double* um, double* up, int32_t out_mode,
                       tf_stream_t stream);

/* flux_body alone (kernels.py:84-93): reads up (a>=0) / um (a<0) of the
 * slot, writes F of the slot.                                              */
int tf_flux_f64(const int32_t* ids, int32_t T, int32_t n,
                double ax, double ay, double az,
                const double* um, const double* up, double* F,
                int32_t out_mode, tf_stream_t stream);

/* update_body (kernels.py:100-111), no FMA contraction: writes the owned
 * region of next_ext[ids[s]] = u_ext - dt_dx * div(F of the slot).         */
int tf_update_f64(const double* pool_ext, const int32_t* ids, int32_t T,
                  int32_t n, const double* F, int32_t out_mode, double dt_dx,
                  double* next_ext, tf_stream_t stream);

/* exchange_ghosts (scenario.py:124-142) for T sub-grids of a periodic
 * per_axis^3 lattice (ids NULL: all per_axis^3 sub-grids).                 */
int tf_ghost_fill_f64(double* pool_ext, const int32_t* ids, int32_t T,
                      int32_t n, int32_t per_axis, tf_stream_t stream);

/* make_state / assemble (scenario.py:83-106) on the device: the global
 * (grid_n^3) field <-> the owned cells of the pool (ghosts untouched).      */
int tf_field_to_pool_f64(const double* field, int32_t grid_n, int32_t n,
                         double* pool_ext, tf_stream_t stream);
int tf_pool_to_field_f64(const double* pool_ext, int32_t grid_n, int32_t n,
                         double* field, tf_stream_t stream);
/* make_state for the sub-grid layers [layer0, layer0+layers) along x only
 * (one chunk of a pipelined host upload).                                  */
int tf_field_to_pool_layers_f64(const double* field, int32_t grid_n,
                                int32_t n, int32_t layer0, int32_t layers,
                                double* pool_ext, tf_stream_t stream);

/* prep_body (kernels.py:69-70): w[slot] = pool_ext[ids[s]].                */
int tf_prep_f64(const double* pool_ext, const int32_t* ids, int32_t T,
                int32_t n, double* w, int32_t out_mode, tf_stream_t stream);

/* reduce_body (kernels.py:96-97): reduce_out[slot] = max(|ax|,|ay|,|az|).  */
int tf_reduce_f64(const int32_t* ids, int32_t T, double ax, double ay,
                  double az, double* reduce_out, int32_t out_mode,
                  tf_stream_t stream);

/* ---- aggregation formation core (reference aggregator.py:247-345) ------- */

typedef struct tf_region tf_region;

typedef struct {
  int32_t parent;      /* parents[arrivals % P]                  (:298)   */
  int32_t executor;    /* executor index the parent is pinned to (:273)   */
  int64_t team;        /* region-local team sequence number              */
  int32_t slice_id;    /* arrival order inside the team          (:303)   */
  int32_t closed;      /* 0 forming, 1 cap, 2 solo fast path, 3 drain     */
  int32_t queried;     /* 1 iff stream_busy was consulted (:316)          */
} tf_enter_result;

/* stream_busy hook (device.py:187-194): return nonzero iff busy.           */
typedef int (*tf_busy_fn)(void* ctx, int32_t executor);

/* AggregationRegion.__init__ (aggregator.py:250-282).                      */
int tf_region_create(const char* name, int32_t max_team,
                     int32_t parent_count, int32_t executors,
                     tf_region** out);
void tf_region_destroy(tf_region* r);
/* executor index of parent i: (crc32(name) % E + i) % E  (:273-277)        */
int32_t tf_region_parent_executor(const tf_region* r, int32_t parent);
/* AggregationRegion.enter (aggregator.py:284-326) minus the task guard.    */
int tf_region_enter(tf_region* r, int64_t tag, tf_busy_fn busy, void* ctx,
                    tf_enter_result* out);
/* Stream drained (device.py:364-370 -> aggregator.py:328-332): closes the
 * forming teams whose parent sits on `executor`, in watch order, at most
 * `cap` of them (their ids written to out_teams); teams beyond cap stay
 * forming and watching, so nothing is closed unreported.  Returns the count
 * (or <0 error).  Size out_teams with tf_region_watch_count.               */
int tf_region_stream_idle(tf_region* r, int32_t executor, int64_t* out_teams,
                          int32_t cap);
/* Number of teams watching `executor`'s stream (an upper bound on what the
 * next tf_region_stream_idle closes).                                      */
int32_t tf_region_watch_count(const tf_region* r, int32_t executor);
/* Team bookkeeping.  release frees a closed team's record. */
int tf_region_release_team(tf_region* r, int64_t team);
int tf_region_team_size(const tf_region* r, int64_t team);
int tf_region_team_members(const tf_region* r, int64_t team, int64_t* tags,
                           int32_t cap);
int tf_region_team_parent(const tf_region* r, int64_t team);
/* RegionStats (aggregator.py:237-244): counters + histogram[1..128].      */
int tf_region_stats(const tf_region* r, int64_t* teams_formed,
                    int64_t* solo_fast_path, int64_t* histogram129);

/* ---- member bookkeeping of a closed team --------------------------------
 * TeamMember._issue / leave / _chain / _maybe_release (aggregator.py:
 * 168-234): the SPMD op-sequence check, lease ownership per step, and the
 * release rule (every member left and no op in flight).  `sig` is the
 * step's signature as the reference formats it (aggregator.py:_fmt_sig,
 * e.g. "alloc:device:<f8:2744", "copy:h2d:21952", "launch:flux:24:1").
 * A mismatch returns TF_E_ORDERING and records "expected\ngot" for
 * tf_region_error (OrderingViolationError(region, cursor, expected, got)).
 * *release == 1 exactly once per team: the caller returns the leases
 * (tf_team_leases) and frees the team with tf_region_release_team.        */
int tf_team_issue(tf_region* r, int64_t team, int32_t cursor, const char* sig,
                  int32_t* step, int32_t* arrivals);
int tf_team_leave(tf_region* r, int64_t team, int32_t cursor,
                  int32_t* release);
int tf_team_op_begin(tf_region* r, int64_t team);
int tf_team_op_end(tf_region* r, int64_t team, int32_t* release);
int tf_team_set_lease(tf_region* r, int64_t team, int32_t step,
                      int64_t lease);
int64_t tf_team_lease(const tf_region* r, int64_t team, int32_t step);
/* leases of the team's steps in step order; returns the count             */
int tf_team_leases(const tf_region* r, int64_t team, int64_t* out,
                   int32_t cap);
int tf_team_step_info(const tf_region* r, int64_t team, int32_t step,
                      int32_t* arrivals, char* sig, int32_t sig_cap);
int64_t tf_region_violations(const tf_region* r);
const char* tf_region_error(const tf_region* r);

/* ---- native HydroSim engine ----------------------------------------------
 * HydroSim.task_iteration (hydro/step.py:83-123) for every sub-grid of a
 * per_axis^3 lattice, driven by driver()'s per-iteration loop
 * (step.py:126-143): five regions in KERNEL_ORDER (prep, reconstruct,
 * flux, reduce, update; parents = max(1, S / max_team), step.py:61), each
 * visit enter -> slice_alloc x4 (pinned/device ext^3 and n^3 staging
 * leases from an exact-size recycling pool) -> h2d copy -> ONE batched
 * kernel per team -> d2h copy -> await -> leave, under the tf_region /
 * tf_team rules, tasks FIFO, streams polled only when no task is runnable
 * (the Python scheduler's order).  `streams` = the executor pool's CUDA
 * streams (NULL: the engine creates them).  w (S,E,E,E), um/up/F
 * (S,3,C,C,C), reduce_out (S): per-sub-grid scratch (HydroSim.scratch).    */
typedef struct tf_hydro tf_hydro;
int tf_hydro_create(int32_t n, int32_t per_axis, int32_t max_team,
                    int32_t executors, const tf_stream_t* streams, double ax,
                    double ay, double az, double dt_dx, double* w, double* um,
                    double* up, double* F, double* reduce_out,
                    tf_hydro** out);
void tf_hydro_destroy(tf_hydro* h);
/* bench.py:142-153 _presize_pools: lease every (kind, len x team size)
 * bucket the run can touch, so the steady state never raw-allocates.       */
int tf_hydro_presize(tf_hydro* h);
/* One iteration: every sub-grid's task through the five regions; u_pool is
 * read (ghosts already exchanged), u_next_pool's owned cells written.
 * Returns when every task has left its last region; `stream` is ordered
 * before (fork) and after (join) the executor streams' work.               */
int tf_hydro_iteration(tf_hydro* h, const double* u_pool, double* u_next_pool,
                       tf_stream_t stream);
/* the engine's region k (KERNEL_ORDER index), for tf_region_stats         */
int tf_hydro_region(const tf_hydro* h, int32_t k, tf_region** out);
/* kernels, copies, bytes copied, raw device allocs, raw pinned allocs
 * (bucket misses, the reference's count), outstanding leases, storage
 * allocation calls past the reserved staging arenas (cudaMalloc /
 * cudaHostAlloc), device polls                                             */
int tf_hydro_counters(const tf_hydro* h, int64_t* out8);
/* host nanoseconds spent issuing device ops, polling without progress, and
 * in tf_hydro_iteration altogether (cumulative)                           */
int tf_hydro_host_times(const tf_hydro* h, int64_t* out3);

/* ---- real-time bulk executor (strategy 3 on real CUDA streams) ---------- */

typedef struct tf_executor tf_executor;

/* An executor pool of `count` streams (executorpool.py:42-60) bound to one
 * region; the region's parents round-robin over them.                      */
int tf_executor_create(tf_region* region, int32_t count, tf_executor** out);
void tf_executor_destroy(tf_executor* ex);
tf_stream_t tf_executor_stream(const tf_executor* ex, int32_t executor);

/* Submit `count` recon+flux task arrivals (sub-grid ids, host memory) in
 * order.  Team formation runs in real time: a parent's stream is busy iff
 * its last recorded CUDA event has not completed (cudaEventQuery); a
 * closed team is one tf_recon_flux_team_f64 launch on its parent's stream.
 * Remaining forming teams are flushed at the end.  Returns launches issued
 * in *launches.  Completion: tf_executor_sync or events on the streams.    */
int tf_executor_run_recon_flux(tf_executor* ex, const double* pool_ext,
                               int64_t pool_slices, const int32_t* ids,
                               int64_t count, int32_t n, double ax, double ay,
                               double az, double* um, double* up, double* F,
                               double* amax, int32_t flux_form,
                               int64_t* launches);
/* Every executor stream waits for the work issued so far on `stream` (call
 * before run when the pool was produced on `stream`).                      */
int tf_executor_fork(tf_executor* ex, tf_stream_t stream);
/* TF_LAUNCH_OVERLAP_PREV: consecutive teams on one executor stream overlap
 * (programmatic dependent launch).                                         */
int tf_executor_set_flags(tf_executor* ex, int32_t flags);
/* Make `stream` wait for all work issued so far on every executor stream.  */
int tf_executor_join(tf_executor* ex, tf_stream_t stream);
int tf_executor_sync(tf_executor* ex);

/* ---- device-queue executor (strategy 3 without per-team launches) ------- */
/* A resident consumer grid drains sub-grid ids that the formation core
 * publishes, one closed team at a time, into a ring in mapped pinned host
 * memory; busy = published slices not yet completed.  The region must have
 * exactly one executor (the queue).  run() returns once every arrival has
 * been published; the consumer runs on `stream` and completes there.
 * Consecutive runs on one stream overlap: run k+1's grid is a programmatic
 * dependent of run k's — its CTAs take the SM slots run k's tail frees,
 * mirror and claim their first slices, and (TF_LAUNCH_OVERLAP_PREV, see
 * tf_qexec_set_flags) load their stencil boxes; every output store waits
 * for run k.  tf_queue_consumer_* are the device side (used by tf_qexec_*).*/
typedef struct tf_qexec tf_qexec;
int tf_qexec_create(tf_region* region, int32_t n, tf_qexec** out);
void tf_qexec_destroy(tf_qexec* q);
/* flags: TF_QUEUE_SORTED (below); TF_LAUNCH_OVERLAP_PREV: a run's first
 * stencil boxes may load while the previous kernel on the stream still runs.  Only valid when that kernel
 * does not produce the run's pool (e.g. it is the previous run, or a team
 * kernel).  Default 0: boxes load after the previous kernel completes.     */
int tf_qexec_set_flags(tf_qexec* q, int32_t flags);
int tf_qexec_run_recon_flux(tf_qexec* q, const double* pool_ext,
                            int64_t pool_slices, const int32_t* ids,
                            int64_t count, double ax, double ay, double az,
                            double* um, double* up, double* F, double* amax,
                            int32_t flux_form, tf_stream_t stream,
                            int64_t* teams_published);
/* slices the consumer has completed so far (host view)                     */
int64_t tf_qexec_completed(const tf_qexec* q);
/* host time summed over runs: {runs, ns waiting for a queue slot's previous
 * run, ns in the launch, ns in the formation + publish loop}               */
int tf_qexec_host_times(const tf_qexec* q, int64_t* out4);
/* Wait for every run in flight; TF_E_TIMEOUT if a consumer grid gave up
 * (its timeout expired with slices unprocessed).  A run reusing a queue
 * slot reports a timeout of that slot's previous run the same way.        */
int tf_qexec_wait(tf_qexec* q);
/* ring_h/ctl_h: mapped pinned host ring of tagged entries (epoch << 32 | id;
 * an entry is published once its tag is this launch's epoch) + control
 * block {published (unused), final_count (host: the count once closed, -1
 * before), completed ((epoch << 32) | slices done, posted by the fetcher
 * CTA), status (1: timed out)}; ring_d:
 * device mirror of the tagged entries, ring_cap of them (the most this
 * launch may publish),
 * zeroed once at allocation; epoch >= 1, new for every launch on that ring; the grid is
 * one fetcher CTA + one CTA per entry (CTA k computes entry k); qdev: {published,
 * final_count, spare, done}, one 128-B line each, zeroed once at allocation
 * and never reset: done is monotonic over the launches on one qdev,
 * done_base = the slices of the earlier launches; final_count is tagged
 * (epoch << 32 | count).
 * flags: TF_QUEUE_CHAIN = launch as a programmatic dependent of the previous
 * kernel on the stream (its first boxes load after that kernel completes),
 * | TF_LAUNCH_OVERLAP_PREV = load them before (see tf_qexec_set_flags).    */
#define TF_QUEUE_CHAIN 2
/* TF_QUEUE_SORTED (tf_queue_consumer_launch, tf_qexec_set_flags): each
 * batch of entries the fetcher mirrors goes to the device ring in sub-grid
 * id order (a counting sort over 1024 id buckets), so consecutive consumer
 * CTAs work on neighbouring sub-grids whatever the teams' member order.    */
#define TF_QUEUE_SORTED 4
int tf_queue_consumer_launch(const double* pool_ext, int64_t pool_slices,
                             int32_t n, const int64_t* ring_h, void* ctl_h,
                             int64_t* ring_d, int64_t ring_cap, void* qdev,
                             uint64_t done_base, int32_t epoch, double ax,
                             double ay, double az, double* um, double* up,
                             double* F, double* amax, int32_t flux_form,
                             int64_t timeout_ns, int32_t flags,
                             tf_stream_t stream);

/* ---- device-launch executor (strategy 3, teams launched by the GPU) ----- */
/* The formation core's closed teams are published (ids + end offset) into
 * mapped pinned memory; a one-CTA launcher kernel, resident for the run,
 * mirrors them to device memory and launches EACH TEAM as its own grid of
 * T CTAs from the device (dynamic parallelism, fire-and-forget) — the
 * reference's one aggregated kernel per team (aggregator.py:157-165)
 * without a host launch.  busy = published slices not all completed.
 * The region must have one executor; n = 8.  run() returns once every
 * arrival is published; the work completes on `stream`.                   */
typedef struct tf_dlexec tf_dlexec;
int tf_dlexec_create(tf_region* region, int32_t n, tf_dlexec** out);
void tf_dlexec_destroy(tf_dlexec* q);
int tf_dlexec_run_recon_flux(tf_dlexec* q, const double* pool_ext,
                             int64_t pool_slices, const int32_t* ids,
                             int64_t count, double ax, double ay, double az,
                             double* um, double* up, double* F, double* amax,
                             int32_t flux_form, tf_stream_t stream,
                             int64_t* teams_published);
/* Wait for every run in flight; TF_E_TIMEOUT if a launcher gave up.       */
int tf_dlexec_wait(tf_dlexec* q);

/* ---- captured team plans (CUDA graphs) ----------------------------------- */

typedef struct tf_plan tf_plan;

/* Capture one iteration's formed teams (flat ids, team_offsets[nteams+1],
 * executor per team) as a CUDA graph: one tf_recon_flux_team_f64 node per
 * team on its executor's branch.  Outputs per sub-grid id (out_mode 1), or
 * with TF_PLAN_TEAM_BUFFERS in flags into the iteration's packed team
 * buffers: team t's slice s at flat index team_offsets[t] + s — the
 * reference's slice_alloc lease layout (aggregator.py:121-128).            */
#define TF_PLAN_TEAM_BUFFERS 2
/* TF_PLAN_REFGEO: capture tf_recon_flux_refgeo_f64 team launches (the
 * reference's launch geometry) instead of the TMA kernel.                  */
#define TF_PLAN_REFGEO 16
int tf_plan_capture_recon_flux(const int32_t* ids, const int64_t* team_offsets,
                               const int32_t* team_executor, int64_t nteams,
                               int32_t executors, const double* pool_ext,
                               int64_t pool_slices, int32_t n, double ax,
                               double ay, double az, double* um, double* up,
                               double* F, double* amax, int32_t flux_form,
                               int32_t flags, tf_plan** out);
/* Same for the fused full step on a padded field (tf_field_step_f64).      */
int tf_plan_capture_field_step(const int32_t* ids, const int64_t* team_offsets,
                               const int32_t* team_executor, int64_t nteams,
                               int32_t executors, const double* padded_in,
                               int32_t X, int32_t Gy, int32_t Gz, int32_t n,
                               double ax, double ay, double az, double dt_dx,
                               double* padded_out, int32_t flags,
                               tf_plan** out);
int tf_plan_launch(tf_plan* plan, tf_stream_t stream);
int64_t tf_plan_kernels(const tf_plan* plan);
void tf_plan_destroy(tf_plan* plan);

/* ---- multi-GPU slab halo (exchange_ghosts across a partition) ----------- */
/* The local pool holds an x-slab of mx sub-grid layers of an m^3 periodic
 * lattice: (mx*m*m, E, E, E), local id = (bx*m + by)*m + bz.  Planes are
 * (3, m*n, m*n) FP64.  pack: lo = the slab's first 3 owned x layers, hi =
 * its last 3.  fill: every ghost cell from the local pool or, in x beyond
 * the slab, from halo_lo (the left neighbour's hi) / halo_hi (the right
 * neighbour's lo).  One rank: halo_lo = own hi, halo_hi = own lo gives
 * exactly exchange_ghosts (scenario.py:124-142).  fill covers local ids
 * [first, first+count) so interior sub-grids can be filled (and computed)
 * while the halo planes are still in flight.                               */
int tf_halo_pack_f64(const double* pool_ext, int32_t n, int32_t mx, int32_t m,
                     double* lo_plane, double* hi_plane, tf_stream_t stream);
int tf_ghost_fill_slab_f64(double* pool_ext, int32_t n, int32_t mx, int32_t m,
                           const double* halo_lo, const double* halo_hi,
                           int32_t first, int32_t count, tf_stream_t stream);

/* ---- fused full iteration on a padded global field (SURVEY §8 f #2) ----- */
/* Padded field P: (X+4, Gy+4, Gz+8) FP64, owned global cell (x,y,z) at
 * P[x+2][y+2][z+4] (X = the slab's x extent; Gy = Gz = grid_n).
 * tf_field_step_f64: for T sub-grids (device ids, or host_ids <= 128 in the
 * launch parameters, or ids == host_ids == NULL: the first T in lexicographic
 * (bx,by,bz) order of the (X/n, Gy/n, Gz/n) lattice), one fused
 * reconstruct+flux+update per sub-grid (kernels.py:73-111, bit-identical):
 * reads the stencil box from padded_in, writes the owned cells of
 * padded_out.  Halo of padded_in must be current.
 * flags: TF_LAUNCH_OVERLAP_PREV as above; n = 8 only, TF_STEP_HALO_YZ /
 * TF_STEP_HALO_X: the step also writes the periodic y/z / x halo layers of
 * padded_out that copy its sub-grids' owned cells (the halo kernel is then
 * unnecessary after a step over every sub-grid; halo edges and corners,
 * which the 6-point stencil never reads, are left as they were).
 * tf_field_halo_f64: periodic y/z halo of every layer; periodic_x != 0 also
 * fills the x halo periodically (one GPU; multi-GPU receives it instead).
 * tf_field_pad_f64 / tf_field_unpad_f64: (X, Gy, Gz) field <-> interior.    */
#define TF_STEP_HALO_YZ 4
#define TF_STEP_HALO_X 8
int tf_field_step_f64(const double* padded_in, int32_t X, int32_t Gy,
                      int32_t Gz, int32_t n, const int32_t* ids,
                      const int32_t* host_ids, int32_t T, double ax, double ay,
                      double az, double dt_dx, double* padded_out,
                      int32_t flags, tf_stream_t stream);
int tf_field_halo_f64(double* padded, int32_t X, int32_t Gy, int32_t Gz,
                      int32_t periodic_x, tf_stream_t stream);
/* Multi-GPU fused step + exchange: as tf_field_step_f64 (device ids), and
 * the slab's 2 lowest / highest owned x layers are ALSO stored into the
 * ring neighbours' next padded fields (peer_lo = left's, peer_hi = right's,
 * NVLink peer pointers from CUDA IPC) at their high / low x halo.  Then
 * tf_peer_barrier publishes `epoch` to both neighbours' flag words
 * (release, system scope) and waits for theirs (acquire); *err = 1 instead
 * of hanging if a neighbour does not arrive within timeout_ns.            */
int tf_field_step_peer_f64(const double* padded_in, int32_t X, int32_t Gy,
                           int32_t Gz, int32_t n, const int32_t* ids,
                           int32_t T, double ax, double ay, double az,
                           double dt_dx, double* padded_out, double* peer_lo,
                           double* peer_hi, tf_stream_t stream);
/* The fused iteration over the WHOLE slab in one launch (every sub-grid of
 * the (X/n, Gy/n, Gz/n) lattice; what tf_field_step_f64 / _peer_f64 do with
 * ids == NULL and T = S), tiled by warp columns instead of sub-grids: a
 * warp marches R (8, or 4 with TF_MARCH_ROWS4) y rows x 32 z cells through
 * xc x planes (0 = 16, or 8 when 16 would leave <= 8192 work items) of the
 * field, one TMA plane box at a time (csrc/field_march.cu).  Same arithmetic, bit-identical.  Needs
 * Gy % R == 0 and Gz % 32 == 0.  flags: TF_STEP_HALO_YZ (also write the
 * next field's periodic y/z halos), TF_STEP_HALO_X (also its periodic x
 * halo: one GPU; peer_lo/peer_hi must then be NULL), TF_MARCH_ROWS4.
 * peer_lo / peer_hi: as tf_field_step_peer_f64 (the ring neighbours' next
 * fields, or NULL).  work: two zeroed uint32 counters private to this
 * launch's stream order (the kernel claims work items from them and leaves
 * them zeroed), or NULL for a static round-robin split.  Replaces the
 * per-sub-grid loop of advect_once / HydroSim's iteration over a whole
 * rank (reference.py:28-52, step.py:125-143) plus exchange_ghosts
 * (scenario.py:124-142) for the x halos.
 * TF_MARCH_PDL_EDGE: launch as a programmatic dependent of the previous
 * kernel on the stream (a peer barrier launched with TF_BARRIER_PDL): the
 * items that read or store x-halo planes wait for it (griddepcontrol.wait),
 * every other item runs at once — the multi-GPU iteration overlaps the
 * ring synchronisation with its interior.
 * TF_MARCH_ALONG_Y: the warps march along y with R x rows per column (the
 * roles of x and y swapped; needs X % R == 0, TF_STEP_HALO_YZ and both x
 * halo destinations): a thin x slab (a rank's share at N >= 4) keeps long
 * columns instead of many short chunks.  Bit-identical (the update's
 * (dFx + dFy) sum is commutative).                                         */
#define TF_MARCH_ROWS4 16
#define TF_MARCH_PDL_EDGE 32
#define TF_MARCH_ALONG_Y 64
int tf_field_march_f64(const double* padded_in, int32_t X, int32_t Gy,
                       int32_t Gz, double ax, double ay, double az,
                       double dt_dx, double* padded_out, double* peer_lo,
                       double* peer_hi, int32_t flags, int32_t xc,
                       uint32_t* work, tf_stream_t stream);
int tf_peer_barrier(long long* my_flags, long long* left_flags,
                    long long* right_flags, long long epoch,
                    long long timeout_ns, int* err, tf_stream_t stream);
/* tf_peer_barrier with flags: TF_BARRIER_PDL = launched as a programmatic
 * dependent of the previous kernel (it publishes the epoch after that
 * kernel completes) and letting the NEXT kernel launch at once (a march
 * with TF_MARCH_PDL_EDGE, whose x-edge items wait for this barrier).       */
#define TF_BARRIER_PDL 1
int tf_peer_barrier_ex(long long* my_flags, long long* left_flags,
                       long long* right_flags, long long epoch,
                       long long timeout_ns, int* err, int32_t flags,
                       tf_stream_t stream);
/* y/z halos of padded layers [first, first+count) only; the periodic x halo
 * (side 1: low halo <- last owned layers, 2: high <- first, 3: both).
 * Used by the chunked host pipeline (FieldIteration.run_host_pipelined).    */
int tf_field_halo_layers_f64(double* padded, int32_t X, int32_t Gy,
                             int32_t Gz, int32_t first, int32_t count,
                             tf_stream_t stream);
int tf_field_halo_xwrap_f64(double* padded, int32_t X, int32_t Gy, int32_t Gz,
                            int32_t side, tf_stream_t stream);
int tf_field_pad_f64(const double* field, int32_t X, int32_t Gy, int32_t Gz,
                     double* padded, tf_stream_t stream);
int tf_field_unpad_f64(const double* padded, int32_t X, int32_t Gy,
                       int32_t Gz, double* field, tf_stream_t stream);
/* Padded layers [first, first+count) (x in padded coordinates, the x halo
 * included) written in full — interior AND periodic y/z halos — straight
 * from a dense (X, Gy, Gz) field: padded (px, py, pz) = field((px-2) mod X,
 * (py-2) mod Gy, (pz-4) mod Gz).  One launch in place of pad + y/z halo +
 * x wrap for a chunk of the host pipeline (scenario.py:124-142 periodic
 * ghosts).  Gy, Gz even.                                                    */
int tf_field_pad_halo_f64(const double* field, int32_t X, int32_t Gy,
                          int32_t Gz, double* padded, int32_t first,
                          int32_t count, tf_stream_t stream);
/* Zero-copy download of the interior into a PINNED host field (cudaHostAlloc /
 * torch pin_memory; TF_E_INVALID otherwise): the kernel's own posted PCIe
 * writes, `ctas` CTAs of 256 threads, Gz even, host_field 16-B aligned.
 * Used by the host pipeline so the copy engines serve only the upload.      */
int tf_field_unpad_host_f64(const double* padded, int32_t X, int32_t Gy,
                            int32_t Gz, double* host_field, int32_t ctas,
                            tf_stream_t stream);

/* ---- device seam ---------------------------------------------------------*/
/* enqueue_copy (reference device.py:237-252) as a real copy: `bytes` from
 * src to dst in stream order; pinned host and device pointers in any
 * combination (cudaMemcpyDefault).                                          */
int tf_memcpy_async(void* dst, const void* src, int64_t bytes,
                    tf_stream_t stream);

/* ---- misc ----------------------------------------------------------------*/
const char* tf_version(void);
/* sm_100a device check: 0 iff device `dev` is compute capability 10.0.    */
int tf_check_device(int32_t dev);

#ifdef __cplusplus
}
#endif
#endif /* TASKFUSE_B200_H */
