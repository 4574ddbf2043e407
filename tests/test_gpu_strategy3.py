"""Strategy-3 bulk paths on the GPU: the formed team plan (CUDA graph) and
the real-time executor must give results independent of team composition —
bit-identical to the oracle (test_hydro.py:195-199 'profile choice does not
change results') — and every arrival must land in exactly one team."""

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cfg2(cuda):
    import torch
    n, grid = 8, 128
    f = HO.sod_field(grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    vel = (1.0, 1.0, 1.0)
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    pool = torch.from_numpy(hp).to(cuda)
    return pool, n, vel, oum, oup, oF


def _outs(S, n, dev):
    import torch
    c = n + 2
    return [torch.full((S, 3, c, c, c), float("nan"), dtype=torch.float64,
                       device=dev) for _ in range(3)]


def test_form_teams_partitions_arrivals():
    from paper_2210_06438_b200.strategy3 import form_teams
    for A in (1, 4, 16, 64, 128):
        teams = form_teams(range(4096), A, executors=8)
        ids = sorted(i for t in teams for i in t.ids)
        assert ids == list(range(4096))
        assert all(1 <= len(t.ids) <= A for t in teams)
        # saturated device: every team closes at the cap, strided members
        assert all(len(t.ids) == A for t in teams)
        P = max(1, 4096 // A)
        assert all(np.all(np.diff(t.ids) == P) for t in teams if len(t.ids) > 1)


@pytest.mark.parametrize("A,E", [(1, 4), (16, 8), (128, 8), (128, 1)])
def test_team_plan_bit_exact(cuda, cfg2, A, E):
    import torch
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    um, up, F = _outs(S, n, cuda)
    amax = torch.full((S,), float("nan"), dtype=torch.float64, device=cuda)
    plan = TeamPlan(form_teams(range(S), A, E), pool, n, vel, um, up, F, E,
                    amax=amax)
    plan.launch()
    plan.launch()   # replay is idempotent
    torch.cuda.synchronize()
    assert plan.kernels == S // A
    assert np.array_equal(F.cpu().numpy(), oF)
    assert np.array_equal(um.cpu().numpy(), oum)
    assert np.array_equal(up.cpu().numpy(), oup)
    assert bool((amax == 1.0).all())


@pytest.mark.parametrize("n,grid,vel", [(8, 32, (-1.0, 0.5, -0.25)),
                                        (16, 64, (0.7, -1.3, 0.0)),
                                        (16, 32, (1.0, 1.0, 1.0))])
@pytest.mark.parametrize("form", [0, 1])
def test_reference_geometry_plan_bit_exact(cuda, n, grid, vel, form):
    """The strategy-1 baseline kernel (the reference's launch geometry:
    ceil((n+2)^3/128) CTAs of 128 threads per slice, stencil from global
    memory) is as exact as the TMA kernel, upwind and KT forms."""
    import torch
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    f = HO.stress_field(grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    if form:
        oF = HO.flux_kt_batch(oum, oup, vel)
    pool = torch.from_numpy(hp).to(cuda)
    S = pool.shape[0]
    um, up, F = _outs(S, n, cuda)
    amax = torch.full((S,), float("nan"), dtype=torch.float64, device=cuda)
    plan = TeamPlan(form_teams(range(S), 1, 2), pool, n, vel, um, up, F, 2,
                    amax=amax, flux_form=form, geometry="reference")
    plan.launch()
    torch.cuda.synchronize()
    assert np.array_equal(um.cpu().numpy(), oum)
    assert np.array_equal(up.cpu().numpy(), oup)
    assert np.array_equal(F.cpu().numpy(), oF)
    assert bool((amax == max(abs(v) for v in vel)).all())


@pytest.mark.parametrize("A,E", [(16, 4), (128, 4)])
def test_team_plan_team_buffers(cuda, cfg2, A, E):
    """Outputs into the packed team leases: flat slot k holds sub-grid
    plan.order[k] (the reference's slice_alloc layout)."""
    import torch
    from paper_2210_06438_b200.strategy3 import TeamPlan, form_teams
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    um, up, F = _outs(S, n, cuda)
    amax = torch.full((S,), float("nan"), dtype=torch.float64, device=cuda)
    plan = TeamPlan(form_teams(range(S), A, E), pool, n, vel, um, up, F, E,
                    amax=amax, team_buffers=True)
    plan.launch()
    torch.cuda.synchronize()
    order = np.asarray(plan.order)
    assert sorted(order.tolist()) == list(range(S))
    assert np.array_equal(F.cpu().numpy(), oF[order])
    assert np.array_equal(um.cpu().numpy(), oum[order])
    assert bool((amax == 1.0).all())


@pytest.mark.parametrize("A", [1, 16, 128])
def test_queue_executor_bit_exact(cuda, cfg2, A):
    """Device-queue strategy 3: every arrival published exactly once, the
    consumer grid completes them all, results bit-exact; runs back to back
    reuse the queue."""
    import torch
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    q = QueueExecutor("reconstruct", A, default_parents(S, A), n)
    for rep in range(2):
        um, up, F = _outs(S, n, cuda)
        order = np.random.default_rng(rep).permutation(S)
        teams = q.run(pool, vel, order, um, up, F)
        torch.cuda.synchronize()
        assert q.completed() == S
        assert np.array_equal(F.cpu().numpy(), oF)
        assert np.array_equal(up.cpu().numpy(), oup)
    st = q.stats()
    assert st["teams_formed"] == sum(st["size_histogram"].values())
    assert sum(k * v for k, v in st["size_histogram"].items()) == 2 * S
    assert max(st["size_histogram"]) <= A


@pytest.mark.parametrize("grid,n,vel", [(32, 8, (1.0, 1.0, 1.0)),
                                        (64, 8, (-1.0, 0.5, -0.25)),
                                        (64, 16, (0.7, -1.3, 0.0))])
def test_aggregated_iteration_host_roundtrip(cuda, grid, n, vel):
    """run_host: host field in -> one device iteration -> host field out ==
    reference_step(u, iterations=1); three chained == one reference step."""
    import torch
    from paper_2210_06438_b200.strategy3 import AggregatedIteration
    f = HO.stress_field(grid)
    it = AggregatedIteration(grid, n, vel, max_team=16, executors=2)
    host_in = torch.from_numpy(f).pin_memory()
    host_out = torch.empty_like(host_in).pin_memory()
    it.run_host(host_in, host_out)
    torch.cuda.synchronize()
    assert np.array_equal(host_out.numpy(), HO.advect_once(f, vel))
    it.run_host(host_in, host_out, iterations=3)
    torch.cuda.synchronize()
    assert np.array_equal(host_out.numpy(), HO.reference_step(f, vel))


@pytest.mark.parametrize("grid,n,vel,layers,cs", [
    (128, 8, (1.0, 1.0, 1.0), (1, 3, 4, 4, 3, 1), 1),
    (128, 8, (-0.6, 1.1, -0.9), (1, 3, 4, 4, 2, 1, 1), 2),
    (128, 8, (0.3, -0.2, 0.9), (16,), 1),
    (128, 8, (0.5, 0.5, -1.0), (1,) * 16, 1),
    (64, 16, (-0.3, 0.8, 0.1), (1, 1, 1, 1), 2),
    (64, 8, (-1.0, 0.5, -0.25), (1, 3, 4, 4, 3, 1), 2),
    (64, 16, (0.7, -1.3, 0.0), (2, 2), 1)])
def test_recon_flux_host_pipelined(cuda, grid, n, vel, layers, cs):
    """The e2e call (host field in, aggregated recon+flux, per-sub-grid max
    signal speed out), plain and pipelined (chunked upload overlapped with
    scatter / ghost fill / team launches, one CUDA graph): the faces in HBM
    equal the oracle's, on every replay."""
    import torch
    from paper_2210_06438_b200.strategy3 import (AggregatedIteration,
                                                 ReconFluxHostPipeline)
    f = HO.stress_field(grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    it = AggregatedIteration(grid, n, vel, max_team=128, executors=2)
    host_in = torch.from_numpy(f).pin_memory()
    amax = torch.empty(it.S, dtype=torch.float64).pin_memory()
    it.recon_flux_host(host_in, amax)
    torch.cuda.synchronize()
    assert np.array_equal(it.F.cpu().numpy(), oF)
    pipe = ReconFluxHostPipeline(it, host_in, amax, layers=layers,
                                 copy_streams=cs)
    for _ in range(2):
        # stale device state must not leak in: the staged field (the last
        # layer's middle planes are scattered before they land, and must
        # not be read by its neighbours' ghost fill) and the pool
        for t in (it.um, it.up, it.F, it.amax, it.field_dev, it.pool):
            t.fill_(float("nan"))
        amax.fill_(float("nan"))
        pipe.run()
        torch.cuda.synchronize()
        assert np.array_equal(it.pool.cpu().numpy(), hp)
        assert np.array_equal(it.um.cpu().numpy(), oum)
        assert np.array_equal(it.up.cpu().numpy(), oup)
        assert np.array_equal(it.F.cpu().numpy(), oF)
        assert bool((amax == max(abs(v) for v in vel)).all())


def test_field_pool_kernels_roundtrip(cuda):
    import torch
    from paper_2210_06438_b200 import ops
    f = HO.initial_field(32)
    field = torch.from_numpy(f).to(cuda)
    pool = torch.full((64, 14, 14, 14), float("nan"), dtype=torch.float64,
                      device=cuda)
    ops.field_to_pool(field, 8, pool)
    assert np.array_equal(pool.cpu().numpy(), HO.make_pool(f, 8),
                          equal_nan=True)
    out = torch.empty_like(field)
    ops.pool_to_field(pool, 8, out)
    assert torch.equal(out, field)


@pytest.mark.parametrize("A,E", [(1, 1), (16, 4), (128, 8)])
def test_realtime_executor_bit_exact(cuda, cfg2, A, E):
    import torch
    from paper_2210_06438_b200.strategy3 import (RealtimeExecutor,
                                                 default_parents)
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    um, up, F = _outs(S, n, cuda)
    ex = RealtimeExecutor("reconstruct", A, E, default_parents(S, A))
    order = np.random.default_rng(A).permutation(S)
    launches = ex.run(pool, n, vel, order, um, up, F)
    torch.cuda.synchronize()
    st = ex.stats()
    assert st["teams_formed"] == launches
    assert sum(k * v for k, v in st["size_histogram"].items()) == S
    assert max(st["size_histogram"]) <= A
    assert np.array_equal(F.cpu().numpy(), oF)
    assert np.array_equal(um.cpu().numpy(), oum)


@pytest.mark.parametrize("sort", [False, True])
@pytest.mark.parametrize("n,vel", [(16, (-0.7, 1.3, 0.2)),
                                   (8, (0.4, -0.9, -1.1))])
def test_queue_executor_other_shapes(cuda, n, vel, sort):
    """The device queue for 16^3 sub-grids (single-buffered consumer) and
    for negative velocity components, stress field, scattered arrivals."""
    import torch
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    grid = 64
    hp = HO.make_pool(HO.stress_field(grid), n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    pool = torch.from_numpy(hp).to(cuda)
    S = pool.shape[0]
    q = QueueExecutor("flux", 8, default_parents(S, 8), n,
                      sorted_dispatch=sort)
    um, up, F = _outs(S, n, cuda)
    amax = torch.zeros(S, dtype=torch.float64, device=cuda)
    q.run(pool, vel, np.random.default_rng(3).permutation(S), um, up, F,
          amax=amax)
    torch.cuda.synchronize()
    assert q.completed() == S
    assert np.array_equal(um.cpu().numpy(), oum)
    assert np.array_equal(up.cpu().numpy(), oup)
    assert np.array_equal(F.cpu().numpy(), oF)
    assert bool((amax == max(abs(v) for v in vel)).all())


def test_queue_executor_back_to_back_runs_of_varying_size(cuda, cfg2):
    """Consecutive real-time runs alternate the two queue slots; each run's
    ring entries carry a new epoch and the previous kernel resets the next
    slot's counters.  Runs of very different sizes (a full iteration, then a
    handful of arrivals, then a large random subset ...) must each process
    exactly their own arrivals — stale entries of a longer earlier run are
    never taken — and leave every other output slot untouched."""
    import torch
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    rng = np.random.default_rng(2210)
    q = QueueExecutor("flux", 32, default_parents(S, 32), n)
    for size in (S, 7, 1500, 1, S, 333):
        ids = rng.choice(S, size=size, replace=False).astype(np.int32)
        um, up, F = _outs(S, n, cuda)
        q.run(pool, vel, ids, um, up, F)
        torch.cuda.synchronize()
        assert q.completed() == size
        Fh = F.cpu().numpy()
        assert np.array_equal(Fh[ids], oF[ids]), size
        rest = np.setdiff1d(np.arange(S), ids)
        assert np.isnan(Fh[rest]).all(), size


def test_queue_consumer_gives_the_gpu_back_when_nothing_arrives(cuda):
    """A queue that is never published to and never closed: the resident
    consumer grid exits after its timeout instead of holding the GPU."""
    import time
    import torch
    from paper_2210_06438_b200 import _lib
    lib = _lib.load()
    n, S = 8, 64
    c = n + 2
    pool = torch.zeros((S, n + 6, n + 6, n + 6), dtype=torch.float64,
                       device=cuda)
    um, up, F = (torch.empty((S, 3, c, c, c), dtype=torch.float64,
                             device=cuda) for _ in range(3))
    ring_h = torch.zeros(S, dtype=torch.int64).pin_memory()  # untagged
    ctl_h = torch.tensor([0, -1, 0, 0, 0], dtype=torch.int64).pin_memory()
    ring_d = torch.zeros(S + 2, dtype=torch.int64, device=cuda)
    qdev = torch.zeros(64, dtype=torch.int64, device=cuda)  # epoch tag 0
    t0 = time.time()
    _lib.check(lib.tf_queue_consumer_launch(
        pool.data_ptr(), S, n, ring_h.data_ptr(), ctl_h.data_ptr(),
        ring_d.data_ptr(), S, qdev.data_ptr(), 0, 1, 1.0, 1.0, 1.0,
        um.data_ptr(), up.data_ptr(), F.data_ptr(), None, 0,
        5_000_000, 0, torch.cuda.current_stream().cuda_stream),
        "tf_queue_consumer_launch")
    torch.cuda.synchronize()
    assert time.time() - t0 < 5.0
    assert int(ctl_h[2]) & 0xFFFFFFFF == 0  # nothing completed (epoch tag)
    assert int(ctl_h[3]) == 1           # the timeout is reported


@pytest.mark.parametrize("A", [1, 16, 128])
def test_device_launch_executor_bit_exact(cuda, cfg2, A):
    """Teams formed in real time, each launched as its own grid FROM THE
    DEVICE (tf_dlexec): every slice of config 2 equals the oracle, on
    back-to-back runs, and every arrival lands in exactly one team."""
    import torch
    from paper_2210_06438_b200.strategy3 import (DeviceLaunchExecutor,
                                                 default_parents)
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    ex = DeviceLaunchExecutor("reconstruct", A, default_parents(S, A), n)
    amax = torch.full((S,), float("nan"), dtype=torch.float64, device=cuda)
    for _ in range(2):
        um, up, F = _outs(S, n, cuda)
        ex.run(pool, vel, np.arange(S, dtype=np.int32), um, up, F, amax=amax)
        ex.wait()
        assert np.array_equal(F.cpu().numpy(), oF)
        assert np.array_equal(um.cpu().numpy(), oum)
        assert np.array_equal(up.cpu().numpy(), oup)
    assert bool((amax == 1.0).all())
    st = ex.stats()
    assert sum(k * v for k, v in st["size_histogram"].items()) == 2 * S
    assert max(st["size_histogram"]) <= A


@pytest.mark.parametrize("early,sort", [(False, False), (True, False),
                                        (True, True)])
def test_queue_executor_overlapped_runs_bit_exact(cuda, cfg2, early, sort):
    """Runs issued back to back with no host synchronisation overlap on the
    device (each consumer grid a programmatic dependent of the previous
    one; slot counters monotonic, never reset).  Runs of varying size over
    two different pools, each into its own outputs, some on a second stream
    (ordered by events), then several runs into the SAME outputs (each
    store waits for the previous run): every output equals its own run's
    oracle."""
    import torch
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    grid = round(S ** (1 / 3)) * n
    hp2 = HO.make_pool(HO.stress_field(grid), n)
    HO.exchange_ghosts_pool(hp2, n, grid // n)
    pool2 = torch.from_numpy(hp2).to(cuda)
    o2 = HO.recon_flux_batch(hp2, n, vel)
    pools = [(pool, (oum, oup, oF)), (pool2, o2)]
    rng = np.random.default_rng(7)
    q = QueueExecutor("flux", 64, default_parents(S, 64), n,
                      early_loads=early, sorted_dispatch=sort)
    side = torch.cuda.Stream()
    runs = []
    for k, size in enumerate((S, 7, 1500, S, 1, S, 333, S, S)):
        ids = rng.choice(S, size=size, replace=False).astype(np.int32)
        p, ref = pools[k % 2]
        um, up, F = _outs(S, n, cuda)
        s = side if k in (3, 4, 7) else torch.cuda.current_stream()
        if s is side:
            side.wait_stream(torch.cuda.current_stream())  # outputs' fill
        q.run(p, vel, ids, um, up, F, stream=s)
        runs.append((ids, ref, F, um, s))
    # same outputs, alternating pools: the last run's values must win
    um, up, F = _outs(S, n, cuda)
    for k in range(6):
        q.run(pools[k % 2][0], vel, np.arange(S, dtype=np.int32), um, up, F)
    q.wait()
    torch.cuda.synchronize()
    for ids, ref, Fo, umo, _ in runs:
        Fh, umh = Fo.cpu().numpy(), umo.cpu().numpy()
        assert np.array_equal(Fh[ids], ref[2][ids])
        assert np.array_equal(umh[ids], ref[0][ids])
        rest = np.setdiff1d(np.arange(S), ids)
        assert np.isnan(Fh[rest]).all()
    last = pools[5 % 2][1]
    assert np.array_equal(F.cpu().numpy(), last[2])
    assert np.array_equal(up.cpu().numpy(), last[1])


def test_queue_executor_rejects_bad_ids_and_stays_usable(cuda, cfg2):
    """An arrival id outside the pool is refused before anything is
    launched or published (ValidationError), and the same queue then runs
    a correct iteration; outputs of the wrong shape are refused too."""
    import torch
    from paper_2210_06438_b200.errors import ValidationError
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    q = QueueExecutor("flux", 16, default_parents(S, 16), n)
    um, up, F = _outs(S, n, cuda)
    bad = np.arange(S, dtype=np.int32)
    bad[7] = S
    with pytest.raises(ValidationError):
        q.run(pool, vel, bad, um, up, F)
    with pytest.raises(ValidationError):
        q.run(pool, vel, np.arange(S, dtype=np.int32), um[: S // 2], up, F)
    q.run(pool, vel, np.arange(S, dtype=np.int32), um, up, F)
    q.wait()
    torch.cuda.synchronize()
    assert q.completed() == S
    assert np.array_equal(F.cpu().numpy(), oF)
    assert np.array_equal(um.cpu().numpy(), oum)


@pytest.mark.parametrize("grid,n,vel", [(64, 8, (1.0, 1.0, 1.0)),
                                        (64, 8, (-1.0, 0.5, -0.25))])
def test_aggregated_iteration_on_the_fly(cuda, grid, n, vel):
    """AggregatedIteration(formation="queue"): the teams formed on the fly
    by the formation core and published to the device queue after each
    ghost fill — recon_flux_host faces and run_host fields equal the
    oracle's / reference_step's, on repeated calls."""
    import torch
    from paper_2210_06438_b200.strategy3 import AggregatedIteration
    f = HO.stress_field(grid)
    hp = HO.make_pool(f, n)
    HO.exchange_ghosts_pool(hp, n, grid // n)
    oum, oup, oF = HO.recon_flux_batch(hp, n, vel)
    it = AggregatedIteration(grid, n, vel, max_team=16, executors=1,
                             formation="queue")
    host_in = torch.from_numpy(f).pin_memory()
    amax = torch.empty(it.S, dtype=torch.float64).pin_memory()
    for _ in range(2):
        it.um.fill_(float("nan"))
        it.recon_flux_host(host_in, amax)
        it.queue.wait()
        torch.cuda.synchronize()
        assert np.array_equal(it.um.cpu().numpy(), oum)
        assert np.array_equal(it.F.cpu().numpy(), oF)
        assert bool((amax == max(abs(v) for v in vel)).all())
    host_out = torch.empty_like(host_in).pin_memory()
    it.run_host(host_in, host_out, iterations=3)
    torch.cuda.synchronize()
    assert np.array_equal(host_out.numpy(), HO.reference_step(f, vel))


def test_queue_executor_bound_call(cuda, cfg2):
    """QueueExecutor.bind: arguments checked once, each call one formation +
    publish run; alternating two bound calls over two pools (back to back,
    overlapped on the device) leaves the last call's outputs, bit-exact."""
    import torch
    from paper_2210_06438_b200.errors import ValidationError
    from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
    pool, n, vel, oum, oup, oF = cfg2
    S = pool.shape[0]
    grid = round(S ** (1 / 3)) * n
    hp2 = HO.make_pool(HO.stress_field(grid), n)
    HO.exchange_ghosts_pool(hp2, n, grid // n)
    pool2 = torch.from_numpy(hp2).to(cuda)
    o2 = HO.recon_flux_batch(hp2, n, vel)
    q = QueueExecutor("flux", 128, default_parents(S, 128), n,
                      early_loads=True)
    um, up, F = _outs(S, n, cuda)
    ids = np.arange(S, dtype=np.int32)
    calls = [q.bind(p, vel, ids, um, up, F) for p in (pool, pool2)]
    for k in range(7):
        assert calls[k % 2]() >= 1
    q.wait()
    torch.cuda.synchronize()
    assert np.array_equal(F.cpu().numpy(), oF)       # call 6: pool
    assert np.array_equal(up.cpu().numpy(), oup)
    calls[1]()
    q.wait()
    torch.cuda.synchronize()
    assert np.array_equal(um.cpu().numpy(), o2[0])
    bad = ids.copy()
    bad[3] = S
    with pytest.raises(ValidationError):
        q.bind(pool, vel, bad, um, up, F)
