"""Fused compute + exchange over peer memory (field.PeerSlabFieldIteration):
the step kernel stores its boundary layers straight into the neighbours'
padded fields through CUDA-IPC mappings, ordered by a device-side peer
barrier.  One rank in-process, and two real processes sharing the one GPU
(IPC within a device, gloo only to swap the handles) — bit-identical to the
whole-grid reference."""

import os
import socket

import numpy as np
import pytest

from oracle import hydro_oracle as HO

pytestmark = pytest.mark.gpu


def test_peer_single_rank(cuda):
    import torch
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    f = HO.stress_field(64)
    vel = (-1.0, 0.5, -0.25)
    r = PeerSlabFieldIteration(SlabPartition(64, 8, 1, 0), f, vel,
                               device=cuda)
    for _ in range(3):
        r.iteration()
    torch.cuda.synchronize()
    r.check()
    assert np.array_equal(r.owned().cpu().numpy(), HO.reference_step(f, vel))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, grid, n, vel, q, axis="auto"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_2210_06438_b200.field import PeerSlabFieldIteration
    from paper_2210_06438_b200.parallel_halo import SlabPartition
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        part = SlabPartition(grid, n, world, rank)
        f = HO.stress_field(grid)
        r = PeerSlabFieldIteration(part, part.slab(f), vel,
                                   device=torch.device("cuda", 0),
                                   march_axis=axis)
        for _ in range(3):
            r.iteration()
        torch.cuda.synchronize()
        r.check()
        q.put((rank, r.owned().cpu().numpy()))
        dist.barrier()   # keep the IPC-shared buffers alive until all read
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("axis", ["x", "y"])
def test_peer_two_processes_one_gpu(cuda, world, axis):
    """Both march axes (y: the ranks' thin slabs marched along y, the
    items on the x faces storing into the neighbours and waiting for the
    overlapped barrier)."""
    import torch.multiprocessing as mp
    grid, n, vel = 64, 8, (0.7, -1.3, 0.0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank,
                         args=(r, world, port, grid, n, vel, q, axis))
             for r in range(world)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs)
    whole = np.concatenate([got[r] for r in range(world)], axis=0)
    assert np.array_equal(whole, HO.reference_step(HO.stress_field(grid),
                                                   vel))


def test_peer_barrier_times_out_instead_of_hanging(cuda):
    """A neighbour that never arrives: the device barrier gives up after its
    timeout and raises the error flag (the host then raises) — it never
    hangs the GPU."""
    import torch
    from paper_2210_06438_b200 import _lib
    lib = _lib.load()
    mine = torch.zeros(2, dtype=torch.int64, device=cuda)
    left = torch.zeros(2, dtype=torch.int64, device=cuda)
    right = torch.zeros(2, dtype=torch.int64, device=cuda)
    err = torch.zeros(1, dtype=torch.int32, device=cuda)
    st = torch.cuda.current_stream().cuda_stream
    # neighbours arrived: both of my flags already at the epoch
    mine.fill_(1)
    _lib.check(lib.tf_peer_barrier(mine.data_ptr(), left.data_ptr(),
                                   right.data_ptr(), 1, 10_000_000,
                                   err.data_ptr(), st), "tf_peer_barrier")
    torch.cuda.synchronize()
    assert int(err.item()) == 0
    assert left.tolist()[1] == 1 and right.tolist()[0] == 1  # I told them
    # epoch 2: nobody writes my flags -> timeout (1 ms), error flag set
    _lib.check(lib.tf_peer_barrier(mine.data_ptr(), left.data_ptr(),
                                   right.data_ptr(), 2, 1_000_000,
                                   err.data_ptr(), st), "tf_peer_barrier")
    torch.cuda.synchronize()
    assert int(err.item()) == 1
