export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_strategy3.py -q -x -k queue > gpurun_out/pytest_queue.log 2>&1; echo "exit $?" >> gpurun_out/pytest_queue.log
timeout 300 python - >> gpurun_out/pytest_queue.log 2>&1 <<'PY'
import sys, time, torch, numpy as np
sys.path.insert(0, '.')
from paper_2210_06438_b200.hydro import sod_field, pool_from_field
from paper_2210_06438_b200 import ops
from paper_2210_06438_b200.strategy3 import QueueExecutor, default_parents
n, grid = 8, 128
f = sod_field(grid, "cuda"); pool = pool_from_field(f, n); ops.ghost_fill(pool, n, grid // n)
S = pool.shape[0]; c = n + 2
um = torch.empty((S,3,c,c,c), dtype=torch.float64, device="cuda"); up = torch.empty_like(um); F = torch.empty_like(um)
arr = np.arange(S, dtype=np.int32)
for A in (1, 4, 16, 64, 128):
    q = QueueExecutor("reconstruct", A, default_parents(S, A), n)
    for _ in range(3): q.run(pool, (1,1,1), arr, um, up, F)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record()
    K = 20
    for _ in range(K): q.run(pool, (1,1,1), arr, um, up, F)
    b.record(); torch.cuda.synchronize(); t1 = time.perf_counter()
    ms = a.elapsed_time(b) / K
    st = q.stats()
    print(f"queue A={A}: {ms:.3f} ms/iter, {S*512/ms/1e6:.2f} G cell-updates/s, host {1e3*(t1-t0)/K:.3f} ms, teams {st['teams_formed']//(K+3)}, mean team {S*(K+3)/st['teams_formed']:.1f}")
PY
echo done
