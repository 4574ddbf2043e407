export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_field.py -q -x -k "pipeline or pipelined" > gpurun_out/pytest_pipe.log 2>&1; echo "exit $?" >> gpurun_out/pytest_pipe.log
timeout 300 python - >> gpurun_out/pytest_pipe.log 2>&1 <<'PY'
import sys, torch
sys.path.insert(0, '.')
from paper_2210_06438_b200.hydro import sod_field
from paper_2210_06438_b200.field import FieldIteration, HostPipeline
it = FieldIteration(128, 8, (1,1,1))
hin = sod_field(128, "cpu").pin_memory(); hout = torch.empty_like(hin).pin_memory()
def t(fn, K=30):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(K): fn()
    b.record(); torch.cuda.synchronize(); return a.elapsed_time(b)/K
print("plain", t(lambda: it.run_host(hin, hout)))
for c in (4, 8, 16):
    print("pipelined", c, t(lambda: it.run_host_pipelined(hin, hout, chunks=c)))
for c in (4, 8, 16):
    p = HostPipeline(it, hin, hout, chunks=c)
    print("graph", c, t(p.run))
PY
echo done
