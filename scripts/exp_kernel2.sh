export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), "alone", round(d["roofline"]["kernel_alone"]["frac"],3))'; }
{
for v in 0 2; do for p in 0 2; do
echo "var=$v persist=$p $(TASKFUSE_RECON_VARIANT=$v TASKFUSE_PERSISTENT=$p q)"
done; done
python - <<'PY'
import torch
x = torch.empty(2**29, dtype=torch.float64, device="cuda")  # 4 GiB
y = torch.empty_like(x)
def t(fn, nbytes, reps=10):
    fn(); torch.cuda.synchronize()
    a=torch.cuda.Event(enable_timing=True); b=torch.cuda.Event(enable_timing=True)
    best=1e9
    for _ in range(reps):
        a.record(); fn(); b.record(); torch.cuda.synchronize(); best=min(best,a.elapsed_time(b))
    return nbytes/best/1e6
print("fill GB/s", t(lambda: x.fill_(1.0), x.numel()*8))
print("copy GB/s", t(lambda: y.copy_(x), 2*x.numel()*8))
z = x[: x.numel()//5]
def ratio():
    # read 1 part, write 4.5 parts (recon+flux ratio ~ 1:4.5)
    y[: z.numel()*4].view(4, -1).copy_(z.expand(4, -1))
print("read1:write4 GB/s", t(ratio, 5*z.numel()*8))
PY
} > gpurun_out/exp_kernel2.log 2>&1
for v in 1 2; do TASKFUSE_RECON_VARIANT=$v TASKFUSE_PERSISTENT=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done >> gpurun_out/exp_kernel2.log
echo done
