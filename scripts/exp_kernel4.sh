export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), "alone", round(d["roofline"]["kernel_alone"]["frac"],3))'; }
{
for t in 128 256 512; do
echo "threads=$t $(TASKFUSE_RECON_THREADS=$t q)"
echo "threads=$t E8 $(TASKFUSE_RECON_THREADS=$t q --executors 8)"
done
} > gpurun_out/exp_kernel4.log 2>&1
for t in 128 512; do TASKFUSE_RECON_THREADS=$t timeout 300 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1; done >> gpurun_out/exp_kernel4.log
echo done
