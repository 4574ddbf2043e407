export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), "alone", round(d["roofline"]["kernel_alone"]["frac"],3))'; }
{
for t in 256 512; do for v in 0 2 4 5; do
echo "threads=$t var=$v $(TASKFUSE_RECON_THREADS=$t TASKFUSE_RECON_VARIANT=$v q)"
done; done
} > gpurun_out/exp_kernel5.log 2>&1
echo done
