export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), "alone", round(d["roofline"]["kernel_alone"]["frac"],3))'; }
{
for v in 2 3; do
echo "var=$v $(TASKFUSE_RECON_VARIANT=$v q)"
echo "var=$v A64 $(TASKFUSE_RECON_VARIANT=$v q --max-team 64)"
done
} > gpurun_out/exp_kernel3.log 2>&1
TASKFUSE_RECON_VARIANT=3 timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_strategy3.py -q -x 2>&1 | tail -3 >> gpurun_out/exp_kernel3.log
echo done
