export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), "alone", round(d["roofline"]["kernel_alone"]["frac"],3), "e2e", round(d["e2e"]["value"]/1e9,2))'; }
{
echo "default $(q)"
echo "nopersist $(TASKFUSE_PERSISTENT=0 q)"
echo "A64 $(q --max-team 64)"
echo "E8 $(q --executors 8)"
} > gpurun_out/exp_kernel.log 2>&1
TASKFUSE_PERSISTENT=2 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x >> gpurun_out/exp_kernel.log 2>&1
echo done
