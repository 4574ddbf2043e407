export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
{
for v in 0 1 2 3; do
echo "step var=$v $(TASKFUSE_STEP_VARIANT=$v timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["ms_per_step"],3), round(d["roofline"]["frac"],3))')"
done
for v in 1 2 3; do TASKFUSE_STEP_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_field.py -q -x 2>&1 | tail -1; done
} > gpurun_out/exp_step.log 2>&1
echo done
