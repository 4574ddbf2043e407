export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_strategy3.py -q -x -k "team_buffers or team_plan" > gpurun_out/exp_plan.log 2>&1
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3))'; }
{
for E in 1 2 3 4 6 8; do
echo "A=128 E=$E sub $(q --executors $E) team $(q --executors $E --team-buffers)"
done
for E in 2 4 8; do
echo "A=64 E=$E sub $(q --max-team 64 --executors $E) team $(q --max-team 64 --executors $E --team-buffers)"
done
} >> gpurun_out/exp_plan.log 2>&1
echo done
