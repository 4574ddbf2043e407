export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
q() { timeout 300 python bench.py --steps 100 --warmup 10 --no-sweep --no-cpu-baseline "$@" 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), d["gpu_launches"])'; }
for A in 128 64 16; do for E in 4 8 16; do
  echo "A=$A E=$E pdl $(q --max-team $A --executors $E) nopdl $(q --max-team $A --executors $E --no-overlap)"
done; done > gpurun_out/exp_pdl.log 2>&1
for A in 128 16; do for E in 1 8; do
  echo "realtime A=$A E=$E pdl $(q --mode realtime --max-team $A --executors $E) nopdl $(q --mode realtime --max-team $A --executors $E --no-overlap)"
done; done >> gpurun_out/exp_pdl.log 2>&1
timeout 120 python -m pytest tests/test_gpu_strategy3.py -q >> gpurun_out/exp_pdl.log 2>&1
echo done
