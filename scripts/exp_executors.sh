export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
for A in 128 64; do for E in 2 4 8 16 32; do
  echo "A=$A E=$E $(timeout 300 python bench.py --steps 100 --warmup 10 --max-team $A --executors $E --no-sweep --no-cpu-baseline 2>&1 | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e9,2), round(d["roofline"]["frac"],3), round(d["roofline"]["kernel_alone"]["frac"],3))')"
done; done > gpurun_out/exp_executors.log 2>&1
echo done
