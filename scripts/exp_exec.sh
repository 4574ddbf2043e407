export TASKFUSE_NO_BUILD=1
for e in 1 2 4; do for a in 64 128; do
  timeout 300 python bench.py --no-sweep --no-cpu-baseline --executors $e --max-team $a --steps 100 > gpurun_out/ex.json 2>/dev/null
  python -c "
import json;d=json.loads(open('gpurun_out/ex.json').read().strip().splitlines()[-1])
print('A=$a executors $e', round(d['value']/1e9,2), round(d['roofline']['frac'],4), round(d['ms_per_step']*1e3,1),'us')"
done; done
