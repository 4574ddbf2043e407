export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
TF_HIB=1 timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_peer.py -q 2>&1 | tail -2
for c in 0 1 0 1; do
  TF_HIB=$c timeout 600 python bench.py --workload cfg5 --steps 20 --warmup 3 > gpurun_out/cfg5_v.json 2>gpurun_out/cfg5_v.err
  python -c "
import json;d=json.loads(open('gpurun_out/cfg5_v.json').read().strip().splitlines()[-1])
print('hib $c cfg5', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms nccl', round(d['nccl_exchange_path']['ms_per_step'],4))" || tail -3 gpurun_out/cfg5_v.err
done
for c in 0 1; do TF_HIB=$c timeout 600 python scripts/exp_e2e.py 2>&1 | grep -E "device step" | sed "s/^/hib $c /"; done
echo done
