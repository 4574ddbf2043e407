export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 600 python bench.py --workload cfg5 --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2>gpurun_out/cfg5.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_cfg5.json').read().strip().splitlines()[-1])
print('cfg5', round(d['value']/1e9,1), 'G', round(d['ms_per_step'],4), 'ms nccl', round(d['nccl_exchange_path']['ms_per_step'],4))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_step_cols8s -s 3 -c 1 -o gpurun_out/prof_step_s python bench.py --workload cfg5 --cfg5-grid 256 --steps 2 --warmup 3 > gpurun_out/ncu_step_s.log 2>&1
echo done
