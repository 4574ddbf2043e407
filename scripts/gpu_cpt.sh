export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
: > gpurun_out/cpt.log
for cpt in 8 4; do
  echo "CPT=$cpt" >> gpurun_out/cpt.log
  TF_COLS8_CPT=$cpt timeout 300 python -m pytest tests/test_gpu_field.py -q -x 2>&1 | tail -1 >> gpurun_out/cpt.log
  TF_COLS8_CPT=$cpt timeout 600 python bench.py --workload cfg5 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cfg5', d['value']/1e9, d['ms_per_step'])" >> gpurun_out/cpt.log
  TF_COLS8_CPT=$cpt timeout 300 python scripts/exp_e2e.py 2>&1 | grep -E "device step|chunks=\[1, 3" >> gpurun_out/cpt.log
done
