export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
for d in 1 2 1 2; do TASKFUSE_QUEUE_DEPTH=$d timeout 300 python scripts/exp_queue_depth.py >> gpurun_out/r2c_queue.log 2>&1; done
timeout 900 python -m pytest tests/test_gpu_hydrosim.py tests/test_gpu_bench_matrix.py tests/test_gpu_fuzz.py tests/test_gpu_strategy3.py -q -x --durations=10 > gpurun_out/r2c_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2c_pytest.log
timeout 600 python - > gpurun_out/r2c_refapi.json 2> gpurun_out/r2c_refapi.err <<'PY'
import json, sys, types
sys.argv=["bench.py"]
import bench
args = types.SimpleNamespace(no_cpu_baseline=False)
print(json.dumps(bench.reference_api_legs(args)))
PY
echo "refapi exit $?" >> gpurun_out/r2c_refapi.err
timeout 300 python -m paper_2210_06438_b200.bench_matrix --executors 1 4 --max-team 1 8 64 --grid-n 64 --steps 2 --format markdown > gpurun_out/r2c_matrix_g64.md 2>&1
echo done
