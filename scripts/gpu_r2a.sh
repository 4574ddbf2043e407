export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2a_pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2a_pytest_gpu.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err; echo "bench exit $?" >> gpurun_out/r2a_bench.err
echo done
