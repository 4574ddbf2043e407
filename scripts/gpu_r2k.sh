export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r2k_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2k_pytest.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2k_bench.json 2> gpurun_out/r2k_bench.err; echo "bench exit $?" >> gpurun_out/r2k_bench.err
echo done
