export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_hydrosim.py tests/test_gpu_bench_matrix.py -q -x --durations=10 > gpurun_out/r2e_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2e_pytest.log
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err; echo "bench exit $?" >> gpurun_out/r2e_bench.err
echo done
