export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_field.py tests/test_gpu_bench_matrix.py -q -x > gpurun_out/pytest_field.log 2>&1; echo "exit $?" >> gpurun_out/pytest_field.log
echo done
