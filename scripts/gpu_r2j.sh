export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 600 compute-sanitizer --tool memcheck --print-limit 5 python -m pytest tests/test_gpu_strategy3.py -q -x -k "device_launch" > gpurun_out/r2j_memcheck.log 2>&1
echo done
