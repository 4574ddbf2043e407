export TASKFUSE_NO_BUILD=1
O=gpurun_out/ppm
mkdir -p $O
timeout 900 python -m pytest tests/test_ppm.py tests/test_gpu_fuzz.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
for v in 0 1 0 1; do TASKFUSE_PPM_LINES=$v timeout 300 python scripts/exp_ppm_lines.py >> $O/ab.log 2>&1; done
echo done
