export TASKFUSE_NO_BUILD=1
O=gpurun_out/${1:-m2}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_march.py tests/test_gpu_fullsize.py -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 python scripts/ab_march.py 8:0:16 > $O/ab.log 2>&1
echo done
