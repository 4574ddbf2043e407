export TASKFUSE_NO_BUILD=1
O=gpurun_out/ec
mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_march.py tests/test_gpu_peer.py tests/test_gpu_fullsize.py tests/test_gpu_bench_line.py -q -x > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 600 python scripts/exp_march_slab.py > $O/slab.log 2>&1
timeout 600 python scripts/ab_march.py 8:0:16 8:0:8 > $O/ab.log 2>&1
echo done
