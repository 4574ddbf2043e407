# Device queue: tests after the epoch fix, and ncu --set full captures of the
# consumer grid (pre-published, exp_consumer.py) and the one-launch kernel.
export TASKFUSE_NO_BUILD=1
O=gpurun_out/q3
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_strategy3.py -q -x -k "queue" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_queue_consumer --launch-skip 8 -c 1 -o $O/consumer -f python scripts/exp_consumer.py > $O/ncu_consumer.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_recon_flux --launch-skip 8 -c 1 -o $O/single -f python scripts/exp_consumer.py > $O/ncu_single.log 2>&1
echo done
