# Queue headline: tests, the consumer's DRAM traffic capture, full bench line.
export TASKFUSE_NO_BUILD=1
O=gpurun_out/q8
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_bench_line.py -q -x -k "queue or bench_line_contract" > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 600 ncu --cache-control none --clock-control none --print-units base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:k_queue_consumer --launch-skip 10 --launch-count 6 --csv python scripts/exp_consumer.py > $O/ncu_queue_consumer.csv 2> $O/ncu_queue_consumer.err
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
echo done
