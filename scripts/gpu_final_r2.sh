# Round-2 evidence on one B200 (gpurun): tests, smoke, every bench arm and
# workload, ncu captures (queue consumer traffic + full, plan graph traffic,
# launch list), sanitizers over the queue / recon / field kernels.
export TASKFUSE_NO_BUILD=1
O=gpurun_out/${FINAL_DIR:-final2}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench.json 2> $O/bench.err; echo "bench exit $?" >> $O/bench.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_ref.json 2> $O/bench_ref.err; echo "ref exit $?" >> $O/bench_ref.err
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 exit $?" >> $O/bench_cfg5.err
TASKFUSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err; echo "2rank exit $?" >> $O/bench_2rank_gloo.err
# the headline's consumer grid: ncu serialises a launch with the host held
# in the launch call, so nothing could be published — captured on a run
# whose slices were all published first (scripts/exp_consumer.py)
timeout 600 ncu --cache-control none --clock-control none --print-units base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum -k regex:k_queue_consumer --launch-skip 10 --launch-count 6 --csv python scripts/exp_consumer.py > $O/ncu_queue_consumer.csv 2> $O/ncu_queue_consumer.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_queue_consumer --launch-skip 8 -c 1 -o $O/consumer_full -f python scripts/exp_consumer.py > $O/ncu_consumer_full.log 2>&1
timeout 900 ncu --graph-profiling graph --cache-control none --clock-control none --print-units base --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --launch-skip 40 --launch-count 6 --csv python bench.py --mode plan --profile-only --steps 20 --warmup 10 > $O/ncu_plan_graph.csv 2> $O/ncu_plan_graph.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --mode plan --profile-only --steps 2 --warmup 3 > $O/launches_plan.csv 2> $O/launches_plan.err
timeout 300 python scripts/exp_consumer_chain.py > $O/consumer_chain.log 2>&1
timeout 300 python scripts/exp_queue.py > $O/queue.log 2>&1
S="compute-sanitizer --error-exitcode 9"
{
echo "== racecheck: queue consumer / recon / field / device launch"; timeout 1200 $S --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_parity.py tests/test_gpu_strategy3.py tests/test_gpu_field.py -q -x -m gpu -k "recon_flux_bit_exact or field_iteration_matches or queue or device_launch" 2>&1 | tail -4
echo "== memcheck: queue executor (overlapped runs, timeouts, shapes)"; timeout 1200 $S --tool memcheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "queue" 2>&1 | tail -3
echo "== synccheck: queue"; timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "queue_executor_bit_exact" 2>&1 | tail -3
} > $O/compute_sanitizer.log 2>&1
echo done
