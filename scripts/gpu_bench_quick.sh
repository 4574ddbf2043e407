export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python bench.py --steps 50 --warmup 10 --no-sweep --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
timeout 900 python bench.py --workload cfg5 --steps 10 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
echo done
