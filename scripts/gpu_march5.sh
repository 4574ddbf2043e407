export TASKFUSE_NO_BUILD=1
O=gpurun_out/${1:-m9}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest exit $?" >> $O/pytest.log
timeout 900 python bench.py --workload cfg5 --steps 20 --warmup 5 > $O/bench_cfg5.json 2> $O/bench_cfg5.err; echo "cfg5 exit $?" >> $O/bench_cfg5.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o $O/march_full -f python scripts/exp_march_one.py 512 > $O/ncu.log 2>&1
timeout 900 python scripts/ab_march.py 8:0:16 8:0:32 > $O/ab.log 2>&1
TASKFUSE_DIST_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err; echo "2rank exit $?" >> $O/bench_2rank_gloo.err
echo done
