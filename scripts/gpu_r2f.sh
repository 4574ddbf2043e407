export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_strategy3.py tests/test_gpu_hydrosim.py -q -x > gpurun_out/r2f_pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/r2f_pytest.log
# DRAM traffic of the TIMED step: the A=128 plan graph replayed as in the bench
timeout 900 ncu --graph-profiling graph --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --launch-skip 40 --launch-count 6 --csv python bench.py --profile-only --steps 20 --warmup 10 > gpurun_out/r2f_ncu_graph.csv 2> gpurun_out/r2f_ncu_graph.err
# launch list of the bench's hot path (gpu__time_duration per launch)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv python bench.py --profile-only --steps 2 --warmup 3 > gpurun_out/r2f_launches.csv 2> gpurun_out/r2f_launches.err
# racecheck with every hazard printed
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 40 python -m pytest tests/test_gpu_parity.py tests/test_ppm.py -q -x -m gpu -k "recon_flux_bit_exact or ppm_matches" > gpurun_out/r2f_race.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2f_bench.json 2> gpurun_out/r2f_bench.err; echo "bench exit $?" >> gpurun_out/r2f_bench.err
echo done
