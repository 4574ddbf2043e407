# The round-2 evidence refresh after the along-y march and the e2e pipeline
# order: everything gpu_final_r2.sh produces, plus the march kernel's
# sanitizer pass (both march axes) and its ncu capture.
export TASKFUSE_NO_BUILD=1
bash scripts/gpu_final_r2.sh
O=gpurun_out/${FINAL_DIR:-final2}
S="compute-sanitizer --error-exitcode 9"
{
echo "== memcheck: march kernel (both axes, every sign, chunk lengths, halos, peer form)"; timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_march.py -q -x 2>&1 | tail -3
echo "== racecheck: march kernel"; timeout 1500 $S --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_march.py -q -x -k "every_sign or chunk_lengths" 2>&1 | tail -3
echo "== memcheck: e2e pipeline"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "pipelined" 2>&1 | tail -3
} > $O/sanitizer_march.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_step_march --launch-skip 2 -c 1 -o $O/march_full -f python scripts/exp_march_one.py 512 > $O/ncu_march.log 2>&1
timeout 300 python scripts/exp_march_slab.py 2>&1 | grep -v Warn > $O/slab.log
timeout 300 python scripts/exp_e2e_tail.py 2>&1 | grep -v Warn > $O/e2e_tail.log
echo done
