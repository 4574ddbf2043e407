export TASKFUSE_NO_BUILD=1
O=gpurun_out/sanm
mkdir -p $O
S="compute-sanitizer --error-exitcode 9"
{
echo "== memcheck: march kernel (every sign, chunk lengths incl. odd / one-plane / one chunk, halos, peer form)"; timeout 1500 $S --tool memcheck python -m pytest tests/test_gpu_march.py -q -x 2>&1 | tail -3
echo "== racecheck: march kernel"; timeout 1500 $S --tool racecheck --racecheck-report all python -m pytest tests/test_gpu_march.py -q -x -k "every_sign or chunk_lengths" 2>&1 | tail -3
echo "== synccheck: march kernel"; timeout 900 $S --tool synccheck python -m pytest tests/test_gpu_march.py -q -x -k "every_sign" 2>&1 | tail -3
echo "== memcheck: host round trips with split copies"; timeout 900 $S --tool memcheck python -m pytest tests/test_gpu_strategy3.py -q -x -k "host" 2>&1 | tail -3
} > $O/sanitizer.log 2>&1
echo done
