export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_recon_flux -s 2 -c 1 -o gpurun_out/prof_single python bench.py --profile-only --mode single --steps 2 --warmup 3 > gpurun_out/ncu_full.log 2>&1
echo done
