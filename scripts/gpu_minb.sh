# march kernel occupancy A/B: libraries built with TASKFUSE_NVCC_EXTRA
# (-DTF_MARCH_MINB=16: <= 128 registers; -DTF_MARCH_CARVEOUT=100: max smem)
export TASKFUSE_NO_BUILD=1
O=gpurun_out/${1:-minb}
mkdir -p $O
cp paper_2210_06438_b200/libtaskfuse_b200.so /tmp/lib_orig.so
for v in $(ls exp_libs | sed 's/lib_//; s/.so//') $(ls exp_libs | sed 's/lib_//; s/.so//'); do
  cp exp_libs/lib_$v.so paper_2210_06438_b200/libtaskfuse_b200.so
  echo "== $v" >> $O/ab.log
  timeout 300 python scripts/ab_march.py 8:0:16 2>&1 | grep -v Warn >> $O/ab.log
done
for v in $(ls exp_libs | sed 's/lib_//; s/.so//'); do
  cp exp_libs/lib_$v.so paper_2210_06438_b200/libtaskfuse_b200.so
  timeout 300 python -m pytest tests/test_gpu_march.py -q -x > $O/pytest_$v.log 2>&1
done
cp /tmp/lib_orig.so paper_2210_06438_b200/libtaskfuse_b200.so
echo done
