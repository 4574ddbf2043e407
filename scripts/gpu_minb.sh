# march kernel register budget A/B: libraries built with -DTF_MARCH_MINB=v
export TASKFUSE_NO_BUILD=1
O=gpurun_out/minb
mkdir -p $O
cp paper_2210_06438_b200/libtaskfuse_b200.so /tmp/lib_orig.so
for v in 1 16 14 1 16 14; do
  cp exp_libs/lib_minb$v.so paper_2210_06438_b200/libtaskfuse_b200.so
  echo "== minb $v" >> $O/ab.log
  timeout 300 python scripts/ab_march.py 8:0:16 2>&1 | grep -v Warn >> $O/ab.log
done
cp /tmp/lib_orig.so paper_2210_06438_b200/libtaskfuse_b200.so
cp exp_libs/lib_minb16.so paper_2210_06438_b200/libtaskfuse_b200.so
timeout 300 python -m pytest tests/test_gpu_march.py -q -x > $O/pytest16.log 2>&1
cp /tmp/lib_orig.so paper_2210_06438_b200/libtaskfuse_b200.so
echo done
