export TASKFUSE_NO_BUILD=1
O=gpurun_out/thr
mkdir -p $O
cp paper_2210_06438_b200/libtaskfuse_b200.so /tmp/lib_cur.so
for v in thr nothr thr nothr; do cp exp_libs/lib_$v.so paper_2210_06438_b200/libtaskfuse_b200.so; echo "== $v" >> $O/q.log; timeout 300 python scripts/exp_queue.py 2>&1 | grep "early=True" | cut -c1-200 >> $O/q.log; done
cp /tmp/lib_cur.so paper_2210_06438_b200/libtaskfuse_b200.so
echo done
