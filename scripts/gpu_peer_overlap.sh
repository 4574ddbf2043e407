export TASKFUSE_NO_BUILD=1
O=gpurun_out/pov2
mkdir -p $O

timeout 600 python scripts/exp_peer_overlap.py > $O/overlap.log 2>&1
cp paper_2210_06438_b200/libtaskfuse_b200.so /tmp/lib_cur.so
for v in nopdl pdl nopdl pdl; do cp exp_libs/lib_$v.so paper_2210_06438_b200/libtaskfuse_b200.so; echo "== $v" >> $O/ab.log; timeout 300 python scripts/ab_march.py 8:0:16 2>&1 | grep -v Warn >> $O/ab.log; done
cp /tmp/lib_cur.so paper_2210_06438_b200/libtaskfuse_b200.so
echo done
