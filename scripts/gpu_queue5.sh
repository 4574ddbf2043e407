export TASKFUSE_NO_BUILD=1
O=gpurun_out/q5
mkdir -p $O
g++ -O2 -I include scripts/form_probe.cpp -L paper_2210_06438_b200 -ltaskfuse_b200 -Wl,-rpath,$PWD/paper_2210_06438_b200 -o scripts/_form_probe && scripts/_form_probe > $O/form.log 2>&1
nproc >> $O/form.log; lscpu | head -20 >> $O/form.log
timeout 300 python scripts/exp_queue.py > $O/queue.log 2>&1
echo done
