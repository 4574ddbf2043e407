# Queue executor breakdown (consumer alone, real-time runs, timeline) and
# the march kernel A/B on one B200.
export TASKFUSE_NO_BUILD=1
O=gpurun_out/probe
mkdir -p $O
timeout 300 python scripts/exp_consumer.py > $O/consumer.log 2>&1
timeout 300 python scripts/exp_queue.py > $O/queue.log 2>&1
timeout 600 python scripts/ab_march.py "$@" > $O/ab.log 2>&1
echo done
