export TASKFUSE_NO_BUILD=1
mkdir -p gpurun_out
export TASKFUSE_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 10 --warmup 3 --no-sweep > gpurun_out/mr_bench.json 2> gpurun_out/mr_bench.err; echo "exit $?" >> gpurun_out/mr_bench.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 > gpurun_out/mr_ref.json 2> gpurun_out/mr_ref.err; echo "exit $?" >> gpurun_out/mr_ref.err
echo done
