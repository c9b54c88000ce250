set -x
export BENCH_DIST_BACKEND=gloo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --workload c3 --steps 3 --warmup 3 > gpurun_out/dry2.json 2> gpurun_out/dry2.err; echo dry2=$?
unset BENCH_DIST_BACKEND
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --workload c3 --steps 3 --warmup 3 > gpurun_out/dry1.json 2> gpurun_out/dry1.err; echo dry1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ref2.json 2> gpurun_out/ref2.err; echo ref2=$?
