mkdir -p gpurun_out/r02c
timeout 1200 python bench.py > gpurun_out/r02c/bench.log 2>&1; echo "bench rc=$?"
tail -c 600 gpurun_out/r02c/bench.log
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02c/bench2.log 2>&1; echo "rc=$?"; tail -c 300 gpurun_out/r02c/bench2.log
