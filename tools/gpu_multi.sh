T=gpurun_out/${TAG:-multi}; mkdir -p $T
timeout 600 python -m pytest tests/test_gpu_fmo.py -q -x > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log; tail -3 $T/tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > $T/bench1.log 2>&1; echo "rc=$?" >> $T/bench1.log; tail -c 300 $T/bench1.log
BENCH_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > $T/bench2.log 2>&1; echo "rc=$?" >> $T/bench2.log; tail -c 300 $T/bench2.log
