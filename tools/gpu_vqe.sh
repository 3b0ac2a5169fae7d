T=gpurun_out/${TAG:-vqe}; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_exact.py -q -x > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log; tail -3 $T/tests.log
timeout 2400 python tools/vqe_config3.py 20000000 400000 > $T/vqe_config3.log 2>&1; echo "rc=$?" >> $T/vqe_config3.log; cat $T/vqe_config3.log
