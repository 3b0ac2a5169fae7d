# full GPU check: gpu tests, smoke, bench (logs under gpurun_out/$TAG)
T=gpurun_out/${TAG:-run}; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $T/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $T/gpu_tests.log 2>&1; echo "tests rc=$?" >> $T/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "smoke rc=$?" >> $T/smoke.log
timeout 900 python bench.py > $T/bench.log 2>&1; echo "bench rc=$?" >> $T/bench.log
tail -3 $T/gpu_tests.log $T/smoke.log; tail -c 600 $T/bench.log
