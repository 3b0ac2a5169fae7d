# round-2 verification: gpu tests, smoke, bench, then launch list + ncu --set full of the top kernel
T=gpurun_out/${TAG:-r02}; mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $T/smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > $T/gpu_tests.log 2>&1; echo "tests rc=$?" >> $T/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1; echo "smoke rc=$?" >> $T/smoke.log
timeout 900 python bench.py > $T/bench.log 2>&1; echo "bench rc=$?" >> $T/bench.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $T/bench_ref.log 2>&1; echo "ref rc=$?" >> $T/bench_ref.log
tail -3 $T/gpu_tests.log $T/smoke.log; tail -c 800 $T/bench.log; tail -c 400 $T/bench_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file $T/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sharded > $T/ncu_bench.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sector_eval_real -c 1 -f -o $T/ncu_real python tools/profile_step.py --batch 148 --reps 1 > $T/ncu_real.log 2>&1
tail -2 $T/ncu_real.log
python tools/phase_real.py 2>&1 | tail -2
