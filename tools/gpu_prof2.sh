# ncu --set full of k_sector_eval_real (148 evaluations) + launch list of the bench step
T=gpurun_out/${TAG:-prof}; mkdir -p $T
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_sector_eval_real -c 1 -f -o $T/ncu_real python tools/profile_step.py --batch 148 --reps 1 > $T/ncu_real.log 2>&1
tail -2 $T/ncu_real.log
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 60 --csv --log-file $T/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-sharded > $T/ncu_bench.log 2>&1
tail -1 $T/ncu_bench.log | cut -c1-200
