# phase clocks + throughput + one ncu --set full capture of k_sector_eval_real (148 evaluations)
set -x
python tools/phase_real.py 2>&1 | tail -2
SWEEP_BATCH=1121 SWEEP_SLAB=256 python tools/sweep.py 2>&1 | tail -1
ncu --set full --import-source on --clock-control none -k regex:k_sector_eval_real -c 1 -f -o gpurun_out/ncu_real_${TAG:-x} python tools/profile_step.py --batch 148 --reps 1 > gpurun_out/ncu_real_${TAG:-x}.log 2>&1
tail -2 gpurun_out/ncu_real_${TAG:-x}.log
