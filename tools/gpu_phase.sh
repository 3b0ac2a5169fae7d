set -x
python tools/phase_real.py 2>&1 | tail -4
PT_BATCH=1 python tools/phase_real.py 2>&1 | tail -3
ncu --set full --import-source on --clock-control none -k regex:k_sector_eval_real -c 1 -o gpurun_out/ncu_real_head python tools/profile_step.py --batch 148 --reps 1 > gpurun_out/ncu_real_head.log 2>&1
tail -3 gpurun_out/ncu_real_head.log
