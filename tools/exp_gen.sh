# generator-step cost breakdown: rebuild with experiment defines on the box, phase clocks
T=gpurun_out/${TAG:-expgen}; mkdir -p $T
for v in "" "-DFFQ_EXP_NOROT" "-DFFQ_EXP_NOROT -DFFQ_EXP_NOPREF"; do
  FFQ_NVCC_EXTRA="$v" python paper_2402_17993_b200/_build.py --force > /dev/null 2>&1
  echo "variant: [$v]"; python tools/phase_real.py 2>&1 | grep sector
done > $T/phase.log 2>&1
cat $T/phase.log
python paper_2402_17993_b200/_build.py --force > /dev/null 2>&1
