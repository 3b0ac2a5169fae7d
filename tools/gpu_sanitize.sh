T=gpurun_out/${TAG:-san}; mkdir -p $T
CS=/usr/local/cuda/bin/compute-sanitizer
for k in real complex runs; do
  for tool in racecheck synccheck; do
    timeout 1200 $CS --tool $tool python tools/sanitize_prod.py $k > $T/${tool}_${k}.log 2>&1; echo "rc=$?" >> $T/${tool}_${k}.log
    tail -4 $T/${tool}_${k}.log
  done
done
timeout 900 $CS --tool memcheck python tools/sanitize_prod.py real > $T/memcheck_real.log 2>&1; echo "rc=$?" >> $T/memcheck_real.log; tail -4 $T/memcheck_real.log
timeout 900 $CS --tool memcheck python tools/sanitize_smoke.py > $T/memcheck_smoke.log 2>&1; echo "rc=$?" >> $T/memcheck_smoke.log; tail -4 $T/memcheck_smoke.log
