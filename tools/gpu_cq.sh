# clique expectation: parity tests of the sector paths, phase clocks (cliques on/off), throughput
T=gpurun_out/${TAG:-cq}; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log
tail -3 $T/tests.log
python tools/phase_real.py > $T/phase_on.log 2>&1; tail -3 $T/phase_on.log
FFQ_CLIQUES=0 python tools/phase_real.py > $T/phase_off.log 2>&1; tail -3 $T/phase_off.log
SWEEP_BATCH=1121 SWEEP_SLAB=256 SWEEP_ENV="FFQ_CLIQUES=1;FFQ_CLIQUES=0" python tools/sweep.py > $T/sweep.log 2>&1; tail -3 $T/sweep.log
