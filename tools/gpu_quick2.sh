# quick check: sector parity tests, phase clocks, 1121-row throughput
T=gpurun_out/${TAG:-q}; mkdir -p $T
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -k "golden or 18_qubit or shift_rows or sector_state or clique or split or repeatable or determinism" > $T/tests.log 2>&1; echo "rc=$?" >> $T/tests.log; tail -2 $T/tests.log
python tools/phase_real.py 2>&1 | grep sector | tail -1
SWEEP_BATCH=1121 SWEEP_SLAB=256 python tools/sweep.py 2>&1 | tail -1
PT_BATCH=1 FFQ_SPLIT=8 python tools/phase_real.py 2>&1 | grep -i "sector\|ms" | tail -2
