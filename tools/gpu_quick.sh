# quick GPU check: parity tests of the sector paths, phase clocks, throughput
set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x 2>&1 | tail -5
python tools/phase_real.py 2>&1 | tail -3
FFQ_BLOCKS=0 python tools/phase_real.py 2>&1 | tail -2
SWEEP_BATCH=1121 SWEEP_SLAB=256 python tools/sweep.py 2>&1 | tail -2
