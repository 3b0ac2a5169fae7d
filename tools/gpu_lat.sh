timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x -k "split or identical or sector or golden" 2>&1 | tail -3
LAT_ENV="FFQ_ROLES=1;FFQ_ROLES=0;FFQ_ROLES=1,FFQ_SPLIT=4" python tools/latency_cold.py
LAT_ENV="FFQ_ROLES=1;FFQ_ROLES=0" python tools/latency.py
PT_BATCH=1 python tools/phase_real.py 2>&1 | tail -2
SWEEP_BATCH=1121 SWEEP_SLAB=256 python tools/sweep.py 2>&1 | tail -2
