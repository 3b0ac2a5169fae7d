timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edges.py tests/test_gpu_fmo.py -q -x 2>&1 | tail -3
python tools/phase_real.py 2>&1 | grep "avg cycles" | tail -1
SWEEP_BATCH=1121 SWEEP_SLAB=256 python tools/sweep.py 2>&1 | tail -1
LAT_ENV="FFQ_ROLES=1" python tools/latency_cold.py
