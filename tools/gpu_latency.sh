# B = 1 latency of the config-3 energy: L2 flushed per call (the bench's b1_ms) and warm,
# with and without role warps / the L2 warm-up pass; phase clocks of one evaluation
LAT_ENV="FFQ_ROLES=1;FFQ_ROLES=0;FFQ_WARM=0;FFQ_ROLES=1,FFQ_SPLIT=4" python tools/latency_cold.py
LAT_ENV="FFQ_ROLES=1;FFQ_ROLES=0" python tools/latency.py
PT_BATCH=1 python tools/phase_real.py 2>&1 | tail -2
