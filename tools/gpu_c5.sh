# compact-layout checks: parity tests, then config 5 at B = 1 and B = 4
set -x
timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -q -x -k "compact or config5" 2>&1 | tail -5
timeout 600 python tools/config5.py 32 1 2>&1 | tail -1
timeout 600 python tools/config5.py 32 4 2>&1 | tail -1
