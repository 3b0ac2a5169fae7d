timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3
timeout 600 python tools/dense_passes.py 2>&1 | tail -4
