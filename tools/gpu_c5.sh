timeout 900 python -m pytest tests/test_gpu_edges.py tests/test_gpu_parity.py -q -x -k "compact or config5" 2>&1 | tail -3
for B in 1 8; do
timeout 600 python tools/config5.py 32 $B 2>&1 | tail -1 | grep -o "rep2.*"
done
timeout 600 python tools/dense_passes.py 2>&1 | tail -4
