timeout 900 python -m pytest tests/test_gpu_rotation_runs.py -q -x 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for R in 2 4 16; do python tools/rot_run.py 28 $R 2>&1 | tail -1; ROT_HIGH=1 python tools/rot_run.py 28 $R 2>&1 | tail -1; done
