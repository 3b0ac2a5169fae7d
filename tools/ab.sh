#!/bin/bash
# A/B: swap in prebuilt variant libraries and run the sweep for each
for v in "$@"; do
  cp variants_tmp/$v/libfragfield_cuda.so paper_2402_17993_b200/lib/libfragfield_cuda.so
  echo "== variant $v"
  SWEEP_BATCH=1121 SWEEP_SLAB=256 SWEEP_ENV="FFQ_PERSIST=0" python tools/sweep.py
done
