# shared-row f source variants of the block expectation: phase clocks per FFQ_BLK_F
for fm in 0 1 2; do echo "FM=$fm"; FFQ_BLK_F=$fm python tools/phase_real.py 2>&1 | tail -2 | head -1; done
FFQ_BLOCKS=0 python tools/phase_real.py 2>&1 | tail -2 | head -1
