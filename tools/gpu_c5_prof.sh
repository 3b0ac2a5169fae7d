# ncu --set full of one list-driven generator pass of config 5 at IL = 1 and IL = 4
T=gpurun_out/c5; mkdir -p $T
for B in 1 4; do
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:^k_compact_gen$ --launch-skip 2600 -c 2 -f -o $T/ncu_c5gen_b$B python tools/config5.py 32 $B > $T/ncu_full_b$B.log 2>&1
tail -1 $T/ncu_full_b$B.log | cut -c1-200
done
