#!/bin/bash
# ncu full capture of one mid-window K1 launch: 1-px default vs 2-px (x2m8).
O=gpurun_out/r2x2p; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
B="python bench.py --workload streams256 --steps 3 --warmup 3 --no-cpu-baseline --traffic off --windows '' --e2e-steps 2"
for v in base x2m8; do
  cp build/$v.so $L
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 100 -c 1 -f -o $O/$v $B > $O/ncu_$v.log 2>&1
done
cp $O/orig.so $L
