#!/bin/bash
# Round 2: occupancy again after the register-relief changes (wall + dst):
# 16 blocks (32 regs), L1-prefetched colour components at 12 / 16 blocks.
O=gpurun_out/r2o; mkdir -p $O
for W in streams256 hd1080 vga; do
  timeout 1800 bash profiles/ab.sh $O/ab_$W $W def8 m16 cl1b cl1bm16 > $O/ab_$W.txt 2>&1
done
