#!/bin/bash
# Round 2: first-round load order (depth component before the colour ones).
O=gpurun_out/r2d; mkdir -p $O
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def2 dfirst > $O/ab_$W.txt 2>&1
done
