#!/bin/bash
O=gpurun_out/r2m16; mkdir -p $O
for W in streams256 rows8k; do
  timeout 1800 bash profiles/ab.sh $O/ab_$W $W def15 m16b > $O/ab_$W.txt 2>&1
done
