#!/bin/bash
O=gpurun_out/r2pf3; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/pfc3.so $L
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_pfc3.log 2>&1; echo "rc=$?" >> $O/pytest_pfc3.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def10 pfc3 > $O/ab_$W.txt 2>&1
done
