#!/bin/bash
O=gpurun_out/r2sk; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/skp.so $L
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "ldg_elide_l1 or random_configs or random_scenes or config3 or config4 or config5 or interleaved" > $O/pytest_skp.log 2>&1; echo "rc=$?" >> $O/pytest_skp.log
cp $O/orig.so $L
for W in streams256 hd1080; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def13 skp > $O/ab_$W.txt 2>&1
done
