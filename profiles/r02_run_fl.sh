#!/bin/bash
# Round 2: where K1 reads its fusion state (out, cpt) -- List 1 after an L1
# prefetch (default), after the depth step (1), in round one (2), List 1
# after an L2 prefetch (3).
O=gpurun_out/r2fl; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/fl3.so $L
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "lean_path or random_configs or processor or fused" > $O/pytest_fl3.log 2>&1; echo "rc=$?" >> $O/pytest_fl3.log
cp $O/orig.so $L
for W in streams256 hd1080; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def4 fl1 fl2 fl3 > $O/ab_$W.txt 2>&1
done
