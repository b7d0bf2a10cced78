#!/bin/bash
# Round 2: colour components 0..1 via one lane-distributed L1 prefetch in round
# one + L1 reads at the colour step (RGBDSEG_CPRE_L1), at 12 and 16 blocks.
O=gpurun_out/r2c; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/cl1.so $L
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "lean_path or random_configs or processor or fused or untouched" > $O/pytest_cl1.log 2>&1; echo "rc=$?" >> $O/pytest_cl1.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def5 cl1 cl1m16 > $O/ab_$W.txt 2>&1
done
