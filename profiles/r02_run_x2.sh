#!/bin/bash
# Round 2: 2-px/thread K1 (k_fused_x2) -- bitwise GPU suite on the x2 build,
# then A/B against the 1-px default at 4/5/6/8 resident blocks.
O=gpurun_out/r2x2; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/x2m6.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_x2m6.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_x2m6.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W base x2m8 x2m6 x2m5 x2m4 > $O/ab_$W.txt 2>&1
done
