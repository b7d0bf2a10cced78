#!/bin/bash
# Round 2: K1 epilogue trims -- kLean instantiation (fused only, no mask
# pointers) and List 1 as selects; GPU suite on the combined build, A/B.
O=gpurun_out/r2l; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/ls.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_ls.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_ls.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def lean sel ls > $O/ab_$W.txt 2>&1
done
