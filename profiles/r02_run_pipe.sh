#!/bin/bash
# Round 2: pipelined persistent K1 (k_fused_pipe) -- bitwise GPU suite on the
# p8 build, A/B vs the one-shot default at 6/8/10/12 resident blocks, ncu of p8.
O=gpurun_out/r2p; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/p8.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_p8.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_p8.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W base p6 p8 p10 p12 > $O/ab_$W.txt 2>&1
done
cp build/p8.so $L
B="python bench.py --workload streams256 --steps 3 --warmup 3 --no-cpu-baseline --traffic off --windows '' --e2e-steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 100 -c 1 -f -o $O/p8 $B > $O/ncu_p8.log 2>&1
cp $O/orig.so $L
