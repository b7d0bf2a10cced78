#!/bin/bash
# Round 2: touched mean/variance stored at a computed address (RGBDSEG_DIRECT_ST)
O=gpurun_out/r2ds; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/dst.so $L
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest_dst.log 2>&1; echo "rc=$?" >> $O/pytest_dst.log
timeout 900 python bench.py --no-cpu-baseline --windows '' --e2e-steps 2 > $O/bench_dst_traffic.json 2> $O/bench_dst_traffic.err
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def7 dst > $O/ab_$W.txt 2>&1
done
