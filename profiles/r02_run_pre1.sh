#!/bin/bash
# Round 2: colour components loaded with the flag words: 1 (component 0 only)
# vs the default 2 -- ncu at frame 100 shows colour component 1 untouched in
# 95% of warps, so the default reads and holds it for nothing there.
O=gpurun_out/r2q; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/pre1.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_pre1.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_pre1.log
cp $O/orig.so $L
for W in streams256 hd1080 vga; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def2 pre1 pre1m16 > $O/ab_$W.txt 2>&1
done
cp build/pre1.so $L
timeout 900 python bench.py --no-cpu-baseline --windows '' --e2e-steps 2 > $O/bench_pre1_traffic.json 2> $O/bench_pre1_traffic.err
timeout 900 python bench.py --start 280 --no-cpu-baseline --windows '' --e2e-steps 2 > $O/bench_pre1_late_traffic.json 2> $O/bench_pre1_late_traffic.err
cp $O/orig.so $L
