#!/bin/bash
# Round 2: weights of steps with >= 2 real components stored without the
# old-bits comparison (RGBDSEG_WSTORE_ALL) -- parity subset + A/B + traffic.
O=gpurun_out/r2w; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/wall.so $L
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "lean_path or random_configs or random_scenes or processor or fused or untouched" > $O/pytest_wall.log 2>&1; echo "rc=$?" >> $O/pytest_wall.log
timeout 900 python bench.py --no-cpu-baseline --windows '' --e2e-steps 2 > $O/bench_wall_traffic.json 2> $O/bench_wall_traffic.err
cp $O/orig.so $L
for W in streams256 hd1080; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W def6 wall > $O/ab_$W.txt 2>&1
done
