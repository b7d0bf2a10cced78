#!/bin/bash
# Round 2: unregistered processor step -- dilation + List 1 in one tiled kernel
# (RGBDSEG_DILATE_FUSE) vs rows16 + cols16 + fuse16.
O=gpurun_out/r2dz; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/dfz.so $L
timeout 1500 python -m pytest tests -m gpu -q -x -k "unregistered or dilate or register or dropin or scenario or eval or acceptance" > $O/pytest_dfz.log 2>&1; echo "rc=$?" >> $O/pytest_dfz.log
for pass in 1 2; do
  for v in def14 dfz; do
    cp build/$v.so $L
    timeout 900 python profiles/bench_paths.py > $O/paths_${v}_$pass.jsonl 2> $O/paths_${v}_$pass.err
  done
done
cp $O/orig.so $L
