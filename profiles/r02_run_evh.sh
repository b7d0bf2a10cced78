#!/bin/bash
O=gpurun_out/r2evh; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/evh.so $L
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "eval or acceptance" > $O/pytest_evh.log 2>&1; echo "rc=$?" >> $O/pytest_evh.log
for pass in 1 2; do
  for v in def16 evh; do
    cp build/$v.so $L
    timeout 900 python profiles/bench_paths.py > $O/paths_${v}_$pass.jsonl 2> $O/paths_${v}_$pass.err
  done
done
cp $O/orig.so $L
