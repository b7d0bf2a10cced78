#!/bin/bash
O=gpurun_out/r2pl; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "planar" > $O/pytest_planar.log 2>&1; echo "rc=$?" >> $O/pytest_planar.log
for W in vga hd1080 streams256; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline --traffic off --windows '' > $O/bench_$W.json 2> $O/bench_$W.err
done
