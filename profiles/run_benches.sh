#!/bin/bash
# The bench lines kept under profiles/ (one B200): default workload with the CPU
# baseline, dense variant, the other BASELINE configs, a late sequence window.
mkdir -p gpurun_out
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
python bench.py --variant ldg --no-cpu-baseline > gpurun_out/bench_dense.json 2> gpurun_out/bench_dense.err
for W in rows8k hd1080 vga; do
  python bench.py --workload $W --no-cpu-baseline > gpurun_out/bench_$W.json 2> gpurun_out/bench_$W.err
done
python bench.py --start 275 --no-cpu-baseline > gpurun_out/bench_late.json 2> gpurun_out/bench_late.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
