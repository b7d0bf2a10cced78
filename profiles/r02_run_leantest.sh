#!/bin/bash
O=gpurun_out/r2t; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "lean_path or tail_and_misaligned" > $O/pytest_lean.log 2>&1; echo "rc=$?" >> $O/pytest_lean.log
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gpus2.json 2> $O/bench_gpus2.err
