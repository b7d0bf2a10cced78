#!/bin/bash
# Round 2: SURVEY 8(f) rows (unregistered path, evaluation epilogue,
# Augmented4, bank API) -- bench lines + per-kernel DRAM bytes/time launch list.
O=gpurun_out/r2paths; mkdir -p $O
timeout 900 python profiles/bench_paths.py > $O/bench_paths.jsonl 2> $O/bench_paths.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/paths_launches.csv python profiles/bench_paths.py --steps 3 --warmup 2 > $O/paths_ncu.log 2>&1
