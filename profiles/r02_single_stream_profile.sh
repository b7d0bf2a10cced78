#!/bin/bash
# Round 2: ncu evidence for the single-stream configs (BASELINE configs[1], [2]):
# full-set capture of one mid-window K1 launch (frame 98) + the launch list.
O=gpurun_out/r2a; mkdir -p $O
for W in vga hd1080; do
  python bench.py --workload $W --no-cpu-baseline --e2e-steps 10 > $O/bench_$W.json 2> $O/bench_$W.err
  B="python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 2"
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 98 -c 1 -f -o $O/ncu_$W $B > $O/ncu_$W.log 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__waves_per_multiprocessor --clock-control none -s 90 -c 60 --csv --log-file $O/launches_$W.csv $B > $O/launches_$W.log 2>&1
done
