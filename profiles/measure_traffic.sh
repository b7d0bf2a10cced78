#!/bin/bash
# per-launch DRAM bytes of the 20 timed K1 launches for every workload/variant
for W in streams256 vga hd1080 rows8k; do for V in auto ldg; do
  B="python bench.py --workload $W --variant $V --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 2"
  $B > gpurun_out/tr_plain_${W}_$V.json 2> gpurun_out/tr_plain_${W}_$V.err || continue
  timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_fused -s 100 -c 20 --csv --log-file gpurun_out/traffic_${W}_$V.csv $B > gpurun_out/tr_ncu_${W}_$V.log 2>&1
done; done
