#!/bin/bash
O=gpurun_out/r2h; mkdir -p $O
B="python bench.py --workload streams256 --variant ws --steps 3 --warmup 3 --no-cpu-baseline --traffic off --windows '' --e2e-steps 2"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused_ws -s 98 -c 1 -f -o $O/ws $B > $O/ncu.log 2>&1
tail -3 $O/ncu.log
