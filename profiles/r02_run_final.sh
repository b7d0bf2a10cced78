#!/bin/bash
# Round 2 checkpoint: GPU suite + smoke, every bench line (default with CPU
# baseline, the other BASELINE configs, late window, reference arm), and the
# ncu evidence of the adopted K1 (launch list + one full capture).
O=gpurun_out/r2f; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
timeout 900 python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for W in rows8k hd1080 vga; do
  timeout 900 python bench.py --workload $W --no-cpu-baseline > $O/bench_$W.json 2> $O/bench_$W.err
done
timeout 900 python bench.py --start 280 --no-cpu-baseline --windows '' > $O/bench_late.json 2> $O/bench_late.err
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --traffic off --windows '' --e2e-steps 2"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file $O/launches_default.csv $B > $O/launches_default.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 100 -c 1 -f -o $O/k1_final $B > $O/ncu_final.log 2>&1
