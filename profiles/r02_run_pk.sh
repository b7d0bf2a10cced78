#!/bin/bash
# Round 2: packed first-round inputs (RGBDSEG_PACK_R1) -- GPU suite on the pk
# build, A/B vs the pre-change default (base) and the current default (cur);
# late-window bench line with its own traffic; 2-rank self-launched bench.
O=gpurun_out/r2k; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
cp build/pk.so $L
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu_pk.log 2>&1; echo "rc=$?" >> $O/pytest_gpu_pk.log
cp $O/orig.so $L
for W in streams256 hd1080; do
  timeout 1500 bash profiles/ab.sh $O/ab_$W $W base cur pk > $O/ab_$W.txt 2>&1
done
timeout 900 python bench.py --start 280 --no-cpu-baseline --windows '' > $O/bench_late.json 2> $O/bench_late.err
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --no-cpu-baseline > $O/bench_gpus2.json 2> $O/bench_gpus2.err
