#!/bin/bash
# Round 2: the L1 form extended to the evaluation-epilogue and interleaved
# K1 instantiations; GPU suite + the 8(f) paths before/after.
O=gpurun_out/r2ev; mkdir -p $O
L=paper_2110_14934_b200/librgbdseg_b200.so
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
cp $L $O/orig.so
for v in prev evpk; do
  cp build/$v.so $L
  timeout 900 python profiles/bench_paths.py > $O/paths_$v.jsonl 2> $O/paths_$v.err
  timeout 900 python bench.py --workload streams256 --no-cpu-baseline --traffic off --windows packed --e2e-steps 0 > $O/bench_$v.json 2> $O/bench_$v.err
done
cp $O/orig.so $L
