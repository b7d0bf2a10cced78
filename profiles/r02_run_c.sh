O=gpurun_out/r2c; mkdir -p $O
python -m pytest tests -m gpu -x -q --durations=15 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
for W in vga hd1080; do python bench.py --workload $W --no-cpu-baseline > $O/bench_$W.json 2> $O/bench_$W.err; done
python bench.py --gpus 2 --no-cpu-baseline > $O/bench_g2.json 2> $O/bench_g2.err; echo "g2 rc=$?"
