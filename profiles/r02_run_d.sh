O=gpurun_out/r2d; mkdir -p $O
python -m pytest tests -m gpu -x -q --durations=20 > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
python profiles/r02_e2e_packed_probe.py > $O/packed_probe.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 100 -c 1 -f -o $O/k1_default python bench.py --steps 3 --warmup 5 --no-cpu-baseline --e2e-steps 2 --traffic off --windows '' > $O/ncu_k1.log 2>&1
echo done
