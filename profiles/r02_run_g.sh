#!/bin/bash
# Round 2: warp-specialised K1 (variant ws) parity + A/B against auto.
O=gpurun_out/r2g; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ws" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/pytest.log
tail -4 $O/pytest.log
for w in streams256 vga hd1080; do for v in auto ws; do
  timeout 300 python bench.py --workload $w --variant $v --no-cpu-baseline --traffic off --windows late --e2e-steps 2 > $O/${w}_$v.json 2> $O/${w}_$v.err
  python -c "import json,sys; d=json.loads(open('$O/${w}_$v.json').read().strip().splitlines()[-1]); print('$w $v', d['value'], d['ms_per_step'], 'late', d['windows']['late']['value'])" || tail -5 $O/${w}_$v.err
done; done
