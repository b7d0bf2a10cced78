#!/bin/bash
# Round 2: min-blocks 16 (32 regs, 64 warps/SM) vs 12 on the three workloads;
# HBM/PCIe ceilings probe; VGA/1080p L2-resident window.
O=gpurun_out/r2f; mkdir -p $O
timeout 300 python profiles/r02_probe_hbm_pcie.py > $O/probe.json 2> $O/probe.err; cat $O/probe.json
L=paper_2110_14934_b200/librgbdseg_b200.so
cp $L $O/orig.so
for pass in 1 2; do for v in base mb16; do for w in vga hd1080 streams256; do
  cp build/$v.so $L
  timeout 300 python bench.py --workload $w --no-cpu-baseline --traffic off --windows late --e2e-steps 2 > $O/${w}_${v}_$pass.json 2> $O/${w}_${v}_$pass.err
  python -c "import json; d=json.loads(open('$O/${w}_${v}_$pass.json').read().strip().splitlines()[-1]); print('$w $v $pass', d['value'], d['ms_per_step'], 'late', d['windows']['late']['value'])"
done; done; done
cp $O/orig.so $L
for w in vga hd1080; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline --traffic off --windows l2,packed > $O/${w}_l2.json 2> $O/${w}_l2.err
  python -c "import json; d=json.loads(open('$O/${w}_l2.json').read().strip().splitlines()[-1]); print('$w', d['value'], 'l2', d['windows'].get('l2_resident'), 'e2e', d['e2e']['value'], 'packed', d['e2e']['interleaved']['value'])"
done
